"""Device time of ONE isolated scan (image resident, stream idle before and after,
CUDA events around the single launch) versus the segment count, full path and
counts path, with and without the unchanged-block skip.
  python scripts/isolated_scan_probe.py [size] [pattern] [k ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 21000
pat = sys.argv[2] if len(sys.argv) > 2 else "hbands"
ks = sys.argv[3:] or [""]
W = H = S
pitch = y.pitch_for(W)
img = y.DeviceBuffer(pitch * H)
y.synth_device(pat, W, H, img.ptr, pitch, bands=147, density=0.5, seed=1307, cell=7)
cap = max(W, 1024)
counts = y.DeviceBuffer(4 * cap)
flags = y.DeviceBuffer(4 * (((cap + 1023) // 1024) * 33 + 32))
bounds = y.DeviceBuffer(4 * cap)
tot = y.DeviceBuffer(64)
for k in ks:
    if k:
        os.environ["YCHG_SEGMENTS"] = k
    else:
        os.environ.pop("YCHG_SEGMENTS", None)
    for skip in (True, False):
        plan = y.Plan(W, H, skip=skip, latency=True)
        info = plan.info()
        plan.set_timing(True)
        for links in (True, False):
            ts = []
            for i in range(25):
                plan.scan_device(img.ptr, pitch, counts.ptr, flags.ptr, bounds.ptr, tot.ptr, with_hyperedges=links)
                ts.append(plan.last_ms()[0] * 1e3)  # synchronises
            print(f"{S}^2 {pat} skip={int(skip)} k={k or 'default'} (grid {info.grid}, seg/strip "
                  f"{info.seg_per_strip}) {'full  ' if links else 'counts'}: median {statistics.median(ts[5:]):.1f} us"
                  f"  min {min(ts[5:]):.1f}", flush=True)
        plan.close()
