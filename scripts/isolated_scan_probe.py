"""Device time of ONE isolated scan (latency plan, image resident, stream idle
before and after) versus the segment count, full path and counts path.
  python scripts/isolated_scan_probe.py [size] [k ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 21000
ks = sys.argv[2:] or [""]
W = H = S
pitch = y.pitch_for(W)
img = y.DeviceBuffer(pitch * H)
y.synth_device("hbands", W, H, img.ptr, pitch, bands=147)
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
    plan = y.Plan(W, H, latency=True)
    info = plan.info()
    plan.set_timing(True)
    for links in (True, False):
        ts = []
        for i in range(25):
            plan.scan_device(img.ptr, pitch, counts.ptr, flags.ptr, bounds.ptr, tot.ptr, with_hyperedges=links)
            ts.append(plan.last_ms()[0] * 1e3)  # synchronises
        print(f"{S}^2 k={k or 'default'} (grid {info.grid}, seg/strip {info.seg_per_strip}) "
              f"{'full  ' if links else 'counts'}: median {statistics.median(ts[5:]):.1f} us  min {min(ts[5:]):.1f}",
              flush=True)
    plan.close()
