"""Per-CTA %globaltimer timelines of the fused scan kernel (Plan.debug_stamps):
an isolated scan and the steady state of a K-scan CUDA graph, for several
segment counts.  Prints phase medians (us) and the graph's per-scan time.
  python scripts/pipe_timeline.py [size] [pattern] [k ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 21000
pat = sys.argv[2] if len(sys.argv) > 2 else "hbands"
ks = sys.argv[3:] or [""]
W = H = S
pitch = y.pitch_for(W)
NB = 10
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(NB)]
st = torch.cuda.current_stream()
for b in bufs:
    y.synth_device(pat, W, H, b.data_ptr(), pitch, bands=147, density=0.5, seed=1307, cell=7, stream=st.cuda_stream)
c = torch.empty(W, dtype=torch.int32, device="cuda")
f = torch.empty(W // 32 + 64, dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda")
t = torch.zeros(4, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def phases(stm, label):
    # stm: (rows, 32) for one scan, ns; rows with entry == 0 did not run this scan
    m = stm[:, 0] > 0
    s = stm[m].astype(np.int64)
    t0 = s[:, 0].min()
    rel = lambda col: (s[:, col][s[:, col] > 0] - t0) / 1e3  # noqa: E731
    life = (s[:, 5] - s[:, 0]) / 1e3
    ramp = (s[:, 6] - s[:, 0]) / 1e3
    strm = (s[:, 7] - s[:, 6]) / 1e3
    merge = (s[:, 2] - s[:, 1]) / 1e3
    fin = s[:, 4] > 0
    fdur = (s[fin, 4] - s[fin, 3]) / 1e3
    print(f"  {label}: CTAs {m.sum()} span {(s[:, 5].max() - t0) / 1e3:.1f} us | entry spread {rel(0).max():.1f} | "
          f"life med {np.median(life):.1f} | ramp(entry->1st stage) med {np.median(ramp):.2f} | "
          f"warp0 stream med {np.median(strm):.1f} | all-warps-done->arrive med {np.median(merge):.2f} | "
          f"finish med {np.median(fdur) if fin.any() else 0:.2f} max {fdur.max() if fin.any() else 0:.2f} | "
          f"last arrive {rel(2).max():.1f} last finish-end {rel(4).max():.1f}", flush=True)
    if fin.any():
        f = s[fin]
        segs = [("loads", 3, 16), ("flags+W2", 16, 17), ("compose", 17, 18), ("lookback", 18, 19),
                ("W4", 19, 20), ("writes+W5", 20, 21), ("tail", 21, 4)]
        print("    finish phases (median us): " + ", ".join(
            f"{nm} {np.median((f[:, b] - f[:, a]) / 1e3):.2f}" for nm, a, b in segs), flush=True)


for k in ks:
    if k:
        os.environ["YCHG_SEGMENTS"] = k
    else:
        os.environ.pop("YCHG_SEGMENTS", None)
    for links in ((True, False) if os.environ.get("YCHG_TL_COUNTS") == "1" else (True,)):
        plan = y.Plan(W, H, latency=os.environ.get("YCHG_TL_LATENCY") == "1")
        info = plan.info()
        print(f"{S}^2 {pat} k={info.seg_per_strip} grid={info.grid} links={links}", flush=True)
        plan.debug_stamps(True)
        n_scans = 0
        for i in range(3):
            n_scans += 1
            plan.scan_device(bufs[i % NB].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(),
                             t.data_ptr(), st.cuda_stream, links)
            torch.cuda.synchronize()
        stm = plan.debug_stamps(True)
        # isolated: the last scan (number 2 -> ring 2)
        phases(stm[2], "isolated")
        for K in (20, 100):
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(st)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    cs = torch.cuda.current_stream().cuda_stream
                    for i in range(K):
                        plan.scan_device(bufs[i % NB].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(),
                                         t.data_ptr(), cs, links)
            st.wait_stream(cap)
            n_scans += 2 * K
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            stm = plan.debug_stamps(True)
            print(f"  graph K={K}: {ms / K * 1e3:.2f} us/scan (total {ms * 1e3:.1f} us)", flush=True)
            # the ring holds the last 4 scans of the replay: take the 4th-last
            phases(stm[(n_scans - 4) % y.STAMP_RING], f"K={K} scan {n_scans - 4}")
        plan.debug_stamps(False)
        plan.close()
