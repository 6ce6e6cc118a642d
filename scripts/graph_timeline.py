"""Per-scan start / end times inside ONE replay of the bench's K-scan graph
(default plan, %globaltimer stamps): where the fill and drain of a K=20 graph go.
  python scripts/graph_timeline.py [K] [pattern] [size]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pat = sys.argv[2] if len(sys.argv) > 2 else "hbands"
S = int(sys.argv[3]) if len(sys.argv) > 3 else 21000
W = H = S
pitch = y.pitch_for(W)
NB = 11
st = torch.cuda.current_stream()
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(NB)]
for b in bufs:
    y.synth_device(pat, W, H, b.data_ptr(), pitch, bands=147, density=0.5, seed=1307, cell=7, stream=st.cuda_stream)
c = torch.empty(W, dtype=torch.int32, device="cuda")
f = torch.empty(W // 32 + 2048, dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda")
t = torch.zeros(4, dtype=torch.int64, device="cuda")
plan = y.Plan(W, H)
info = plan.info()
plan.debug_stamps(True)
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
cap.wait_stream(st)
with torch.cuda.stream(cap):
    with torch.cuda.graph(g, stream=cap):
        cs = torch.cuda.current_stream().cuda_stream
        for i in range(K):
            plan.scan_device(bufs[i % NB].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), cs)
st.wait_stream(cap)
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
n0 = K  # scans 0..K-1 were the first replay, K..2K-1 the timed one
rows = []
for sc in range(K, 2 * K):
    s = stm[sc % y.STAMP_RING].astype(np.int64)
    m = s[:, 8] > 0
    arr = s[:, 8] == sc + 1
    sel = s[arr] if arr.any() else s[m]
    rows.append((sc - K, sel[:, 0].min(), sel[:, 0].max(), sel[:, 2].max(), sel[:, 5].max()))
t0 = rows[0][1]
print(f"{pat} {S}^2 k={info.seg_per_strip} grid={info.grid}: K={K} graph {ms * 1e3 / K:.2f} us/scan, "
      f"total {ms * 1e3:.1f} us (events)")
print(" scan | first CTA in | last CTA in | last arrival | last exit (us from scan 0's first CTA)")
for i, a, b, c2, d in rows:
    print(f" {i:4d} | {(a - t0) / 1e3:11.1f} | {(b - t0) / 1e3:10.1f} | {(c2 - t0) / 1e3:11.1f} | {(d - t0) / 1e3:8.1f}")
