"""Graph time vs the number of scans K (default plan, K-scan CUDA graph, CUDA events,
best of 5 replays): T(K) = fixed + slope * K separates the per-scan steady state
from the fixed ramp / drain / launch part.  python scripts/graph_kfit.py [pattern] [size]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

pat = sys.argv[1] if len(sys.argv) > 1 else "hbands"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 21000
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
Ks = (1, 2, 3, 5, 10, 20, 40, 100)
us = []
for K in Ks:
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(st)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            cs = torch.cuda.current_stream().cuda_stream
            for i in range(K):
                plan.scan_device(bufs[i % NB].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(),
                                 t.data_ptr(), cs)
    st.wait_stream(cap)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    us.append(best)
    print(f"K={K}: {best:.1f} us ({best / K:.2f} us/scan)", flush=True)
k = np.array(Ks[-3:], dtype=float)
slope, fixed = np.polyfit(k, np.array(us[-3:]), 1)
mask_bytes = H * ((W + 7) // 8)
print(f"{pat} {S}^2: T(K) ~ {fixed:.1f} us + {slope:.2f} us * K (K >= {Ks[-3]}); steady state "
      f"{mask_bytes / (slope * 1e-6) / 1e9:.0f} GB/s", flush=True)
