"""The bench's timed workload as ONE CUDA graph (K scans of 21000^2 hbands(147) on
rotating device copies, one plan), replayed twice -- for
`ncu --graph-profiling graph`, which profiles each graph launch as one workload:
its DRAM bytes should be ~K x 55.7 MB and its duration ~K x the bench's
ms_per_step (shows the ~55 MB per step is read once while scans overlap).
  python scripts/graph_profile.py [K] [pattern]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
pat = sys.argv[2] if len(sys.argv) > 2 else "hbands"
W = H = 21000
pitch = y.pitch_for(W)
NB = 11
st = torch.cuda.current_stream()
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(NB)]
for b in bufs:
    y.synth_device(pat, W, H, b.data_ptr(), pitch, bands=147, density=0.5, seed=1307, stream=st.cuda_stream)
c = torch.empty(W, dtype=torch.int32, device="cuda")
f = torch.empty(y.boundary_flag_words(W), dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda")
t = torch.zeros(4, dtype=torch.int64, device="cuda")
plan = y.Plan(W, H)
for i in range(3):
    plan.scan_device(bufs[i].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
cap.wait_stream(st)
with torch.cuda.stream(cap):
    with torch.cuda.graph(g, stream=cap):
        cs = torch.cuda.current_stream().cuda_stream
        for i in range(K):
            plan.scan_device(bufs[i % NB].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), cs)
st.wait_stream(cap)
for _ in range(2):
    g.replay()
torch.cuda.synchronize()
print("hyperedges", t.cpu().tolist())
