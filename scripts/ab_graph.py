"""A/B of K-scan CUDA-graph throughput (us/scan) between library builds (YCHG_LIB)
and segment counts (YCHG_SEGMENTS), no stamps: python scripts/ab_graph.py size pattern"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 21000
pat = sys.argv[2] if len(sys.argv) > 2 else "random"
W = H = S
pitch = y.pitch_for(W)
NB = 11 if S <= 32768 else 3
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
res = []
for K in (20, 100):
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
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K * 1e3)
    res.append(f"K={K} {best:.2f}")
print(f"{os.path.basename(os.environ.get('YCHG_LIB', 'default'))} seg={os.environ.get('YCHG_SEGMENTS', '-')} "
      f"{pat} grid={info.grid} k={info.seg_per_strip}: " + "  ".join(res) + f"  he={t.cpu().tolist()[2]}", flush=True)
