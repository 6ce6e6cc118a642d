"""H2D bandwidth vs number of concurrent copy streams/chunks (55 MB pinned)."""
import time, sys, torch
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y
n = 55125000
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host.random_(0, 255)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def run(nstreams, nchunks):
    ch = (n + nchunks - 1) // nchunks
    for i in range(nchunks):
        s = streams[i % nstreams]
        a = i * ch; b = min(n, a + ch)
        y._lib.ychg_memcpy(dev.data_ptr() + a, host.data_ptr() + a, b - a, s.cuda_stream)
    torch.cuda.synchronize()
for ns, nc in [(1, 1), (1, 8), (2, 2), (2, 8), (4, 4), (4, 16), (8, 8), (8, 32)]:
    run(ns, nc)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); run(ns, nc); ts.append(time.perf_counter() - t0)
    t = sorted(ts)[5]
    print(f"streams {ns} chunks {nc:3d}: {t*1e3:.3f} ms  {n/t/1e9:.1f} GB/s")
