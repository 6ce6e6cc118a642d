"""H2D options for a 21000x21000 packed mask (55 MB, 2625-B rows)."""
import time, torch, sys
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y
W = H = 21000
rb = (W + 7) // 8
pitch = y.pitch_for(W)
host = torch.empty(rb * H, dtype=torch.uint8, pin_memory=True)
host.random_(0, 255)
pageable = host.clone().numpy()
dense = torch.empty(rb * H, dtype=torch.uint8, device="cuda")
pitched = torch.empty(pitch * H, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return sorted(ts)[n // 2] * 1e3
import ctypes
L = y._lib
f1 = lambda: L.ychg_memcpy(dense.data_ptr(), host.data_ptr(), rb * H, s.cuda_stream)
f2 = lambda: L.ychg_memcpy_2d(pitched.data_ptr(), pitch, host.data_ptr(), rb, rb, H, s.cuda_stream)
f3 = lambda: (L.ychg_memcpy(dense.data_ptr(), host.data_ptr(), rb * H, s.cuda_stream),
              L.ychg_memcpy_2d(pitched.data_ptr(), pitch, dense.data_ptr(), rb, rb, H, s.cuda_stream))
f4 = lambda: L.ychg_memcpy_2d(pitched.data_ptr(), pitch, dense.data_ptr(), rb, rb, H, s.cuda_stream)
pg = pageable.ctypes.data
f5 = lambda: L.ychg_memcpy(dense.data_ptr(), pg, rb * H, s.cuda_stream)
for name, fn in [("H2D 1D pinned", f1), ("H2D 2D pinned", f2), ("H2D 1D + D2D 2D", f3), ("D2D 2D repitch", f4), ("H2D 1D pageable", f5)]:
    ms = t(fn)
    print(f"{name:18s} {ms:8.3f} ms  {rb*H/ms/1e6:7.1f} GB/s")
