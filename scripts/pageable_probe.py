"""e2e of ychg_scan_host from pageable vs pinned host memory (21000^2 hbands(147))."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402

W = H = 21000
img = y.synth("hbands", W, H, bands=147)
rows = img.bytes().reshape(H, -1)[:, : (W + 7) // 8]
pin = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
pin.numpy()[:] = rows
page = np.ascontiguousarray(rows).copy()
for name, arr in (("pinned", pin.numpy()), ("pageable", page)):
    im = y.BinaryImage(W, H, arr)
    for _ in range(3):
        y.scan(im)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        r = y.scan(im)
        ts.append(time.perf_counter() - t0)
    t = sorted(ts)[5]
    print(f"{name}: {t * 1e3:.3f} ms  {W * H / t / 1e9:.1f} Gpix/s  hyperedges {r.hyperedges}")
dev = torch.empty_like(pin, device="cuda")
for name, src in (("pinned", pin), ("pageable", torch.from_numpy(page))):
    fl = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        fl.append(time.perf_counter() - t0)
    print(f"bare H2D {name}: {sorted(fl)[5] * 1e3:.3f} ms")
