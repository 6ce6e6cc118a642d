"""Host-path overhead: ychg_scan_host wall time on a tiny image (pure API/launch cost)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402

for W, H in ((64, 64), (2000, 2000), (21000, 21000)):
    img = y.synth("hbands", W, H, bands=min(147, H // 2))
    host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
    host.copy_(torch.from_numpy(img.bytes().reshape(H, -1)[:, : (W + 7) // 8]))
    himg = y.BinaryImage(W, H, host.numpy())
    for _ in range(5):
        y.scan(himg)
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        y.scan(himg)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{W}x{H}: scan_host wall min {ts[0]*1e6:.0f} us med {ts[25]*1e6:.0f} us", flush=True)
