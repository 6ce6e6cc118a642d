"""e2e breakdown: ychg_scan_host wall time over 40 calls (min/median/max), then a
few calls with YCHG_HOST_TIMING=1 (device-side H2D / repitch / scan / D2H), and a
raw pinned cudaMemcpy H2D of the same 55 MB for the PCIe ceiling."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402

W = H = 21000
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
host.copy_(torch.from_numpy(img.bytes().reshape(H, -1)[:, : (W + 7) // 8]))
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3):
    y.scan(himg)
ts = []
for _ in range(40):
    t0 = time.perf_counter()
    y.scan(himg)
    ts.append(time.perf_counter() - t0)
ts.sort()
print("e2e ms min %.3f med %.3f max %.3f" % (ts[0] * 1e3, ts[len(ts) // 2] * 1e3, ts[-1] * 1e3))
dev = torch.empty(host.numel(), dtype=torch.uint8, device="cuda")
hv = host.view(-1)
for _ in range(3):
    dev.copy_(hv, non_blocking=True)
torch.cuda.synchronize()
tt = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.copy_(hv, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    tt.append(e0.elapsed_time(e1))
tt.sort()
print("raw pinned H2D 55 MB: ms min %.3f med %.3f -> %.1f GB/s" % (tt[0], tt[len(tt) // 2], host.numel() / tt[len(tt) // 2] / 1e6))
