"""Per-CTA timeline of the streaming kernel in steady state (last 4 scans of a burst):
duration, warp imbalance (last - first warp done), merge (publish - last warp),
exit - publish."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402

W = H = 21000
links = not (len(sys.argv) > 1 and sys.argv[1] == "counts")
torch.cuda.set_device(0)
pitch = y.pitch_for(W)
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(6)]
for b in bufs:
    y.synth_device("hbands", W, H, b.data_ptr(), pitch, bands=147)
c = torch.empty(W, dtype=torch.int32, device="cuda"); f = torch.empty(W // 32 + 64, dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda"); t = torch.zeros(4, dtype=torch.int64, device="cuda")
plan = y.Plan(W, H)
info = plan.info()
s = torch.cuda.current_stream().cuda_stream
plan.debug_stamps(True)
for i in range(24):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
st = plan.debug_stamps(True).astype(np.float64)
G = info.grid
for ring in range(4):
    e = st[ring, :G]
    nw = 4 if links else 8  # streaming CTA width per path (ychg_device.cuh scan_warps)
    warps = e[:, 1:1 + nw]
    dur = (e[:, 23] - e[:, 0]) / 1e3
    imb = (warps.max(1) - warps.min(1)) / 1e3
    first = (warps.min(1) - e[:, 0]) / 1e3
    merge = (e[:, 20] - warps.max(1)) / 1e3
    flw = (e[:, 11] - e[:, 10]) / 1e3
    tail = (e[:, 23] - e[:, 20]) / 1e3
    print(f"ring {ring}: CTA dur med {np.median(dur):6.2f} max {dur.max():6.2f} | first warp done med {np.median(first):6.2f}"
          f" | warp imbalance med {np.median(imb):5.2f} max {imb.max():5.2f} | merge med {np.median(merge):5.2f}"
          f" (fin_loaded wait med {np.median(flw):5.2f}) | publish->exit {np.median(tail):5.2f} us")
