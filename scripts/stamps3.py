"""Finisher (B) timeline per strip for the last scan of a burst: stamps 21 segs
seen, 24 loads done, 26 tree compose, 27 look-back, 25 outputs, 22 done."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y

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
s = torch.cuda.current_stream().cuda_stream
for i in range(8):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
plan.debug_stamps(False); plan.debug_stamps(True)
for i in range(4):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
st = plan.debug_stamps(True).astype(np.int64)  # (4, grid, 32)
nstr = plan.info().n_strips
ring = int(np.argmax(np.nanmax(np.where(st[:, :, 0] > 0, st[:, :, 0], 0), axis=1)))
e = st[ring].astype(np.float64)
t0 = e[:, 0][e[:, 0] > 0].min()
rel = np.where(e > 0, (e - t0) / 1000.0, np.nan)
print("A: entry max %.2f warps-done med %.2f max %.2f published max %.2f exit max %.2f" % (
    np.nanmax(rel[:, 0]), np.nanmedian(rel[:, 1:9]), np.nanmax(rel[:, 1:9]), np.nanmax(rel[:, 20]), np.nanmax(rel[:, 23])))
for sidx in range(nstr):
    r = rel[sidx]
    print("B strip %2d: segs %6.2f loads %6.2f tree %6.2f lookback %6.2f outputs %6.2f done %6.2f" % (
        sidx, r[21], r[24], r[26], r[27], r[25], r[22]))
