"""Pipelined timeline: a burst of back-to-back scans, per-CTA stamps of the last 4."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 21000
pattern = sys.argv[2] if len(sys.argv) > 2 else "hbands"
links = not (len(sys.argv) > 3 and sys.argv[3] == "counts")
torch.cuda.set_device(0)
pitch = y.pitch_for(W)
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(6)]
for b in bufs:
    y.synth_device(pattern, W, H, b.data_ptr(), pitch, bands=147, density=0.5, seed=1307)
c = torch.empty(W, dtype=torch.int32, device="cuda"); f = torch.empty(W // 32 + 64, dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda"); t = torch.zeros(4, dtype=torch.int64, device="cuda")
plan = y.Plan(W, H)
s = torch.cuda.current_stream().cuda_stream
for i in range(8):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
plan.debug_stamps(False); plan.debug_stamps(True)
for i in range(8):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
st = plan.debug_stamps(True).astype(np.int64)  # (4, grid, 32)
nstr = plan.info().n_strips
t0 = st[:, :, 0][st[:, :, 0] > 0].min()
rel = np.where(st > 0, (st - t0) / 1000.0, np.nan)
order = np.argsort(np.nanmin(rel[:, :, 0], axis=1))
for r in order:
    e = rel[r]
    print(f"scan ring {r}: A entry {np.nanmin(e[:,0]):7.2f}..{np.nanmax(e[:,0]):7.2f}  warps done med {np.nanmedian(e[:,1:9]):7.2f} max {np.nanmax(e[:,1:9]):7.2f}"
          f"  published max {np.nanmax(e[:,20]):7.2f}  A exit max {np.nanmax(e[:,23]):7.2f} | B segs seen {np.nanmax(e[:nstr,21]):7.2f} loads {np.nanmax(e[:nstr,24]):7.2f} done {np.nanmax(e[:nstr,22]):7.2f}")
print("totals", t.tolist())
