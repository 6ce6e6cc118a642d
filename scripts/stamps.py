"""Per-CTA timeline of one scan from %globaltimer stamps (diagnostics)."""
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
for i in range(5):
    plan.scan_device(bufs[i % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
for i in range(3):
    plan.debug_stamps(False)
    plan.debug_stamps(True)
    plan.scan_device(bufs[(5 + i) % 6].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
    torch.cuda.synchronize()
st = plan.debug_stamps(True).astype(np.int64)
t0 = st[:, 0].min()
rel = (st - t0) / 1000.0
print("ctas", st.shape[0], "totals", t.tolist())
def q(x): return f"min {x.min():7.2f} med {np.median(x):7.2f} max {x.max():7.2f}"
print("entry        ", q(rel[:, 0]))
nw = int(sys.argv[4]) if len(sys.argv) > 4 else 8
wd = rel[:, 1:1 + min(nw, 16)]
print("warp done    ", q(wd))
print("warp spread per CTA (max-min)", q(wd.max(1) - wd.min(1)))
print("merged (9)   ", q(rel[:, 20]))
print("fin start(21)", q(rel[:21, 21]))
isf = st[:, 22] > 0
fin = rel[isf, 22]
print("finish (11)  ", q(fin) if fin.size else "-", "finishers", fin.size)
print("finish dur   ", q(rel[isf, 22] - rel[isf, 21]))
print("exit (12)    ", q(rel[:, 23]))
for name, a_, b_ in (("segs->loads", 21, 24), ("loads->tree", 24, 26), ("tree->wait", 26, 27), ("wait->sync", 27, 25), ("sync->done", 25, 22)):
    print(f"{name:18s}", q(rel[isf, b_] - rel[isf, a_]))
order = np.argsort(rel[isf, 21])
print("finisher ticket->finish (sorted by ticket):", [f"{a:.1f}->{b:.1f}" for a, b in zip(rel[isf, 21][order], rel[isf, 22][order])])
print("per-warp-index mean done:", " ".join(f"{x:.2f}" for x in wd.mean(0)))
print("per-CTA mean done, by CTA index deciles:", " ".join(f"{x:.2f}" for x in [wd[i:i+15].mean() for i in range(0, wd.shape[0], 15)]))
start = rel[:, 0]
print("CTA entry spread", q(start))
