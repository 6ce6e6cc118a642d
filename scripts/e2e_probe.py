import time, sys, torch
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y
W = H = 21000
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
host.copy_(torch.from_numpy(img.bytes()))
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3): r = y.scan(himg)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); r = y.scan(himg); ts.append(time.perf_counter() - t0)
print("e2e scan median %.3f ms min %.3f ms  HE %d" % (sorted(ts)[7] * 1e3, min(ts) * 1e3, r.hyperedges))
ts = []
for _ in range(15):
    t0 = time.perf_counter(); c = y.cut_vertex_counts(himg); ts.append(time.perf_counter() - t0)
print("e2e counts median %.3f ms" % (sorted(ts)[7] * 1e3))
