import time, sys, torch, os
sys.path.insert(0, ".")
import paper_1307_2560_b200 as y
W = H = 21000
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
host.copy_(torch.from_numpy(img.bytes()))
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3): r = y.scan(himg)
ts = []
for _ in range(8):
    t0 = time.perf_counter(); r = y.scan(himg); ts.append(time.perf_counter() - t0)
print("e2e scan", [round(t * 1e3, 3) for t in ts])
