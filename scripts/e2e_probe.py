import time, torch, numpy as np, os, sys
sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y
W=H=21000
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W+7)//8), dtype=torch.uint8, pin_memory=True)
host.numpy()[:] = img.bytes().reshape(H, -1)[:, :(W+7)//8]
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3): y.scan(himg)
ts=[]
for _ in range(10):
    t0=time.perf_counter(); r=y.scan(himg); ts.append(time.perf_counter()-t0)
print("scan e2e ms", sorted(ts)[5]*1e3, r.hyperedges)
dev = torch.empty_like(host, device="cuda")
fl=[]
for _ in range(10):
    torch.cuda.synchronize(); t0=time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize(); fl.append(time.perf_counter()-t0)
print("copy floor ms", sorted(fl)[5]*1e3)
# two half copies
fl=[]
for _ in range(10):
    torch.cuda.synchronize(); t0=time.perf_counter(); dev[:H//2].copy_(host[:H//2], non_blocking=True); dev[H//2:].copy_(host[H//2:], non_blocking=True); torch.cuda.synchronize(); fl.append(time.perf_counter()-t0)
print("2-chunk copy ms", sorted(fl)[5]*1e3)
