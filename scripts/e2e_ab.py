"""A/B of the host entry point's end-to-end time between two builds of
libychg_b200.so (YCHG_LIB), alternating processes on one box.
  python scripts/e2e_ab.py <libA.so> <libB.so> [rounds] [size]"""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, time, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y
W = H = int(os.environ.get("AB_SIZE", "21000"))
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
host.numpy()[:] = img.bytes().reshape(H, -1)[:, :(W + 7) // 8]
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3):
    y.scan(himg)
ts = []
for _ in range(40):
    t0 = time.perf_counter(); r = y.scan(himg); ts.append(time.perf_counter() - t0)
ts.sort()
dev = torch.empty_like(host, device="cuda")
fl = []
for _ in range(40):
    torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
    fl.append(time.perf_counter() - t0)
fl.sort()
print(f"median {ts[20]*1e3:.3f} ms  p10 {ts[4]*1e3:.3f}  copy floor median {fl[20]*1e3:.3f}  HE {r.hyperedges}")
"""
a, b = sys.argv[1], sys.argv[2]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
size = sys.argv[4] if len(sys.argv) > 4 else "21000"
for i in range(rounds):
    for lib in (a, b):
        env = dict(os.environ, YCHG_LIB=os.path.abspath(lib), AB_SIZE=size)
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        print(f"{os.path.basename(lib):28s} {size}: {p.stdout.strip() or p.stderr[-500:]}", flush=True)
