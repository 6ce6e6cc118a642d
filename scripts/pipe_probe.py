"""Distinct images, full/counts-only interleaved, each scan into its own outputs:
graph vs eager; prints every scan whose totals differ from the oracle."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1307_2560_b200 as y  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
pattern = sys.argv[2] if len(sys.argv) > 2 else "mix"   # mix: every third scan counts-only; full: all full
orc = Oracle()
W, H = 3100, 2600
specs = [Spec.random(W, H, 0.5, 21), Spec.hbands(W, H, 40), Spec.checker(W, H, 5), Spec.random(W, H, 0.3, 22),
         Spec.frame(W, H)]
pitch = y.pitch_for(W)
imgs = []
for sp in specs:
    bits = orc.synth(sp)
    dev = np.zeros((H, pitch), np.uint8)
    dev[:, : bits.shape[1]] = bits
    he, runs, links = orc.hyperedges(bits, W)
    imgs.append((torch.from_numpy(dev).cuda(), he, runs, links))
plan = y.Plan(W, H)
print("plan", plan.info().grid, plan.info().seg_per_strip, flush=True)
n = 24
full = [(i % 3 != 2) if pattern == "mix" else True for i in range(n)]
outs = [(torch.full((W,), -7, dtype=torch.int32, device="cuda"), torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda"),
         torch.full((W,), -7, dtype=torch.int32, device="cuda"), torch.zeros(4, dtype=torch.int64, device="cuda"))
        for _ in range(n)]
stream = torch.cuda.current_stream()


def launch(cs):
    for i in range(n):
        c, f, b, t = outs[i]
        plan.scan_device(imgs[i % len(imgs)][0].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(),
                         t.data_ptr(), cs, full[i])


if mode == "graph":
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            launch(torch.cuda.current_stream().cuda_stream)
    stream.wait_stream(cap)
for rep in range(3):
    if mode == "graph":
        g.replay()
    else:
        launch(stream.cuda_stream)
    torch.cuda.synchronize()
    bad = []
    for i in range(n):
        _, he, runs, links = imgs[i % len(imgs)]
        tt = outs[i][3].cpu().tolist()
        want = [runs, links if full[i] else 0, he if full[i] else -1]
        if tt[:3] != want:
            bad.append((i, i % len(imgs), tt[:3], want))
    print(mode, pattern, "rep", rep, "bad", len(bad), bad[:6], flush=True)
