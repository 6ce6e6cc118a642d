"""Long randomized stress of the pipelined scan (not part of the test suite):
random geometries, segment counts and grids, latency / default plans, the
unchanged-block skip on and off, random / banded / checker content; CUDA graphs
of back-to-back scans of distinct images, full and counts-only mixed; every
output checked against the oracle; a stall aborts after 20 s.  Usage: python scripts/pipeline_stress.py [trials] [seed]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
orc = Oracle()
t_start = time.time()
for trial in range(trials):
    W = int(rng.choice([1, 7, 31, 32, 33, 1023, 1024, 1025, 2048, 2049, 3000, 4096, 5000, 9000]))
    H = int(rng.choice([1, 2, 31, 32, 33, 63, 64, 65, 257, 1000, 2500, 4000]))
    os.environ["YCHG_SEGMENTS"] = str(int(rng.integers(1, 12)))
    os.environ["YCHG_GRID"] = str(int(rng.choice([1, 2, 3, 5, 1000])))
    def pick():
        kind = int(rng.integers(0, 4))
        if kind == 1 and H >= 2:
            return Spec.hbands(W, H, int(rng.integers(1, max(2, H // 2 + 1))))
        if kind == 2:
            return Spec.checker(W, H, int(rng.choice([1, 3, 7, 33, 100])))
        return Spec.random(W, H, float(rng.choice([0.05, 0.3, 0.5, 0.7, 0.95])), int(rng.integers(0, 1 << 40)))
    specs = [pick() for _ in range(3)]
    pitch = y.pitch_for(W)
    imgs = []
    for sp in specs:
        bits = orc.synth(sp)
        dev = np.zeros((H, pitch), np.uint8)
        dev[:, : bits.shape[1]] = bits
        counts = orc.counts(bits, W)
        imgs.append((torch.from_numpy(dev).cuda(), counts, orc.boundaries(counts), orc.hyperedges(bits, W)[0]))
    try:
        plan = y.Plan(W, H, latency=bool(rng.integers(0, 2)), skip=bool(rng.integers(0, 4)))
    except y.ValidationError:
        continue  # e.g. more segments per CTA than supported with a tiny forced grid
    n = int(rng.integers(2, 13))
    full = [bool(rng.integers(0, 2)) for _ in range(n)]
    outs = [(torch.full((W,), -7, dtype=torch.int32, device="cuda"), torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda"),
             torch.full((W,), -7, dtype=torch.int32, device="cuda"), torch.zeros(4, dtype=torch.int64, device="cuda"))
            for _ in range(n)]
    stream = torch.cuda.current_stream()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            cs = torch.cuda.current_stream().cuda_stream
            for i in range(n):
                c, f, b, t = outs[i]
                plan.scan_device(imgs[i % 3][0].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(),
                                 t.data_ptr(), cs, full[i])
    stream.wait_stream(cap)
    for rep in range(int(rng.integers(1, 4))):
        g.replay()
        t0 = time.time()
        while not stream.query():
            if time.time() - t0 > 20:
                print(f"STALL trial {trial}: {W}x{H} seg={os.environ['YCHG_SEGMENTS']} grid={os.environ['YCHG_GRID']}",
                      flush=True)
                os._exit(3)
            time.sleep(0.002)
    for i in range(n):
        c, _, b, t = outs[i]
        _, counts, bounds, he = imgs[i % 3]
        tt = t.cpu().tolist()
        ok = (np.array_equal(c.cpu().numpy(), counts) and tt[3] == bounds.size
              and np.array_equal(b.cpu().numpy()[: bounds.size], bounds) and tt[2] == (he if full[i] else -1))
        if not ok:
            print(f"MISMATCH trial {trial} scan {i}: {W}x{H} seg={os.environ['YCHG_SEGMENTS']} "
                  f"grid={os.environ['YCHG_GRID']} full={full[i]} got {tt} want he={he}", flush=True)
            os._exit(4)
    plan.close()
print(f"pipeline stress: {trials} trials ok in {time.time() - t_start:.0f} s", flush=True)
