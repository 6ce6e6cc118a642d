"""Pipeline fill/drain of a short CUDA-graph burst (K=4 scans after an idle GPU):
per scan, streaming CTAs' entry / exit spread and the finisher's completion,
relative to the first CTA entry of scan 0 (per-CTA %globaltimer stamps)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402

W = H = 21000
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4   # with K > 4 the stamp ring holds the last 4 scans
links = not (len(sys.argv) > 2 and sys.argv[2] == "counts")
torch.cuda.set_device(0)
pitch = y.pitch_for(W)
bufs = [torch.empty((H, pitch), dtype=torch.uint8, device="cuda") for _ in range(min(K, 8))]
for b in bufs:
    y.synth_device("hbands", W, H, b.data_ptr(), pitch, bands=147)
c = torch.empty(W, dtype=torch.int32, device="cuda"); f = torch.empty(W // 32 + 64, dtype=torch.int32, device="cuda")
bd = torch.empty(W, dtype=torch.int32, device="cuda"); t = torch.zeros(4, dtype=torch.int64, device="cuda")
plan = y.Plan(W, H)
info = plan.info()
plan.debug_stamps(True)
g = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
with torch.cuda.stream(cap):
    with torch.cuda.graph(g, stream=cap):
        s = torch.cuda.current_stream().cuda_stream
        for i in range(K):
            plan.scan_device(bufs[i % len(bufs)].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), bd.data_ptr(), t.data_ptr(), s, links)
torch.cuda.synchronize()
for rep in range(3):
    g.replay()
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    st = plan.debug_stamps(True).astype(np.float64)
    G = info.grid
    nS = info.n_strips
    base = None
    rows = []
    for sc in range(max(0, K - 4), K):
        e = st[sc % 4]
        ent = e[:G, 0]
        ext = e[:G, 23]
        fin = e[:nS, 22]
        pub = e[:G, 20]
        if base is None:
            base = ent.min()
        fs = [(e[:nS, j].max() - base) / 1e3 for j in (21, 24, 26, 27, 25, 22)]
        life = np.median(ext - ent) / 1e3
        rows.append((sc, life, (ent.min() - base) / 1e3, (ent.max() - base) / 1e3, (np.median(ext) - base) / 1e3,
                     (ext.max() - base) / 1e3, (pub.max() - base) / 1e3, *fs))
    print(f"rep {rep}: graph {e0.elapsed_time(e1) * 1e3:.1f} us (K={K})")
    for r in rows:
        print("  scan %d: CTA life med %5.1f | entry %6.1f..%6.1f  exit med %6.1f max %6.1f | last publish %6.1f | finisher (max over strips)"
              " seen %6.1f loads %6.1f k3 %6.1f lookback %6.1f outputs %6.1f done %6.1f" % r)
