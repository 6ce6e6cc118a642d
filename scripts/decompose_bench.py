"""Device decompose vs the reference's decompose(build_profile(img)) (CPU, serial).
GPU numbers: end-to-end wall time of y.decompose(image) (H2D, profile, decompose,
D2H of all three arrays into pageable memory) and the device time of the
decomposition kernels alone.  Prints one JSON line per image."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1307_2560_b200 as y  # noqa: E402

CASES = [("checker", 21000, 21000, dict(cell=7)), ("hbands", 21000, 21000, dict(bands=147)),
         ("random", 8000, 8000, dict(density=0.5, seed=1307)), ("random", 21000, 21000, dict(density=0.5, seed=1307)),
         ("checker", 21000, 21000, dict(cell=21))]
ref = None
try:
    from oracle import Reference
    ref = Reference()
except Exception as e:  # noqa: BLE001
    print(json.dumps({"reference": "unavailable", "why": str(e)[:200]}))

for pat, w, h, kw in CASES:
    img = y.synth(pat, w, h, **kw)
    y.decompose(img)  # warm-up (allocations)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        hg = y.decompose(img)
        t.append(time.perf_counter() - t0)
    buf = y.HypergraphBuffers(hg.edge_runs.shape[0])
    y.decompose(img, out=buf)
    tp = []
    for _ in range(3):
        t0 = time.perf_counter()
        hgp = y.decompose(img, out=buf)
        tp.append(time.perf_counter() - t0)
    assert np.array_equal(hgp.edge_runs, hg.edge_runs) and np.array_equal(hgp.run_to_edge, hg.run_to_edge)
    row = {"image": f"{pat}{kw} {w}x{h}", "runs": int(hg.edge_runs.shape[0]), "edges": hg.edge_count,
           "gpu_e2e_s": min(t), "gpu_e2e_pinned_out_s": min(tp), "gpu_decompose_kernels_ms": hg.device_ms}
    if ref is not None and hg.edge_runs.shape[0] < 40_000_000:
        ri = ref.image(img.bytes(), w)
        t0 = time.perf_counter()
        d = ri.decompose()
        row["ref_s"] = time.perf_counter() - t0
        row["identical"] = bool(np.array_equal(d.edge_runs, hg.edge_runs) and np.array_equal(d.edge_offsets, hg.edge_offsets)
                                and np.array_equal(d.run_to_edge, hg.run_to_edge))
        row["speedup_e2e"] = row["ref_s"] / row["gpu_e2e_s"]
        row["speedup_e2e_pinned_out"] = row["ref_s"] / row["gpu_e2e_pinned_out_s"]
        buf.close()
    buf.close()
    print(json.dumps(row), flush=True)
