"""One device decompose per workload at 21000^2 (for an ncu launch list of the
profile + decomposition kernels): python scripts/decompose_launches.py [pattern...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1307_2560_b200 as y  # noqa: E402

CASES = {"checker7": ("checker", dict(cell=7)), "random": ("random", dict(density=0.5, seed=1307)),
         "hbands": ("hbands", dict(bands=147)), "checker21": ("checker", dict(cell=21))}
for name in sys.argv[1:] or list(CASES):
    pat, kw = CASES[name]
    img = y.synth(pat, 21000, 21000, **kw)
    hg = y.decompose(img)
    d = hashlib.sha1(np.ascontiguousarray(hg.edge_runs).tobytes() + np.ascontiguousarray(hg.run_to_edge).tobytes()
                     + np.ascontiguousarray(hg.edge_offsets).tobytes()).hexdigest()[:16]
    print(name, hg.edge_offsets.shape[0] - 1, d, flush=True)
