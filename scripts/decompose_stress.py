"""Randomized stress of the device decompose / build_profile vs the oracle (not part
of the test suite).  Usage: python scripts/decompose_stress.py [trials] [seed]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1307_2560_b200 as y  # noqa: E402
from oracle import Oracle, Spec  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
orc = Oracle()
t0 = time.time()
for t in range(trials):
    W, H = int(rng.integers(1, 3000)), int(rng.integers(1, 1500))
    kind = int(rng.integers(0, 4))
    if kind == 0:
        sp = Spec.random(W, H, float(rng.choice([0.02, 0.2, 0.5, 0.8, 0.98])), int(rng.integers(0, 1 << 40)))
    elif kind == 1 and H >= 2:
        sp = Spec.hbands(W, H, int(rng.integers(1, H // 2 + 1)))
    elif kind == 2:
        sp = Spec.checker(W, H, int(rng.integers(1, 40)))
    else:
        sp = Spec.frame(W, H)
    bits = orc.synth(sp)
    img = y.BinaryImage(W, H, bits)
    prof = y.build_profile(img)
    want_p = orc.profile(bits, W)
    if not np.array_equal(prof.runs_flat, want_p):
        print("PROFILE MISMATCH", t, sp, flush=True)
        sys.exit(3)
    got = y.decompose(img)
    want = orc.decompose(bits, W)
    if not (np.array_equal(got.edge_runs, want.edge_runs) and np.array_equal(got.edge_offsets, want.edge_offsets)
            and np.array_equal(got.run_to_edge, want.run_to_edge)):
        print("DECOMPOSE MISMATCH", t, sp, flush=True)
        sys.exit(4)
    if got.edge_count != y.scan(img).hyperedges:
        print("K3 vs decompose MISMATCH", t, sp, flush=True)
        sys.exit(5)
print(f"decompose stress: {trials} trials ok in {time.time() - t0:.0f} s", flush=True)
