"""One build_profile per workload (for an ncu launch list of profile_fill_kernel);
YCHG_LIB selects the library build; the printed profile digests must agree
across builds."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1307_2560_b200 as y  # noqa: E402

for pat, w, h, kw in [("checker", 21000, 21000, dict(cell=7)), ("random", 21000, 21000, dict(density=0.5, seed=1307)),
                      ("hbands", 21000, 21000, dict(bands=147)), ("checker", 21000, 21000, dict(cell=21))]:
    img = y.synth(pat, w, h, **kw)
    prof = y.build_profile(img)
    runs = np.ascontiguousarray(prof.runs_flat)
    print(pat, runs.shape, hashlib.sha1(runs.tobytes()).hexdigest()[:16], flush=True)
