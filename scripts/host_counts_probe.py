"""Wall-clock distribution of the host entry point ychg_cut_vertex_counts on a
4096^2 pageable image (the reference acceptance criterion 5 workload), per library
build: python scripts/host_counts_probe.py lib.so [lib2.so ...]"""
import ctypes
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from oracle import Oracle, Spec  # noqa: E402  (input generation only)

orc = Oracle()
imgs = {name: orc.synth(sp) for name, sp in [("hbands1", Spec.hbands(4096, 4096, 1)),
                                            ("hbands2048", Spec.hbands(4096, 4096, 2048)),
                                            ("checker1", Spec.checker(4096, 4096, 1))]}
for lib_path in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(lib_path))
    f = lib.ychg_cut_vertex_counts
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                  ctypes.c_void_p]
    out = np.zeros(4096, np.int32)
    for name, bits in imgs.items():
        b = np.ascontiguousarray(bits)
        ts = []
        for i in range(40):
            t0 = time.perf_counter()
            rc = f(b.ctypes.data, 4096, 4096, 512, 0, 1, out.ctypes.data)
            ts.append((time.perf_counter() - t0) * 1e6)
            assert rc == 0
        ts = ts[5:]
        print(f"{os.path.basename(lib_path)} {name}: median {statistics.median(ts):.0f} us  min {min(ts):.0f}  "
              f"max {max(ts):.0f}  p25 {np.percentile(ts, 25):.0f} p75 {np.percentile(ts, 75):.0f}", flush=True)
