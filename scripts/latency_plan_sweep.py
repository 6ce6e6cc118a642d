"""Isolated-scan latency of the host entry point (YCHG_PLAN_LATENCY plans) versus
the segment count: one process per YCHG_SEGMENTS value (plans are cached per
geometry), per-phase device times from YCHG_HOST_TIMING=1.  Usage:
  python scripts/latency_plan_sweep.py [k ...]      (no k: the default plan)"""
import os
import subprocess
import sys

CHILD = r"""
import os, sys, time, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_1307_2560_b200 as y
W = H = int(os.environ.get("SWEEP_SIZE", "21000"))
img = y.synth("hbands", W, H, bands=147)
host = torch.empty((H, (W + 7) // 8), dtype=torch.uint8, pin_memory=True)
host.numpy()[:] = img.bytes().reshape(H, -1)[:, :(W + 7) // 8]
himg = y.BinaryImage(W, H, host.numpy())
for _ in range(3):
    y.scan(himg)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); r = y.scan(himg); ts.append(time.perf_counter() - t0)
print("e2e_ms", round(statistics.median(ts) * 1e3, 3), "hyperedges", r.hyperedges, flush=True)
"""

ks = sys.argv[1:] or [""]
for k in ks:
    env = dict(os.environ, YCHG_HOST_TIMING="1")
    if k:
        env["YCHG_SEGMENTS"] = k
    p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    lines = [l for l in p.stderr.splitlines() if l.startswith("[ychg host]")]
    scan_us = sorted(float(l.split("scan ")[1].split(" us")[0]) for l in lines[-15:]) if lines else []
    med = scan_us[len(scan_us) // 2] if scan_us else None
    print(f"k={k or 'default'} {p.stdout.strip()} isolated scan median {med} us  (rc {p.returncode})", flush=True)
    if p.returncode:
        print(p.stderr[-2000:])
