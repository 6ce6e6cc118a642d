"""GPU parity at the BASELINE configs, element-wise (SURVEY §8c large-scale plan):

* 21000^2 hbands(147) and random(0.5, 1307) -- BASELINE config 2 -- with the
  default plan (the bench's own launch shape), the unchanged-block skip on and off,
  and the host entry point; counts and boundaries against the reference compiled
  from /root/reference (oracle/_ref: cut_vertex_counts(parallel(nproc)) +
  detect_boundary_columns, runscan.cpp:122-153), hyperedges against the
  reference's hyperedge_count(decompose(build_profile)) (hypergraph.cpp:94-192)
  where it fits (hbands) and otherwise against the C restatements pinned to it;
* 65536^2 random(0.5, 1307) -- BASELINE config 5's mask on one GPU -- counts and
  boundaries against the reference, hyperedges against the C a7 restatement
  (decompose would need tens of GB here; tests/test_oracle.py pins the
  restatement to decompose);
* the N=2 column-strip path of bench.py (multigpu.py, K0 with a global column
  offset, all-gather + all-reduce + K2 over the gathered counts) on one GPU over
  gloo, checked by bench.py's own parity block and against the one-GPU scan.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import Spec

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NPROC = os.cpu_count() or 1


def device_image(y, torch, pattern, W, H, **kw):
    pitch = y.pitch_for(W)
    d = torch.empty((H, pitch), dtype=torch.uint8, device="cuda")
    y.synth_device(pattern, W, H, d.data_ptr(), pitch, **kw)
    torch.cuda.synchronize()
    return d, pitch


def scan_plan(y, torch, d, pitch, W, H, skip=True, links=True):
    c = torch.full((W,), -7, dtype=torch.int32, device="cuda")
    f = torch.zeros(y.boundary_flag_words(W), dtype=torch.int32, device="cuda")
    b = torch.full((W,), -7, dtype=torch.int32, device="cuda")
    t = torch.zeros(4, dtype=torch.int64, device="cuda")
    plan = y.Plan(W, H, skip=skip)
    for _ in range(2):  # the second scan runs on a warm plan (tickets, parity halves)
        plan.scan_device(d.data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(), t.data_ptr(),
                         torch.cuda.current_stream().cuda_stream, links)
    torch.cuda.synchronize()
    tt = t.cpu().tolist()
    plan.close()
    return c.cpu().numpy(), b.cpu().numpy()[: tt[3]], tt


@pytest.mark.parametrize("pattern", ["hbands", "random"])
def test_21000_baseline_config_elementwise(gpu, orc, ref, pattern):
    import torch
    y = gpu
    W = H = 21000
    kw = dict(bands=147) if pattern == "hbands" else dict(density=0.5, seed=1307)
    sp = Spec.hbands(W, H, 147) if pattern == "hbands" else Spec.random(W, H, 0.5, 1307)
    d, pitch = device_image(y, torch, pattern, W, H, **kw)
    bits = d[:, : (W + 7) // 8].cpu().numpy()
    assert np.array_equal(bits, orc.synth(sp)), "K0 synth != reference synth restatement"
    rimg = ref.image(bits, W)
    want_c = rimg.counts(1, NPROC)                      # reference cut_vertex_counts(parallel(nproc))
    want_b = ref.boundaries(want_c)                     # reference detect_boundary_columns
    runs = int(want_c.astype(np.int64).sum())
    if pattern == "hbands":
        want_he = rimg.hyperedges(1, NPROC)             # reference hyperedge_count(decompose(build_profile))
        assert want_he == 147
    else:
        want_he, oruns, olinks = orc.hyperedges(bits, W)  # decompose restatement (pinned, test_oracle.py)
        assert oruns == runs and runs - orc.a7_links(bits, W) == want_he
    for skip in (True, False):
        c, b, t = scan_plan(y, torch, d, pitch, W, H, skip=skip)
        assert np.array_equal(c, want_c), (pattern, skip)
        assert np.array_equal(b, want_b), (pattern, skip)
        assert t == [runs, runs - want_he, want_he, want_b.size], (pattern, skip)
    c2, b2, t2 = scan_plan(y, torch, d, pitch, W, H, links=False)
    assert np.array_equal(c2, want_c) and np.array_equal(b2, want_b) and t2[2] == -1
    r = y.scan(y.BinaryImage(W, H, bits))               # host entry point (pageable rows)
    assert np.array_equal(r.counts, want_c) and np.array_equal(r.boundaries, want_b)
    assert (r.total_runs, r.hyperedges) == (runs, want_he)


def test_65536_random_elementwise(gpu, orc, ref):
    import torch
    y = gpu
    W = H = 65536
    d, pitch = device_image(y, torch, "random", W, H, density=0.5, seed=1307)
    bits = d[:, : W // 8].cpu().numpy()
    assert np.array_equal(bits, orc.synth(Spec.random(W, H, 0.5, 1307))), "K0 synth != reference synth restatement"
    want_c = ref.image(bits, W).counts(1, NPROC)
    want_b = ref.boundaries(want_c)
    runs = int(want_c.astype(np.int64).sum())
    links = orc.a7_links(bits, W)
    c, b, t = scan_plan(y, torch, d, pitch, W, H)
    assert np.array_equal(c, want_c)
    assert np.array_equal(b, want_b)
    assert t == [runs, links, runs - links, want_b.size]


@pytest.mark.parametrize("width,pattern", [(5000, "random"), (8192, "hbands")])
def test_bench_two_rank_strip_path_on_one_gpu(gpu, orc, width, pattern):
    """bench.py --gpus 2 under torch.distributed.run with both ranks on cuda:0
    (YCHG_BENCH_SHARE_GPU=1, gloo): unequal strips at 5000 columns, K0 strips with
    a global column offset, the exchange and K2 over the gathered counts; its parity
    block (vs the reference) must hold and its totals equal the one-GPU scan's."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, YCHG_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--size", str(width), "--steps", "3", "--warmup", "1", "--pattern", pattern, "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    p = line["parity"]
    assert p["counts_sha256_match"] and p["boundaries_match"] and p["hyperedges_match"], p
    sp = Spec.random(width, width, 0.5, 1307) if pattern == "random" else Spec.hbands(width, width, 147)
    bits = orc.synth(sp)
    r = gpu.scan(gpu.BinaryImage(width, width, bits))
    assert line["totals"] == {"total_runs": r.total_runs, "links": r.links, "hyperedges": r.hyperedges,
                              "n_boundaries": int(r.boundaries.size)}
    assert line["config"]["strip_width_per_gpu"] in (2048, 2952, 4096)
