"""GPU parity: the sm_100a path, called through the C ABI, against the oracle and
the reference golden fixtures.  Bit-exact for everything (integer work)."""
import hashlib
import os
import subprocess

import numpy as np
import pytest

from golden_io import acceptance2, corpus, large, spec_of
from oracle import Spec, branch_example

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAT = {0: "full", 1: "empty", 2: "frame", 3: "hbands", 4: "checker", 5: "random"}


def sha(a):
    return hashlib.sha256(np.asarray(a, dtype="<i4").tobytes()).hexdigest()


def image(y, orc, sp):
    return y.BinaryImage(sp.width, sp.height, orc.synth(sp))


def test_known_answers(gpu):
    y = gpu
    assert y.cut_vertex_counts(y.synth("full", 4, 4)).tolist() == [1, 1, 1, 1]
    assert y.cut_vertex_counts(y.synth("frame", 5, 5)).tolist() == [1, 2, 2, 2, 1]
    assert y.cut_vertex_counts(y.BinaryImage(3, 3)).tolist() == [0, 0, 0]
    br = y.BinaryImage(2, 7, branch_example())
    assert y.cut_vertex_counts(br).tolist() == [2, 2]
    assert y.cut_vertex_counts(y.BinaryImage(0, 0)).tolist() == []
    assert y.cut_vertex_counts(y.synth("hbands", 8, 11, bands=3)).tolist() == [3] * 8
    for counts, want in [([1, 2, 2, 2, 1], [0, 1, 4]), ([0, 0, 0], []), ([], []), ([0, 1], [1]), ([3], [0]),
                         ([2, 2], [0])]:
        assert y.detect_boundary_columns(counts).tolist() == want
    r = y.scan(br)
    assert (r.counts.tolist(), r.boundaries.tolist(), r.hyperedges) == ([2, 2], [0], 4)
    f = y.scan(y.synth("frame", 5, 5))
    assert (f.boundaries.tolist(), f.hyperedges, f.total_runs) == ([0, 1, 4], 4, 8)


def test_strategies_identical_and_validated(gpu, orc):
    y = gpu
    img = image(y, orc, Spec.random(3, 50, 0.5, 8))
    base = y.cut_vertex_counts(img, y.ScanStrategy.serial())
    for t in (1, 2, 4, 8, 16):
        assert np.array_equal(y.cut_vertex_counts(img, y.ScanStrategy.parallel(t)), base)
    with pytest.raises(y.ValidationError):
        y.cut_vertex_counts(img, y.ScanStrategy.parallel(0))


@pytest.mark.parametrize("small", ["1", "0"])
def test_small_image_kernel_vs_oracle(gpu, orc, monkeypatch, small):
    """One-off scans of images of one strip and <= 512 rows take the single-CTA
    kernel (YCHG_NO_SMALL=1 forces the pipelined one): both against the oracle at
    its geometry edges -- 1 row / 1 column, widths off the byte and word, exactly
    1024 columns / 512 rows, one past them (pipelined), every pattern, counts-only."""
    y = gpu
    monkeypatch.setenv("YCHG_NO_SMALL", "0" if small == "1" else "1")
    geoms = [(1, 1), (7, 3), (8, 512), (9, 1), (31, 33), (32, 64), (33, 511), (513, 257), (1000, 500),
             (1023, 512), (1024, 512), (1024, 1), (1025, 100), (600, 513)]
    rng = np.random.default_rng(77)
    for w, h in geoms:
        specs = [Spec.random(w, h, float(rng.choice([0.1, 0.5, 0.9])), int(rng.integers(0, 1 << 62))),
                 Spec.checker(w, h, int(rng.integers(1, 9)))]
        if h >= 2:
            specs.append(Spec.hbands(w, h, min(147, h // 2)))
        for sp in specs:
            bits = orc.synth(sp)
            img = y.BinaryImage(w, h, bits)
            r = y.scan(img)
            c = orc.counts(bits, w)
            assert np.array_equal(r.counts, c), sp
            assert np.array_equal(r.boundaries, orc.boundaries(c)), sp
            assert r.hyperedges == orc.hyperedges(bits, w)[0], sp
            assert np.array_equal(y.cut_vertex_counts(img), c), sp


def test_golden_corpus(gpu, orc):
    y = gpu
    for row in corpus():
        sp = spec_of(row["spec"])
        r = y.scan(image(y, orc, sp))
        assert r.counts.tolist() == row["counts"], row["name"]
        assert r.boundaries.tolist() == row["boundaries"], row["name"]
        assert r.hyperedges == row["hyperedges"], row["name"]
        assert r.total_runs == sum(row["counts"]), row["name"]


def test_counts_only_path_matches(gpu, orc):
    y = gpu
    for row in corpus()[::11]:
        sp = spec_of(row["spec"])
        assert y.cut_vertex_counts(image(y, orc, sp)).tolist() == row["counts"], row["name"]


def test_byte_boundary_widths(gpu, orc):
    # test_runscan.cpp:51-64 widths, plus word/strip edges of the GPU layout
    y = gpu
    for w in (1, 7, 8, 9, 16, 17, 31, 32, 33, 63, 64, 65, 70, 1023, 1024, 1025, 1031, 2047, 2049):
        for seed in (5, 6):
            sp = Spec.random(w, 33, 0.5, seed)
            bits = orc.synth(sp)
            r = y.scan(y.BinaryImage(w, 33, bits))
            c = orc.counts(bits, w)
            assert np.array_equal(r.counts, c), w
            assert np.array_equal(r.boundaries, orc.boundaries(c)), w
            assert r.hyperedges == orc.hyperedges(bits, w)[0], w


def test_acceptance2_512(gpu, orc):
    y = gpu
    for row in acceptance2():
        sp = spec_of(row["spec"])
        r = y.scan(image(y, orc, sp))
        assert sha(r.counts) == row["counts_sha256"]
        assert r.boundaries.size == row["n_boundaries"]
        assert r.hyperedges == row["hyperedges"]


@pytest.mark.parametrize("idx", range(10))
def test_large_golden(gpu, orc, idx):
    y = gpu
    row = large()[idx]
    sp = spec_of(row["spec"])
    dev = y.synth(PAT[sp.pattern], sp.width, sp.height, bands=sp.bands, cell=sp.cell, density=sp.density,
                  seed=sp.seed)
    r = y.scan(dev)
    assert sha(r.counts) == row["counts_sha256"]
    assert sha(r.boundaries) == row["boundaries_sha256"]
    assert r.n_boundaries == row["n_boundaries"]
    assert r.hyperedges == row["hyperedges"]
    assert r.total_runs == row["total_runs"]


def test_random_geometries_vs_oracle(gpu, orc):
    y = gpu
    rng = np.random.default_rng(2024)
    for _ in range(60):
        w, h = int(rng.integers(1, 5000)), int(rng.integers(1, 700))
        sp = Spec.random(w, h, float(rng.choice([0.05, 0.3, 0.5, 0.8, 0.97])), int(rng.integers(0, 1 << 62)))
        bits = orc.synth(sp)
        r = y.scan(y.BinaryImage(w, h, bits))
        c = orc.counts(bits, w)
        assert np.array_equal(r.counts, c), sp
        assert np.array_equal(r.boundaries, orc.boundaries(c)), sp
        assert r.hyperedges == orc.hyperedges(bits, w)[0], sp


def test_device_synth_bit_exact(gpu, orc):
    y = gpu
    for sp in [Spec.random(1001, 77, 0.37, 123456789), Spec.random(64, 64, 1.0, 3), Spec.random(64, 64, 0.0, 3),
               Spec.hbands(333, 100, 7), Spec.checker(129, 65, 3), Spec.frame(17, 9), Spec.full(9, 3),
               Spec.empty(40, 4)]:
        d = y.synth(PAT[sp.pattern], sp.width, sp.height, bands=sp.bands, cell=sp.cell, density=sp.density,
                    seed=sp.seed)
        assert np.array_equal(d.bytes(), orc.synth(sp)), sp
    with pytest.raises(y.ValidationError):
        y.synth("hbands", 10, 10, bands=6)


def test_garbage_padding_bits_ignored(gpu, orc):
    # counts never look at columns >= W (runscan.cpp:41-74); neither may the pair step
    y = gpu
    sp = Spec.random(37, 64, 0.5, 77)
    bits = orc.synth(sp)
    dirty = bits.copy()
    dirty[:, -1] |= 0x07  # the 3 padding bits of the last byte
    r = y.scan(y.BinaryImage(37, 64, dirty))
    c = orc.counts(bits, 37)
    assert np.array_equal(r.counts, c)
    assert r.hyperedges == orc.hyperedges(bits, 37)[0]


def test_device_api_and_halo_strips(gpu, orc):
    """Column strips with a right halo (multi-GPU layout) computed through ychg_scan_device."""
    y = gpu
    W, H = 5000, 900
    bits = orc.synth(Spec.random(W, H, 0.5, 4242))
    counts = orc.counts(bits, W)
    pair = orc.pair_links(bits, W)
    bounds = [0, 2048, 3072, W]
    total_links = 0
    for i in range(3):
        c0, c1 = bounds[i], bounds[i + 1]
        halo = 8 if c1 < W else 0
        wimg = (c1 - c0) + halo
        sub = np.unpackbits(bits, axis=1)[:, c0:c0 + wimg]
        sub = np.packbits(sub, axis=1)
        pitch = y.pitch_for(wimg)
        dev = np.zeros((H, pitch), np.uint8)
        dev[:, : sub.shape[1]] = sub
        dbits = y.DeviceBuffer(dev.nbytes)
        dbits.from_host(dev)
        n = c1 - c0
        dc, df, db = y.DeviceBuffer(4 * n), y.DeviceBuffer(4 * ((n + 31) // 32 + 32)), y.DeviceBuffer(4 * n)
        dt = y.DeviceBuffer(32)
        plan = y.Plan(wimg, H, width_cnt=n)
        plan.scan_device(dbits.ptr, pitch, dc.ptr, df.ptr, db.ptr, dt.ptr)
        got = dc.to_host(np.zeros(n, np.int32))
        tot = dt.to_host(np.zeros(4, np.int64))
        assert np.array_equal(got, counts[c0:c1])
        assert tot[0] == counts[c0:c1].sum()
        assert tot[1] == pair[c0:c1].sum()
        total_links += int(tot[1])
        plan.close()
    assert counts.sum() - total_links == orc.hyperedges(bits, W)[0]


def test_timing_hooks(gpu):
    y = gpu
    W = H = 2048
    pitch = y.pitch_for(W)
    d = y.DeviceBuffer(pitch * H)
    y.synth_device("random", W, H, d.ptr, pitch, density=0.5, seed=1)
    dc, df, db, dt = y.DeviceBuffer(4 * W), y.DeviceBuffer(4 * (W // 32 + 64)), y.DeviceBuffer(4 * W), y.DeviceBuffer(32)
    plan = y.Plan(W, H)
    plan.set_timing(True)
    plan.scan_device(d.ptr, pitch, dc.ptr, df.ptr, db.ptr, dt.ptr)
    a, b = plan.last_ms()
    assert a > 0 and b == 0.0  # one kernel per scan (the strip finish is fused)
    info = plan.info()
    assert info.kernels_per_scan == 1 and info.grid >= 1


def test_cxx_dropin_binary(gpu, ref):
    """The reference's test_runscan.cpp vectors through the C++ drop-in, and its
    ValidationError::what() texts equal to the live reference's (runscan.cpp:25-26,
    105-107): no prefix added by the shim."""
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    ours = dict(ln.split("\t")[1:3] for ln in out.stdout.splitlines() if ln.startswith("WHAT\t"))
    full3 = ref.image(np.full((50, 1), 0xE0, np.uint8), 3)
    full4 = ref.image(np.full((4, 1), 0xF0, np.uint8), 4)

    def ref_what(fn):
        with pytest.raises(ValueError) as e:
            fn()
        return str(e.value)

    want = {"parallel0": ref_what(lambda: full3.counts(1, 0)),
            "parallel-2": ref_what(lambda: full3.counts(1, -2)),
            "column_runs4": ref_what(lambda: full4.column_runs(4)),
            "column_runs-1": ref_what(lambda: full4.column_runs(-1))}
    assert want["parallel0"] == "scan: parallel strategy needs threads >= 1, got 0"
    assert want["column_runs4"] == "column_runs: column 4 out of range [0, 4)"
    for k, v in want.items():
        assert ours[k] == v, (k, ours[k], v)
    assert ours["build_profile_parallel0"] == want["parallel0"]


def test_back_to_back_scans_pipelined(gpu, orc):
    """Consecutive scans on one plan overlap (programmatic dependent launch): each
    scan's finisher runs while the next scan streams.  Launch a burst with no host
    synchronisation, each scan into its own outputs, then check every one."""
    import torch

    y = gpu
    W, H = 3000, 700
    specs = [Spec.random(W, H, 0.5, 11), Spec.hbands(W, H, 50), Spec.checker(W, H, 3), Spec.random(W, H, 0.2, 12)]
    pitch = y.pitch_for(W)
    imgs = []
    for sp in specs:
        bits = orc.synth(sp)
        dev = np.zeros((H, pitch), np.uint8)
        dev[:, : bits.shape[1]] = bits
        imgs.append((torch.from_numpy(dev).cuda(), bits))
    plan = y.Plan(W, H)
    outs = []
    stream = torch.cuda.current_stream().cuda_stream
    for rep in range(3):
        for i, (d, _) in enumerate(imgs):
            c = torch.full((W,), -7, dtype=torch.int32, device="cuda")
            f = torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda")
            b = torch.full((W,), -7, dtype=torch.int32, device="cuda")
            t = torch.zeros(4, dtype=torch.int64, device="cuda")
            plan.scan_device(d.data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(), t.data_ptr(), stream)
            outs.append((i, c, b, t))
    torch.cuda.synchronize()
    for i, c, b, t in outs:
        bits = imgs[i][1]
        counts = orc.counts(bits, W)
        bounds = orc.boundaries(counts)
        he = orc.hyperedges(bits, W)[0]
        tt = t.cpu().tolist()
        assert np.array_equal(c.cpu().numpy(), counts), i
        assert tt[3] == bounds.size and np.array_equal(b.cpu().numpy()[: bounds.size], bounds), i
        assert tt[2] == he, i
    plan.close()


def test_build_profile_known_answers(gpu):
    y = gpu
    fr = y.build_profile(y.synth("frame", 5, 5))
    assert fr.counts.tolist() == [1, 2, 2, 2, 1]
    assert fr.runs(0).tolist() == [[0, 0, 4]]
    assert fr.runs(2).tolist() == [[2, 0, 0], [2, 4, 4]]
    assert fr.total_runs() == 8
    br = y.BinaryImage(2, 7, branch_example())
    assert y.build_profile(br, y.ScanStrategy.parallel(4)).runs_flat.tolist() == [[0, 0, 1], [0, 3, 6], [1, 0, 4],
                                                                                 [1, 6, 6]]
    assert y.column_runs(br, 1).tolist() == [[1, 0, 4], [1, 6, 6]]
    assert y.column_runs(y.BinaryImage(3, 3), 0).tolist() == []
    with pytest.raises(y.ValidationError):
        y.column_runs(y.synth("full", 4, 4), 4)
    with pytest.raises(y.ValidationError):
        y.column_runs(y.synth("full", 4, 4), -1)
    with pytest.raises(y.ValidationError):
        y.build_profile(br, y.ScanStrategy.parallel(0))


def test_build_profile_golden_corpus(gpu, orc):
    y = gpu
    for row in corpus():
        sp = spec_of(row["spec"])
        bits = orc.synth(sp)
        p = y.build_profile(y.BinaryImage(sp.width, sp.height, bits))
        assert p.counts.tolist() == row["counts"], row["name"]
        assert np.array_equal(p.runs_flat, orc.profile(bits, sp.width)), row["name"]


def test_build_profile_invariants_and_large(gpu, orc):
    # test_runscan.cpp:93-123: sorted, separated by background, conservation of pixels
    y = gpu
    for sp in [Spec.random(4096, 3000, 0.5, 99), Spec.random(1025, 700, 0.9, 3), Spec.hbands(5000, 600, 147),
               Spec.checker(777, 513, 1), Spec.random(33, 2000, 0.3, 1)]:
        bits = orc.synth(sp)
        p = y.build_profile(y.BinaryImage(sp.width, sp.height, bits))
        want = orc.profile(bits, sp.width)
        assert np.array_equal(p.runs_flat, want), sp
        r = p.runs_flat
        assert (r[:, 1] <= r[:, 2]).all()
        same = r[1:, 0] == r[:-1, 0]
        assert (r[1:, 1][same] >= r[:-1, 2][same] + 2).all()
        assert int((r[:, 2] - r[:, 1] + 1).sum()) == int(np.unpackbits(bits).sum())
        for c in (0, sp.width // 2, sp.width - 1):
            assert np.array_equal(y.column_runs(y.BinaryImage(sp.width, sp.height, bits), c), p.runs(c)), (sp, c)


@pytest.mark.parametrize("kind", ["direct", "rowwise", "staged", "band"])
def test_build_profile_each_fill_kernel(gpu, orc, monkeypatch, kind):
    """The four fill kernels (band-staged by default; YCHG_FILL_KERNEL forces one)
    on the golden corpus and on band / width / height edges: 255/256/257 and
    511/513 rows (partial bands and chunks), widths off the 32-column word, the
    8-column byte and the band kernel's 4-word group, runs crossing bands, open at
    the last row, one-row masks, 128 runs per column and band (checker(1))."""
    y = gpu
    monkeypatch.setenv("YCHG_FILL_KERNEL", kind)
    specs = [spec_of(row["spec"]) for row in corpus()]
    specs += [Spec.random(1000, 257, 0.5, 5), Spec.random(37, 256, 0.7, 6), Spec.random(65, 255, 0.3, 7),
              Spec.random(1031, 513, 0.95, 8), Spec.random(9, 511, 0.05, 9), Spec.hbands(100, 1000, 3),
              Spec.checker(301, 700, 1), Spec.checker(64, 600, 300), Spec.random(257, 1, 0.5, 10),
              Spec.random(3000, 2000, 0.5, 11)]
    for sp in specs:
        bits = orc.synth(sp)
        p = y.build_profile(y.BinaryImage(sp.width, sp.height, bits))
        assert np.array_equal(p.runs_flat, orc.profile(bits, sp.width)), (kind, sp)


def test_reference_acceptance_on_gpu_library(gpu):
    """The reference's own acceptance suite (tests/acceptance.cpp), compiled from the
    reference sources and headers with libychg.so linked in place of runscan.cpp
    (oracle/Makefile `dropin`).  Criteria 4 and 6 assert CPU-thread scaling and are
    reported, not required."""
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/acceptance_dropin not built (needs /root/reference at build time)")
    for crit in (1, 2, 3, 5, 7):
        out = subprocess.run([exe, str(crit)], capture_output=True, text=True, timeout=600)
        line = out.stdout.strip().splitlines()[0] if out.stdout.strip() else out.stderr
        assert out.returncode == 0 and line.startswith("[PASS]"), line


def checker_hyperedges(w, h, c):
    """checker(c): every foreground cell is a rectangle and its own hyperedge (cells
    only touch diagonally); cell (0,0) is foreground (synth.cpp checker rule)."""
    cx, cy = -(-w // c), -(-h // c)
    return (cx * cy + 1) // 2


@pytest.mark.parametrize("pattern", ["hbands", "checker"])
def test_max_size_65536(gpu, orc, ref, pattern):
    """BASELINE config 5 geometry on one GPU (512 MiB mask, 64 strips x k segments):
    counts bit-exact vs the unmodified reference (parallel, all host cores), the
    boundary list vs the reference's detect_boundary_columns, and the hyperedge total
    vs its closed form (validated against the oracle on small sizes below)."""
    y = gpu
    for w, h, c in [(20, 20, 7), (65, 70, 7), (100, 33, 7)]:
        assert orc.hyperedges(orc.synth(Spec.checker(w, h, c)), w)[0] == checker_hyperedges(w, h, c)
    n = 65536
    sp = Spec.hbands(n, n, 147) if pattern == "hbands" else Spec.checker(n, n, 7)
    img = y.synth(pattern, n, n, bands=147 if pattern == "hbands" else 0, cell=7 if pattern == "checker" else 0)
    r = y.scan(img)
    rimg = ref.image_synth(sp)
    assert np.array_equal(rimg.bytes(), img.bytes().reshape(n, -1)[:, : (n + 7) // 8])
    want = rimg.counts(1, os.cpu_count() or 1)
    assert np.array_equal(r.counts, want)
    assert np.array_equal(r.boundaries, ref.boundaries(want))
    assert r.total_runs == int(want.sum())
    assert r.hyperedges == (147 if pattern == "hbands" else checker_hyperedges(n, n, 7))


@pytest.mark.parametrize("segments", [None, 2, 3, 4])
def test_pipelined_graph_distinct_images(gpu, orc, segments, monkeypatch):
    """CUDA-graph replays of back-to-back scans of DISTINCT images, full and
    counts-only interleaved, each into its own outputs, with forced row-segment
    counts (regression: a cross-scan race once let scan t overwrite segment flags
    scan t-2's finisher had not read -- a stall -- and scan tickets could be drawn
    out of launch order -- mixed images).  A stall fails after 20 s."""
    import time

    import torch

    y = gpu
    if segments is not None:
        monkeypatch.setenv("YCHG_SEGMENTS", str(segments))
    W, H = 3100, 2600
    specs = [Spec.random(W, H, 0.5, 21), Spec.hbands(W, H, 40), Spec.checker(W, H, 5), Spec.random(W, H, 0.3, 22),
             Spec.frame(W, H)]
    pitch = y.pitch_for(W)
    imgs = []
    for sp in specs:
        bits = orc.synth(sp)
        dev = np.zeros((H, pitch), np.uint8)
        dev[:, : bits.shape[1]] = bits
        counts = orc.counts(bits, W)
        imgs.append((torch.from_numpy(dev).cuda(), counts, orc.boundaries(counts), orc.hyperedges(bits, W)[0]))
    plan = y.Plan(W, H)
    n = 24
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
                plan.scan_device(imgs[i % len(imgs)][0].data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(),
                                 t.data_ptr(), cs, i % 3 != 2)
    stream.wait_stream(cap)
    for rep in range(4):
        g.replay()
        t0 = time.time()
        while not stream.query():
            assert time.time() - t0 < 20, f"pipelined graph stalled (replay {rep}, segments {segments})"
            time.sleep(0.01)
    for i in range(n):
        c, _, b, t = outs[i]
        _, counts, bounds, he = imgs[i % len(imgs)]
        tt = t.cpu().tolist()
        assert np.array_equal(c.cpu().numpy(), counts), i
        assert tt[3] == bounds.size and np.array_equal(b.cpu().numpy()[: bounds.size], bounds), i
        assert tt[2] == (he if i % 3 != 2 else -1), i
    plan.close()


def test_pipelined_graph_random_geometries(gpu, orc, monkeypatch):
    """Random geometries (strip / word / byte edges, tall and wide), each captured as
    a CUDA graph of back-to-back scans of distinct images with random segment counts
    and full / counts-only mixed; every scan's outputs checked against the oracle."""
    import time

    import torch

    y = gpu
    rng = np.random.default_rng(777)
    for trial in range(12):
        W = int(rng.choice([1, 31, 33, 1023, 1025, 2049, 3000, 5000]))
        H = int(rng.choice([1, 2, 31, 33, 257, 1000, 2500]))
        monkeypatch.setenv("YCHG_SEGMENTS", str(int(rng.integers(1, 9))))
        # some trials with a tiny grid: every CTA then streams several segments
        monkeypatch.setenv("YCHG_GRID", str(int(rng.choice([1, 2, 3, 1000]))))
        specs = [Spec.random(W, H, float(rng.choice([0.1, 0.5, 0.9])), int(rng.integers(0, 1 << 40))) for _ in range(3)]
        pitch = y.pitch_for(W)
        imgs = []
        for sp in specs:
            bits = orc.synth(sp)
            dev = np.zeros((H, pitch), np.uint8)
            dev[:, : bits.shape[1]] = bits
            counts = orc.counts(bits, W)
            imgs.append((torch.from_numpy(dev).cuda(), counts, orc.boundaries(counts), orc.hyperedges(bits, W)[0]))
        plan = y.Plan(W, H)
        n = 9
        full = [bool(rng.integers(0, 2)) for _ in range(n)]
        outs = [(torch.full((W,), -7, dtype=torch.int32, device="cuda"),
                 torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda"),
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
        for rep in range(2):
            g.replay()
            t0 = time.time()
            while not stream.query():
                assert time.time() - t0 < 20, f"stall: {W}x{H} trial {trial}"
                time.sleep(0.005)
        for i in range(n):
            c, _, b, t = outs[i]
            _, counts, bounds, he = imgs[i % 3]
            tt = t.cpu().tolist()
            assert np.array_equal(c.cpu().numpy(), counts), (W, H, i)
            assert tt[3] == bounds.size and np.array_equal(b.cpu().numpy()[: bounds.size], bounds), (W, H, i)
            assert tt[2] == (he if full[i] else -1), (W, H, i)
        plan.close()


def test_scan_sharded_matches_single_device(gpu, orc):
    """ychg_scan_host_sharded (column strips + halos, gathered counts, one K2 pass,
    summed runs/links): identical to the single-device scan and the oracle for 1..5
    strips, with every strip on device 0 (the strip/merge logic is the same for
    several devices)."""
    y = gpu
    rng = np.random.default_rng(99)
    for sp in [Spec.random(5000, 700, 0.5, 3), Spec.hbands(4100, 600, 37), Spec.checker(3333, 500, 3),
               Spec.random(1024, 300, 0.4, 4), Spec.random(1, 50, 0.5, 5), Spec.frame(2049, 9)]:
        bits = orc.synth(sp)
        img = y.BinaryImage(sp.width, sp.height, bits)
        want = y.scan(img)
        counts = orc.counts(bits, sp.width)
        assert np.array_equal(want.counts, counts)
        for n in (1, 2, 3, 5):
            got = y.scan_sharded(img, n, devices=[0] * int(rng.integers(1, 3)))
            assert np.array_equal(got.counts, want.counts), (sp, n)
            assert np.array_equal(got.boundaries, want.boundaries), (sp, n)
            assert (got.total_runs, got.links, got.hyperedges) == (want.total_runs, want.links, want.hyperedges), (sp, n)
        c = y.scan_sharded(img, 3, with_hyperedges=False)
        assert np.array_equal(c.counts, counts) and c.hyperedges == -1


def test_very_wide_and_very_tall(gpu, orc):
    """Extreme aspect ratios: ~977 strips of one row segment each (a long
    finisher look-back chain), and one strip of 4M rows (128 segments per strip)."""
    y = gpu
    for sp in (Spec.random(1_000_000, 40, 0.5, 17), Spec.random(40, 4_000_000, 0.5, 18)):
        bits = orc.synth(sp)
        r = y.scan(y.BinaryImage(sp.width, sp.height, bits))
        counts = orc.counts(bits, sp.width)
        assert np.array_equal(r.counts, counts)
        assert np.array_equal(r.boundaries, orc.boundaries(counts))
        assert r.hyperedges == orc.hyperedges(bits, sp.width)[0]


def test_sync_inputs_image_written_by_preceding_kernel(gpu, orc):
    """YCHG_PLAN_SYNC_INPUTS: each image is written by the synth kernel launched right
    before the scan on the same stream, into one reused buffer, with no host sync in
    between -- the streaming kernel must wait for that grid before its first load."""
    import torch
    y = gpu
    W, H = 5000, 3000
    pitch = y.pitch_for(W)
    d = torch.zeros((H, pitch), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    specs = [Spec.random(W, H, 0.5, 31), Spec.hbands(W, H, 40), Spec.checker(W, H, 2), Spec.random(W, H, 0.1, 32)] * 2
    for latency in (False, True):
        plan = y.Plan(W, H, latency=latency, sync_inputs=True)
        outs = []
        for sp in specs:
            name = {v: k for k, v in y.PATTERNS.items()}[sp.pattern]
            y.synth_device(name, W, H, d.data_ptr(), pitch, bands=sp.bands, cell=sp.cell, density=sp.density,
                           seed=sp.seed, stream=stream)
            c = torch.full((W,), -7, dtype=torch.int32, device="cuda")
            f = torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda")
            b = torch.full((W,), -7, dtype=torch.int32, device="cuda")
            t = torch.zeros(4, dtype=torch.int64, device="cuda")
            plan.scan_device(d.data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(), t.data_ptr(), stream)
            outs.append((sp, c, t))
        torch.cuda.synchronize()
        for sp, c, t in outs:
            bits = orc.synth(sp)
            assert np.array_equal(c.cpu().numpy(), orc.counts(bits, W)), sp
            assert t.cpu().tolist()[2] == orc.hyperedges(bits, W)[0], sp
        plan.close()


def test_host_path_pageable_pinned_and_strided_inputs(gpu, orc, monkeypatch):
    """ychg_scan_host from pageable rows (pinned staging ring, several 1 MB chunks
    with a partial tail), from pinned rows (direct DMA) and from strided rows
    (driver 2-D copy): identical results, equal to the oracle."""
    import torch
    monkeypatch.setenv("YCHG_STAGE_MB", "1")  # read once per process: only effective if first
    y = gpu
    W, H = 9001, 2999
    sp = Spec.random(W, H, 0.45, 4242)
    bits = orc.synth(sp)
    rb = bits.shape[1]
    want_c = orc.counts(bits, W)
    want_b = orc.boundaries(want_c)
    want_h = orc.hyperedges(bits, W)[0]
    pin = torch.empty((H, rb), dtype=torch.uint8, pin_memory=True)
    pin.numpy()[:] = bits
    strided = np.zeros((H, rb + 5), np.uint8)
    strided[:, :rb] = bits
    import ctypes
    for arr in (bits.copy(), pin.numpy(), strided):
        for _ in range(2):  # the second call reuses the staging ring and device buffers
            counts = np.zeros(W, np.int32)
            bounds = np.zeros(W, np.int32)
            t = y.Totals()
            y._check(y._lib.ychg_scan_host(arr.ctypes.data_as(ctypes.c_void_p), W, H, arr.strides[0], 1,
                                           counts.ctypes.data_as(ctypes.c_void_p),
                                           bounds.ctypes.data_as(ctypes.c_void_p), ctypes.byref(t)), "scan")
            assert np.array_equal(counts, want_c), arr.strides
            assert t.n_boundaries == want_b.size and np.array_equal(bounds[: t.n_boundaries], want_b)
            assert t.hyperedges == want_h


def test_host_path_output_buffers_grow_and_shrink(gpu, orc):
    """The host entry point's mapped output block is reallocated as images widen
    (counts | boundaries | totals written by the finisher straight into host
    memory): alternate narrow / wide / narrow images, counts-only and full path,
    every result equal to the oracle (also after a shrink, with stale data from
    the wider scan still in the block)."""
    y = gpu
    for k, (W, H, dens) in enumerate([(100, 37, 0.5), (40000, 64, 0.3), (1500, 900, 0.6), (70001, 33, 0.5),
                                      (9, 5, 0.5), (2049, 2049, 0.45)]):
        sp = Spec.random(W, H, dens, 99 + k)
        bits = orc.synth(sp)
        img = y.BinaryImage(W, H, bits)
        want_c = orc.counts(bits, W)
        want_b = orc.boundaries(want_c)
        for links in (True, False):
            r = y.scan(img, with_hyperedges=links)
            assert np.array_equal(r.counts, want_c), (W, H, links)
            assert np.array_equal(r.boundaries, want_b), (W, H, links)
            if links:
                assert r.hyperedges == orc.hyperedges(bits, W)[0], (W, H)
        assert np.array_equal(y.cut_vertex_counts(img), want_c)


def _scan_plan(y, bits, W, H, skip=True, links=True):
    """One device scan of host rows `bits` through a fresh plan -> (counts, boundaries, totals)."""
    import torch
    pitch = y.pitch_for(W)
    dev = np.zeros((H, pitch), np.uint8)
    dev[:, : bits.shape[1]] = bits
    d = torch.from_numpy(dev).cuda()
    c = torch.full((W,), -7, dtype=torch.int32, device="cuda")
    f = torch.zeros(W // 32 + 64, dtype=torch.int32, device="cuda")
    b = torch.full((W,), -7, dtype=torch.int32, device="cuda")
    t = torch.zeros(4, dtype=torch.int64, device="cuda")
    plan = y.Plan(W, H, skip=skip)
    plan.scan_device(d.data_ptr(), pitch, c.data_ptr(), f.data_ptr(), b.data_ptr(), t.data_ptr(),
                     torch.cuda.current_stream().cuda_stream, links)
    torch.cuda.synchronize()
    tt = t.cpu().tolist()
    plan.close()
    return c.cpu().numpy(), b.cpu().numpy()[: tt[3]], tt


def _row_image(W, H, row_fn):
    """Rows built column-wise: row_fn(y) -> bool array of W columns."""
    px = np.stack([row_fn(yy) for yy in range(H)]).astype(np.uint8)
    return np.packbits(px, axis=1)


@pytest.mark.parametrize("case", ["halo_only", "lane_edge", "sparse_rows", "one_pixel", "strip_edge_pair"])
def test_skip_unchanged_blocks_exact(gpu, orc, case):
    """The skip of 32-row blocks equal to the row above (default on) must be exact,
    including changes that only the right-halo bit of lane 31 sees (column 1024k,
    the next strip's first column), changes at lane (32-column) edges, and single
    changed pixels; compared with the oracle and with YCHG_PLAN_NO_SKIP."""
    y = gpu
    W, H = 3100, 2100
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    base = rng.random(W) < 0.5
    if case == "halo_only":          # only columns 1024 and 2048 ever change
        toggles = set(int(v) for v in rng.integers(0, H, 120))
        state = {1024: False, 2048: True}
        rows = []
        for yy in range(H):
            if yy in toggles:
                for c in state:
                    state[c] = not state[c]
            r = base.copy()
            for c, v in state.items():
                r[c] = v
            rows.append(r)
        bits = np.packbits(np.stack(rows).astype(np.uint8), axis=1)
    elif case == "lane_edge":        # only columns 31/32 and 1023 change, at random rows
        cols = [31, 32, 1023]
        bits = _row_image(W, H, lambda yy: np.where(np.isin(np.arange(W), cols), (yy * 7919 % 97) < 40, base))
    elif case == "sparse_rows":      # a handful of changing rows, everything else constant
        change = set(int(v) for v in rng.integers(0, H, 9))
        rows, cur = [], base.copy()
        for yy in range(H):
            if yy in change:
                cur = rng.random(W) < 0.5
            rows.append(cur.copy())
        bits = np.packbits(np.stack(rows).astype(np.uint8), axis=1)
    elif case == "one_pixel":        # constant rows + single isolated pixels
        px = np.tile(base, (H, 1))
        for _ in range(40):
            px[int(rng.integers(0, H)), int(rng.integers(0, W))] ^= True
        bits = np.packbits(px.astype(np.uint8), axis=1)
    else:                            # vertical pairs straddling the strip edge, toggled together
        px = np.zeros((H, W), bool)
        on = False
        for yy in range(H):
            if yy % 61 == 0:
                on = not on
            px[yy, 1023] = on
            px[yy, 1024] = (yy % 13) < 9
        bits = np.packbits(px.astype(np.uint8), axis=1)
    want_c = orc.counts(bits, W)
    want_b = orc.boundaries(want_c)
    he, runs, links = orc.hyperedges(bits, W)
    for skip in (True, False):
        c, b, t = _scan_plan(y, bits, W, H, skip=skip)
        assert np.array_equal(c, want_c), (case, skip)
        assert np.array_equal(b, want_b), (case, skip)
        assert t[:3] == [runs, links, he], (case, skip)


def test_column_runs_byte_column_path(gpu, orc, ref):
    """column_runs moves one byte column (O(height)) and rebases Run.col: every
    column of odd widths (partial last byte, garbage padding bits), and a column of
    > 65536 runs (the second, exact-size call), against the live reference."""
    y = gpu
    for sp in (Spec.random(37, 301, 0.5, 5), Spec.random(1031, 77, 0.3, 6), Spec.checker(19, 40, 3)):
        bits = orc.synth(sp)
        rimg = ref.image(bits, sp.width)
        noisy = bits.copy()
        if sp.width % 8:
            noisy[:, -1] |= np.uint8((1 << (8 - sp.width % 8)) - 1)  # padding bits set: must be ignored
        for img in (y.BinaryImage(sp.width, sp.height, bits), y.BinaryImage(sp.width, sp.height, noisy)):
            for col in range(sp.width):
                assert np.array_equal(y.column_runs(img, col), rimg.column_runs(col)), (sp, col)
    tall = Spec.random(9, 300_000, 0.5, 7)
    bits = orc.synth(tall)
    rimg = ref.image(bits, 9)
    img = y.BinaryImage(9, tall.height, bits)
    for col in (0, 4, 8):
        got = y.column_runs(img, col)
        assert got.shape[0] > 65536 and np.array_equal(got, rimg.column_runs(col)), col


def test_scan_sharded_restores_caller_device(gpu, orc):
    """ychg_scan_host_sharded switches devices internally (peer access, the gathering
    device); the caller's current device must be the same afterwards."""
    import ctypes
    y = gpu
    sp = Spec.random(3000, 200, 0.5, 8)
    img = y.BinaryImage(sp.width, sp.height, orc.synth(sp))
    drv = ctypes.CDLL("libcuda.so.1")  # the driver's current context is the thread's current device
    n = y.device_count()
    for dev in range(min(n, 2)):
        y._check(y._lib.ychg_set_device(dev), "set_device")
        y.scan_sharded(img, 3, devices=list(range(n))[:2])
        cur = ctypes.c_int(-1)
        assert drv.cuCtxGetDevice(ctypes.byref(cur)) == 0
        assert cur.value == dev
    y._check(y._lib.ychg_set_device(0), "set_device")


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2", reason="needs two GPUs (peer stores over NVLink)")
def test_scan_sharded_peer_gather_two_devices(gpu, orc):
    """Strips on two devices: the finishers on device 1 store their counts straight
    into the gathering array on device 0 (peer pointers), bit-exact with one device."""
    y = gpu
    for sp in (Spec.random(9000, 700, 0.5, 12), Spec.hbands(5000, 600, 37)):
        img = y.BinaryImage(sp.width, sp.height, orc.synth(sp))
        want = y.scan(img)
        for n in (2, 3, 4):
            got = y.scan_sharded(img, n, devices=[0, 1])
            assert np.array_equal(got.counts, want.counts) and np.array_equal(got.boundaries, want.boundaries)
            assert (got.total_runs, got.links, got.hyperedges) == (want.total_runs, want.links, want.hyperedges)
