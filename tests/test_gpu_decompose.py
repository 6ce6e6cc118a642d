"""GPU parity of the device decomposition: decompose
(hypergraph.cpp:94-170) through the C ABI, bit-exact against the reference's own
known answers (test_hypergraph.cpp), the golden digests of the unmodified
reference (tests/golden/decompose_ref.json.gz) and the oracle restatement."""
import numpy as np
import pytest

from golden_io import decompose as golden_decompose
from golden_io import decomposition_digest, spec_of
from oracle import Decomposition, Spec, branch_example

pytestmark = pytest.mark.gpu


def gpu_decompose(y, orc, sp):
    return y.decompose(y.BinaryImage(sp.width, sp.height, orc.synth(sp)))


def as_tuple(hg):
    return Decomposition(hg.edge_runs, hg.edge_offsets, hg.run_to_edge)


def test_decompose_known_answers(gpu):
    y = gpu
    # test_hypergraph.cpp:24-35 full image -> one edge
    hg = y.decompose(y.synth("full", 4, 4))
    assert hg.edge_count == 1 and hg.edge(0).tolist() == [[0, 0, 3], [1, 0, 3], [2, 0, 3], [3, 0, 3]]
    # :37-57 frame
    hg = y.decompose(y.synth("frame", 5, 5))
    assert hg.edge_offsets.tolist() == [0, 1, 4, 7, 8]
    assert hg.edge(1).tolist() == [[1, 0, 0], [2, 0, 0], [3, 0, 0]]
    assert hg.edge(2).tolist() == [[1, 4, 4], [2, 4, 4], [3, 4, 4]]
    assert hg.run_to_edge.tolist() == [0, 1, 2, 1, 2, 1, 2, 3]
    # :59-73 branch example: four single-run edges
    hg = y.decompose(y.BinaryImage(2, 7, branch_example()))
    assert hg.edge_runs.tolist() == [[0, 0, 1], [0, 3, 6], [1, 0, 4], [1, 6, 6]]
    assert hg.edge_offsets.tolist() == [0, 1, 2, 3, 4]
    # :75-88 pattern counts, empty images
    for k in (1, 3, 7):
        assert y.decompose(y.synth("hbands", 20, 20, bands=k)).edge_count == k
    assert y.decompose(y.synth("checker", 8, 8, cell=1)).edge_count == 32
    assert y.decompose(y.synth("empty", 3, 3)).edge_count == 0
    assert y.decompose(y.BinaryImage(0, 0)).edge_count == 0


def test_decompose_golden_reference_digests(gpu, orc):
    # every corpus image and the large images, digests of the reference's own output
    y = gpu
    for row in golden_decompose():
        sp = spec_of(row["spec"])
        got = decomposition_digest(as_tuple(gpu_decompose(y, orc, sp)))
        assert got == {k: row[k] for k in got}, (row["name"], row["spec"])


def test_decompose_random_geometries_vs_oracle(gpu, orc):
    y = gpu
    rng = np.random.default_rng(2024)
    for _ in range(80):
        w, h = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        sp = Spec.random(w, h, float(rng.choice([0.05, 0.3, 0.5, 0.7, 0.95])), int(rng.integers(0, 1 << 62)))
        want = orc.decompose(orc.synth(sp), w)
        got = gpu_decompose(y, orc, sp)
        for a, b in zip(as_tuple(got), want):
            assert np.array_equal(a, b), sp


@pytest.mark.parametrize("sp", [Spec.hbands(21000, 600, 147), Spec.checker(3000, 3000, 1),
                                Spec.random(6000, 5000, 0.5, 1307), Spec.full(70000, 3), Spec.frame(3, 70000)],
                         ids=["long-chains", "checker1", "random", "one-wide-chain", "tall"])
def test_decompose_large_vs_oracle(gpu, orc, sp):
    y = gpu
    bits = orc.synth(sp)
    want = orc.decompose(bits, sp.width)
    got = y.decompose(y.BinaryImage(sp.width, sp.height, bits))
    for a, b in zip(as_tuple(got), want):
        assert np.array_equal(a, b)
    assert got.edge_count == orc.hyperedges(bits, sp.width)[0]


@pytest.mark.parametrize("cell", [1, 7, 23, 24, 25, 48, 200])
def test_decompose_chain_lengths_around_the_walk(gpu, orc, cell):
    """Chains of `cell` runs (checker(cell): every chain exactly cell columns long)
    around the emit kernel's walk length (24: heads walk their chains and stage a
    warp's output stretch in shared memory; longer chains are finished run by run
    by decomp_long_kernel), plus ragged edges (widths not a multiple of cell)."""
    y = gpu
    for w, h in ((cell * 11 + 5, 257), (cell * 3 + 1, 1000)):
        sp = Spec.checker(w, h, cell)
        bits = orc.synth(sp)
        want = orc.decompose(bits, sp.width)
        got = y.decompose(y.BinaryImage(sp.width, sp.height, bits))
        for a, b in zip(as_tuple(got), want):
            assert np.array_equal(a, b), (cell, w, h)


def test_decompose_profile_input_and_validation(gpu, orc):
    y = gpu
    sp = Spec.random(97, 61, 0.4, 5)
    img = y.BinaryImage(sp.width, sp.height, orc.synth(sp))
    prof = y.build_profile(img)
    assert y.decompose(prof) == y.decompose(img)
    assert np.array_equal(y.decompose(prof).run_to_edge, y.decompose(img).run_to_edge)

    def bad(mutate, msg):
        runs = prof.runs_flat.copy()
        mutate(runs)
        with pytest.raises(y.ValidationError, match=msg):
            y.decompose(y.ColumnProfile(prof.width, prof.height, prof.counts.copy(), runs))

    # hypergraph.cpp:74-86 messages; the first failing run in profile order wins
    c0 = int(np.argmax(prof.counts > 1))
    o = int(prof.col_off[c0])
    bad(lambda r: r.__setitem__((o, 0), c0 + 1), f"run in column list {c0} claims column {c0 + 1}")
    bad(lambda r: r.__setitem__((o, 2), sp.height), f"outside height {sp.height}")
    bad(lambda r: r.__setitem__((o + 1, 1), int(r[o, 2]) + 1), f"runs in column {c0} must be sorted")
    with pytest.raises(y.ValidationError):
        y.decompose(y.ColumnProfile(-1, 3, np.zeros(0, np.int32), np.zeros((0, 3), np.int32)))
    with pytest.raises(y.ValidationError):
        y.decompose(y.ColumnProfile(3, 3, np.zeros(2, np.int32), np.zeros((0, 3), np.int32)))
    # an empty profile is fine
    assert y.decompose(y.ColumnProfile(4, 4, np.zeros(4, np.int32), np.zeros((0, 3), np.int32))).edge_count == 0


def test_decompose_live_reference(gpu, orc, ref):
    # when oracle/_ref travelled with the repo: the unmodified reference itself
    y = gpu
    for sp in [Spec.checker(2049, 1500, 7), Spec.random(1500, 1700, 0.6, 77), Spec.hbands(4000, 4000, 147)]:
        bits = orc.synth(sp)
        want = ref.image(bits, sp.width).decompose()
        got = y.decompose(y.BinaryImage(sp.width, sp.height, bits))
        for a, b in zip(as_tuple(got), want):
            assert np.array_equal(a, b)


def test_decompose_max_size_65536_vs_reference(gpu, ref):
    """BASELINE config-5 geometry (65536^2 hbands(147): 9.6M runs in 147 chains of
    65536 runs, every one longer than the emit kernel's walk): the device
    decomposition element-wise against the unmodified reference's decompose."""
    y = gpu
    n = 65536
    sp = Spec.hbands(n, n, 147)
    img = y.synth("hbands", n, n, bands=147)
    got = y.decompose(img)
    want = ref.image_synth(sp).decompose()
    assert got.edge_count == 147
    for a, b in zip(as_tuple(got), want):
        assert np.array_equal(a, b)


def test_decompose_cxx_dropin(gpu):
    """ychg::b200::decompose returns the reference's own Hypergraph type, equal to
    ychg::decompose (tests/cpp/decompose_dropin.cpp, built by `make -C oracle dropin`)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                       "decompose_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/decompose_dropin not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "[PASS]" in out.stdout


def test_decompose_into_pinned_buffers(gpu, orc):
    """decompose(..., out=HypergraphBuffers): views into reusable pinned arrays equal
    the freshly allocated result; too small a buffer falls back to fresh arrays."""
    y = gpu
    buf = y.HypergraphBuffers(200_000)
    for sp in (Spec.random(500, 400, 0.5, 1), Spec.checker(300, 333, 3), Spec.random(500, 400, 0.5, 1)):
        img = y.BinaryImage(sp.width, sp.height, orc.synth(sp))
        fresh = y.decompose(img)
        got = y.decompose(img, out=buf)
        for a, b in zip(as_tuple(got), as_tuple(fresh)):
            assert np.array_equal(a, b)
    small = y.HypergraphBuffers(10)
    img = y.BinaryImage(500, 400, orc.synth(Spec.random(500, 400, 0.5, 2)))
    assert y.decompose(img, out=small) == y.decompose(img)
    buf.close()
    small.close()


def test_profile_and_decompose_tall(gpu, orc):
    """Columns with > 65535 runs (tall masks): build_profile and decompose vs the oracle."""
    y = gpu
    sp = Spec.random(37, 300_001, 0.5, 23)
    bits = orc.synth(sp)
    img = y.BinaryImage(sp.width, sp.height, bits)
    prof = y.build_profile(img)
    assert np.array_equal(prof.runs_flat, orc.profile(bits, sp.width))
    assert prof.counts.max() > 65535
    got = y.decompose(img)
    for a, b in zip(as_tuple(got), orc.decompose(bits, sp.width)):
        assert np.array_equal(a, b)
