"""CPU: pin the oracle restatement to the reference's own known answers and to
the golden fixtures generated from the unmodified reference (oracle/_ref)."""
import hashlib

import numpy as np
import pytest

from golden_io import acceptance2, corpus, decompose, decomposition_digest, large, spec_of
from oracle import Spec, a7_links, branch_example, full_corpus


def test_splitmix64_frozen_vector(orc):
    # test_imagekit.cpp:81-91
    assert orc.splitmix64(1234567, 5) == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                                          4593380528125082431, 16408922859458223821]
    assert orc.splitmix64(0, 1) == [16294208416658607535]


def test_bit_layout_msb_first(orc):
    # test_imagekit.cpp:49-53: x=0 is 0x80; frame 5x5 P4 payload (test_imagekit.cpp:198-209)
    assert orc.synth(Spec.frame(5, 5))[:, 0].tolist() == [0xF8, 0x88, 0x88, 0x88, 0xF8]


def test_counts_known_answers(orc):
    # test_runscan.cpp:35-49
    assert orc.counts(orc.synth(Spec.full(4, 4)), 4).tolist() == [1, 1, 1, 1]
    assert orc.counts(orc.synth(Spec.frame(5, 5)), 5).tolist() == [1, 2, 2, 2, 1]
    assert orc.counts(orc.synth(Spec.empty(3, 3)), 3).tolist() == [0, 0, 0]
    assert orc.counts(branch_example(), 2).tolist() == [2, 2]
    assert orc.counts(np.zeros((0, 0), np.uint8), 0).tolist() == []
    assert orc.counts(orc.synth(Spec.hbands(8, 11, 3)), 8).tolist() == [3] * 8


def test_boundaries_known_answers(orc):
    # test_runscan.cpp:129-143
    cases = [([1, 2, 2, 2, 1], [0, 1, 4]), ([0, 0, 0], []), ([], []), ([0, 1], [1]), ([3], [0]), ([2, 2], [0])]
    for counts, want in cases:
        assert orc.boundaries(np.array(counts, np.int32)).tolist() == want


def test_hyperedge_known_answers(orc):
    # acceptance.cpp:101-121, test_hypergraph.cpp:75-88, test_bench.cpp:139-160, test_cli.cpp:176-193
    assert orc.hyperedges(branch_example(), 2)[0] == 4
    assert orc.hyperedges(orc.synth(Spec.frame(5, 5)), 5)[0] == 4
    for k in (1, 3, 7):
        assert orc.hyperedges(orc.synth(Spec.hbands(20, 20, k)), 20)[0] == k
    assert orc.hyperedges(orc.synth(Spec.checker(8, 8, 1)), 8)[0] == 32
    assert orc.hyperedges(orc.synth(Spec.empty(3, 3)), 3)[0] == 0
    assert orc.hyperedges(np.zeros((0, 0), np.uint8), 0)[0] == 0
    for k, want in ((1, 1), (2, 2), (4, 4)):
        assert orc.hyperedges(orc.synth(Spec.hbands(64, 64, k)), 64)[0] == want
    assert orc.hyperedges(orc.synth(Spec.checker(64, 64, 1)), 64)[0] == 2048
    assert orc.hyperedges(orc.synth(Spec.checker(16, 16, 1)), 16)[0] == 128


def test_oracle_matches_reference_golden_corpus(orc):
    rows = corpus()
    assert len(rows) == 1170
    for row in rows:
        sp = spec_of(row["spec"])
        bits = orc.synth(sp)
        c = orc.counts(bits, sp.width)
        assert c.tolist() == row["counts"], row["name"]
        assert orc.boundaries(c).tolist() == row["boundaries"], row["name"]
        assert orc.hyperedges(bits, sp.width)[0] == row["hyperedges"], row["name"]


def test_corpus_generator_matches_golden():
    names = [n for n, _ in full_corpus()]
    assert names == [r["name"] for r in corpus()]


def test_oracle_matches_reference_acceptance2(orc):
    for row in acceptance2()[:40]:
        sp = spec_of(row["spec"])
        bits = orc.synth(sp)
        c = orc.counts(bits, sp.width)
        assert hashlib.sha256(c.astype("<i4").tobytes()).hexdigest() == row["counts_sha256"]
        assert orc.boundaries(c).size == row["n_boundaries"]
        assert orc.hyperedges(bits, sp.width)[0] == row["hyperedges"]


@pytest.mark.parametrize("idx", [1, 5, 7, 9])
def test_oracle_matches_reference_large(orc, idx):
    row = large()[idx]
    sp = spec_of(row["spec"])
    bits = orc.synth(sp)
    c = orc.counts(bits, sp.width)
    assert hashlib.sha256(c.astype("<i4").tobytes()).hexdigest() == row["counts_sha256"]
    assert orc.hyperedges(bits, sp.width)[0] == row["hyperedges"]


def test_a7_streaming_rule_equals_decompose(orc):
    # runs - links(strip components with exactly two runs) == decompose count
    for name, sp in full_corpus()[::7]:
        bits = orc.synth(sp)
        he, runs, links = orc.hyperedges(bits, sp.width)
        assert a7_links(bits, sp.width) == links, name


def test_c_a7_restatement_pinned(orc):
    """yo_a7_links (the C streaming restatement the 65536^2 parity test relies on,
    where decompose does not fit) equals the decompose-based link count on the whole
    corpus and on the reference-pinned large fixtures, whose hyperedge totals come
    from the reference's own decompose (tests/golden/large_ref.json)."""
    for name, sp in full_corpus():
        bits = orc.synth(sp)
        he, runs, links = orc.hyperedges(bits, sp.width)
        assert orc.a7_links(bits, sp.width) == links, name
    for row in large():
        sp = spec_of(row["spec"])
        bits = orc.synth(sp)
        runs = int(orc.counts(bits, sp.width).astype(np.int64).sum())
        assert runs - orc.a7_links(bits, sp.width) == row["hyperedges"], row["spec"]


def test_threaded_synth_matches_serial_draws(orc):
    """yo_synth splits rows over threads; the random pattern's row start state
    seed + y*w*golden must reproduce the sequential SplitMix64 stream exactly."""
    sp = Spec.random(5003, 900, 0.37, 987654321)
    bits = orc.synth(sp)
    draws = orc.splitmix64(sp.seed, 3 * sp.width)   # the first three rows, sequentially
    thr = int(0.37 * 2.0 ** 64)
    for y in range(3):
        row = np.array([d < thr for d in draws[y * sp.width:(y + 1) * sp.width]], dtype=np.uint8)
        assert np.array_equal(np.packbits(row), bits[y]), y
    tall = Spec.random(40, 9000, 0.5, 11)   # > 4096 rows: the threaded path
    tb = orc.synth(tall)
    dr = orc.splitmix64(tall.seed, 40 * 9000)
    want = np.packbits(np.array([d < 2 ** 63 for d in dr], dtype=np.uint8).reshape(9000, 40), axis=1)
    assert np.array_equal(tb, want)


def test_oracle_against_live_reference(orc, ref):
    # When oracle/_ref is present: random geometries straddling byte/word edges.
    rng = np.random.default_rng(5)
    for _ in range(60):
        w, h = int(rng.integers(1, 200)), int(rng.integers(1, 120))
        sp = Spec.random(w, h, float(rng.choice([0.1, 0.5, 0.9])), int(rng.integers(0, 1 << 62)))
        bits = ref.synth(sp)
        assert np.array_equal(bits, orc.synth(sp))
        img = ref.image(bits, w)
        c = img.counts(1, 4)
        assert np.array_equal(c, orc.counts(bits, w))
        assert img.hyperedges() == orc.hyperedges(bits, w)[0]


def test_profile_restatement_matches_reference(orc, ref):
    # build_profile (runscan.cpp:130-143) via the compiled reference vs the oracle restatement
    for name, sp in full_corpus()[::5]:
        bits = orc.synth(sp)
        img = ref.image(bits, sp.width)
        assert np.array_equal(orc.profile(bits, sp.width), img.profile(1, 4)), name


def test_profile_known_answers(orc):
    # test_runscan.cpp:17-33, 116-123
    fr = orc.profile(orc.synth(Spec.frame(5, 5)), 5)
    assert fr.tolist() == [[0, 0, 4], [1, 0, 0], [1, 4, 4], [2, 0, 0], [2, 4, 4], [3, 0, 0], [3, 4, 4], [4, 0, 4]]
    br = orc.profile(branch_example(), 2)
    assert br.tolist() == [[0, 0, 1], [0, 3, 6], [1, 0, 4], [1, 6, 6]]


def test_decompose_known_answers(orc):
    # test_hypergraph.cpp:37-57 (frame) and :59-73 (branch example)
    d = orc.decompose(orc.synth(Spec.frame(5, 5)), 5)
    assert d.edge_offsets.tolist() == [0, 1, 4, 7, 8]
    assert d.edge_runs.tolist() == [[0, 0, 4], [1, 0, 0], [2, 0, 0], [3, 0, 0], [1, 4, 4], [2, 4, 4], [3, 4, 4],
                                    [4, 0, 4]]
    assert d.run_to_edge.tolist() == [0, 1, 2, 1, 2, 1, 2, 3]  # edge_of(0,0)=0, (1,0)=1, (1,1)=2, (4,0)=3
    b = orc.decompose(branch_example(), 2)
    assert b.edge_offsets.tolist() == [0, 1, 2, 3, 4]
    assert b.edge_runs.tolist() == [[0, 0, 1], [0, 3, 6], [1, 0, 4], [1, 6, 6]]
    # test_hypergraph.cpp:75-88: hbands(20,20,k) -> k edges; empty -> 0
    for k in (1, 3, 7):
        assert orc.decompose(orc.synth(Spec.hbands(20, 20, k)), 20).edge_count == k
    assert orc.decompose(orc.synth(Spec.empty(3, 3)), 3).edge_count == 0


def test_decompose_matches_reference_golden(orc):
    # digests of the reference's decompose on the 1170-image corpus + the small large images
    for row in decompose():
        sp = spec_of(row["spec"])
        if sp.width * sp.height > 5_000_000:
            continue
        got = decomposition_digest(orc.decompose(orc.synth(sp), sp.width))
        want = {k: row[k] for k in got}
        assert got == want, row["name"]


def test_decompose_against_live_reference(orc, ref):
    rng = np.random.default_rng(11)
    for _ in range(40):
        w, h = int(rng.integers(1, 150)), int(rng.integers(1, 100))
        sp = Spec.random(w, h, float(rng.choice([0.2, 0.5, 0.8])), int(rng.integers(0, 1 << 62)))
        bits = orc.synth(sp)
        a, b = orc.decompose(bits, w), ref.image(bits, w).decompose()
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
