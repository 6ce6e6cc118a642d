"""CPU: the GPU kernel's K3 band-stitching algorithm, replayed bit-exactly by
tests/kernel_model.py, reproduces the reference hyperedge totals under many
band splits (tiny blocks, many segments and strips)."""
import numpy as np
import pytest

from golden_io import corpus, spec_of
from kernel_model import model_hyperedges
from oracle import Spec

SPLITS = [(1, 1, 1), (2, 3, 1), (3, 2, 2), (5, 1, 1), (32, 1, 32)]


@pytest.mark.parametrize("block_rows,k,strip_words", SPLITS)
def test_model_matches_golden_corpus(orc, block_rows, k, strip_words):
    for row in corpus()[::3]:
        sp = spec_of(row["spec"])
        bits = orc.synth(sp)
        nb = (sp.height + block_rows - 1) // block_rows
        runs, links = model_hyperedges(bits, sp.width, block_rows=block_rows, seg_per_strip=min(k, nb),
                                       strip_words=strip_words)
        assert runs - links == row["hyperedges"], row["name"]


def test_model_strip_halo_width(orc):
    # multi-GPU strips: count [0, wc) of a wider buffer; pairs use the halo column
    bits = orc.synth(Spec.random(300, 97, 0.5, 99))
    he_full, runs_full, links_full = orc.hyperedges(bits, 300)
    pair = orc.pair_links(bits, 300)
    counts = orc.counts(bits, 300)
    for wc in (64, 100, 257):
        runs, links = model_hyperedges(bits, 300, block_rows=4, seg_per_strip=3, strip_words=1, width_cnt=wc)
        assert runs == int(counts[:wc].sum())
        assert links == int(pair[:wc].sum())


@pytest.mark.parametrize("spec", [Spec.random(512, 512, 0.5, 50000), Spec.hbands(700, 300, 147),
                                  Spec.checker(333, 257, 7), Spec.full(90, 200)])
def test_model_medium(orc, spec):
    bits = orc.synth(spec)
    he, runs, links = orc.hyperedges(bits, spec.width)
    r, l = model_hyperedges(bits, spec.width, block_rows=8, seg_per_strip=5, strip_words=4)
    assert (r, l) == (runs, links)
