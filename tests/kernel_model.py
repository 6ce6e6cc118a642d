"""Bit-exact Python model of the ychg_scan_kernel K3 algorithm (test infrastructure).

It replays, with 32-bit Python ints, exactly the per-lane bit-sliced state
machine of paper_1307_2560_b200/csrc/ychg_scan.cu (row_step, head mode, warp
band summaries, compose_summary, the strip stitch and the bottom closing) over
an arbitrary split of the rows into bands.  CPU tests drive it with tiny block
heights so that every image of the corpus is cut into many bands, which
exercises the band-stitching logic far harder than the 32-row GPU blocks do,
and compare the hyperedge total with the oracle.
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF


def words_of_row(row: np.ndarray, nwords: int) -> tuple[list[int], list[int]]:
    """(a, b) words for one row: a = columns 32w..32w+31 with column j at bit 31-j
    (byte-swapped load); b = the same shifted by one column (column c+1 at c's bit)."""
    nbytes = row.size
    pad = np.zeros(nwords * 4 + 1, dtype=np.uint8)
    pad[:nbytes] = row
    a = [int.from_bytes(pad[4 * w:4 * w + 4].tobytes(), "big") for w in range(nwords)]
    b = [((a[w] << 1) & M32) | (int(pad[4 * w + 4]) >> 7) for w in range(nwords)]
    return a, b


def word_mask(gw: int, limit: int) -> int:
    n = limit - 32 * gw
    if n >= 32:
        return M32
    if n <= 0:
        return 0
    return (~(M32 >> n)) & M32


def popc(x: int) -> int:
    return bin(x & M32).count("1")


class Summary:
    __slots__ = ("O", "E", "h1", "h2", "OE", "T2", "T3")

    def __init__(self, O=0, E=0, h1=0, h2=0, OE=0, T2=0, T3=0):
        self.O, self.E, self.h1, self.h2, self.OE, self.T2, self.T3 = O, E, h1, h2, OE, T2, T3


def compose(A: Summary, B: Summary) -> tuple[Summary, int]:
    n = lambda x: (~x) & M32  # noqa: E731
    Ap = A.O & n(A.E)
    Bp = B.O & n(B.E)
    s1 = A.h1 | B.h1
    s2 = A.h2 | B.h2 | (A.h1 & B.h1)
    J = n(Ap) & A.OE
    resolved = J & B.E & ((n(A.T2) & B.h1 & n(B.h2)) | (A.T2 & n(A.T3) & n(B.h1)))
    C = Summary(
        O=A.O,
        E=(Ap & B.E) | (n(Ap) & A.E),
        h1=(Ap & s1) | (n(Ap) & A.h1),
        h2=(Ap & s2) | (n(Ap) & A.h2),
        OE=B.OE,
        T2=(Bp & (A.T2 | B.h1)) | (n(Bp) & B.T2),
        T3=(Bp & (A.T3 | (A.T2 & B.h1) | B.h2)) | (n(Bp) & B.T3),
    )
    return C, popc(resolved)


def band(a_rows, b_rows, halo_a, halo_b, mk3, block_rows):
    """Run one lane over a band; returns (Summary, links).  Head pairs start
    poisoned at N >= 3 (G2 = G3 = 1) so their closing never counts locally."""
    n = lambda x: (~x) & M32  # noqa: E731
    pa, pb = halo_a, halo_b
    O = pa | pb
    Hd = O
    G2 = G3 = O
    pab = pa & pb
    h1 = h2 = 0
    links = 0
    for start in range(0, len(a_rows), block_rows):
        head = (Hd & mk3) != 0  # per lane; the kernel decides per warp, results are identical
        lks = []
        for a, b in zip(a_rows[start:start + block_rows], b_rows[start:start + block_rows]):
            ab = a & b
            cont = (a & pa) | (b & pb)
            lk = n(cont) & G2 & n(G3)
            # G2 & f == ab & G2 & ~pab: G2 implies pa | pb, and f = ab & (pa ^ pb)
            assert G2 & ~(pa | pb) == 0 and pab & ~G2 == 0
            if head:
                Hd &= cont
                t = Hd & ab & n(pab)  # Hd <= G2
                assert t == Hd & ab & (pa ^ pb)
                h2 |= h1 & t
                h1 |= t
            g3 = (cont & G3) | (ab & G2 & n(pab))
            assert g3 == (cont & G3) | (G2 & ab & (pa ^ pb))
            G2 = ab | (cont & G2)
            G3 = g3
            pa, pb, pab = a, b, ab
            lks.append(lk)
        links += sum(popc(x & mk3) for x in lks)
    m = mk3
    return Summary(O & m, O & n(Hd) & m, h1 & m, h2 & m, (pa | pb) & m, G2 & m, G3 & m), links


def model_hyperedges(bits: np.ndarray, width: int, *, block_rows: int = 32, seg_per_strip: int = 1,
                     warps: int = 8, strip_words: int = 32, width_cnt: int | None = None) -> tuple[int, int]:
    """(total_runs, links) as the GPU pipeline computes them for this band split."""
    h = bits.shape[0]
    wc = width if width_cnt is None else width_cnt
    if wc == 0 or h == 0:
        return 0, 0
    nwords = (wc + 31) // 32
    nw_all = (width + 31) // 32 + 1
    rows_a, rows_b = [], []
    for y in range(h):
        a, b = words_of_row(bits[y], nw_all)
        rows_a.append(a)
        rows_b.append(b)
    n_blocks = (h + block_rows - 1) // block_rows
    # virtual zero rows up to the block-aligned end (TMA zero fill beyond H)
    zero = [0] * nw_all
    while len(rows_a) < n_blocks * block_rows:
        rows_a.append(zero)
        rows_b.append(zero)
    n_strips = (wc + 32 * strip_words - 1) // (32 * strip_words)
    k = seg_per_strip
    total_links = 0
    for s in range(n_strips):
        for lane in range(strip_words):
            gw = s * strip_words + lane
            if gw >= nwords:
                continue
            mk3 = word_mask(gw, min(wc, width - 1))
            strip_sum, strip_links = None, 0
            for j in range(k):
                sb0, sb1 = (j * n_blocks) // k, ((j + 1) * n_blocks) // k
                nseg = sb1 - sb0
                seg_sum, seg_links = None, 0
                for w in range(warps):
                    wb0 = sb0 + (w * nseg) // warps
                    wb1 = sb0 + ((w + 1) * nseg) // warps
                    if wb1 <= wb0:
                        continue
                    y0, y1 = wb0 * block_rows, wb1 * block_rows
                    ha = rows_a[y0 - 1][gw] if y0 > 0 else 0
                    hb = rows_b[y0 - 1][gw] if y0 > 0 else 0
                    sm, lk = band([r[gw] for r in rows_a[y0:y1]], [r[gw] for r in rows_b[y0:y1]],
                                  ha, hb, mk3, block_rows)
                    seg_links += lk
                    if seg_sum is None:
                        seg_sum = sm
                    else:
                        seg_sum, r = compose(seg_sum, sm)
                        seg_links += r
                if seg_sum is None:
                    continue
                strip_links += seg_links
                if strip_sum is None:
                    strip_sum = seg_sum
                else:
                    strip_sum, r = compose(strip_sum, seg_sum)
                    strip_links += r
            strip_links += popc(strip_sum.OE & strip_sum.T2 & (~strip_sum.T3 & M32))
            total_links += strip_links
    px = np.unpackbits(bits, axis=1)[:, :wc].astype(np.int64)
    prev = np.vstack([np.zeros((1, wc), dtype=np.int64), px[:-1]])
    runs = int(((px == 1) & (prev == 0)).sum())
    return runs, total_links
