"""Column-strip sharding of the yCHG pass across the GPUs of one node.

Columns are independent (one result slot per column, runscan.cpp:14-17), so the
mask is cut into vertical strips, one per rank:

* rank r counts columns [c0, c1) (c0, c1 multiples of 8, so strips are whole
  bytes of every packed row) and holds ONE extra byte column on the right (the
  halo) so that the K3 pair step sees column c1 for the pair (c1-1, c1);
* the per-column counts are all-gathered (NCCL over NVLink on GPUs, gloo in the
  CPU tests) -- every rank then owns the full count array;
* the boundary flag of a strip's first column needs counts[c0-1] from the
  left neighbour: after the all-gather it is simply read;
* links and Σcounts are all-reduced (sum); hyperedges = Σcounts - Σlinks.

The strip computation itself is injected (`compute`): the sm_100a kernels through
the C ABI in production (bench.py), the oracle restatement in the CPU tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Strip:
    rank: int
    c0: int          # first counted column
    c1: int          # one past the last counted column
    halo_cols: int   # columns present to the right of c1 (0 on the last strip, else 8)

    @property
    def width_cnt(self) -> int:
        return self.c1 - self.c0

    @property
    def width_img(self) -> int:
        return self.c1 - self.c0 + self.halo_cols


def plan_strips(width: int, world: int, align: int = 1024) -> list[Strip]:
    """Equal strips, boundaries on multiples of `align` columns (>= 8, a multiple of 8)."""
    assert align % 8 == 0 and world >= 1
    units = (width + align - 1) // align
    strips = []
    for r in range(world):
        u0, u1 = (r * units) // world, ((r + 1) * units) // world
        c0, c1 = min(width, u0 * align), min(width, u1 * align)
        halo = min(8, width - c1)
        strips.append(Strip(r, c0, c1, halo))
    return strips


def strip_bits(bits: np.ndarray, width: int, s: Strip) -> np.ndarray:
    """Packed rows of columns [c0, c1 + halo) (c0 is a multiple of 8 -> a byte slice)."""
    b0 = s.c0 // 8
    b1 = (s.c0 + s.width_img + 7) // 8
    out = np.ascontiguousarray(bits[:, b0:b1])
    # zero bits of the last byte that lie beyond the strip's image width
    tail = s.width_img % 8
    if tail and out.shape[1]:
        out[:, -1] &= np.uint8((0xFF << (8 - tail)) & 0xFF)
    return out


def merge_boundaries(counts: np.ndarray) -> np.ndarray:
    """detect_boundary_columns on the gathered counts (runscan.cpp:145-153)."""
    prev = np.concatenate([[0], counts[:-1]]) if counts.size else counts
    return np.nonzero(counts != prev)[0].astype(np.int32)


def run_sharded(bits: np.ndarray, width: int, height: int, compute, dist=None):
    """One sharded pass.  `compute(sub_bits, width_img, width_cnt, height) ->
    (counts[width_cnt] int32, links int)`; `dist` is torch.distributed (or None
    for a single process).  Returns (counts, boundaries, total_runs, links,
    hyperedges) on every rank."""
    import torch

    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    strips = plan_strips(width, world)
    s = strips[rank]
    sub = strip_bits(bits, width, s)
    counts, links = compute(sub, s.width_img, s.width_cnt, height)
    # all-gather the per-column counts (padded to the widest strip)
    wmax = max(t.width_cnt for t in strips)
    buf = torch.zeros(wmax, dtype=torch.int32)
    buf[: s.width_cnt] = torch.from_numpy(np.asarray(counts, dtype=np.int32))
    if dist:
        gathered = [torch.zeros(wmax, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gathered, buf)
        lk = torch.tensor([int(links)], dtype=torch.int64)
        dist.all_reduce(lk)
        links_total = int(lk.item())
    else:
        gathered = [buf]
        links_total = int(links)
    full = np.concatenate([g.numpy()[: t.width_cnt] for g, t in zip(gathered, strips)])
    total = int(full.sum())
    return full, merge_boundaries(full), total, links_total, total - links_total
