"""Column-strip sharding of the yCHG pass across the GPUs of one node (SURVEY §8e,
BASELINE config 5: 65536^2 on 2/4/8 B200), one process per GPU.

Columns are independent (one result slot per column, runscan.cpp:14-17), and the
reference's own parallelism is exactly this column chunking (for_column_chunks,
runscan.cpp:18-34), so the mask is cut into vertical strips, one per rank:

* rank r counts columns [c0, c1) (multiples of 1024: whole strips of the device
  layout) and holds one extra byte column on the right (the halo) so that the K3
  pair step sees column c1 for the pair (c1-1, c1);
* per step the strip counts are all-gathered (NCCL over NVLink on GPUs, gloo in
  the CPU tests) into the global count array, and (runs, links) all-reduced;
* the boundary flag of a strip's first column needs counts[c0-1] from the left
  neighbour (runscan.cpp:147-149): the global boundary list is therefore K2 over
  the gathered counts (``detect_boundaries_device`` on GPUs, ``merge_boundaries``
  here for the tests), which is the strip-edge fix-up;
* hyperedges = sum(runs) - sum(links).

``bench.py`` drives ``StripExchange`` with device tensors and NCCL for N > 1;
``tests/test_multigpu.py`` drives the same class with CPU tensors and gloo
(world 2 and 3), the strips computed by the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Strip:
    rank: int
    c0: int          # first counted column
    c1: int          # one past the last counted column
    halo_cols: int   # columns present to the right of c1 (0 on the last strip, else <= 8)

    @property
    def width_cnt(self) -> int:
        return self.c1 - self.c0

    @property
    def width_img(self) -> int:
        return self.c1 - self.c0 + self.halo_cols


def plan_strips(width: int, world: int, align: int = 1024) -> list[Strip]:
    """Equal strips, boundaries on multiples of `align` columns (a multiple of 8)."""
    assert align % 8 == 0 and world >= 1
    units = (width + align - 1) // align
    strips = []
    for r in range(world):
        u0, u1 = (r * units) // world, ((r + 1) * units) // world
        c0, c1 = min(width, u0 * align), min(width, u1 * align)
        strips.append(Strip(r, c0, c1, min(8, width - c1)))
    return strips


def strip_bits(bits: np.ndarray, width: int, s: Strip) -> np.ndarray:
    """Packed rows of columns [c0, c1 + halo) of a host image (c0 is a multiple of 8)."""
    b0 = s.c0 // 8
    b1 = (s.c0 + s.width_img + 7) // 8
    out = np.ascontiguousarray(bits[:, b0:b1])
    tail = s.width_img % 8  # zero bits of the last byte beyond the strip's image width
    if tail and out.shape[1]:
        out[:, -1] &= np.uint8((0xFF << (8 - tail)) & 0xFF)
    return out


def merge_boundaries(counts: np.ndarray) -> np.ndarray:
    """detect_boundary_columns on the gathered counts (runscan.cpp:145-153)."""
    prev = np.concatenate([[0], counts[:-1]]) if counts.size else counts
    return np.nonzero(counts != prev)[0].astype(np.int32)


class StripExchange:
    """The per-step exchange of one rank over torch.distributed: all-gather of the
    strip counts into the global count array (padded to the widest strip when the
    strips differ), all-reduce (sum) of the int64 pair (runs, links) in place.
    Buffers live on `device` (a CUDA device for NCCL, "cpu" for gloo)."""

    def __init__(self, dist, strips: list[Strip], rank: int, device="cpu"):
        import torch

        self.dist, self.strips, self.rank = dist, strips, rank
        self.world = len(strips)
        self.width = strips[-1].c1
        self.wmax = max(s.width_cnt for s in strips)
        self.equal = all(s.width_cnt == self.wmax for s in strips)
        self.send = torch.zeros(self.wmax, dtype=torch.int32, device=device)
        self.gathered = torch.zeros(self.world * self.wmax, dtype=torch.int32, device=device)
        self.counts = (self.gathered[: self.width] if self.equal
                       else torch.zeros(self.width, dtype=torch.int32, device=device))

    def run(self, counts_local, sums):
        """counts_local: this rank's width_cnt int32 counts; sums: int64 [runs, links],
        all-reduced in place.  Returns the global counts (a view owned by self)."""
        s = self.strips[self.rank]
        src = counts_local
        if not self.equal:
            self.send[: s.width_cnt].copy_(counts_local)
            src = self.send
        self.dist.all_gather_into_tensor(self.gathered, src)
        self.dist.all_reduce(sums)
        if not self.equal:
            for r, t in enumerate(self.strips):
                self.counts[t.c0:t.c1].copy_(self.gathered[r * self.wmax:r * self.wmax + t.width_cnt])
        return self.counts


def run_sharded(bits: np.ndarray, width: int, height: int, compute, dist=None):
    """One sharded pass over a host image (the CPU tests' entry point).
    `compute(sub_bits, width_img, width_cnt, height) -> (counts[width_cnt], links)`.
    Returns (counts, boundaries, total_runs, links, hyperedges) on every rank."""
    import torch

    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    strips = plan_strips(width, world)
    s = strips[rank]
    counts, links = compute(strip_bits(bits, width, s), s.width_img, s.width_cnt, height)
    local = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int32))
    sums = torch.tensor([int(np.asarray(counts, dtype=np.int64).sum()), int(links)], dtype=torch.int64)
    if dist:
        full = StripExchange(dist, strips, rank).run(local, sums).numpy().copy()
    else:
        full = local.numpy().copy()
    runs, lk = (int(v) for v in sums.tolist())
    return full, merge_boundaries(full), runs, lk, runs - lk
