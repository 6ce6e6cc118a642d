"""Column-strip sharding of the yCHG pass across the GPUs of one node (SURVEY §8e,
BASELINE config 5: 65536^2 on 2/4/8 B200), one process per GPU.

Columns are independent (one result slot per column, runscan.cpp:14-17), and the
reference's own parallelism is exactly this column chunking (for_column_chunks,
runscan.cpp:18-34), so the mask is cut into vertical strips, one per rank:

* rank r counts columns [c0, c1) (multiples of 1024: whole strips of the device
  layout) and holds one extra byte column on the right (the halo) so that the K3
  pair step sees column c1 for the pair (c1-1, c1);
* per step ONE all-gather (NCCL over NVLink on GPUs, gloo in the CPU tests)
  collects every strip's counts AND its (runs, links) totals (written by the
  scan next to its counts), from which the global count array and the sums
  follow;
* the boundary flag of a strip's first column needs counts[c0-1] from the left
  neighbour (runscan.cpp:147-149): the global boundary list is therefore K2 over
  the gathered counts (``detect_boundaries_device`` on GPUs, ``merge_boundaries``
  here for the tests), which is the strip-edge fix-up;
* hyperedges = sum(runs) - sum(links).

``bench.py`` drives ``StripExchange`` with device tensors and NCCL for N > 1
(then ``assemble_strips_device``: global counts + boundary list + sums in two
small kernels);
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
    """The per-step exchange of one rank over torch.distributed (NCCL on GPUs, gloo
    in the CPU tests): ONE all-gather.  Every rank contributes a segment of
    `seg` int32 -- its strip's counts at [0, width_cnt) (the scan writes them
    there directly) and its ychg_totals {total_runs, links, hyperedges,
    n_boundaries} (4 int64) at int offset `tot_off` -- so the global counts AND
    the (runs, links) sums follow from the gathered buffer without a second
    collective (`assemble_strips_device` on GPUs, `host_assemble` here)."""

    def __init__(self, dist, strips: list[Strip], rank: int, device="cpu"):
        import torch

        self.dist, self.strips, self.rank = dist, strips, rank
        self.world = len(strips)
        self.width = strips[-1].c1
        wmax = max(s.width_cnt for s in strips)
        self.tot_off = (wmax + 1) // 2 * 2          # 8-byte aligned ychg_totals
        self.seg = self.tot_off + 8
        self.c0 = [s.c0 for s in strips] + [self.width]
        self.send = torch.zeros(self.seg, dtype=torch.int32, device=device)
        self.gathered = torch.zeros(self.world * self.seg, dtype=torch.int32, device=device)

    @property
    def totals_view(self):
        """This rank's ychg_totals slot in the send buffer (4 int64)."""
        return self.send[self.tot_off:self.tot_off + 8].view(__import__("torch").int64)

    def run(self):
        self.dist.all_gather_into_tensor(self.gathered, self.send)
        return self.gathered

    def host_assemble(self):
        """(global counts, total runs, links) from the gathered buffer (host copy)."""
        g = self.gathered.cpu().numpy()
        counts = np.concatenate([g[r * self.seg:r * self.seg + (self.c0[r + 1] - self.c0[r])]
                                 for r in range(self.world)])
        tot = np.stack([g[r * self.seg + self.tot_off:r * self.seg + self.tot_off + 8].view(np.int64)
                        for r in range(self.world)])
        return counts, int(tot[:, 0].sum()), int(tot[:, 1].sum())


def run_sharded(bits: np.ndarray, width: int, height: int, compute, dist=None):
    """One sharded pass over a host image (the CPU tests' entry point).
    `compute(sub_bits, width_img, width_cnt, height) -> (counts[width_cnt], links)`.
    Returns (counts, boundaries, total_runs, links, hyperedges) on every rank."""
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    strips = plan_strips(width, world)
    s = strips[rank]
    counts, links = compute(strip_bits(bits, width, s), s.width_img, s.width_cnt, height)
    counts = np.ascontiguousarray(counts, dtype=np.int32)
    runs = int(counts.astype(np.int64).sum())
    if not dist:
        return counts.copy(), merge_boundaries(counts), runs, int(links), runs - int(links)
    import torch

    x = StripExchange(dist, strips, rank)
    x.send[: s.width_cnt] = torch.from_numpy(counts)
    x.totals_view[:] = torch.tensor([runs, int(links), runs - int(links), 0], dtype=torch.int64)
    x.run()
    full, runs_all, links_all = x.host_assemble()
    return full, merge_boundaries(full), runs_all, links_all, runs_all - links_all
