"""CPU: the column-strip sharding host logic (paper_1307_2560_b200/multigpu.py: plan_strips,
StripExchange) over torch.distributed gloo with world_size 2 and 3, strips computed by the
oracle; bench.py drives the same StripExchange with NCCL and the C ABI per GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import Oracle, Spec
from paper_1307_2560_b200.multigpu import merge_boundaries, plan_strips, run_sharded, strip_bits


def oracle_strip(orc):
    def compute(sub, width_img, width_cnt, height):
        counts = orc.counts(sub, width_img)[:width_cnt]
        links = int(orc.pair_links(sub, width_img)[:width_cnt].sum())
        return counts, links
    return compute


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        bits = orc.synth(spec)
        out = run_sharded(bits, spec.width, spec.height, oracle_strip(orc), dist)
        q.put((rank, out[0].tolist(), out[1].tolist(), out[2], out[3], out[4]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec", [(2, Spec.random(3000, 200, 0.5, 17)), (3, Spec.checker(5000, 64, 3)),
                                        (2, Spec.hbands(2100, 300, 7)), (3, Spec.random(1500, 90, 0.3, 5))])
def test_sharded_matches_oracle(orc, world, spec):
    bits = orc.synth(spec)
    counts = orc.counts(bits, spec.width)
    he, runs, links = orc.hyperedges(bits, spec.width)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, c, b, total, lk, h in res:
        assert c == counts.tolist()
        assert b == orc.boundaries(counts).tolist()
        assert (total, lk, h) == (runs, links, he)


def test_plan_strips_cover_and_align():
    for width in (1, 7, 1024, 1025, 21000, 65536):
        for world in (1, 2, 3, 8):
            st = plan_strips(width, world)
            assert st[0].c0 == 0 and st[-1].c1 == width
            for a, b in zip(st, st[1:]):
                assert a.c1 == b.c0 and a.c1 % 8 == 0
                assert a.halo_cols == min(8, width - a.c1)
            assert st[-1].halo_cols == 0


def test_strip_bits_halo(orc):
    spec = Spec.random(2500, 40, 0.5, 9)
    bits = orc.synth(spec)
    full = np.unpackbits(bits, axis=1)[:, :2500]
    for s in plan_strips(2500, 2):
        sub = strip_bits(bits, 2500, s)
        got = np.unpackbits(sub, axis=1)[:, : s.width_img]
        assert np.array_equal(got, full[:, s.c0:s.c0 + s.width_img])


def test_merge_boundaries():
    assert merge_boundaries(np.array([1, 2, 2, 2, 1])).tolist() == [0, 1, 4]
    assert merge_boundaries(np.array([0, 0])).tolist() == []
