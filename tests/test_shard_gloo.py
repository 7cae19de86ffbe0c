"""World-size-2 (gloo, CPU) tests of the multi-GPU sharding logic.

Each rank quantizes its shard of a global tensor with index_base = the
shard's first global index -- here through the CPU oracle, since this host
has no GPU; on B200 the same shard_range/index_base drive lpq_quantize -- and
the gathered shards must equal the single-process result bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_lib import STOCHASTIC, NEAREST_EVEN, Oracle, bits, block_fmt, fixed_fmt


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_04540_b200.shard import shard_range
    o = Oracle()
    ok = []
    # elementwise: fixed(8,4) stochastic over a global tensor of 10_001 elements
    n = 10_001
    lo, hi = shard_range(n, rank, world)
    x = o.random_uniform(hi - lo, 2, 0, -10.0, 10.0, index_base=lo)
    st, y = o.quantize(x, fixed_fmt(8, 4), STOCHASTIC, seed=0x15EED, call=0, index_base=lo)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, y))
    # per-row block format: shards aligned to rows
    R, L = 37, 64
    lo_r, hi_r = shard_range(R * L, rank, world, unit=L)
    xb = o.random_uniform(hi_r - lo_r, 3, 0, -1.0, 1.0, index_base=lo_r).reshape(-1, L)
    st, yb = o.quantize(xb, block_fmt(8, 0), STOCHASTIC, seed=9, call=2, index_base=lo_r)
    parts_b = [None] * world
    dist.all_gather_object(parts_b, (lo_r, yb))
    if rank == 0:
        whole_x = o.random_uniform(n, 2, 0, -10.0, 10.0)
        st, whole = o.quantize(whole_x, fixed_fmt(8, 4), STOCHASTIC, seed=0x15EED, call=0)
        got = np.concatenate([p[1] for p in sorted(parts, key=lambda t: t[0])])
        ok.append(bool(np.array_equal(bits(got), bits(whole))))
        wx = o.random_uniform(R * L, 3, 0, -1.0, 1.0).reshape(R, L)
        st, wb = o.quantize(wx, block_fmt(8, 0), STOCHASTIC, seed=9, call=2)
        gb = np.concatenate([p[1] for p in sorted(parts_b, key=lambda t: t[0])])
        ok.append(bool(np.array_equal(bits(gb), bits(wb))))
        # max-over-ranks timing reduction, as bench.py does
        t = torch.tensor([1.0 + rank])
        out.put(ok)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put(float(t.item()))
    dist.destroy_process_group()


def test_sharded_equals_whole_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok == [True, True]
    assert tmax == 2.0


@pytest.mark.parametrize("n,world,unit", [(10, 3, 1), (4096 * 7, 4, 4096), (5, 8, 1)])
def test_shard_range_partitions(n, world, unit):
    from paper_1910_04540_b200.shard import shard_range
    spans = [shard_range(n, r, world, unit) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    assert all((hi - lo) % unit == 0 for lo, hi in spans)
    sizes = [hi - lo for lo, hi in spans]
    assert max(sizes) - min(sizes) <= unit
