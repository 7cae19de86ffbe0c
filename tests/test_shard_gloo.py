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
    # blocks spanning shards: the exchange step of
    # shard.quantize_block_split -- local maxima, ONE all_reduce(MAX), apply
    # with the global maxima and the shard's index_base -- here with the
    # oracle's two halves of fused_block in place of the device kernels
    G = (6, 5, 7)  # global shape, sharded along dim 0
    per = (G[0] // world) * G[1] * G[2]
    xs = o.random_uniform(per, 4, 0, -3.0, 3.0, index_base=rank * per)
    xs = xs.reshape(G[0] // world, G[1], G[2])
    xs[0, 2, 3] = 50.0 if rank == 1 else xs[0, 2, 3]  # a block max on rank 1 only
    split = []
    for dim in (None, 1, 2):
        st, mx = o.reduce_max_abs(xs, dim)
        mt = torch.from_numpy(mx.copy())
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        st, ys = o.quantize_block_given_max(xs, block_fmt(8, dim), STOCHASTIC, mt.numpy(),
                                            seed=11, call=4, index_base=rank * per)
        gl = [None] * world
        dist.all_gather_object(gl, (rank, ys, xs))
        split.append(gl)
    if rank == 0:
        for dim, gl in zip((None, 1, 2), split):
            gl = sorted(gl, key=lambda t: t[0])
            wx = np.concatenate([g[2] for g in gl])
            st, want = o.quantize(wx, block_fmt(8, dim), STOCHASTIC, seed=11, call=4)
            got = np.concatenate([g[1] for g in gl])
            ok.append(bool(st == 0 and np.array_equal(bits(got), bits(want))))
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
    assert ok == [True, True, True, True, True]
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


def test_block_split_refuses_row_blocks():
    # block_dim 0 blocks are whole dim-0 slices: shard by rows, no exchange
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.shard import block_unit, quantize_block_split
    spec = q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode.NearestEven, 1)
    with pytest.raises(ValueError):
        quantize_block_split(q, None, spec, 0, 0)
    assert block_unit((4, 5, 6), 0) == 30
    assert block_unit((4, 5, 6), None) is None and block_unit((4, 5, 6), 2) is None
