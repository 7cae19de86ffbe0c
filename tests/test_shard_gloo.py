"""World-size-2 (gloo, CPU) tests of the multi-GPU sharding logic.

Each rank quantizes its shard of a global tensor with index_base = the
shard's first global index -- here through the CPU oracle, since this host
has no GPU; on B200 the same shard_range/index_base drive lpq_quantize -- and
the gathered shards must equal the single-process result bit for bit.

The shard module's own functions run here with two ranks: quantize_block_split
(its max exchange and its collective error semantics) is driven through a
stand-in quantizer module whose block_absmax / quantize_block_apply are the
oracle's two halves of fused_block; gemm_rows, broadcast_operand and binpack
are exercised as bench.py uses them for C4 and C5.
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


class _OracleQ:
    """The two device entry points quantize_block_split calls, restated by
    the oracle (reduce_max_abs + the apply pass with given maxima)."""

    def __init__(self, o):
        from paper_1910_04540_b200 import InvalidInputError
        self.o = o
        self.InvalidInputError = InvalidInputError

    def block_absmax(self, x, fmt):
        st, mx = self.o.reduce_max_abs(x.numpy(), fmt.block_dim)
        return torch.from_numpy(mx.view(np.int32).copy())

    def quantize_block_apply(self, x, spec, call, m, index_base=0):
        st, y = self.o.quantize_block_given_max(
            x.numpy(), block_fmt(spec.format.wl, spec.format.block_dim), int(spec.mode),
            m.numpy().view(np.float32), seed=spec.seed, call=call, index_base=index_base)
        if st != 0:
            raise self.InvalidInputError("quantize: non-finite input")
        return torch.from_numpy(y)


def _shard_module_checks(rank, world, o, ok):
    """shard.quantize_block_split / gemm_rows / broadcast_operand / binpack
    with two real ranks."""
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.shard import (binpack, broadcast_operand, gemm_rows,
                                             quantize_block_split, shard_range)
    from oracle_lib import float_fmt
    fq = _OracleQ(o)
    G = (8, 3, 5)
    per = (G[0] // world) * G[1] * G[2]
    xs = o.random_uniform(per, 14, 0, -2.0, 2.0, index_base=rank * per).reshape(-1, *G[1:])
    if rank == 1:
        xs[1, 0, 4] = -77.0  # a block maximum held by rank 1 only
    res = []
    for dim in (None, 1, 2):
        spec = q.QuantSpec(q.BlockFloatFormat(8, dim), q.RoundingMode.Stochastic, 31)
        y = quantize_block_split(fq, torch.from_numpy(xs.copy()), spec, 6, rank * per)
        gl = [None] * world
        dist.all_gather_object(gl, (rank, y.numpy(), xs))
        res.append(gl)
    # a NaN on rank 1 only: block maxima skip it, so only rank 1's apply pass
    # sees it -- and every rank must raise
    xn = xs.copy()
    if rank == 1:
        xn[0, 1, 1] = np.nan
    spec = q.QuantSpec(q.BlockFloatFormat(8), q.RoundingMode.NearestEven, 1)
    raised = False
    try:
        quantize_block_split(fq, torch.from_numpy(xn), spec, 0, rank * per)
    except q.InvalidInputError:
        raised = True
    flags = [None] * world
    dist.all_gather_object(flags, raised)
    # GEMM row shards with B broadcast from rank 0 (per-op GEMM, stochastic,
    # global variate index via row_base)
    M, K, N = 7, 9, 6
    a = o.random_uniform(M * K, 21, 0, -1.0, 1.0).reshape(M, K)
    b = (o.random_uniform(K * N, 22, 0, -1.0, 1.0).reshape(K, N) if rank == 0
         else np.zeros((K, N), np.float32))
    bt = broadcast_operand(torch.from_numpy(b))
    lo, hi = gemm_rows(M, rank, world)
    f = float_fmt(5, 2)
    st, c = o.quant_gemm(np.ascontiguousarray(a[lo:hi]), bt.numpy(), f, f, STOCHASTIC,
                         seed=5, call=3, row_base=lo)
    gl = [None] * world
    dist.all_gather_object(gl, (lo, c))
    # bin-packing plan: identical on every rank, a partition of the items
    w = [int(v) for v in (o.random_uniform(40, 33, 0, 1.0, 1000.0) ** 2)]
    plan = binpack(w, world)
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    if rank == 0:
        for dim, g in zip((None, 1, 2), res):
            g = sorted(g, key=lambda t: t[0])
            wx = np.concatenate([t[2] for t in g])
            st, want = o.quantize(wx, block_fmt(8, dim), STOCHASTIC, seed=31, call=6)
            ok.append(bool(st == 0 and np.array_equal(
                bits(np.concatenate([t[1] for t in g])), bits(want))))
        ok.append(flags == [True] * world)
        bw = o.random_uniform(K * N, 22, 0, -1.0, 1.0).reshape(K, N)
        st, want = o.quant_gemm(a, bw, f, f, STOCHASTIC, seed=5, call=3)
        got = np.concatenate([t[1] for t in sorted(gl, key=lambda t: t[0])])
        ok.append(bool(np.array_equal(bits(got), bits(want))))
        flat = sorted(i for p in plan for i in p)
        loads = [sum(w[i] for i in p) for p in plan]
        ok.append(plans[0] == plans[1] and flat == list(range(len(w)))
                  and max(loads) - min(loads) <= max(w))
        ok.append(shard_range(M, 1, world) == gemm_rows(M, 1, world))


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
    _shard_module_checks(rank, world, o, ok)
    if rank == 0:
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
    assert ok == [True] * 12, ok
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
