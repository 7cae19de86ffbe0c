"""Multi-GPU sharding of the quantizer hot path (one process per GPU).

The per-element result depends only on (x_i, format, mode, seed, call, the
GLOBAL flat index i) -- proj/src/quant_ops.cpp:13-31 draws the variate of
element i as uniform_variate(seed, call, i) -- so a tensor sharded into
contiguous flat ranges (or whole rows, for per-row block formats) is
quantized by each rank independently with index_base = the shard's first
global index, bit-identical to the single-GPU result, with no communication
on the data path.  torch.distributed (NCCL) is used only to gather results
for verification and to take the max of per-rank timings -- plus the two
real exchanges of SURVEY §8(e): the block-maximum all_reduce of a block that
spans shards (quantize_block_split) and the one broadcast of the replicated
GEMM operand B (broadcast_operand).

Partition plans (pure functions, tested with world-size-2 gloo):
    shard_range   contiguous flat ranges (elementwise formats, whole rows)
    gemm_rows     output-row blocks of a GEMM (A and C rows, row_base)
    binpack       a list of work items (e.g. the C5 sweep's quantizations)
                  spread over ranks by bytes
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int, unit: int = 1):
    """[lo, hi) of the flat range rank owns: contiguous, aligned to `unit`
    (e.g. a row length, so no block straddles two ranks), sizes differing by
    at most one unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if unit < 1 or n % unit:
        raise ValueError("n must be a multiple of unit")
    units = n // unit
    base, extra = divmod(units, world)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return lo_u * unit, hi_u * unit


def block_unit(shape, block_dim):
    """Elements per shardable unit for a block format: a whole block row
    (block_dim == 0 on any shape); None when blocks span the tensor (whole
    tensor / inner dims), which needs the max-exchange step of
    quantize_block_split instead."""
    if block_dim is None:
        return None
    if block_dim == 0:
        n = 1
        for s in shape[1:]:
            n *= int(s)
        return n
    return None


def quantize_shard(q, x_local, spec, call, index_base):
    """Quantize this rank's shard (device tensor) of a larger tensor."""
    return q.quantize_fused_at(x_local, spec, call, index_base=index_base)


def quantize_block_split(q, x_local, spec, call, index_base, group=None):
    """A block format whose blocks span shards: the whole
    tensor (block_dim None; any flat sharding) or blocks along dim d >= 1 of a
    tensor sharded along dim 0 (whole dim-0 slices per rank).  One exchange
    step: each rank reduces its part of every block maximum on the device
    (lpq_block_absmax), the [extent] maxima are combined with ONE
    all_reduce(MAX) over NCCL (non-negative fp32 bits order like the floats),
    and each rank quantizes its shard with the global maxima
    (lpq_quantize_block_apply) -- bit-identical to quantizing the gathered
    tensor on one GPU (fused_block, quant_ops.cpp:68-115).

    Errors are collective, as the whole-tensor call throws as a unit
    (quant_ops.cpp:28-29): a non-finite element on any rank (block maxima skip
    NaN, so only the rank holding it sees it in the apply pass) raises
    InvalidInputError on EVERY rank, after one all_reduce(MAX) of the ranks'
    error flags.  `q` is the quantizer module (the package), passed in so the
    exchange logic is testable without a GPU."""
    import torch
    import torch.distributed as dist
    fmt = spec.format
    if fmt.block_dim == 0:
        raise ValueError("block_dim 0: blocks are whole dim-0 slices; shard by rows "
                         "(block_unit) and quantize locally, no exchange needed")
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    m = q.block_absmax(x_local, fmt)
    if multi:
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    err, y = None, None
    try:
        y = q.quantize_block_apply(x_local, spec, call, m, index_base=index_base)
    except q.InvalidInputError as e:
        err = e
    if multi:
        flag = torch.tensor([0 if err is None else 1], dtype=torch.int32, device=m.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        if err is None and int(flag.item()):
            raise q.InvalidInputError(
                "quantize: non-finite input on another rank (block split)")
    if err is not None:
        raise err
    return y


def gemm_rows(m: int, rank: int, world: int):
    """[lo, hi) of the output rows rank owns in a GEMM sharded by rows (A and
    C row blocks; B replicated).  The per-op GEMM's variate index of output
    (i, j) is the GLOBAL i*N + j, so rank passes row_base = lo and its rows
    equal the single-GPU result's bit for bit."""
    return shard_range(m, rank, world)


def broadcast_operand(t, src: int = 0, group=None):
    """The replicated GEMM operand B: ONE broadcast from `src` (NCCL over
    NVLink on B200), outside any timed region.  Returns t (filled in place)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(t, src=src, group=group)
    return t


def binpack(weights, world: int):
    """Spread work items over `world` ranks by weight (e.g. algorithmic bytes
    of each quantization in the C5 sweep): longest-processing-time greedy --
    items in descending weight, each to the currently lightest rank (ties to
    the lower rank), deterministic, so every rank computes the same plan with
    no communication.  Returns one list of item indices per rank, each in
    ascending item order (so a rank's launches keep the sweep's order)."""
    if world < 1:
        raise ValueError("bad world")
    load = [0] * world
    plan = [[] for _ in range(world)]
    for i in sorted(range(len(weights)), key=lambda k: (-weights[k], k)):
        r = min(range(world), key=lambda k: (load[k], k))
        plan[r].append(i)
        load[r] += weights[i]
    return [sorted(p) for p in plan]


def gather(y_local, group=None):
    """Verification only: all_gather the shards (equal sizes) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.empty_like(y_local) for _ in range(world)]
    dist.all_gather(parts, y_local.contiguous(), group=group)
    return torch.cat([p.reshape(-1) for p in parts])
