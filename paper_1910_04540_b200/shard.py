"""Multi-GPU sharding of the quantizer hot path (one process per GPU).

The per-element result depends only on (x_i, format, mode, seed, call, the
GLOBAL flat index i) -- proj/src/quant_ops.cpp:13-31 draws the variate of
element i as uniform_variate(seed, call, i) -- so a tensor sharded into
contiguous flat ranges (or whole rows, for per-row block formats) is
quantized by each rank independently with index_base = the shard's first
global index, bit-identical to the single-GPU result, with no communication
on the data path.  torch.distributed (NCCL) is used only to gather results
for verification and to take the max of per-rank timings.
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
    tensor on one GPU (fused_block, quant_ops.cpp:68-115)."""
    import torch.distributed as dist
    fmt = spec.format
    if fmt.block_dim == 0:
        raise ValueError("block_dim 0: blocks are whole dim-0 slices; shard by rows "
                         "(block_unit) and quantize locally, no exchange needed")
    m = q.block_absmax(x_local, fmt)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    return q.quantize_block_apply(x_local, spec, call, m, index_base=index_base)


def gather(y_local, group=None):
    """Verification only: all_gather the shards (equal sizes) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [torch.empty_like(y_local) for _ in range(world)]
    dist.all_gather(parts, y_local.contiguous(), group=group)
    return torch.cat([p.reshape(-1) for p in parts])
