"""Host-side mirror of the reference quantizer API (lpsim, C++) over liblpq.

Names, argument meaning and error behaviour follow
proj/include/lpsim/quant_ops.hpp:14-46 and formats.hpp:14-80:

    spec = QuantSpec(FixedFormat(8, 4), RoundingMode.Stochastic, seed=5)
    q = quantize_fused(t, spec)          # advances spec.call_counter (stochastic)
    q = quantize_fused_at(t, spec, 7)    # pure form
    c = quantized_matmul(a, b, spec)     # Q(matmul(a, b)), fused epilogue
    c = quant_gemm(a, b, fmt_mul, fmt_add, mode)   # per-op-rounded GEMM

A tensor is either a CUDA torch.Tensor (device path: lpq_quantize on the
current torch stream, synchronised only to read the status word) or a numpy
array / host torch tensor (host path: lpq_quantize_host, which streams it
through the GPU with the copies overlapped).  Every path runs the sm_100a
kernels; there is no CPU implementation behind this module.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from ._lib import (FormatError, InvalidInputError, InvalidValueError,
                   LpqFormat, ShapeError, UnsupportedFormatError, check, lib,
                   shape_array)

try:  # torch is plumbing for device memory and streams, not a dependency of the math
    import torch
except Exception:  # pragma: no cover
    torch = None


class RoundingMode(enum.IntEnum):
    """formats.hpp:14-19 (same order)."""
    Stochastic = 0
    NearestEven = 1
    NearestAway = 2
    NearestTowardZero = 3


@dataclass(frozen=True)
class FloatFormat:
    """formats.hpp:36-49: exp_bits exponent bits, man_bits mantissa bits,
    no denormals/inf/nan, top exponent code normal, max_exp capped at 127."""
    exp_bits: int = 8
    man_bits: int = 23

    def bias(self):
        return (1 << (self.exp_bits - 1)) - 1

    def min_exp(self):
        return 1 - self.bias()

    def max_exp(self):
        return min((1 << self.exp_bits) - 1 - self.bias(), 127)

    def max_value(self):
        return float(np.ldexp(2.0 - np.ldexp(1.0, -self.man_bits), self.max_exp()))

    def c(self):
        return LpqFormat(0, self.exp_bits, self.man_bits, 0, 0, 0, 0, -1)


@dataclass(frozen=True)
class FixedFormat:
    """formats.hpp:54-67: k * 2^-fl, k a wl-bit two's-complement integer."""
    wl: int = 8
    fl: int = 4
    symmetric: bool = False
    saturate: bool = True

    def step(self):
        return float(np.ldexp(1.0, -self.fl))

    def k_max(self):
        return (1 << (self.wl - 1)) - 1

    def k_min(self):
        return -self.k_max() if self.symmetric else -(1 << (self.wl - 1))

    def c(self):
        return LpqFormat(1, 0, 0, self.wl, self.fl, int(self.symmetric),
                         int(self.saturate), -1)


@dataclass(frozen=True)
class BlockFloatFormat:
    """formats.hpp:73-78: shared exponent per block; block_dim None = whole
    tensor, d = slices at a fixed index along dimension d."""
    wl: int = 8
    block_dim: Optional[int] = None

    def c(self):
        d = -1 if self.block_dim is None else int(self.block_dim)
        if self.block_dim is not None and self.block_dim < 0:
            d = -2  # rejected by validate like formats.hpp:105-107
        return LpqFormat(2, 0, 0, self.wl, 0, 0, 0, d)


NumberFormat = Union[FloatFormat, FixedFormat, BlockFloatFormat]


@dataclass
class QuantSpec:
    """quant_ops.hpp:14-19."""
    format: NumberFormat = field(default_factory=FloatFormat)
    mode: RoundingMode = RoundingMode.NearestEven
    seed: int = 0
    call_counter: int = 0


def validate(fmt: NumberFormat) -> None:
    """formats.hpp:82-112 (via lpq_validate_format)."""
    check(lib.lpq_validate_format(C.byref(fmt.c())), "validate")


def pass_count() -> int:
    return int(lib.lpq_pass_count())


def reset_pass_count() -> None:
    lib.lpq_reset_pass_count()


def launch_count() -> int:
    return int(lib.lpq_launch_count())


# ---- device plumbing ---------------------------------------------------------

_status_bufs = {}
_ws_bufs = {}
_tls = threading.local()


def _is_device(t) -> bool:
    return torch is not None and isinstance(t, torch.Tensor) and t.is_cuda


def _stream_key(device):
    # status words and workspaces are per (device, stream): calls on
    # different streams may run concurrently and must not share them
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return idx, torch.cuda.current_stream(idx).cuda_stream


def _status_buf(device):
    key = _stream_key(device)
    buf = _status_bufs.get(key)
    if buf is None:
        buf = torch.zeros(1, dtype=torch.int32, device=device)
        _status_bufs[key] = buf
    return buf


def _workspace(device, nbytes):
    if nbytes == 0:
        return None
    key = _stream_key(device)
    buf = _ws_bufs.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _ws_bufs[key] = buf
    return buf


def _stream_ptr(device):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def fetch_status(device=None) -> None:
    """Synchronise the current stream and raise if a kernel flagged an error."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    st = lib.lpq_status_fetch(C.c_void_p(_status_buf(device).data_ptr()),
                              _stream_ptr(device))
    check(st, "quantize")


# ---- quantize ----------------------------------------------------------------

def _check_out(out, like):
    """An `out` tensor is written through a raw pointer: it must be a
    contiguous fp32 CUDA tensor of the input's element count on its device."""
    if (not isinstance(out, torch.Tensor) or out.dtype != torch.float32
            or not out.is_contiguous() or out.device != like.device
            or out.numel() != like.numel()):
        raise ValueError("out: a contiguous float32 tensor with the input's "
                         "element count on the input's device is required")


def _quantize_device(t, spec: QuantSpec, call: int, out=None, index_base=0,
                     sync=True):
    if t.dtype != torch.float32:
        raise TypeError("quantize: tensors are fp32 (proj/include/lpsim/tensor.hpp:16)")
    x = t.contiguous()
    if out is not None:
        _check_out(out, x)
    y = torch.empty_like(x) if out is None else out
    fmt = spec.format.c()
    shape = shape_array(x.shape)
    nbytes = lib.lpq_workspace_size(C.byref(fmt), shape, x.dim())
    ws = _workspace(x.device, nbytes)
    with torch.cuda.device(x.device):
        st = lib.lpq_quantize(
            C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), shape, x.dim(),
            int(index_base), C.byref(fmt), int(spec.mode), int(spec.seed),
            int(call), C.c_void_p(ws.data_ptr() if ws is not None else 0),
            nbytes, C.c_void_p(_status_buf(x.device).data_ptr()),
            _stream_ptr(x.device))
        check(st, "quantize")
        if sync:
            fetch_status(x.device)
    return y


def _quantize_host(t, spec: QuantSpec, call: int, index_base=0, device=-1):
    is_torch = torch is not None and isinstance(t, torch.Tensor)
    x = t.detach().contiguous().numpy() if is_torch else np.ascontiguousarray(t)
    if x.dtype != np.float32:
        raise TypeError("quantize: tensors are fp32")
    y = np.empty_like(x)
    fmt = spec.format.c()
    st = lib.lpq_quantize_host(
        C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data),
        shape_array(x.shape), x.ndim, int(index_base), C.byref(fmt),
        int(spec.mode), int(spec.seed), int(call), int(device))
    check(st, "quantize")
    return torch.from_numpy(y) if is_torch else y


def quantize_fused_at(t, spec: QuantSpec, call: int, *, out=None,
                      index_base: int = 0, sync: bool = True):
    """quantize_fused_at (quant_ops.cpp:154-164): pure, explicit call id."""
    if _is_device(t):
        return _quantize_device(t, spec, call, out=out, index_base=index_base,
                                sync=sync)
    return _quantize_host(t, spec, call, index_base=index_base)


def _block_extent(x, fmt):
    if not isinstance(fmt, BlockFloatFormat):
        raise UnsupportedFormatError("block maxima need a block format")
    if fmt.block_dim is None:
        return 1
    if fmt.block_dim >= x.dim():
        raise ShapeError("block_dim out of range")
    return int(x.shape[fmt.block_dim])


def block_absmax(t, fmt: "BlockFloatFormat"):
    """This tensor's part of every block maximum of `fmt` (the first half of
    fused_block, quant_ops.cpp:68-115; reduce_max_abs, tensor.cpp:320-353):
    an int32 CUDA tensor [extent] of max|x| fp32 bits (NaN ignored).  For a
    block split across shards, combine the shards' results with an
    elementwise max (torch.distributed.all_reduce(op=MAX)), then call
    quantize_block_apply -- lpq_block_absmax in include/lpq.h."""
    x = t.contiguous()
    if x.dtype != torch.float32 or not x.is_cuda:
        raise TypeError("block_absmax: a float32 CUDA tensor is required")
    extent = _block_extent(x, fmt)
    m = torch.zeros(max(extent, 1), dtype=torch.int32, device=x.device)
    f = fmt.c()
    with torch.cuda.device(x.device):
        check(lib.lpq_block_absmax(C.c_void_p(x.data_ptr()), shape_array(x.shape), x.dim(),
                                   C.byref(f), C.c_void_p(m.data_ptr()),
                                   _stream_ptr(x.device)), "block_absmax")
    return m[:extent]


def quantize_block_apply(t, spec: QuantSpec, call: int, maxima, *, out=None,
                         index_base: int = 0, sync: bool = True):
    """The quantization pass of fused_block with given block maxima (e.g.
    all-reduced across shards); bit-identical to quantize_fused_at of the
    whole tensor when `maxima` are the whole tensor's block maxima and
    `index_base` is this shard's first global flat index."""
    x = t.contiguous()
    if x.dtype != torch.float32 or not x.is_cuda:
        raise TypeError("quantize_block_apply: a float32 CUDA tensor is required")
    extent = _block_extent(x, spec.format)
    if not isinstance(maxima, torch.Tensor) or maxima.dtype != torch.int32:
        raise TypeError("maxima: the int32 fp32-bit tensor block_absmax returns "
                        "(combine shards with an elementwise max of those bits)")
    m = maxima.to(device=x.device).contiguous()
    if m.numel() != extent:
        raise ValueError(f"maxima: {extent} block maxima expected, got {m.numel()}")
    if out is not None:
        _check_out(out, x)
    y = torch.empty_like(x) if out is None else out
    f = spec.format.c()
    with torch.cuda.device(x.device):
        st = lib.lpq_quantize_block_apply(
            C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), shape_array(x.shape),
            x.dim(), int(index_base), C.byref(f), int(spec.mode), int(spec.seed), int(call),
            C.c_void_p(m.data_ptr()), C.c_void_p(_status_buf(x.device).data_ptr()),
            _stream_ptr(x.device))
        check(st, "quantize")
        if sync:
            fetch_status(x.device)
    return y


def quantize_fused(t, spec: QuantSpec, **kw):
    """quantize_fused (quant_ops.cpp:179-183): uses and (for stochastic
    rounding only) advances spec.call_counter."""
    out = quantize_fused_at(t, spec, spec.call_counter, **kw)
    if spec.mode == RoundingMode.Stochastic:
        spec.call_counter += 1
    return out


def quantize_composed_at(t, spec: QuantSpec, call: int, *, index_base: int = 0,
                         sync: bool = True):
    """quantize_composed_at (quant_ops.cpp:166-177): the many-kernel baseline
    (one kernel and HBM pass per tensor op).  Float formats raise
    UnsupportedFormatError."""
    fmt = spec.format.c()
    if _is_device(t):
        x = t.contiguous()
        y = torch.empty_like(x)
        shape = shape_array(x.shape)
        nbytes = lib.lpq_composed_workspace_size(C.byref(fmt), shape, x.dim())
        ws = _workspace(x.device, nbytes)
        with torch.cuda.device(x.device):
            st = lib.lpq_quantize_composed(
                C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), shape,
                x.dim(), int(index_base), C.byref(fmt), int(spec.mode),
                int(spec.seed), int(call),
                C.c_void_p(ws.data_ptr() if ws is not None else 0), nbytes,
                C.c_void_p(_status_buf(x.device).data_ptr()), _stream_ptr(x.device))
            check(st, "quantize_composed")
            if sync:
                fetch_status(x.device)
        return y
    is_torch = torch is not None and isinstance(t, torch.Tensor)
    x = t.detach().contiguous().numpy() if is_torch else np.ascontiguousarray(t)
    y = np.empty_like(x)
    st = lib.lpq_quantize_composed_host(
        C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data),
        shape_array(x.shape), x.ndim, int(index_base), C.byref(fmt),
        int(spec.mode), int(spec.seed), int(call), -1)
    check(st, "quantize_composed")
    return torch.from_numpy(y) if is_torch else y


def quantize_composed(t, spec: QuantSpec, **kw):
    out = quantize_composed_at(t, spec, spec.call_counter, **kw)
    if spec.mode == RoundingMode.Stochastic:
        spec.call_counter += 1
    return out


def quantize_fused_many(tensors, spec: QuantSpec, *, outs=None, sync=True):
    """quantize_fused over a list of CUDA tensors, in order (the call counter
    advances once per tensor for stochastic rounding, as a loop of
    quantize_fused calls would), in as few launches as possible
    (lpq_quantize_grouped: up to 64 tensors per launch)."""
    if not tensors:
        return []
    xs = [t.contiguous() for t in tensors]
    ys = [torch.empty_like(x) for x in xs] if outs is None else list(outs)
    dev = xs[0].device
    stoch = spec.mode == RoundingMode.Stochastic
    descs = (_lib.LpqTensorDesc * len(xs))()
    keep = []
    ws_need = 0
    fmt = spec.format.c()
    for i, (x, y) in enumerate(zip(xs, ys)):
        shp = shape_array(x.shape)
        keep.append(shp)
        ws_need = max(ws_need, lib.lpq_workspace_size(C.byref(fmt), shp, x.dim()))
        descs[i] = _lib.LpqTensorDesc(x.data_ptr(), y.data_ptr(), shp, x.dim(), 0,
                                      0, spec.call_counter + (i if stoch else 0))
    ws = _workspace(dev, ws_need)
    with torch.cuda.device(dev):
        st = lib.lpq_quantize_grouped(descs, len(xs), C.byref(fmt), int(spec.mode),
                                      int(spec.seed),
                                      C.c_void_p(ws.data_ptr() if ws is not None else 0),
                                      ws_need, C.c_void_p(_status_buf(dev).data_ptr()),
                                      _stream_ptr(dev))
        check(st, "quantize_grouped")
        if sync:
            fetch_status(dev)
    if stoch:
        spec.call_counter += len(xs)
    return ys


def quantized_op(op, spec: QuantSpec):
    """quantized_op (quant_ops.hpp:36-42): quantize_fused appended to op."""
    def run(*args, **kwargs):
        return quantize_fused(op(*args, **kwargs), spec)
    return run


# ---- GEMMs -----------------------------------------------------------------

def _as_dev(a, device):
    if _is_device(a):
        return a.contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(device)


def quant_gemm(a, b, fmt_mul: FloatFormat, fmt_add: FloatFormat,
               mode: RoundingMode = RoundingMode.NearestEven, seed: int = 0,
               call: int = 0, *, row_base: int = 0, out=None, sync=True):
    """Per-op-rounded GEMM (include/lpq.h lpq_quant_gemm)."""
    host = not (_is_device(a) and _is_device(b))
    if host and not _is_device(a) and not _is_device(b):
        A = np.ascontiguousarray(a, dtype=np.float32)
        B = np.ascontiguousarray(b, dtype=np.float32)
        M, K = A.shape
        K2, N = B.shape
        if K != K2:
            raise ShapeError("quant_gemm: inner dimensions disagree")
        Cm = np.empty((M, N), dtype=np.float32)
        st = lib.lpq_quant_gemm_host(
            C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data),
            C.c_void_p(Cm.ctypes.data), M, N, K, int(row_base),
            C.byref(fmt_mul.c()), C.byref(fmt_add.c()), int(mode), int(seed),
            int(call), -1)
        check(st, "quant_gemm")
        return Cm
    dev = a.device if _is_device(a) else b.device
    A, B = _as_dev(a, dev), _as_dev(b, dev)
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
        raise ShapeError("quant_gemm: operands must be rank-2 with matching inner dims")
    M, K = A.shape
    N = B.shape[1]
    if out is not None:
        _check_out(out, torch.empty((M, N), dtype=torch.float32, device=dev))
    Cd = torch.empty((M, N), dtype=torch.float32, device=dev) if out is None else out
    nbytes = lib.lpq_quant_gemm_workspace_size(M, N, K)
    ws = _workspace(dev, nbytes)
    with torch.cuda.device(dev):
        st = lib.lpq_quant_gemm(
            C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
            C.c_void_p(Cd.data_ptr()), M, N, K, int(row_base),
            C.byref(fmt_mul.c()), C.byref(fmt_add.c()), int(mode), int(seed),
            int(call), C.c_void_p(ws.data_ptr()), nbytes,
            C.c_void_p(_status_buf(dev).data_ptr()), _stream_ptr(dev))
        check(st, "quant_gemm")
        if sync:
            fetch_status(dev)
    return Cd


def quantized_matmul_at(a, b, spec: QuantSpec, call: int, *, row_base=0,
                        out=None, sync=True):
    """quantized_matmul (quant_ops.cpp:191-193) with an explicit call id:
    double-accumulated matmul, quantizer fused into the epilogue."""
    if not (_is_device(a) or _is_device(b)):
        A = np.ascontiguousarray(a, dtype=np.float32)
        B = np.ascontiguousarray(b, dtype=np.float32)
        if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
            raise ShapeError("matmul: operands must be rank-2 with matching inner dims")
        M, K = A.shape
        N = B.shape[1]
        Cm = np.empty((M, N), dtype=np.float32)
        st = lib.lpq_matmul_q_host(
            C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data),
            C.c_void_p(Cm.ctypes.data), M, N, K, C.byref(spec.format.c()),
            int(spec.mode), int(spec.seed), int(call), -1)
        check(st, "quantized_matmul")
        return Cm
    dev = a.device if _is_device(a) else b.device
    A, B = _as_dev(a, dev), _as_dev(b, dev)
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
        raise ShapeError("matmul: operands must be rank-2 with matching inner dims")
    M, K = A.shape
    N = B.shape[1]
    if out is not None:
        _check_out(out, torch.empty((M, N), dtype=torch.float32, device=dev))
    Cd = torch.empty((M, N), dtype=torch.float32, device=dev) if out is None else out
    fmt = spec.format.c()
    nbytes = lib.lpq_workspace_size(C.byref(fmt), shape_array((M, N)), 2)
    ws = _workspace(dev, nbytes)
    with torch.cuda.device(dev):
        st = lib.lpq_matmul_q(
            C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
            C.c_void_p(Cd.data_ptr()), M, N, K, int(row_base), C.byref(fmt),
            int(spec.mode), int(spec.seed), int(call),
            C.c_void_p(ws.data_ptr() if ws is not None else 0), nbytes,
            C.c_void_p(_status_buf(dev).data_ptr()), _stream_ptr(dev))
        check(st, "quantized_matmul")
        if sync:
            fetch_status(dev)
    return Cd


def quantized_matmul(a, b, spec: QuantSpec, **kw):
    out = quantized_matmul_at(a, b, spec, spec.call_counter, **kw)
    if spec.mode == RoundingMode.Stochastic:
        spec.call_counter += 1
    return out


# ---- generators ----------------------------------------------------------------

def random_uniform(shape, seed: int, call: int, lo: float, hi: float, *,
                   device="cuda", index_base: int = 0):
    """random_uniform (tensor.cpp:430-440), generated on the device."""
    shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    y = torch.empty(shape, dtype=torch.float32, device=device)
    with torch.cuda.device(y.device):
        check(lib.lpq_uniform(C.c_void_p(y.data_ptr()), y.numel(),
                              int(index_base), int(seed), int(call),
                              float(lo), float(hi), _stream_ptr(y.device)),
              "random_uniform")
    return y


def variate_tensor(shape, seed: int, call: int, *, device="cuda",
                   index_base: int = 0):
    """variate_tensor (tensor.cpp:281-290), generated on the device."""
    shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    y = torch.empty(shape, dtype=torch.float32, device=device)
    with torch.cuda.device(y.device):
        check(lib.lpq_variates(C.c_void_p(y.data_ptr()), y.numel(),
                               int(index_base), int(seed), int(call),
                               _stream_ptr(y.device)), "variate_tensor")
    return y


__all__ = [
    "RoundingMode", "FloatFormat", "FixedFormat", "BlockFloatFormat",
    "NumberFormat", "QuantSpec", "validate", "quantize_fused",
    "quantize_fused_at", "quantize_fused_many", "quantize_composed",
    "quantize_composed_at", "block_absmax", "quantize_block_apply",
    "quantized_op", "quantized_matmul",
    "quantized_matmul_at", "quant_gemm", "random_uniform", "variate_tensor",
    "pass_count", "reset_pass_count", "launch_count", "fetch_status",
    "InvalidInputError", "InvalidValueError", "ShapeError", "FormatError",
    "UnsupportedFormatError",
]
