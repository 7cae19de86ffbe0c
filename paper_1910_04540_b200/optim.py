"""Low-precision SGD with momentum, the training-loop caller of the
quantizers, mirroring the reference's
LowPrecisionOptimizer (proj/include/lpsim/train.hpp, proj/src/train.cpp:
130-178) on device tensors.  Each parameter's whole update -- four
quantizations and four elementwise ops in the reference -- is ONE fused
kernel (lpq_sgd_step).  Call counters advance exactly as in the reference:
gradient +1, accumulator +2 (velocity and accumulator), weight +1 per
parameter, each only for stochastic specs.
"""
from __future__ import annotations

import copy
import ctypes as C

import numpy as np
from typing import Optional, Sequence

from . import _lib
from ._lib import FormatError, LpqQuantSlot, LpqSgdTensor, ShapeError, check, lib
from .quant import (BlockFloatFormat, QuantSpec, RoundingMode, _status_buf,
                    _stream_ptr, fetch_status, quantize_fused)


def _slot(spec: Optional[QuantSpec], call_offset: int = 0) -> LpqQuantSlot:
    if spec is None:
        return LpqQuantSlot()
    s = LpqQuantSlot()
    s.format = spec.format.c()
    s.mode = int(spec.mode)
    s.enabled = 1
    s.seed = int(spec.seed)
    s.call = int(spec.call_counter) + call_offset
    return s


def _advance(spec: Optional[QuantSpec], k: int) -> None:
    if spec is not None and spec.mode == RoundingMode.Stochastic:
        spec.call_counter += k


def _check_tensor(t, first, what):
    """The fused kernel reads and writes every pointer as n fp32 values on one
    device: anything else is rejected before it reaches the launch."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32 or not t.is_cuda:
        raise TypeError(f"optimizer: {what} must be float32 CUDA tensors "
                        "(proj/include/lpsim/tensor.hpp:16)")
    if t.device != first.device:
        raise TypeError(f"optimizer: {what} must be on {first.device}, got {t.device}")


def _is_block(spec: Optional[QuantSpec]) -> bool:
    return spec is not None and isinstance(spec.format, BlockFloatFormat)


def _sgd_dtype():
    return np.dtype({"names": [n for n, _ in LpqSgdTensor._fields_],
                     "formats": [np.uint64 if t is not C.c_int64 else np.int64
                                 for _, t in LpqSgdTensor._fields_],
                     "offsets": [getattr(LpqSgdTensor, n).offset for n, _ in LpqSgdTensor._fields_],
                     "itemsize": C.sizeof(LpqSgdTensor)})


_SGD_DTYPE = _sgd_dtype()


class LowPrecisionOptimizer:
    """LowPrecisionOptimizer(model, lr, momentum, cfg) over a list of CUDA
    parameter tensors (updated in place, like the Linear weights/biases)."""

    def __init__(self, params: Sequence, lr: float, momentum: float,
                 weight: Optional[QuantSpec] = None,
                 accumulator: Optional[QuantSpec] = None,
                 gradient: Optional[QuantSpec] = None):
        import torch
        if lr < 0.0:
            raise FormatError("learning rate must be non-negative")  # train.cpp:134
        if not (0.0 <= momentum < 1.0):
            raise FormatError("momentum must be in [0, 1)")          # train.cpp:135-136
        self.lr = float(lr)
        self.momentum = float(momentum)
        self.weight_spec = copy.deepcopy(weight)
        self.acc_spec = copy.deepcopy(accumulator)
        self.grad_spec = copy.deepcopy(gradient)
        self.params = list(params)
        for p in self.params:
            _check_tensor(p, self.params[0], "parameters")
            if not p.is_contiguous():
                raise ValueError("parameters must be contiguous")
        self.acc = [p.detach().clone().contiguous() for p in self.params]
        self.vel = [torch.zeros_like(p) for p in self.params]

    @classmethod
    def from_config(cls, params: Sequence, lr: float, momentum: float, cfg):
        """LowPrecisionOptimizer(model, lr, momentum, cfg) with a QuantConfig
        (io.parse_quant_config); uses its weight/accumulator/gradient specs
        (train.cpp:130-146)."""
        return cls(params, lr, momentum, weight=cfg.weight,
                   accumulator=cfg.accumulator, gradient=cfg.gradient)

    def accumulators(self):
        return self.acc

    def step(self, grads: Sequence, *, sync: bool = True) -> None:
        """LowPrecisionOptimizer::step (train.cpp:148-178): every parameter's
        update in one grouped launch (lpq_sgd_step_grouped, up to 64 tensors
        per launch), with the call ids the reference's per-parameter loop
        would give each of its four quantizations.  sync=True (the
        reference's behaviour) raises a non-finite update before returning;
        sync=False leaves the launch asynchronous and the error in the device
        status word for the next synchronising call (fetch_status)."""
        if len(grads) != len(self.params):
            raise ShapeError("optimizer step: gradient count mismatch")
        if not self.params:
            return
        acc_stoch = self.acc_spec is not None and self.acc_spec.mode == RoundingMode.Stochastic
        for p, g in zip(self.params, grads):  # validate before any state changes
            if tuple(p.shape) != tuple(g.shape):
                raise ShapeError("optimizer step: gradient shape mismatch")
            if not p.is_contiguous():
                raise ValueError("parameters must be contiguous")
            _check_tensor(g, self.params[0], "gradients")
        if any(_is_block(s) for s in (self.grad_spec, self.acc_spec, self.weight_spec)):
            return self._step_unfused(grads, sync)
        # the tensor table, filled column-wise (the per-step host cost of
        # a Python loop over ctypes structs exceeds the kernel's)
        cnt = len(self.params)
        if getattr(self, "_table", None) is None:
            self._table = np.zeros(cnt, dtype=_SGD_DTYPE)
            self._table["vel"] = [v.data_ptr() for v in self.vel]
            self._table["acc"] = [a.data_ptr() for a in self.acc]
            self._table["weight"] = [p.data_ptr() for p in self.params]
            self._table["n"] = [p.numel() for p in self.params]
        t = self._table
        gs = [g if g.is_contiguous() else g.contiguous() for g in grads]
        t["grad"] = [g.data_ptr() for g in gs]
        j = np.arange(cnt, dtype=np.uint64)

        def calls(spec, per):
            if spec is None:
                return np.zeros(cnt, np.uint64)
            step = per if spec.mode == RoundingMode.Stochastic else 0
            return np.uint64(spec.call_counter) + j * np.uint64(step)
        t["call_grad"] = calls(self.grad_spec, 1)
        t["call_vel"] = calls(self.acc_spec, 2)
        t["call_acc"] = t["call_vel"] + np.uint64(1 if acc_stoch else 0)
        t["call_weight"] = calls(self.weight_spec, 1)
        descs = t.ctypes.data_as(C.POINTER(LpqSgdTensor))
        dev = self.params[0].device
        qg, qv, qw = _slot(self.grad_spec), _slot(self.acc_spec), _slot(self.weight_spec)
        st = lib.lpq_sgd_step_grouped(descs, len(self.params), self.momentum, self.lr,
                                      C.byref(qg), C.byref(qv), C.byref(qv), C.byref(qw),
                                      C.c_void_p(_status_buf(dev).data_ptr()),
                                      _stream_ptr(dev))
        check(st, "optimizer step")
        # the counters advance only once the launch was accepted (a rejected
        # step leaves the specs as they were)
        _advance(self.grad_spec, cnt)
        _advance(self.acc_spec, 2 * cnt)
        _advance(self.weight_spec, cnt)
        if sync:
            fetch_status(dev)

    def _step_unfused(self, grads, sync):
        """Block floating point in any slot (the fused kernel has no per-block
        reduction): the reference's per-parameter sequence (train.cpp:161-174)
        as quantize_fused launches and fp32 elementwise ops on the device --
        scale(vel, float(momentum)) + g, then acc - scale(v, float(lr)), each a
        separately rounded fp32 op as in tensor.cpp:140-168 -- with the call
        counters advancing per quantization exactly as quantize_fused does."""
        import torch
        m32 = float(np.float32(self.momentum))
        lr32 = float(np.float32(self.lr))
        for k, (p, g) in enumerate(zip(self.params, grads)):
            g = g.contiguous()
            if self.grad_spec is not None:
                g = quantize_fused(g, self.grad_spec, sync=sync)
            v = torch.add(torch.mul(self.vel[k], m32), g)
            if self.acc_spec is not None:
                v = quantize_fused(v, self.acc_spec, sync=sync)
            self.vel[k].copy_(v)
            a = torch.sub(self.acc[k], torch.mul(v, lr32))
            if self.acc_spec is not None:
                a = quantize_fused(a, self.acc_spec, sync=sync)
            self.acc[k].copy_(a)
            if self.weight_spec is not None:
                quantize_fused(a, self.weight_spec, out=p, sync=sync)
            else:
                p.copy_(a)
