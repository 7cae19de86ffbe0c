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
from typing import Optional, Sequence

from . import _lib
from ._lib import FormatError, LpqQuantSlot, ShapeError, check, lib
from .quant import QuantSpec, RoundingMode, _status_buf, _stream_ptr, fetch_status


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

    def step(self, grads: Sequence) -> None:
        """LowPrecisionOptimizer::step (train.cpp:148-178)."""
        if len(grads) != len(self.params):
            raise ShapeError("optimizer step: gradient count mismatch")
        for p, g, a, v in zip(self.params, grads, self.acc, self.vel):
            if tuple(p.shape) != tuple(g.shape):
                raise ShapeError("optimizer step: gradient shape mismatch")
            if not p.is_contiguous():
                raise ValueError("parameters must be contiguous")
            g = g.contiguous()
            acc_stoch = self.acc_spec is not None and self.acc_spec.mode == RoundingMode.Stochastic
            qg = _slot(self.grad_spec)
            qv = _slot(self.acc_spec)
            qa = _slot(self.acc_spec, 1 if acc_stoch else 0)
            qw = _slot(self.weight_spec)
            dev = p.device
            st = lib.lpq_sgd_step(
                C.c_void_p(g.data_ptr()), C.c_void_p(v.data_ptr()),
                C.c_void_p(a.data_ptr()), C.c_void_p(p.data_ptr()), p.numel(),
                self.momentum, self.lr, C.byref(qg), C.byref(qv), C.byref(qa),
                C.byref(qw), 0, C.c_void_p(_status_buf(dev).data_ptr()),
                _stream_ptr(dev))
            check(st, "optimizer step")
            _advance(self.grad_spec, 1)
            _advance(self.acc_spec, 2)
            _advance(self.weight_spec, 1)
        if self.params:
            fetch_status(self.params[0].device)
