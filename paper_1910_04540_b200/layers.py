"""Quantizer layers on either side of the path: the
reference's ActivationQuant / ErrorQuant layers and inject_quantizers
(proj/include/lpsim/train.hpp, proj/src/train.cpp:54-128) as torch modules
over CUDA tensors.  Every quantization is one lpq_quantize launch
(quant.quantize_fused); autograd is plumbing.

* ActivationQuant: forward y = quantize_fused(x, spec) (train.cpp:64-65),
  backward passes the gradient straight through (train.cpp:98).
* ErrorQuant: identity forward (train.cpp:67), backward
  g = quantize_fused(g, spec) (train.cpp:93-95).
Each layer owns a copy of its spec, so its call counter advances per
quantization exactly like the reference layer's (stochastic only).
"""
from __future__ import annotations

import copy

import torch

from ._lib import LpsimError
from .quant import QuantSpec, quantize_fused


class InjectionError(LpsimError):
    """injection_error (errors.hpp:46-49)."""


class _ActFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, layer):
        return quantize_fused(x.contiguous(), layer.spec)

    @staticmethod
    def backward(ctx, g):
        return g, None


class _ErrFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, layer):
        ctx.layer = layer
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        layer = ctx.layer
        q = quantize_fused(g.contiguous(), layer.spec)
        if layer.trace is not None:
            layer.trace.append(q)  # BackwardTrace::error_signals
        return q, None


class ActivationQuant(torch.nn.Module):
    def __init__(self, spec: QuantSpec):
        super().__init__()
        self.spec = copy.deepcopy(spec)

    def forward(self, x):
        return _ActFn.apply(x, self)

    def extra_repr(self):
        return f"{self.spec.format}, {self.spec.mode.name}"


class ErrorQuant(torch.nn.Module):
    def __init__(self, spec: QuantSpec):
        super().__init__()
        self.spec = copy.deepcopy(spec)
        self.trace = None  # set to a list to record the quantized errors

    def forward(self, x):
        return _ErrFn.apply(x, self)

    def extra_repr(self):
        return f"{self.spec.format}, {self.spec.mode.name}"


def has_quantizer_layers(model: torch.nn.Sequential) -> bool:
    """train.cpp:31-37."""
    return any(isinstance(m, (ActivationQuant, ErrorQuant)) for m in model)


def inject_quantizers(model: torch.nn.Sequential, cfg) -> torch.nn.Sequential:
    """inject_quantizers (train.cpp:103-128): after every Linear an ErrorQuant
    (cfg.error), then the Linear's ReLU if one follows, then an
    ActivationQuant (cfg.activation).  The Linear/ReLU modules are shared with
    `model` (the reference copies them by value; parameters here are the
    caller's).  Raises InjectionError on an already-injected model."""
    if getattr(model, "_lpq_injected", False) or has_quantizer_layers(model):
        raise InjectionError("model already has quantizers injected")
    layers = list(model)
    out = []
    i = 0
    while i < len(layers):
        if isinstance(layers[i], torch.nn.Linear):
            out.append(layers[i])
            if cfg.error is not None:
                out.append(ErrorQuant(cfg.error))
            if i + 1 < len(layers) and isinstance(layers[i + 1], torch.nn.ReLU):
                out.append(layers[i + 1])
                i += 2
            else:
                i += 1
            if cfg.activation is not None:
                out.append(ActivationQuant(cfg.activation))
        else:
            out.append(layers[i])
            i += 1
    seq = torch.nn.Sequential(*out)
    seq._lpq_injected = True
    return seq
