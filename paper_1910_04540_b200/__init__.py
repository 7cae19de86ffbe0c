"""B200-native fused quantization simulator (QPyTorch / arXiv 1910.04540 hot path).

The product is liblpq.so (include/lpq.h): hand-written sm_100a kernels behind
a C ABI that mirrors the reference's quantizer API (lpsim,
proj/include/lpsim/quant_ops.hpp).  This package is its Python binding and a
mirror of the reference interface (quant.py); see DESIGN.md.
"""
from .quant import *  # noqa: F401,F403
from .quant import __all__  # noqa: F401

__version__ = "0.1.0"
