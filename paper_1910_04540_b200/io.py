"""The data formats on either side of the path,
mirroring proj/include/lpsim/io.hpp: LPT1 tensor files, the format and
rounding spec strings, and `lpsim quantize` (tools/lpsim_main.cpp:23-34) as
quantize_file -- all through liblpq.so (include/lpq.h)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import LpqFormat, check, lib, shape_array
from .quant import (BlockFloatFormat, FixedFormat, FloatFormat, QuantSpec,
                    RoundingMode)


def _from_c(f: LpqFormat):
    if f.kind == 0:
        return FloatFormat(f.exp_bits, f.man_bits)
    if f.kind == 1:
        return FixedFormat(f.wl, f.fl, bool(f.symmetric), bool(f.saturate))
    return BlockFloatFormat(f.wl, None if f.block_dim < 0 else f.block_dim)


def parse_format(text: str):
    """parse_format (io.cpp:132-181)."""
    f = LpqFormat()
    check(lib.lpq_parse_format(text.encode(), C.byref(f)), "parse_format")
    return _from_c(f)


def parse_rounding(text: str) -> RoundingMode:
    """parse_rounding (io.cpp:200-206)."""
    m = C.c_int()
    check(lib.lpq_parse_rounding(text.encode(), C.byref(m)), "parse_rounding")
    return RoundingMode(m.value)


def format_to_string(fmt) -> str:
    """format_to_string (io.cpp:183-198)."""
    buf = C.create_string_buffer(64)
    lib.lpq_format_to_string(C.byref(fmt.c()), buf, 64)
    return buf.value.decode()


def read_tensor_file(path: str) -> np.ndarray:
    """read_tensor_file (io.cpp:96-99)."""
    shape = (C.c_int64 * 8)()
    rank = C.c_int()
    check(lib.lpq_tensor_file_info(path.encode(), shape, C.byref(rank)), "read_tensor_file")
    shp = tuple(shape[d] for d in range(rank.value))
    out = np.empty(shp, dtype=np.float32)
    check(lib.lpq_load_tensor_file(path.encode(), C.c_void_p(out.ctypes.data), out.size),
          "read_tensor_file")
    return out


def write_tensor_file(path: str, t) -> None:
    """write_tensor_file (io.cpp:89-94)."""
    a = np.asarray(t, dtype=np.float32, order="C")  # keeps rank 0
    check(lib.lpq_save_tensor_file(path.encode(), C.c_void_p(a.ctypes.data),
                                   shape_array(a.shape), a.ndim), "write_tensor_file")


def quantize_file(in_path: str, out_path: str, spec: QuantSpec, *, device: int = -1) -> None:
    """`lpsim quantize IN OUT --format F --rounding R --seed S` on the GPU
    (quantize_fused with spec.call_counter, advanced for stochastic)."""
    check(lib.lpq_quantize_file(in_path.encode(), out_path.encode(),
                                C.byref(spec.format.c()), int(spec.mode), int(spec.seed),
                                int(spec.call_counter), int(device)), "quantize_file")
    if spec.mode == RoundingMode.Stochastic:
        spec.call_counter += 1
