"""ctypes binding of liblpq.so (include/lpq.h).

This is the Python-side reference binding of the C ABI (INTEGRATION.md shows
the same stub for a maintainer).  There is no fallback: if the library is
missing the import fails loudly, and every status code maps to the exception
type the reference raises (proj/include/lpsim/errors.hpp:9-55).
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "liblpq.so")

OK = 0
ERR_FORMAT, ERR_SHAPE, ERR_INVALID_INPUT, ERR_UNSUPPORTED = 1, 2, 3, 4
ERR_BLOCK_RANGE, ERR_ARGUMENT, ERR_WORKSPACE, ERR_CUDA, ERR_NO_DEVICE = 5, 6, 7, 8, 9
ERR_INVALID_VALUE = 10


class LpqFormat(C.Structure):
    """lpq_format (include/lpq.h) -- one NumberFormat as a flat struct."""
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "exp_bits", "man_bits", "wl", "fl", "symmetric", "saturate",
        "block_dim")]


# ---- exception taxonomy of the reference (errors.hpp) ----------------------
class LpsimError(RuntimeError):
    pass


class InvalidInputError(LpsimError):
    """invalid_input_error: non-finite input or block maximum out of range."""


class ShapeError(LpsimError):
    """shape_error."""


class FormatError(LpsimError):
    """format_error."""


class UnsupportedFormatError(LpsimError):
    """unsupported_format_error."""


class InvalidValueError(LpsimError):
    """invalid_value_error: non-finite result of a composed-chain op."""


class DeviceError(LpsimError):
    """CUDA runtime failure inside liblpq (no reference counterpart)."""


_EXC = {
    ERR_FORMAT: FormatError, ERR_SHAPE: ShapeError,
    ERR_INVALID_INPUT: InvalidInputError, ERR_BLOCK_RANGE: InvalidInputError,
    ERR_UNSUPPORTED: UnsupportedFormatError, ERR_ARGUMENT: ValueError,
    ERR_WORKSPACE: ValueError, ERR_CUDA: DeviceError, ERR_NO_DEVICE: DeviceError,
    ERR_INVALID_VALUE: InvalidValueError,
}

class LpqQuantSlot(C.Structure):
    """lpq_quant_slot (include/lpq.h)."""
    _fields_ = [("format", LpqFormat), ("mode", C.c_int32), ("enabled", C.c_int32),
                ("seed", C.c_uint64), ("call", C.c_uint64)]


class LpqTensorDesc(C.Structure):
    """lpq_tensor_desc (include/lpq.h)."""
    _fields_ = [("x", C.c_void_p), ("y", C.c_void_p),
                ("shape", C.POINTER(C.c_int64)), ("rank", C.c_int32),
                ("reserved", C.c_int32), ("index_base", C.c_uint64),
                ("call", C.c_uint64)]


class LpqSgdTensor(C.Structure):
    """lpq_sgd_tensor (include/lpq.h)."""
    _fields_ = [("grad", C.c_void_p), ("vel", C.c_void_p), ("acc", C.c_void_p),
                ("weight", C.c_void_p), ("n", C.c_int64), ("index_base", C.c_uint64),
                ("call_grad", C.c_uint64), ("call_vel", C.c_uint64),
                ("call_acc", C.c_uint64), ("call_weight", C.c_uint64)]


_F = C.POINTER(LpqFormat)
_S = C.POINTER(LpqQuantSlot)
_I64P = C.POINTER(C.c_int64)
_VP = C.c_void_p

_PROTOS = {
    "lpq_abi_version": (C.c_int, []),
    "lpq_status_string": (C.c_char_p, [C.c_int]),
    "lpq_validate_format": (C.c_int, [_F]),
    "lpq_workspace_size": (C.c_size_t, [_F, _I64P, C.c_int]),
    "lpq_launch_count": (C.c_uint64, []),
    "lpq_pass_count": (C.c_uint64, []),
    "lpq_reset_pass_count": (None, []),
    "lpq_last_cuda_error": (C.c_char_p, []),
    "lpq_quantize": (C.c_int, [_VP, _VP, _I64P, C.c_int, C.c_uint64, _F,
                               C.c_int, C.c_uint64, C.c_uint64, _VP,
                               C.c_size_t, _VP, _VP]),
    "lpq_status_fetch": (C.c_int, [_VP, _VP]),
    "lpq_block_absmax": (C.c_int, [_VP, _I64P, C.c_int, _F, _VP, _VP]),
    "lpq_quantize_block_apply": (C.c_int, [_VP, _VP, _I64P, C.c_int, C.c_uint64, _F,
                                           C.c_int, C.c_uint64, C.c_uint64, _VP, _VP,
                                           _VP]),
    "lpq_quant_gemm_workspace_size": (C.c_size_t, [C.c_int64, C.c_int64,
                                                   C.c_int64]),
    "lpq_quant_gemm": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64,
                                 C.c_int64, C.c_int64, _F, _F, C.c_int,
                                 C.c_uint64, C.c_uint64, _VP, C.c_size_t, _VP,
                                 _VP]),
    "lpq_matmul_q": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64,
                               C.c_int64, C.c_int64, _F, C.c_int, C.c_uint64,
                               C.c_uint64, _VP, C.c_size_t, _VP, _VP]),
    "lpq_uniform": (C.c_int, [_VP, C.c_int64, C.c_uint64, C.c_uint64,
                              C.c_uint64, C.c_float, C.c_float, _VP]),
    "lpq_variates": (C.c_int, [_VP, C.c_int64, C.c_uint64, C.c_uint64,
                               C.c_uint64, _VP]),
    "lpq_quantize_host": (C.c_int, [_VP, _VP, _I64P, C.c_int, C.c_uint64, _F,
                                    C.c_int, C.c_uint64, C.c_uint64,
                                    C.c_int]),
    "lpq_quant_gemm_host": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int64, _F, _F, C.c_int,
                                      C.c_uint64, C.c_uint64, C.c_int]),
    "lpq_matmul_q_host": (C.c_int, [_VP, _VP, _VP, C.c_int64, C.c_int64,
                                    C.c_int64, _F, C.c_int, C.c_uint64,
                                    C.c_uint64, C.c_int]),
    "lpq_composed_workspace_size": (C.c_size_t, [_F, _I64P, C.c_int]),
    "lpq_quantize_composed": (C.c_int, [_VP, _VP, _I64P, C.c_int, C.c_uint64,
                                        _F, C.c_int, C.c_uint64, C.c_uint64,
                                        _VP, C.c_size_t, _VP, _VP]),
    "lpq_quantize_composed_host": (C.c_int, [_VP, _VP, _I64P, C.c_int,
                                             C.c_uint64, _F, C.c_int,
                                             C.c_uint64, C.c_uint64, C.c_int]),
    "lpq_sgd_step": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int64, C.c_float,
                               C.c_float, _S, _S, _S, _S, C.c_uint64, _VP,
                               _VP]),
    "lpq_sgd_step_grouped": (C.c_int, [C.POINTER(LpqSgdTensor), C.c_int, C.c_float,
                                       C.c_float, _S, _S, _S, _S, _VP, _VP]),
    "lpq_quantize_grouped": (C.c_int, [C.POINTER(LpqTensorDesc), C.c_int, _F,
                                       C.c_int, C.c_uint64, _VP, C.c_size_t,
                                       _VP, _VP]),
    "lpq_host_bytes_per_element": (None, [_F, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "lpq_parse_format": (C.c_int, [C.c_char_p, _F]),
    "lpq_parse_rounding": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
    "lpq_format_to_string": (C.c_int, [_F, C.c_char_p, C.c_size_t]),
    "lpq_tensor_file_info": (C.c_int, [C.c_char_p, _I64P, C.POINTER(C.c_int)]),
    "lpq_load_tensor_file": (C.c_int, [C.c_char_p, _VP, C.c_int64]),
    "lpq_save_tensor_file": (C.c_int, [C.c_char_p, _VP, _I64P, C.c_int]),
    "lpq_quantize_file": (C.c_int, [C.c_char_p, C.c_char_p, _F, C.c_int,
                                    C.c_uint64, C.c_uint64, C.c_int]),
    "lpq_shutdown": (None, []),
}

# the symbols include/lpq.h declares (tests check every one is exported)
EXPORTED = tuple(_PROTOS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"liblpq.so not built ({LIB_PATH}); run "
            "`python -m paper_1910_04540_b200._build` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _LazyLib:
    """liblpq.so, loaded on first use (so the build recipe can import the
    package before the library exists); a missing library raises loudly."""

    _lib = None

    def __getattr__(self, name):
        if _LazyLib._lib is None:
            _LazyLib._lib = _load()
        return getattr(_LazyLib._lib, name)


lib = _LazyLib()


def status_string(st: int) -> str:
    return lib.lpq_status_string(st).decode()


def check(st: int, what: str = "lpq") -> None:
    """Raise the reference's exception type for a non-OK status."""
    if st == OK:
        return
    msg = f"{what}: {status_string(st)}"
    if st in (ERR_CUDA, ERR_NO_DEVICE):
        msg += f" ({lib.lpq_last_cuda_error().decode()})"
    raise _EXC.get(st, LpsimError)(msg)


def shape_array(shape):
    arr = (C.c_int64 * max(1, len(shape)))(*[int(s) for s in shape])
    return arr
