"""The data formats on either side of the path,
mirroring proj/include/lpsim/io.hpp: LPT1 tensor files, the format and
rounding spec strings, the JSON quantization config, and `lpsim quantize` (tools/lpsim_main.cpp:23-34) as
quantize_file -- all through liblpq.so (include/lpq.h)."""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._lib import FormatError, LpqFormat, check, lib, shape_array
from .quant import (BlockFloatFormat, FixedFormat, FloatFormat, QuantSpec,
                    RoundingMode, validate)


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


# ---------------------------------------------------------------------------
# JSON quantization config (io.hpp:29-36, io.cpp:208-329)

_CATEGORIES = ("weight", "accumulator", "gradient", "activation", "error")
_FIELDS = ("kind", "rounding", "seed", "exp", "man", "wl", "fl", "symmetric",
           "saturate", "block")
_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    """splitmix64 finalizer (rng.hpp:17-22); host-side seed derivation."""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class ConfigTypeError(TypeError):
    """A JSON value of the wrong type where the reference's json library raises
    its type_error (e.g. "kind": 3, "symmetric": "yes")."""


@dataclass
class QuantConfig:
    """QuantConfig (train.hpp:16-22): one optional QuantSpec per category."""
    weight: Optional[QuantSpec] = None
    accumulator: Optional[QuantSpec] = None
    gradient: Optional[QuantSpec] = None
    activation: Optional[QuantSpec] = None
    error: Optional[QuantSpec] = None


def _is_int(v) -> bool:
    # nlohmann number_integer / number_unsigned; integers beyond 64 bits parse
    # as floating point there
    return (isinstance(v, int) and not isinstance(v, bool)
            and -(1 << 63) <= v <= _M64)


def _as_int32(v: int) -> int:
    # get<int>() of a 64-bit JSON integer: static_cast, two's-complement wrap
    return ((v + (1 << 31)) & 0xFFFFFFFF) - (1 << 31)


def _as_u64(v) -> int:
    # get<std::uint64_t>(): integers wrap mod 2^64, floats truncate, booleans
    # and everything else are type errors (nlohmann 3.11 from_json)
    if _is_int(v):
        return v & _M64
    if isinstance(v, float):
        return int(v) & _M64
    raise ConfigTypeError("type must be number, but is " + type(v).__name__)


def _as_bool(v) -> bool:
    if not isinstance(v, bool):
        raise ConfigTypeError("type must be boolean, but is " + type(v).__name__)
    return v


def _as_str(v) -> str:
    if not isinstance(v, str):
        raise ConfigTypeError("type must be string, but is " + type(v).__name__)
    return v


def _spec_entry(j, category: str, default_seed: int, index: int) -> QuantSpec:
    """parse_spec_entry (io.cpp:212-290)."""
    if not isinstance(j, dict):
        raise FormatError(f"config key '{category}' must be an object")
    for k in j:
        if k not in _FIELDS:
            raise FormatError(f"config key '{category}': unknown field '{k}'")
    if "kind" not in j:
        raise FormatError(f"config key '{category}': missing 'kind'")
    kind = _as_str(j["kind"])

    def get_int(field):
        if field not in j:
            raise FormatError(f"config key '{category}': missing '{field}'")
        if not _is_int(j[field]):
            raise FormatError(f"config key '{category}': '{field}' must be an integer")
        return _as_int32(j[field])

    def forbid(*fields):
        for field in fields:
            if field in j:
                raise FormatError(f"config key '{category}': field '{field}' "
                                  f"does not apply to kind '{kind}'")

    if kind == "float":
        forbid("wl", "fl", "symmetric", "saturate", "block")
        fmt = FloatFormat(get_int("exp"), get_int("man"))
    elif kind == "fixed":
        forbid("exp", "man", "block")
        wl, fl = get_int("wl"), get_int("fl")
        sym = _as_bool(j["symmetric"]) if "symmetric" in j else False
        sat = _as_bool(j["saturate"]) if "saturate" in j else True
        fmt = FixedFormat(wl, fl, sym, sat)
    elif kind == "block":
        forbid("exp", "man", "fl", "symmetric", "saturate")
        wl = get_int("wl")
        dim = None
        if "block" in j:
            b = j["block"]
            if b == "tensor" and isinstance(b, str):
                dim = None
            elif isinstance(b, dict) and len(b) == 1 and "dim" in b and _is_int(b["dim"]):
                dim = _as_int32(b["dim"])
            else:
                raise FormatError(f"config key '{category}': 'block' must be "
                                  "\"tensor\" or {\"dim\": d}")
        fmt = BlockFloatFormat(wl, dim)
    else:
        raise FormatError(f"config key '{category}': unknown kind '{kind}'")
    validate(fmt)  # formats.hpp:82-112, through liblpq
    mode = (parse_rounding(_as_str(j["rounding"])) if "rounding" in j
            else RoundingMode.NearestEven)
    seed = (_as_u64(j["seed"]) if "seed" in j
            else _mix64((default_seed & _M64) ^ _mix64(index)))
    return QuantSpec(fmt, mode, seed, 0)


def _reject_constant(name):
    raise FormatError(f"config is not valid JSON: {name}")


def parse_quant_config(json_text: str, default_seed: int) -> QuantConfig:
    """parse_quant_config (io.cpp:294-321): optional keys weight / accumulator /
    gradient / activation / error; unknown keys are rejected; entries without
    a seed get mix64(default_seed ^ mix64(category index))."""
    try:
        j = json.loads(json_text, parse_constant=_reject_constant)
    except (ValueError, RecursionError) as e:
        if isinstance(e, FormatError):
            raise
        raise FormatError(f"config is not valid JSON: {e}") from None
    if not isinstance(j, dict):
        raise FormatError("config must be a JSON object")
    for k in j:
        if k not in _CATEGORIES:
            raise FormatError(f"unknown config key '{k}'")
    cfg = QuantConfig()
    for index, name in enumerate(_CATEGORIES):
        if name in j:
            setattr(cfg, name, _spec_entry(j[name], name, default_seed, index))
    return cfg


def load_quant_config(path: str, default_seed: int) -> QuantConfig:
    """load_quant_config (io.cpp:323-329)."""
    try:
        with open(path, "r", encoding="utf-8", errors="surrogateescape") as fh:
            text = fh.read()
    except OSError:
        raise FormatError(f"cannot open config {path}") from None
    return parse_quant_config(text, default_seed)
