"""liblpq.so loads, exports every symbol include/lpq.h declares, and its
host-only helpers behave without a GPU (no compute calls here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lpq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lpq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1910_04540_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 19
    for n in names:
        assert hasattr(_lib.lib, n), n
    assert set(names) == set(_lib.EXPORTED)


def test_library_is_sm100a_and_loads():
    from paper_1910_04540_b200 import _lib
    assert _lib.lib.lpq_abi_version() == 1
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


@pytest.mark.parametrize("fmt,ok", [
    ("float:8:23", True), ("float:0:2", False), ("float:9:2", False),
    ("float:5:24", False), ("float:1:0", True), ("fixed:2:0", True),
    ("fixed:1:0", False), ("fixed:25:0", False), ("fixed:8:-120", True),
    ("fixed:8:-121", False), ("fixed:8:126", True), ("fixed:8:127", False),
    ("block:8", True), ("block:1", False), ("block:25", False),
])
def test_validate_matches_reference_rules(fmt, ok):
    # formats.hpp:82-112
    import paper_1910_04540_b200 as q
    kind, *a = fmt.split(":")
    a = [int(v) for v in a]
    f = {"float": q.FloatFormat, "fixed": q.FixedFormat, "block": q.BlockFloatFormat}[kind](*a)
    if ok:
        q.validate(f)
    else:
        with pytest.raises(q.FormatError):
            q.validate(f)


def test_block_dim_negative_rejected():
    import paper_1910_04540_b200 as q
    with pytest.raises(q.FormatError):
        q.validate(q.BlockFloatFormat(8, -3))


def test_workspace_and_status_strings():
    from paper_1910_04540_b200 import _lib
    import paper_1910_04540_b200 as q
    f = q.BlockFloatFormat(8, 1).c()
    shp = _lib.shape_array((3, 1000, 7))
    assert _lib.lib.lpq_workspace_size(C.byref(f), shp, 3) >= 1000 * 4
    assert _lib.lib.lpq_workspace_size(C.byref(q.FixedFormat(8, 4).c()), shp, 3) == 0
    for s in range(10):
        assert _lib.status_string(s)
    assert "non-finite" in _lib.status_string(3)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200._lib import DeviceError
    with pytest.raises(DeviceError):
        q.quantize_fused_at(np.ones(16, np.float32), q.QuantSpec(q.FixedFormat(8, 4)), 0)


def test_shape_checks_before_any_device_work():
    # argument and shape errors come back before the library touches a GPU
    from paper_1910_04540_b200 import _lib
    import paper_1910_04540_b200 as q
    f = q.FixedFormat(8, 4).c()
    L = _lib.lib

    def call(shape):
        return L.lpq_quantize(None, None, _lib.shape_array(shape), len(shape), 0,
                              C.byref(f), 0, 0, 0, None, 0, None, None)
    assert call((1 << 40, 1 << 40)) == _lib.ERR_SHAPE     # element count overflows
    assert call((1 << 31, 1 << 31)) == _lib.ERR_SHAPE     # byte count overflows
    assert call((-1, 4)) == _lib.ERR_SHAPE
    assert call((0, 1 << 62)) == 0                        # empty: nothing to do
    assert call((4, 4)) == _lib.ERR_ARGUMENT              # null pointers
    bf = q.BlockFloatFormat(8, 2).c()
    assert L.lpq_quantize(None, None, _lib.shape_array((4, 4)), 2, 0, C.byref(bf), 0, 0, 0,
                          None, 0, None, None) == _lib.ERR_SHAPE  # block_dim >= rank


def test_block_split_entry_points_validate_first():
    # lpq_block_absmax / lpq_quantize_block_apply: format, shape and argument
    # errors before any device work
    from paper_1910_04540_b200 import _lib
    import paper_1910_04540_b200 as q
    L = _lib.lib
    shp = _lib.shape_array((4, 6))
    fx = q.FixedFormat(8, 4).c()
    b1 = q.BlockFloatFormat(8, 1).c()
    b5 = q.BlockFloatFormat(8, 5).c()
    bad = q.BlockFloatFormat(30, 1).c()
    assert L.lpq_block_absmax(None, shp, 2, C.byref(fx), None, None) == _lib.ERR_UNSUPPORTED
    assert L.lpq_block_absmax(None, shp, 2, C.byref(b5), None, None) == _lib.ERR_SHAPE
    assert L.lpq_block_absmax(None, shp, 2, C.byref(bad), None, None) == _lib.ERR_FORMAT
    assert L.lpq_block_absmax(None, shp, 2, C.byref(b1), None, None) == _lib.ERR_ARGUMENT
    assert L.lpq_block_absmax(None, _lib.shape_array((0, 6)), 2, C.byref(b1), None,
                              None) == _lib.ERR_ARGUMENT  # extent 6 still needs maxima

    def apply(fmt, shape, mode=0):
        return L.lpq_quantize_block_apply(None, None, _lib.shape_array(shape), len(shape), 0,
                                          C.byref(fmt), mode, 0, 0, None, None, None)
    assert apply(fx, (4, 6)) == _lib.ERR_UNSUPPORTED
    assert apply(b5, (4, 6)) == _lib.ERR_SHAPE
    assert apply(b1, (4, 6), mode=7) == _lib.ERR_ARGUMENT
    assert apply(b1, (0, 6)) == 0  # empty: nothing to do
    assert apply(b1, (4, 6)) == _lib.ERR_ARGUMENT
