"""LPT1 files and spec strings against the reference's
own io.cpp (compiled into oracle/_ref) and the cases of
proj/tests/test_io.cpp:29-97.  Host-only: no GPU."""
import os

import numpy as np
import pytest

from oracle_lib import bits

CASES_OK = ["float:5:2", "fixed:3:1", "fixed:8:4:symmetric", "fixed:8:4:wrap",
            "fixed:8:4:symmetric:wrap", "block:8", "block:8:tensor", "block:6:dim1",
            "float", "fixed", "block", "float:8:23", "float:1:0", "fixed:24:126",
            "fixed:2:-126", "block:24:dim0", "float: 5:2", "fixed:+8:4"]
CASES_BAD = ["decimal:3", "float:9:2", "fixed:30:1", "fixed:8", "fixed:8:x",
             "block:8:diag", "float:5", "float:5:2:1", "fixed:8:4:odd", "block:8:dim",
             "block:8:dim-1", "block:1", "fixed:8:127", "", "float:5:2 ", "block:8:tensor:x"]


@pytest.mark.parametrize("text", CASES_OK + CASES_BAD)
def test_parse_format_matches_reference(ref, text):
    from paper_1910_04540_b200 import io as lio
    from paper_1910_04540_b200._lib import FormatError
    st, rf = ref.parse_format(text)
    if st != 0:
        with pytest.raises(FormatError):
            lio.parse_format(text)
        return
    f = lio.parse_format(text).c()
    for name, _ in f._fields_:
        assert getattr(f, name) == getattr(rf, name), (text, name)


def test_format_strings_round_trip():
    from paper_1910_04540_b200 import io as lio
    for text in ["float:4:3", "fixed:8:4:symmetric:wrap", "block:6:dim1", "block:8:tensor"]:
        assert lio.format_to_string(lio.parse_format(text)) == text
    assert lio.format_to_string(lio.parse_format("block:8")) == "block:8:tensor"
    import paper_1910_04540_b200 as q
    assert lio.parse_rounding("stochastic") == q.RoundingMode.Stochastic
    assert lio.parse_rounding("nearest_zero") == q.RoundingMode.NearestTowardZero
    with pytest.raises(q.FormatError):
        lio.parse_rounding("nearest")


@pytest.mark.parametrize("shape", [(), (7,), (3, 5), (2, 3, 4, 1), (0, 4)])
def test_lpt1_interop_with_reference(ref, tmp_path, shape):
    from paper_1910_04540_b200 import io as lio
    rng = np.random.default_rng(len(shape))
    x = rng.standard_normal(shape).astype(np.float32)
    a, b = str(tmp_path / "ref.lpt"), str(tmp_path / "ours.lpt")
    assert ref.write_tensor_file(a, x) == 0
    got = lio.read_tensor_file(a)                      # reference writes, we read
    assert got.shape == x.shape and np.array_equal(bits(got), bits(x))
    lio.write_tensor_file(b, x)                        # we write, reference reads
    st, y, shp = ref.read_tensor_file(b, x.size)
    assert st == 0 and shp == x.shape and np.array_equal(bits(y), bits(x.reshape(-1)))
    assert open(a, "rb").read() == open(b, "rb").read()  # byte-identical files


def test_lpt1_errors(tmp_path):
    from paper_1910_04540_b200 import io as lio
    from paper_1910_04540_b200._lib import FormatError
    p = str(tmp_path / "t.lpt")
    lio.write_tensor_file(p, np.ones((4, 4), np.float32))
    data = open(p, "rb").read()
    open(p, "wb").write(data[:-3])                    # truncated payload
    with pytest.raises(FormatError):
        lio.read_tensor_file(p)
    open(p, "wb").write(b"LPT2" + data[4:])           # bad magic
    with pytest.raises(FormatError):
        lio.read_tensor_file(p)
    open(p, "wb").write(b"LPT1" + (9).to_bytes(4, "little"))  # rank > 8
    with pytest.raises(FormatError):
        lio.read_tensor_file(p)
    with pytest.raises(FormatError):
        lio.read_tensor_file(str(tmp_path / "missing.lpt"))
    with pytest.raises(ValueError):
        lio.write_tensor_file(p, np.ones((1,) * 9, np.float32))


# ---------------------------------------------------------------------------
# JSON quantization config (io.cpp:208-329) against the reference parser, with
# the cases of proj/tests/test_io.cpp plus type/edge cases
CONFIGS = [
    '{}',
    '{"weight": {"kind": "float", "exp": 5, "man": 2}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "rounding": "stochastic", "seed": 9}}',
    '{"gradient": {"kind": "fixed", "wl": 8, "fl": 4, "symmetric": true, "saturate": false}}',
    '{"activation": {"kind": "block", "wl": 8, "block": "tensor"}, "error": {"kind": "block", "wl": 6, "block": {"dim": 1}}}',
    '{"accumulator": {"kind": "float", "exp": 8, "man": 23, "rounding": "nearest_zero"}}',
    '{"weight": {"kind": "block", "wl": 8}, "accumulator": {"kind": "fixed", "wl": 16, "fl": 8},'
    ' "gradient": {"kind": "float", "exp": 5, "man": 2, "rounding": "nearest_away"},'
    ' "activation": {"kind": "fixed", "wl": 8, "fl": 4}, "error": {"kind": "float", "exp": 4, "man": 3}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "seed": 18446744073709551615}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "seed": -1}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "seed": 3.75}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "seed": true}}',
    '{"weight": {"kind": "fixed", "wl": 4294967304, "fl": 4}}',      # wraps to 8
    '{"weight": {"kind": "float", "exp": 5, "man": 2}, "weight": {"kind": "fixed", "wl": 8, "fl": 4}}',
    # rejected
    '[]', '3', 'not json', '{"weight": 3}', '{"bias": {"kind": "float", "exp": 5, "man": 2}}',
    '{"weight": {"exp": 5, "man": 2}}', '{"weight": {"kind": "decimal"}}',
    '{"weight": {"kind": "float", "exp": 5}}', '{"weight": {"kind": "float", "exp": 5.0, "man": 2}}',
    '{"weight": {"kind": "float", "exp": 9, "man": 2}}',
    '{"weight": {"kind": "float", "exp": 5, "man": 2, "wl": 8}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "block": "tensor"}}',
    '{"weight": {"kind": "block", "wl": 8, "fl": 1}}',
    '{"weight": {"kind": "block", "wl": 8, "block": {"dim": -1}}}',
    '{"weight": {"kind": "block", "wl": 8, "block": {"dim": 1, "x": 2}}}',
    '{"weight": {"kind": "block", "wl": 8, "block": "rows"}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "rounding": "up"}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "colour": 1}}',
    '{"weight": {"kind": "float", "exp": NaN, "man": 2}}',
    # type errors (the reference's json library throws type_error)
    '{"weight": {"kind": 3}}', '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "symmetric": 1}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "seed": "7"}}',
    '{"weight": {"kind": "fixed", "wl": 8, "fl": 4, "rounding": 0}}',
]


@pytest.mark.parametrize("text", CONFIGS)
@pytest.mark.parametrize("default_seed", [0, 0x15EED, 2**64 - 1])
def test_quant_config_matches_reference(ref, text, default_seed):
    from paper_1910_04540_b200 import io as lio
    from paper_1910_04540_b200._lib import FormatError
    st, want = ref.parse_quant_config(text, default_seed)
    if st == 1:
        with pytest.raises(FormatError):
            lio.parse_quant_config(text, default_seed)
        return
    if st == 7:
        with pytest.raises(lio.ConfigTypeError):
            lio.parse_quant_config(text, default_seed)
        return
    assert st == 0
    cfg = lio.parse_quant_config(text, default_seed)
    for name, w in zip(("weight", "accumulator", "gradient", "activation", "error"), want):
        got = getattr(cfg, name)
        if w is None:
            assert got is None, name
            continue
        wf, wmode, wseed = w
        f = got.format.c()
        for field, _ in f._fields_:
            assert getattr(f, field) == getattr(wf, field), (text, name, field)
        assert int(got.mode) == wmode and got.seed == wseed and got.call_counter == 0


def test_load_quant_config(tmp_path):
    from paper_1910_04540_b200 import io as lio
    from paper_1910_04540_b200._lib import FormatError
    p = tmp_path / "cfg.json"
    p.write_text('{"gradient": {"kind": "fixed", "wl": 8, "fl": 4, "rounding": "stochastic"}}')
    cfg = lio.load_quant_config(str(p), 5)
    assert cfg.weight is None and cfg.gradient.format.wl == 8
    assert cfg.gradient.seed == lio._mix64(5 ^ lio._mix64(2))
    with pytest.raises(FormatError):
        lio.load_quant_config(str(tmp_path / "missing.json"), 5)
