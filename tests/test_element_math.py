"""The kernels' per-element arithmetic (paper_1910_04540_b200/csrc/
quant_math.cuh), compiled for the host CPU, swept against the oracle.

The same source is inlined into every sm_100a quantizer kernel, so this pins
the exactness arguments of DESIGN.md §3 on ~10^6 inputs per (format, mode)
without a GPU: random bit patterns over the whole finite fp32 range, random
magnitudes 2^-150..2^127, uniform values, and hand-picked edges.  The GPU
tests then only have to show the kernels apply it to the right elements.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle_lib import (ALL_MODES, block_fmt, bits, f32_from_bits, fixed_fmt,
                        float_fmt, Fmt)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hm():
    from paper_1910_04540_b200._build import build_host_math
    path = build_host_math()
    L = C.CDLL(path)
    fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
    up = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
    L.hm_quant.argtypes = [fp, up, fp, C.c_int64, C.POINTER(Fmt), C.c_int]
    L.hm_quant_block.argtypes = [fp, up, fp, C.c_int64, C.c_int, C.c_uint32, C.c_int]
    L.hm_quant_block.restype = C.c_int
    L.hm_variate24.restype = C.c_uint32
    L.hm_variate24.argtypes = [C.c_uint64, C.c_uint64]
    L.hm_stream_key.restype = C.c_uint64
    L.hm_stream_key.argtypes = [C.c_uint64, C.c_uint64]
    L.hm_variates24.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_variates24_balanced.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_variates24_fma.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_variates24_x4.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_variates24_x4_top.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_variates24_x4_topw.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, up]
    L.hm_quant_float_bits_top.argtypes = [fp, up, fp, C.c_int64, C.c_int, C.c_int]
    L.hm_quant_float_bits.argtypes = [fp, up, fp, C.c_int64, C.c_int, C.c_int]
    return L


def variates(hm, seed, call, n):
    v = np.empty(n, np.uint32)
    hm.hm_variates24(hm.hm_stream_key(seed, call), 0, n, v)
    return v


def inputs(n=1 << 18, seed=7):
    rng = np.random.default_rng(seed)
    b = f32_from_bits(rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32))
    mags = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-150, 128, n)).astype(np.float32)
    u = rng.uniform(-20, 20, n).astype(np.float32)
    sp = np.array([0.0, -0.0, 0.5, -0.5, 1.5, 2.5, -2.5, 1e-45, -1e-45, 3.99,
                   0.25, -0.25, 0.75, 114688.0, 122880.0, 3.4028235e38], np.float32)
    x = np.concatenate([sp, b, mags, u])
    return x[np.isfinite(x)]


FORMATS = [float_fmt(5, 2), float_fmt(8, 7), float_fmt(8, 23), float_fmt(1, 0),
           float_fmt(2, 1), float_fmt(4, 3), float_fmt(1, 23), float_fmt(8, 0),
           float_fmt(3, 2), float_fmt(7, 12),
           fixed_fmt(8, 4), fixed_fmt(3, 1), fixed_fmt(8, 4, True),
           fixed_fmt(6, 2, False, False), fixed_fmt(5, 2, True, False),
           fixed_fmt(24, 126), fixed_fmt(2, -126), fixed_fmt(24, -104, False, False),
           fixed_fmt(24, 100, True, False), fixed_fmt(12, 60, False, False),
           fixed_fmt(4, -20, False, False)]


def test_variate24_matches_reference_rng(hm, oracle):
    for seed, call in [(1, 0), (0x15EED, 0), (77, 5), (2**64 - 1, 2**63 + 5)]:
        key = hm.hm_stream_key(seed, call)
        assert key == oracle.L.lpqo_stream_key(seed, call)
        for i in list(range(300)) + [2**40 + 3, 2**64 - 1]:
            assert hm.hm_variate24(key, i) * 2.0**-24 == oracle.variate(seed, call, i)


def test_balanced_variate_form_is_identical(hm):
    for key, base in [(0, 0), (0x5E41AB087439611E, 2**40), (2**64 - 1, 2**63)]:
        a = np.empty(1 << 16, np.uint32)
        b = np.empty(1 << 16, np.uint32)
        hm.hm_variates24(key, base, a.size, a)
        hm.hm_variates24_balanced(key, base, b.size, b)
        assert np.array_equal(a, b)
        hm.hm_variates24_fma(key, base, b.size, b)
        assert np.array_equal(a, b)


def test_float4_variate_form_is_identical(hm):
    # variate24_x4 shares the high word of key ^ (idx + q) + C0 across the 4
    # lanes; cover its carry fallback (low word of w within 3 of 2^32) too
    C0 = 0x9E3779B97F4A7C15
    near = []
    for d in range(0, 8):  # key ^ idx with (z & ~3) + C0 ending at 2^32 - 1 - d
        z = ((1 << 32) - 1 - d - (C0 & 0xFFFFFFFF)) & 0xFFFFFFFF | (0x12345 << 32)
        near.append((z & ~3 & (2**64 - 1), 0))
    for top2 in range(4):  # ... and the shared >> 30 word (no carry past bit 29)
        for d in range(0, 8):
            wlo = (top2 << 30) | (0x3FFFFFFF - d)
            z = ((wlo - (C0 & 0xFFFFFFFF)) & 0xFFFFFFFF) | (0xABCDE << 32)
            near.append((z & ~3 & (2**64 - 1), 0))
            near.append((0, z & ~3 & (2**64 - 1)))
    cases = [(0, 0), (0x5E41AB087439611E, 2**40), (2**64 - 1, 2**63), (3, 4), (6, 2**32 - 4)] + near
    for key, base in cases:
        n = 1 << 12
        a = np.empty(n, np.uint32)
        b = np.empty(n, np.uint32)
        hm.hm_variates24(key, base, n, a)
        hm.hm_variates24_x4(key, base, n, b)
        assert np.array_equal(a, b), (key, base)
        hm.hm_variates24_x4_top(key, base, n, b)
        assert np.array_equal(a, b), (key, base, "top")
        hm.hm_variates24_x4_topw(key, base, n, b)
        assert np.array_equal(a, b), (key, base, "topw")


@pytest.mark.parametrize("em", [(5, 2), (4, 3), (2, 1), (7, 12), (3, 0), (8, 22)])
def test_float_bits_top_form_is_identical(hm, em):
    # quant_float_bits_top(top) == quant_float_bits<stochastic>(top >> 8) for
    # every sign, whatever the top word's low 8 bits hold
    rng = np.random.default_rng(em[0] * 31 + em[1])
    x = inputs(1 << 16, seed=em[0])
    v = rng.integers(0, 1 << 24, size=x.size, dtype=np.uint64).astype(np.uint32)
    junk = rng.integers(0, 256, size=x.size, dtype=np.uint64).astype(np.uint32)
    v[:4] = [0, (1 << 24) - 1, 1, (1 << 23)]
    top = (v << np.uint32(8)) | junk
    a = np.empty_like(x)
    b = np.empty_like(x)
    hm.hm_quant_float_bits(x, v, a, x.size, *em)
    hm.hm_quant_float_bits_top(x, top, b, x.size, *em)
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("fmt", FORMATS, ids=repr)
@pytest.mark.parametrize("mode", ALL_MODES)
def test_elementwise_math_vs_oracle(hm, oracle, fmt, mode):
    x = inputs()
    seed, call = 9 + mode, 3
    st, want = oracle.quantize(x, fmt, mode, seed=seed, call=call)
    assert st == 0
    v = variates(hm, seed, call, x.size) if mode == 0 else np.zeros(x.size, np.uint32)
    got = np.empty_like(x)
    hm.hm_quant(x, v, got, x.size, C.byref(fmt), mode)
    bad = bits(got) != bits(want)
    assert not bad.any(), (x[bad][:4], got[bad][:4], want[bad][:4])


@pytest.mark.parametrize("wl", [2, 3, 4, 8, 12, 24])
@pytest.mark.parametrize("mode", ALL_MODES)
def test_block_math_vs_oracle(hm, oracle, wl, mode):
    rng = np.random.default_rng(wl * 10 + mode)
    for trial in range(40):
        e = int(rng.integers(-160, 128))
        x = (rng.uniform(-1, 1, 301) * 2.0**e).astype(np.float32)
        if trial % 5 == 0:
            x[:150] = 0.0
        if trial == 3:
            x[:] = 0.0
        if not np.isfinite(x).all():
            continue
        seed, call = 5, trial
        st, want = oracle.quantize(x, block_fmt(wl), mode, seed=seed, call=call)
        v = variates(hm, seed, call, x.size)
        got = np.empty_like(x)
        badblk = hm.hm_quant_block(x, v, got, x.size, wl,
                                   int(bits(np.abs(x)).max()), mode)
        if st == 3:
            assert badblk
            continue
        assert st == 0 and not badblk
        assert np.array_equal(bits(got), bits(want)), (wl, mode, e)


UNDER_FMTS = [float_fmt(5, 2), float_fmt(2, 1), float_fmt(4, 3), float_fmt(3, 2),
              float_fmt(7, 12), float_fmt(6, 0), float_fmt(2, 22), float_fmt(8, 7)]


def _underflow_cases(fmt):
    """Inputs at the underflow boundaries of `fmt` and, per input, variates at
    the stochastic decision boundary (T = |x| * 2^(24 - min_exp))."""
    min_exp = 1 - ((1 << (fmt.exp_bits - 1)) - 1)
    half, mn = 2.0 ** (min_exp - 1), 2.0 ** min_exp
    mags = [half, np.nextafter(np.float32(half), np.float32(0)),
            np.nextafter(np.float32(half), np.float32(1)),
            np.nextafter(np.float32(mn), np.float32(0)), mn, 1e-45, 2e-45,
            2.0 ** (min_exp - 24), 3 * 2.0 ** (min_exp - 24), 2.0 ** (min_exp - 2),
            (2 ** 24 - 1) * 2.0 ** (min_exp - 24), 1.5 * 2.0 ** (min_exp - 24),
            0.75 * mn, 0.3 * mn]
    xs, vs = [], []
    for m in mags:
        m = np.float32(m)
        if not np.isfinite(m) or m == 0:
            continue
        t = float(m) * 2.0 ** (24 - min_exp)
        cand = {0, 1, 2 ** 24 - 1}
        for c in (np.floor(t), np.ceil(t)):
            if c < 2 ** 25:
                c = int(c)
                cand |= {c - 1, c, c + 1, 2 ** 24 - c - 1, 2 ** 24 - c, 2 ** 24 - c + 1}
        for v in sorted(c for c in cand if 0 <= c < 2 ** 24):
            for sgn in (1.0, -1.0):
                xs.append(np.float32(sgn * m))
                vs.append(v)
    return np.array(xs, np.float32), np.array(vs, np.uint32)


@pytest.mark.parametrize("fmt", UNDER_FMTS, ids=repr)
@pytest.mark.parametrize("mode", [0, 1])
def test_underflow_decision_boundaries(hm, oracle, fmt, mode):
    """The kernels' element math on the underflow two-point grid against the
    restated scalar quantizer with the SAME explicit variate u = v * 2^-24, at
    the round-to-nearest tie and at the stochastic decision boundary on both
    signs (v = T, T +- 1, 2^24 - T ...); the reference's own scalar API too
    when oracle/_ref is built."""
    x, v = _underflow_cases(fmt)
    got = np.empty_like(x)
    hm.hm_quant(x, v, got, x.size, C.byref(fmt), mode)
    u = (v.astype(np.float64) * 2.0 ** -24).astype(np.float32)
    want = np.array([oracle.quant_scalar(float(a), fmt, mode, float(b)) for a, b in zip(x, u)],
                    np.float32)
    bad = bits(got) != bits(want)
    assert not bad.any(), (x[bad][:4], v[bad][:4], got[bad][:4], want[bad][:4])
    from oracle_lib import RefLib
    if RefLib.available():
        st, ref = RefLib().quant_scalar_many(x, fmt, mode, u if mode == 0 else None)
        assert st == 0 and np.array_equal(bits(got), bits(ref))
