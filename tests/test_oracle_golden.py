"""Pin the C restatement (oracle/lpq_oracle.c) before trusting it.

1. Known-answer values transcribed from the reference's own unit tests
   (proj/tests/test_rng_rounding.cpp, test_scalar_quant.cpp) and KATs computed
   from the reference.
2. Every golden fixture in tests/golden/golden_v1.npz, which the reference
   library itself produced (tests/golden/make_golden.py).
"""
import numpy as np
import pytest

import golden_cases
from oracle_lib import (NEAREST_AWAY, NEAREST_EVEN, NEAREST_ZERO, STOCHASTIC,
                        block_fmt, bits, fixed_fmt, float_fmt)


# ---- rounding: test_rng_rounding.cpp:11-75 ----------------------------------
@pytest.mark.parametrize("r,mode,u,want", [
    (1.48, NEAREST_EVEN, 0, 1.0), (1.48, NEAREST_AWAY, 0, 1.0),
    (-2.75, NEAREST_EVEN, 0, -3.0), (5.0, NEAREST_ZERO, 0, 5.0),
    (0.5, NEAREST_EVEN, 0, 0.0), (0.5, NEAREST_AWAY, 0, 1.0),
    (0.5, NEAREST_ZERO, 0, 0.0), (-0.5, NEAREST_AWAY, 0, -1.0),
    (-0.5, NEAREST_EVEN, 0, 0.0), (-0.5, NEAREST_ZERO, 0, 0.0),
    (1.5, NEAREST_EVEN, 0, 2.0), (2.5, NEAREST_EVEN, 0, 2.0),
    (-1.5, NEAREST_EVEN, 0, -2.0), (-1.5, NEAREST_ZERO, 0, -1.0),
    (0.25, STOCHASTIC, 0.25, 0.0), (0.25, STOCHASTIC, 0.2499, 1.0),
    (0.25, STOCHASTIC, 0.9, 0.0), (3.0, STOCHASTIC, 0.0, 3.0),
    (-3.0, STOCHASTIC, 0.0, -3.0),
    (2.0**51 + 0.5, NEAREST_EVEN, 0, 2.0**51), (2.0**51 + 1.5, NEAREST_EVEN, 0, 2.0**51 + 2),
    (2.0**51 + 2.5, NEAREST_EVEN, 0, 2.0**51 + 2), (-(2.0**51 + 0.5), NEAREST_EVEN, 0, -(2.0**51)),
    (2.0**51 + 0.5, NEAREST_AWAY, 0, 2.0**51 + 1), (-(2.0**51 + 0.5), NEAREST_AWAY, 0, -(2.0**51 + 1)),
    (2.0**51 + 0.5, NEAREST_ZERO, 0, 2.0**51), (2.0**51 + 0.5, STOCHASTIC, 0.25, 2.0**51 + 1),
    (2.0**51 + 0.5, STOCHASTIC, 0.75, 2.0**51), (2.0**52, NEAREST_EVEN, 0, 2.0**52),
    (2.0**100, STOCHASTIC, 0.0, 2.0**100),
])
def test_round_integer_kats(oracle, r, mode, u, want):
    assert oracle.round_integer(r, mode, u) == want


def test_signed_zero_rules(oracle):
    # SURVEY.md Appendix A (verified against rounding.hpp): even/stochastic +0,
    # away -0 iff r<0, toward-zero -0 iff r>=0
    sb = lambda v: np.signbit(v)
    assert not sb(oracle.round_integer(-0.3, NEAREST_EVEN))
    assert sb(oracle.round_integer(-0.3, NEAREST_AWAY))
    assert not sb(oracle.round_integer(0.3, NEAREST_AWAY))
    assert sb(oracle.round_integer(0.3, NEAREST_ZERO))
    assert sb(oracle.round_integer(-0.0, NEAREST_ZERO))
    assert not sb(oracle.round_integer(-0.3, NEAREST_ZERO))
    assert not sb(oracle.round_integer(-0.3, STOCHASTIC, 0.1))  # -1 + 1 = +0


# ---- rng: test_rng_rounding.cpp:86-115 + KATs --------------------------------
def test_rng_kats(oracle):
    L = oracle.L
    assert L.lpqo_stream_key(1, 0) == 0x5E41AB087439611E
    v = [oracle.variate(0x15EED, 0, i) for i in range(3)]
    assert v == pytest.approx([0.83390957, 0.08302921, 0.60927117], abs=1e-7)
    u = [oracle.variate(3, 5, i) for i in range(1000)]
    assert all(0 <= x < 1 and x * 16777216.0 == int(x * 16777216.0) for x in u)


def test_rng_pinned_mean(oracle):
    # test_rng_rounding.cpp:107-115: mean of u(seed 1, call 0, i < 1e6)
    y = oracle.random_uniform(1_000_000, 1, 0, 0.0, 1.0)
    assert abs(float(np.mean(y.astype(np.float64))) - 0.500005285987) < 1e-9


# ---- scalar quantizer goldens: test_scalar_quant.cpp:60-147 -----------------
def test_fixed_examples(oracle):
    f31 = fixed_fmt(3, 1)
    assert oracle.quant_scalar(0.74, f31, NEAREST_EVEN) == 0.5
    assert oracle.quant_scalar(-5.0, f31, NEAREST_EVEN) == -2.0
    assert oracle.quant_scalar(0.25, f31, NEAREST_AWAY) == 0.5
    assert oracle.quant_scalar(0.25, f31, NEAREST_EVEN) == 0.0
    wrap = fixed_fmt(3, 1, False, False)
    assert oracle.quant_scalar(-5.0, wrap, NEAREST_EVEN) == -1.0
    assert oracle.quant_scalar(1.5, wrap, NEAREST_EVEN) == 1.5


def test_float_examples(oracle):
    assert oracle.quant_scalar(1.3, float_fmt(5, 2), NEAREST_EVEN) == 1.25
    assert oracle.quant_scalar(100.0, float_fmt(2, 1), NEAREST_EVEN) == 6.0
    assert oracle.quant_scalar(-100.0, float_fmt(2, 1), NEAREST_EVEN) == -6.0
    tiny = 2.0**-6
    f43 = float_fmt(4, 3)
    assert oracle.quant_scalar(np.float32(0.4 * tiny), f43, NEAREST_EVEN) == 0.0
    assert oracle.quant_scalar(np.float32(0.6 * tiny), f43, NEAREST_EVEN) == tiny
    assert oracle.quant_scalar(0.5 * tiny, f43, NEAREST_EVEN) == 0.0
    assert oracle.quant_scalar(0.5 * tiny, f43, NEAREST_AWAY) == tiny
    assert oracle.quant_scalar(-0.5 * tiny, f43, NEAREST_AWAY) == -tiny
    assert oracle.quant_scalar(0.5 * tiny, f43, NEAREST_ZERO) == 0.0


def test_block_examples(oracle):
    b8 = block_fmt(8)
    st, y = oracle.quantize(np.array([1.0, 3.0], np.float32), b8, NEAREST_EVEN)
    assert st == 0 and list(y) == [1.0, 3.0]
    st, y = oracle.quantize(np.array([0.7, 3.0], np.float32), b8, NEAREST_EVEN)
    assert list(y) == [0.6875, 3.0]
    st, y = oracle.quantize(np.array([0.0, 0.0], np.float32), b8, NEAREST_EVEN)
    assert list(y) == [0.0, 0.0]
    st, y = oracle.quantize(np.array([3.99], np.float32), b8, NEAREST_EVEN)
    assert y[0] == 127.0 * 0.03125


def test_identity_format_is_bit_exact(oracle):
    rng = np.random.default_rng(5)
    x = rng.standard_normal(100_000).astype(np.float32)
    st, y = oracle.quantize(x, float_fmt(8, 23), NEAREST_EVEN)
    assert st == 0 and np.array_equal(bits(x), bits(y))


def test_nonfinite_and_block_range(oracle):
    st, _ = oracle.quantize(np.array([1.0, np.inf], np.float32), fixed_fmt(8, 4), NEAREST_EVEN)
    assert st == 3
    st, _ = oracle.quantize(np.array([1.0, 2.0**127], np.float32), block_fmt(8), NEAREST_EVEN)
    assert st == 3
    st, _ = oracle.quantize(np.ones((4, 4), np.float32), block_fmt(8, 3), NEAREST_EVEN)
    assert st == 2


# ---- every reference-produced fixture -----------------------------------------
def test_oracle_matches_reference_fixtures(oracle):
    z = golden_cases.load()
    n = 0
    for i, fmt, mode, seed, call, st, x, y in golden_cases.quantize_cases(z):
        ost, oy = oracle.quantize(x, fmt, mode, seed=seed, call=call)
        assert ost == st, (i, fmt, mode)
        if st == 0:
            assert np.array_equal(bits(oy), bits(y)), (i, fmt, mode)
        n += 1
    assert n > 300
    assert np.array_equal(oracle.random_uniform(4097, 7, 0, -4.0, 4.0), z["uniform_s7_m4_4"])
    assert np.array_equal(oracle.random_uniform(1000, 2, 0, -10.0, 10.0), z["uniform_s2_m10_10"])
    v = np.array([oracle.variate(0x15EED, 0, i) for i in range(1000)], np.float32)
    assert np.array_equal(v, z["variates_15eed"])
    assert np.array_equal(oracle.matmul(z["mm_a"], z["mm_b"]), z["mm_c"])


# ---- the per-op GEMM's rounding order, pinned to the reference itself ----------
def _gemm_inputs(seed, m, k, n, scale_a=1.0, scale_b=1.0):
    rng = np.random.default_rng(seed)
    a = (rng.uniform(-1, 1, (m, k)) * scale_a).astype(np.float32)
    b = (rng.uniform(-1, 1, (k, n)) * scale_b).astype(np.float32)
    # edge values: zeros, exact powers of two, products on rounding ties,
    # magnitudes that underflow / saturate the narrow formats
    a.flat[::7] = 0.0
    b.flat[3::11] = np.float32(-0.0)
    a.flat[1::13] = np.float32(2.0 ** -9)
    b.flat[2::17] = np.float32(1.5)
    a.flat[5::19] = np.float32(3.0e4)
    b.flat[4::23] = np.float32(-1.0e-6)
    return a, b


GEMM_CASES = [  # (fmt_mul, fmt_add, m, k, n, scale_a, scale_b)
    ((8, 7), (8, 7), 6, 40, 5, 1.0, 1.0),
    ((5, 2), (5, 2), 5, 33, 7, 1.0, 1.0),
    ((4, 3), (4, 3), 4, 29, 6, 4.0, 0.25),
    ((5, 2), (8, 7), 3, 64, 4, 16.0, 16.0),     # saturating products, wider adds
    ((8, 23), (5, 10), 4, 17, 3, 1.0, 1.0),     # identity multiply, fp16-like adds
    ((2, 1), (3, 0), 3, 12, 3, 1.0, 1.0),       # tiny formats (max 6, 2-point grids)
]


@pytest.mark.parametrize("case", GEMM_CASES, ids=str)
@pytest.mark.parametrize("mode", [NEAREST_EVEN, NEAREST_AWAY, NEAREST_ZERO, STOCHASTIC])
def test_quant_gemm_restatement_equals_reference_composition(oracle, ref, case, mode):
    """The restated per-op GEMM (oracle/lpq_oracle.c lpqo_quant_gemm, which
    the device kernels are checked against) equals, bit for bit, the
    reference's OWN composition per k: mul -> quantize_fused_at(call+2k) ->
    add -> quantize_fused_at(call+2k+1) (tensor.cpp:140-156,
    quant_ops.cpp:154-164) -- so the rounding order and the
    stochastic call mapping are pinned to the reference library."""
    (em, mm), (ea, ma), m, k, n, sa, sb = case
    a, b = _gemm_inputs(hash((case, mode)) % 2**32, m, k, n, sa, sb)
    fm, fa = float_fmt(em, mm), float_fmt(ea, ma)
    st, want = ref.quant_gemm_composed(a, b, fm, fa, mode, seed=0x15EED, call=9)
    assert st == 0
    st, got = oracle.quant_gemm(a, b, fm, fa, mode, seed=0x15EED, call=9)
    assert st == 0
    assert np.array_equal(bits(got), bits(want)), (case, mode)


def test_oracle_quant_gemm_matches_reference_gemm_fixtures(oracle):
    """The restated per-op GEMM vs every fixture the reference produced
    through its own tensor-op composition (tests/golden/golden_gemm_v1.npz)."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "golden_gemm_v1.npz"))
    for ci, em, mm, ea, ma, mode, seed, call in z["meta"]:
        st, got = oracle.quant_gemm(z[f"a{ci}"], z[f"b{ci}"], float_fmt(int(em), int(mm)),
                                    float_fmt(int(ea), int(ma)), int(mode), seed=int(seed),
                                    call=int(call))
        assert st == 0 and np.array_equal(bits(got), bits(z[f"c{ci}_{mode}"])), (ci, mode)
