"""GPU parity of the GEMMs.

* quant_gemm (per-op-rounded, lpq_quant_gemm) vs the reference's OWN
  composition (mul -> quantize_fused_at -> add -> quantize_fused_at per k,
  tests/golden/golden_gemm_v1.npz, made by tests/golden/make_golden_gemm.py
  through oracle/_ref) and vs the restated oracle lpqo_quant_gemm (itself
  pinned to that composition on the CPU, test_oracle_golden.py): bit-exact,
  both kernels (hardware-bf16 fast path and the general path), every rounding
  mode, and 64 sampled rows of the 4096^3 BASELINE problem.
* quantized_matmul (lpq_matmul_q) vs the reference library's own
  quantized_matmul outputs (golden fixtures) and the oracle's double matmul.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import golden_cases
from oracle_lib import (ALL_MODES, NEAREST_EVEN, STOCHASTIC, bits, fixed_fmt,
                        float_fmt)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1910_04540_b200 as q
    return q


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def bf16_operands(oracle, shape, seed, lo=-1.0, hi=1.0):
    n = int(np.prod(shape))
    x = oracle.random_uniform(n, seed, 0, lo, hi)
    st, xq = oracle.quantize(x, float_fmt(8, 7), NEAREST_EVEN)
    return xq.reshape(shape)


@pytest.mark.parametrize("M,N,K", [(64, 64, 64), (200, 300, 257), (1, 7, 3),
                                   (129, 131, 1000), (256, 256, 16)])
def test_quant_gemm_bf16_path_vs_oracle(q, oracle, M, N, K):
    a = bf16_operands(oracle, (M, K), 1)
    b = bf16_operands(oracle, (K, N), 2)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    assert st == 0
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


def test_quant_gemm_general_path_non_bf16_inputs(q, oracle):
    rng = np.random.default_rng(4)
    a = rng.uniform(-1, 1, (70, 90)).astype(np.float32)   # not bf16-exact
    b = rng.uniform(-1, 1, (90, 50)).astype(np.float32)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


@pytest.mark.parametrize("M,N,K,seed", [(70, 50, 90, 4), (128, 128, 64, 5), (131, 257, 129, 6),
                                        (1, 3, 2, 7), (256, 128, 1000, 8)])
def test_quant_gemm_raw_fp32_operands(q, oracle, M, N, K, seed):
    # operands that are NOT bf16-exact (float(8,7) nearest): the raw kernel
    # (FMUL pairs rounded by cvt.rn.bf16x2, then HADD2) under the pre-scan
    # proof; zeros of both signs included
    rng = np.random.default_rng(seed)
    a = rng.uniform(-3, 3, (M, K)).astype(np.float32)
    b = rng.uniform(-3, 3, (K, N)).astype(np.float32)
    a.reshape(-1)[:: 7] = 0.0
    b.reshape(-1)[1:: 11] = -0.0
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    assert st == 0
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


@pytest.mark.parametrize("case", ["tiny", "subnormal", "huge"])
def test_quant_gemm_raw_guards(q, oracle, case):
    # raw operands outside the raw kernel's proof: products near 2^-126, a
    # subnormal operand, sums near the top of the range -> the general kernel
    rng = np.random.default_rng(17)
    a = rng.uniform(-1, 1, (40, 60)).astype(np.float32)
    b = rng.uniform(-1, 1, (60, 30)).astype(np.float32)
    if case == "tiny":
        a *= np.float32(2.0**-60)
        b *= np.float32(2.0**-58)
    elif case == "subnormal":
        a[3, 5] = np.float32(2.0**-140)
    else:
        a *= np.float32(2.0**66)
        b *= np.float32(2.0**60)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want)), case


@pytest.mark.parametrize("fm,fa,K", [((8, 7), (8, 7), 300), ((8, 10), (8, 3), 200),
                                     ((5, 10), (5, 10), 64), ((5, 2), (5, 2), 12),
                                     ((4, 3), (6, 5), 8)])
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
@pytest.mark.parametrize("N", [64, 30])
def test_quant_gemm_bit_domain_kernel(q, oracle, fm, fa, K, mode, N):
    # operands in [0.5, 2) with random signs keep every product and sum
    # inside both formats' normal ranges for these K, so the pre-scan selects
    # k_qgemm_bits (bit-domain Q after every op); N = 30 takes its scalar-
    # variate form (flat indices of a thread's 4 columns not 4-aligned)
    rng = np.random.default_rng(fm[0] * 100 + fa[1] * 10 + mode + N)
    M = 70
    a = (rng.uniform(0.5, 2.0, (M, K)) * rng.choice([-1, 1], (M, K))).astype(np.float32)
    b = (rng.uniform(0.5, 2.0, (K, N)) * rng.choice([-1, 1], (K, N))).astype(np.float32)
    st, want = oracle.quant_gemm(a, b, float_fmt(*fm), float_fmt(*fa), mode,
                                 seed=1234, call=6, row_base=3)
    assert st == 0
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(*fm), q.FloatFormat(*fa),
                       q.RoundingMode(mode), 1234, 6, row_base=3)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (fm, fa, mode, N)


def test_quant_gemm_underflow_guard(q, oracle):
    # bf16-exact operands whose products fall below 2^-126: the device-side
    # pre-scan must route to the general kernel (two-point underflow grid)
    a = bf16_operands(oracle, (40, 60), 5) * np.float32(2.0**-70)
    b = bf16_operands(oracle, (60, 30), 6) * np.float32(2.0**-60)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


def test_quant_gemm_overflow_guard(q, oracle):
    a = bf16_operands(oracle, (20, 64), 7) * np.float32(2.0**70)
    b = bf16_operands(oracle, (64, 20), 8) * np.float32(2.0**62)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


@pytest.mark.parametrize("fm,fa", [((5, 2), (5, 2)), ((8, 7), (8, 7)),
                                   ((4, 3), (8, 10)), ((8, 23), (8, 23))])
@pytest.mark.parametrize("mode", ALL_MODES)
def test_quant_gemm_formats_modes(q, oracle, fm, fa, mode):
    rng = np.random.default_rng(fm[0] * 10 + fa[1] + mode)
    a = rng.uniform(-2, 2, (33, 47)).astype(np.float32)
    b = rng.uniform(-2, 2, (47, 29)).astype(np.float32)
    st, want = oracle.quant_gemm(a, b, float_fmt(*fm), float_fmt(*fa), mode,
                                 seed=99, call=4, row_base=5)
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(*fm), q.FloatFormat(*fa),
                       q.RoundingMode(mode), 99, 4, row_base=5)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


def test_quant_gemm_host_path(q, oracle):
    a = bf16_operands(oracle, (50, 70), 11)
    b = bf16_operands(oracle, (70, 40), 12)
    st, want = oracle.quant_gemm(a, b, float_fmt(8, 7), float_fmt(8, 7))
    got = q.quant_gemm(a, b, q.FloatFormat(8, 7), q.FloatFormat(8, 7))
    assert np.array_equal(bits(got), bits(want))


def test_quant_gemm_identity_format_is_fp32_sequential(q):
    # float(8,23) Q is the identity on normal values: the per-op GEMM then
    # equals a plain fp32 mul/add chain in ascending k
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, (16, 40)).astype(np.float32)
    b = rng.uniform(-1, 1, (40, 12)).astype(np.float32)
    want = np.zeros((16, 12), np.float32)
    for k in range(40):
        want = (want + (a[:, k:k + 1] * b[k:k + 1, :]).astype(np.float32)).astype(np.float32)
    got = q.quant_gemm(dev(a), dev(b), q.FloatFormat(8, 23), q.FloatFormat(8, 23))
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


GOLDEN_GEMM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "golden_gemm_v1.npz")


def test_quant_gemm_vs_reference_composition_goldens(q):
    """Every case the reference library produced through its own tensor ops
    (bf16-exact inputs take k_qgemm_bf16, the rest k_qgemm_general), on the
    device path and the host path."""
    z = np.load(GOLDEN_GEMM)
    n = 0
    for ci, em, mm, ea, ma, mode, seed, call in z["meta"]:
        a, b, want = z[f"a{ci}"], z[f"b{ci}"], z[f"c{ci}_{mode}"]
        args = (q.FloatFormat(int(em), int(mm)), q.FloatFormat(int(ea), int(ma)),
                q.RoundingMode(int(mode)), int(seed), int(call))
        got = q.quant_gemm(dev(a), dev(b), *args).cpu().numpy()
        assert np.array_equal(bits(got), bits(want)), (ci, mode)
        got_h = q.quant_gemm(a, b, *args)
        assert np.array_equal(bits(got_h), bits(want)), (ci, mode, "host")
        n += 1
    assert n == len(z["meta"]) >= 25


def _sampled_rows(n, count=64, seed=0):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, 127, 128, 255, 256, n // 2, n - 129, n - 128, n - 1]
    extra = rng.choice(n, count - len(fixed), replace=False)
    return sorted(set(fixed) | set(int(r) for r in extra))[:count]


def _parallel_rows(fn, rows):
    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        return list(ex.map(fn, rows))


@pytest.mark.parametrize("operands", ["f87", "raw"])
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_c4_quant_gemm_4096_sampled_rows(q, oracle, mode, operands):
    """C4 (4096^3, float(8,7) after every multiply and add; bench configs
    c4 / c4raw / c4s): 64 sampled output rows (tile borders included) vs the
    oracle, rows in parallel host threads.  Nearest runs the exact-bf16 kernel
    on float(8,7) operands and the raw-bf16 kernel on raw fp32 ones;
    stochastic runs the bit-domain kernel."""
    n = 4096
    a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
    b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
    if operands == "f87":
        f87 = q.QuantSpec(q.FloatFormat(8, 7))
        a = q.quantize_fused_at(a, f87, 0)
        b = q.quantize_fused_at(b, f87, 0)
    c = q.quant_gemm(a, b, q.FloatFormat(8, 7), q.FloatFormat(8, 7), q.RoundingMode(mode),
                     0x15EED, 2).cpu().numpy()
    ah, bh = a.cpu().numpy(), b.cpu().numpy()
    rows = _sampled_rows(n, 64, seed=mode)

    def one(r):
        st, want = oracle.quant_gemm(ah[r:r + 1], bh, float_fmt(8, 7), float_fmt(8, 7),
                                     mode, seed=0x15EED, call=2, row_base=r)
        return r, st == 0 and np.array_equal(bits(c[r:r + 1]), bits(want))
    bad = [r for r, ok in _parallel_rows(one, rows) if not ok]
    assert len(rows) == 64 and not bad, bad


def test_matmul_q_4096_sampled_rows(q, oracle):
    """The reference quantized_matmul at bench size (bench.py --config c4ref:
    4096^3, fixed(8,4) stochastic, FP64 tensor-core DMMA + fused Q): 64
    sampled rows vs the oracle's double matmul (tensor.cpp:355-376) and
    quantizer with the rows' global index base."""
    n = 4096
    a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
    b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
    spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 0x15EED)
    c = q.quantized_matmul_at(a, b, spec, 0).cpu().numpy()
    ah, bh = a.cpu().numpy(), b.cpu().numpy()
    rows = _sampled_rows(n, 64, seed=7)

    def one(r):
        acc = oracle.matmul(ah[r:r + 1], bh)
        st, want = oracle.quantize(acc, fixed_fmt(8, 4), STOCHASTIC, seed=0x15EED, call=0,
                                   index_base=r * n)
        return r, st == 0 and np.array_equal(bits(c[r:r + 1]), bits(want))
    bad = [r for r, ok in _parallel_rows(one, rows) if not ok]
    assert not bad, bad


def test_matmul_q_vs_reference_goldens(q, oracle):
    z = golden_cases.load()
    a, b = z["mm_a"], z["mm_b"]
    ident = q.QuantSpec(q.FloatFormat(8, 23))
    assert np.array_equal(bits(q.quantized_matmul(dev(a), dev(b), ident).cpu().numpy()),
                          bits(z["mm_c"]))
    s = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 11, 3)
    got = q.quantized_matmul(dev(a), dev(b), s).cpu().numpy()
    assert np.array_equal(bits(got), bits(z["qmm_fixed84_stoch_s11_c3"]))
    assert s.call_counter == 4
    s = q.QuantSpec(q.FloatFormat(5, 2))
    got = q.quantized_matmul(a, b, s)  # host path
    assert np.array_equal(bits(got), bits(z["qmm_float52_even"]))


@pytest.mark.parametrize("M,N,K", [(100, 90, 513), (256, 128, 64), (3, 5, 7)])
def test_matmul_q_vs_oracle(q, oracle, M, N, K):
    rng = np.random.default_rng(M + N + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    c = oracle.matmul(a, b)
    for fmt, qf in [(fixed_fmt(8, 4), q.FixedFormat(8, 4)), (float_fmt(5, 2), q.FloatFormat(5, 2))]:
        for mode in ALL_MODES:
            st, want = oracle.quantize(c, fmt, mode, seed=3, call=1)
            got = q.quantized_matmul_at(dev(a), dev(b), q.QuantSpec(qf, q.RoundingMode(mode), 3), 1)
            assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (fmt, mode)
    from oracle_lib import block_fmt
    st, want = oracle.quantize(c, block_fmt(8, 0), NEAREST_EVEN)
    got = q.quantized_matmul_at(dev(a), dev(b), q.QuantSpec(q.BlockFloatFormat(8, 0)), 0)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


def test_gemm_empty_inner_dimension(q, oracle):
    # K = 0: every output is the empty sum, +0 (acc starts at +0; the
    # reference matmul's double accumulator is 0.0, quantized to +0)
    a = np.zeros((5, 0), np.float32)
    b = np.zeros((0, 7), np.float32)
    f87 = q.FloatFormat(8, 7)
    got = q.quant_gemm(dev(a), dev(b), f87, f87).cpu().numpy()
    assert got.shape == (5, 7) and np.array_equal(bits(got), np.zeros((5, 7), np.uint32))
    for fmt in (q.FloatFormat(5, 2), q.FixedFormat(8, 4), q.BlockFloatFormat(8, 0)):
        got = q.quantized_matmul_at(dev(a), dev(b), q.QuantSpec(fmt), 0).cpu().numpy()
        assert np.array_equal(bits(got), np.zeros((5, 7), np.uint32)), fmt


@pytest.mark.parametrize("M,N,K", [(131, 77, 1001), (256, 256, 512)])
def test_matmul_q_adversarial_accumulation(q, oracle, M, N, K):
    # exponents over 2^-40..2^40 and sign-alternating near-cancelling terms:
    # any deviation from the ascending-k DFMA chain of the reference
    # (tensor.cpp:355-376) -- e.g. a reordered or single-rounding k-group sum
    # in the FP64 tensor-core path -- shows up in the rounded result
    rng = np.random.default_rng(M * N + K)
    a = (rng.uniform(1, 2, (M, K)) * 2.0 ** rng.integers(-40, 41, (M, K))
         * rng.choice([-1, 1], (M, K))).astype(np.float32)
    b = (rng.uniform(1, 2, (K, N)) * 2.0 ** rng.integers(-40, 41, (K, N))).astype(np.float32)
    b[1::2] = -b[::2][: b[1::2].shape[0]]  # pairs that nearly cancel
    c = oracle.matmul(a, b)
    got = q.quantized_matmul_at(dev(a), dev(b), q.QuantSpec(q.FloatFormat(8, 23)), 0)
    st, want = oracle.quantize(c, float_fmt(8, 23), NEAREST_EVEN)
    assert st == 0 and np.array_equal(bits(got.cpu().numpy()), bits(want))
