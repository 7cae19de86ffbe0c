"""GPU parity against the UNMODIFIED reference library itself.

The other GPU suites check the device path against the C restatement
(oracle/lpq_oracle.c), which the CPU suite pins to the reference.  These tests
skip the restatement: the device results are compared bit for bit with
oracle/_ref/liblpsim_ref.so -- the reference's own quant_ops.cpp / tensor.cpp
compiled unchanged (oracle/Makefile) -- through its lpsim::quantize_fused_at,
quantize_composed_at, quantized_matmul and its mul/quantize/add per-op GEMM
composition (oracle/ref_capi.cpp), on BASELINE-shaped inputs at sizes the
reference finishes in seconds.  The library travels with the tree (it is
built by build(), git-ignored, not gpurun-ignored); without it these tests
skip.
"""
import numpy as np
import pytest

from oracle_lib import (ALL_MODES, NEAREST_EVEN, STOCHASTIC, RefLib, bits,
                        block_fmt, fixed_fmt, float_fmt)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1910_04540_b200 as q
    return q


@pytest.fixture(scope="module")
def ref():
    if not RefLib.available():
        pytest.skip("oracle/_ref/liblpsim_ref.so not built")
    r = RefLib()
    r.set_num_threads(8)
    return r


def spec_of(q, fmt, mode, seed):
    if fmt.kind == 0:
        f = q.FloatFormat(fmt.exp_bits, fmt.man_bits)
    elif fmt.kind == 1:
        f = q.FixedFormat(fmt.wl, fmt.fl, bool(fmt.symmetric), bool(fmt.saturate))
    else:
        f = q.BlockFloatFormat(fmt.wl, None if fmt.block_dim < 0 else fmt.block_dim)
    return q.QuantSpec(f, q.RoundingMode(mode), seed, 0)


CASES = [
    # (format, shape): the BASELINE configs' formats at reduced sizes, and the
    # block plans (rows in registers, chunk rendezvous, two-pass segments and
    # columns, whole tensor)
    (float_fmt(5, 2), (1 << 20,)),
    (fixed_fmt(8, 4), (1 << 20,)),
    (fixed_fmt(8, 4, False, False), (100_003,)),       # wrap mode, ragged
    (float_fmt(8, 7), (333, 777)),
    (float_fmt(4, 3), (4099,)),
    (block_fmt(8, 0), (512, 4096)),                    # C3 rows
    (block_fmt(8, 0), (8, 200_000)),                   # chunk rendezvous
    (block_fmt(8, None), (1 << 20,)),                  # whole tensor (chunk plan)
    (block_fmt(8, None), (3_000_001,)),                # whole tensor, two-pass segments
    (block_fmt(6, 1), (64, 300, 33)),                  # columns
]


@pytest.mark.parametrize("fmt,shape", CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("mode", ALL_MODES)
def test_fused_vs_reference_library(q, ref, fmt, shape, mode):
    x = ref.random_uniform(shape, 7, 0, -4.0, 4.0)
    if fmt.kind == 2 and fmt.block_dim >= 0:  # blocks of different magnitudes
        rng = np.random.default_rng(5)
        scale = (2.0 ** rng.integers(-20, 20, shape[fmt.block_dim])).astype(np.float32)
        sh = [1] * len(shape)
        sh[fmt.block_dim] = shape[fmt.block_dim]
        x = (x * scale.reshape(sh)).astype(np.float32)
    st, want = ref.quantize(x, fmt, mode, seed=0x15EED, call=3)
    assert st == 0
    got = q.quantize_fused_at(torch.from_numpy(x).cuda(), spec_of(q, fmt, mode, 0x15EED), 3)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (fmt, shape, mode)
    # the host entry point (staged copies, byte-coded copy-back where it applies)
    got_h = q.quantize_fused_at(x, spec_of(q, fmt, mode, 0x15EED), 3)
    assert np.array_equal(bits(got_h), bits(want))


@pytest.mark.parametrize("fmt", [fixed_fmt(8, 4), block_fmt(8, 0), block_fmt(8, None)],
                         ids=str)
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_composed_vs_reference_library(q, ref, fmt, mode):
    x = ref.random_uniform((257, 1000), 9, 0, -4.0, 4.0)
    st, want = ref.quantize_composed(x, fmt, mode, seed=11, call=2)
    assert st == 0
    got = q.quantize_composed_at(torch.from_numpy(x).cuda(), spec_of(q, fmt, mode, 11), 2)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


@pytest.mark.parametrize("fmt", [fixed_fmt(8, 4), float_fmt(5, 2), block_fmt(8, None)],
                         ids=str)
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_quantized_matmul_vs_reference_library(q, ref, fmt, mode):
    a = ref.random_uniform((96, 200), 1, 0, -1.0, 1.0)
    b = ref.random_uniform((200, 72), 2, 0, -1.0, 1.0)
    st, want, _ = ref.quantized_matmul(a, b, fmt, mode, seed=3, call=1)
    assert st == 0
    spec = spec_of(q, fmt, mode, 3)
    got = q.quantized_matmul_at(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), spec, 1)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


@pytest.mark.parametrize("fm,fa", [((8, 7), (8, 7)), ((5, 2), (5, 2)), ((4, 3), (8, 10))])
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
@pytest.mark.parametrize("operands", ["raw", "bf16"])
def test_quant_gemm_vs_reference_composition(q, ref, fm, fa, mode, operands):
    # the per-op GEMM against the reference's OWN tensor ops per k:
    # mul -> quantize_fused_at(call + 2k) -> add -> quantize_fused_at(call + 2k + 1)
    # (tensor.cpp:140-156, quant_ops.cpp:154-164); raw and float(8,7)-exact
    # operands reach every kernel of the launch (exact / raw bf16, bits, general)
    a = ref.random_uniform((24, 40), 3, 0, -1.0, 1.0)
    b = ref.random_uniform((40, 20), 4, 0, -1.0, 1.0)
    if operands == "bf16":
        _, a = ref.quantize(a, float_fmt(8, 7), NEAREST_EVEN)
        _, b = ref.quantize(b, float_fmt(8, 7), NEAREST_EVEN)
    st, want = ref.quant_gemm_composed(a, b, float_fmt(*fm), float_fmt(*fa), mode, seed=5, call=7)
    assert st == 0
    got = q.quant_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                       q.FloatFormat(*fm), q.FloatFormat(*fa), q.RoundingMode(mode), 5, 7)
    assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (fm, fa, mode, operands)
