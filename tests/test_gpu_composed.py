"""The many-kernel GPU baseline (lpq_quantize_composed) -- the reference's
quantize_composed (proj/src/quant_ops.cpp:117-150) on B200.

Mirrors proj/tests/test_quant_ops.cpp:119-181: fused and composed agree
bitwise for fixed and block formats in every rounding mode over assorted
shapes; float formats are rejected; the composed chain makes >= 4 (fixed) /
>= 6 (block) data passes while fused makes <= 2.
"""
import numpy as np
import pytest

from oracle_lib import bits

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1910_04540_b200 as q
    return q


def random_shape(rng):
    return tuple(int(v) for v in rng.integers(1, 7, size=int(rng.integers(1, 5))))


def formats(q):
    return [q.FixedFormat(8, 4), q.FixedFormat(3, 1), q.FixedFormat(8, 4, True),
            q.FixedFormat(6, 2, False, False), q.FixedFormat(5, 2, True, False),
            q.BlockFloatFormat(8), q.BlockFloatFormat(4), q.BlockFloatFormat(8, 0),
            q.BlockFloatFormat(6, 1)]


def test_fused_equals_composed_bitwise(q, oracle):
    rng = np.random.default_rng(7000)
    checked = 0
    for fmt in formats(q):
        for mode in q.RoundingMode:
            spec = q.QuantSpec(fmt, mode, 123)
            for rep in range(12):
                shape = random_shape(rng)
                if isinstance(fmt, q.BlockFloatFormat) and fmt.block_dim is not None \
                        and fmt.block_dim >= len(shape):
                    shape = shape + (2,) * (fmt.block_dim + 1 - len(shape))
                x = rng.uniform(-30, 30, shape).astype(np.float32)
                xd = torch.from_numpy(x).cuda()
                fused = q.quantize_fused_at(xd, spec, rep).cpu().numpy()
                comp = q.quantize_composed_at(xd, spec, rep).cpu().numpy()
                assert np.array_equal(bits(fused), bits(comp)), (fmt, mode, shape)
                checked += 1
    assert checked > 400


def test_composed_large_and_host(q):
    x = q.random_uniform((1 << 22,), 9, 0, -10.0, 10.0)
    for fmt in (q.FixedFormat(8, 4), q.BlockFloatFormat(8), q.BlockFloatFormat(8, 0)):
        xx = x.view(1024, 4096) if isinstance(fmt, q.BlockFloatFormat) else x
        spec = q.QuantSpec(fmt, q.RoundingMode.Stochastic, 0x15EED)
        f = q.quantize_fused_at(xx, spec, 0)
        c = q.quantize_composed_at(xx, spec, 0)
        assert torch.equal(f.view(torch.int32), c.view(torch.int32))
        h = q.quantize_composed_at(xx.cpu().numpy(), spec, 0)
        assert np.array_equal(bits(h), bits(f.cpu().numpy()))


def test_composed_rejects_float_and_counts_passes(q):
    t = torch.from_numpy(np.random.default_rng(71).uniform(-4, 4, (32, 32))
                         .astype(np.float32)).cuda()
    with pytest.raises(q.UnsupportedFormatError):
        q.quantize_composed(t, q.QuantSpec(q.FloatFormat(5, 2)))
    q.reset_pass_count()
    q.quantize_composed_at(t, q.QuantSpec(q.FixedFormat(8, 4)), 0)
    assert q.pass_count() >= 4
    q.reset_pass_count()
    q.quantize_composed_at(t, q.QuantSpec(q.BlockFloatFormat(8)), 0)
    assert q.pass_count() >= 6
    q.reset_pass_count()
    q.quantize_fused_at(t, q.QuantSpec(q.BlockFloatFormat(8)), 0)
    assert q.pass_count() <= 2


def test_composed_validation_errors(q):
    # tensor.cpp map_elements: a non-finite result raises invalid_value_error
    bad = torch.tensor([1.0, float("inf")], device="cuda")
    with pytest.raises(q.InvalidValueError):
        q.quantize_composed(bad, q.QuantSpec(q.FixedFormat(8, 4)))
    with pytest.raises(q.InvalidValueError):
        q.quantize_composed(bad, q.QuantSpec(q.BlockFloatFormat(8)))
