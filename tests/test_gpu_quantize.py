"""GPU parity: the sm_100a quantizer kernels through the C ABI vs the oracle.

Bar: bit-exact (memcmp of the fp32 bit patterns) for every format and all
four rounding modes, stochastic included (the kernels draw the reference's
own variates).  Checked against (a) the reference library's own outputs
(tests/golden fixtures), (b) the C restatement on seeded inputs of assorted
shapes, alignments and block plans, and (c) at BASELINE sizes, on sampled
windows plus size-independent properties.
"""
import numpy as np
import pytest

import golden_cases
from oracle_lib import (ALL_MODES, NEAREST_EVEN, STOCHASTIC, block_fmt, bits,
                        fixed_fmt, float_fmt)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def q():
    import paper_1910_04540_b200 as q
    return q


def spec_of(q, fmt, mode, seed=0):
    if fmt.kind == 0:
        f = q.FloatFormat(fmt.exp_bits, fmt.man_bits)
    elif fmt.kind == 1:
        f = q.FixedFormat(fmt.wl, fmt.fl, bool(fmt.symmetric), bool(fmt.saturate))
    else:
        f = q.BlockFloatFormat(fmt.wl, None if fmt.block_dim < 0 else fmt.block_dim)
    return q.QuantSpec(f, q.RoundingMode(mode), seed, 0)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def same_bits(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return np.array_equal(bits(a), bits(b))


# ---- (a) the reference's own outputs ---------------------------------------------
def test_golden_fixtures_device(q):
    n = 0
    for i, fmt, mode, seed, call, st, x, y in golden_cases.quantize_cases():
        spec = spec_of(q, fmt, mode, seed)
        if st != 0:
            with pytest.raises(q.InvalidInputError):
                q.quantize_fused_at(dev(x), spec, call)
            continue
        got = q.quantize_fused_at(dev(x), spec, call)
        assert same_bits(got, y), (i, fmt, mode)
        n += 1
    assert n > 300


def test_golden_fixtures_host_path(q):
    for i, fmt, mode, seed, call, st, x, y in golden_cases.quantize_cases():
        if i % 3:
            continue
        spec = spec_of(q, fmt, mode, seed)
        if st != 0:
            with pytest.raises(q.InvalidInputError):
                q.quantize_fused_at(x, spec, call)
            continue
        assert same_bits(q.quantize_fused_at(x, spec, call), y), (i, fmt, mode)


def test_generators_match_reference(q):
    z = golden_cases.load()
    u = q.random_uniform((4097,), 7, 0, -4.0, 4.0)
    assert same_bits(u, z["uniform_s7_m4_4"])
    u = q.random_uniform((1000,), 2, 0, -10.0, 10.0)
    assert same_bits(u, z["uniform_s2_m10_10"])
    v = q.variate_tensor((1000,), 0x15EED, 0)
    assert same_bits(v, z["variates_15eed"])


# ---- (b) seeded inputs vs the C restatement -----------------------------------------
ELEM_FMTS = [float_fmt(5, 2), float_fmt(8, 7), float_fmt(4, 3), float_fmt(1, 0),
             float_fmt(8, 23), fixed_fmt(8, 4), fixed_fmt(3, 1, True),
             fixed_fmt(6, 2, False, False), fixed_fmt(24, 100, True, False),
             fixed_fmt(2, -126)]


def mixed_inputs(rng, n):
    m = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-150, 127, n)).astype(np.float32)
    u = rng.uniform(-30, 30, n).astype(np.float32)
    x = np.where(rng.random(n) < 0.5, m, u).astype(np.float32)
    x[: min(n, 8)] = np.array([0.0, -0.0, 0.5, -0.5, 2.5, -2.5, 1e-45, 3.99],
                              np.float32)[: min(n, 8)]
    return x


@pytest.mark.parametrize("fmt", ELEM_FMTS, ids=repr)
@pytest.mark.parametrize("mode", ALL_MODES)
def test_elementwise_vs_oracle_ragged(q, oracle, fmt, mode):
    rng = np.random.default_rng(fmt.wl * 100 + fmt.exp_bits * 10 + mode)
    spec = spec_of(q, fmt, mode, seed=1234)
    for n in (1, 3, 4, 17, 1023, 4096 + 5, 300_001):
        x = mixed_inputs(rng, n)
        st, want = oracle.quantize(x, fmt, mode, seed=1234, call=n)
        assert st == 0
        got = q.quantize_fused_at(dev(x), spec, n)
        assert same_bits(got, want), (fmt, mode, n)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_elementwise_misaligned_and_inplace(q, oracle, offset):
    rng = np.random.default_rng(offset)
    n = 100_003
    x = mixed_inputs(rng, n)
    fmt = fixed_fmt(8, 4)
    st, want = oracle.quantize(x, fmt, STOCHASTIC, seed=5, call=9)
    spec = spec_of(q, fmt, STOCHASTIC, seed=5)
    big = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
    big[offset:offset + n] = dev(x)
    got = q.quantize_fused_at(big[offset:offset + n], spec, 9)
    assert same_bits(got, want)
    # output at a different misalignment than the input: scalar path
    out = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
    xv = big[offset:offset + n]
    q.quantize_fused_at(xv, spec, 9, out=out[(offset + 1) % 4:(offset + 1) % 4 + n])
    assert same_bits(out[(offset + 1) % 4:(offset + 1) % 4 + n], want)
    # in place
    q.quantize_fused_at(xv, spec, 9, out=xv)
    assert same_bits(xv, want)


BLOCK_CASES = [
    # (shape, block_dim): covers all three plans
    ((300, 4096), 0),       # rows in registers, 1024x4
    ((64, 100), 0),         # rows, 128 threads
    ((7, 20000), 0),        # rows, 1024 x 8 float4
    ((5, 40000), 0),        # few rows of 40K: chunk rendezvous (3 chunks per row)
    ((300, 40000), 0),      # many rows of 40K: 2-CTA clusters (DSMEM max exchange)
    ((80, 200000), 0),      # chunk rendezvous, 13 chunks per row (ragged last)
    ((40, 802816), 0),      # ResNet-50 conv1 per-sample block, 49 chunks per row
    ((1, 300, 40000), 1),   # clusters along dim 1 (leading 1)
    ((256, 50176), 0),      # ResNet-50 [256, 256, 14, 14] per-sample rows: clusters
    ((2, 65540), 0),        # 5 chunks of 13108 floats (uneven split)
    ((1 << 20,), None),     # whole tensor, one row of 64 chunks
    ((4096, 64), 0),        # short rows: 16 lanes per row
    ((999, 12), 0),         # short rows: 4 lanes per row
    ((77, 400), 0),         # short rows: 32 lanes x 4 float4
    ((33, 4), 0),           # short rows: 1 lane per row
    ((2, 3, 99_999), 2),    # last dim of odd length -> two-pass columns
    ((1000,), None),        # whole tensor, rows plan (1 row)
    ((1_000_003,), None),   # whole tensor, two-pass segments, odd length
    ((50, 70, 30), 1),      # columns plan (stride 30)
    ((40, 33), 1),          # last dim, stride 1
    ((3, 5, 2048), 1),      # segments with outer > 1
    ((6, 5, 9), 2),
    ((1, 3, 256), 1),       # leading 1: rows plan along dim 1
    ((257, 3), 0),          # stride 3 (< 64): columns plan along dim 0
    ((70_001, 8), 1),       # narrow columns plan: 2 threads per row lane, 128 lanes
    ((30_001, 6), 1),       # narrow, W % 4 != 0 (scalar loads), ragged lanes
    ((9_000, 3, 20), 1),    # narrow, stride 20 inside a 60-float row
]


@pytest.mark.parametrize("shape,dim", BLOCK_CASES, ids=str)
@pytest.mark.parametrize("mode", ALL_MODES)
@pytest.mark.parametrize("wl", [8, 4])
def test_block_plans_vs_oracle(q, oracle, shape, dim, mode, wl):
    rng = np.random.default_rng(hash((shape, dim, mode, wl)) % 2**32)
    x = rng.uniform(-1, 1, shape).astype(np.float32)
    # per-slice exponents that vary, and some all-zero slices
    if dim is not None:
        sl = [slice(None)] * len(shape)
        for b in range(shape[dim]):
            sl[dim] = b
            x[tuple(sl)] *= np.float32(2.0 ** int(rng.integers(-30, 30)))
        sl[dim] = 0
        x[tuple(sl)] = 0.0
    fmt = block_fmt(wl, dim)
    st, want = oracle.quantize(x, fmt, mode, seed=77, call=3)
    assert st == 0
    got = q.quantize_fused_at(dev(x), spec_of(q, fmt, mode, seed=77), 3)
    assert same_bits(got, want), (shape, dim, mode, wl)
    # host path (streamed rows / resident two-pass)
    got_h = q.quantize_fused_at(x, spec_of(q, fmt, mode, seed=77), 3)
    assert same_bits(got_h, want)


CLUSTER_CASES = [((300, 40000), 0), ((80, 200000), 0), ((40, 802816), 0), ((6, 1 << 20), 0)]


@pytest.mark.parametrize("shape,dim", CLUSTER_CASES, ids=str)
@pytest.mark.parametrize("mode", ALL_MODES)
def test_block_rows_without_workspace_take_the_cluster_plan(q, oracle, shape, dim, mode):
    # lpq_quantize with ws = NULL: the rows of 32K..1M floats that the chunk
    # plan would take run on the workspace-free cluster plan (DSMEM maxima)
    import ctypes as C
    from paper_1910_04540_b200 import _lib
    rng = np.random.default_rng(hash((shape, mode)) % 2**32)
    x = rng.uniform(-1, 1, shape).astype(np.float32)
    x *= (2.0 ** rng.integers(-20, 20, (shape[0], 1))).astype(np.float32)
    fmt = block_fmt(8, dim)
    st, want = oracle.quantize(x, fmt, mode, seed=5, call=2)
    assert st == 0
    xd = dev(x)
    y = torch.empty_like(xd)
    spec = spec_of(q, fmt, mode, seed=5)
    status = q.quant._status_buf(xd.device)
    shp = _lib.shape_array(xd.shape)
    rc = _lib.lib.lpq_quantize(C.c_void_p(xd.data_ptr()), C.c_void_p(y.data_ptr()), shp,
                               xd.dim(), 0, C.byref(spec.format.c()), mode, 5, 2,
                               C.c_void_p(0), 0, C.c_void_p(status.data_ptr()),
                               C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    q.fetch_status(xd.device)
    assert same_bits(y, want), (shape, mode)


def test_block_chunk_plan_many_rows_and_index_base(q, oracle):
    # [256, 100352] (ResNet-50 layer-4 activation rows, 7 chunks each) with a
    # flat-index base that is not a multiple of 4 (scalar variate path), and
    # rows whose maxima sit in different chunks
    R, L = 256, 100352
    x = q.random_uniform((R, L), 11, 0, -1.0, 1.0)
    for r in range(0, R, 17):
        x[r, (r * 7919) % L] = 3.0 + r
    xh = x.cpu().numpy()
    for mode, base in ((STOCHASTIC, 0), (STOCHASTIC, 6), (NEAREST_EVEN, 3)):
        spec = q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode(mode), 21)
        y = q.quantize_fused_at(x, spec, 1, index_base=base)
        for r in (0, 17, 100, 255):
            st, want = oracle.quantize_block_given_max(
                xh[r:r + 1], block_fmt(8, 0), mode, np.abs(xh[r:r + 1]).max(axis=1),
                seed=21, call=1, index_base=base + r * L)
            assert st == 0 and same_bits(y[r:r + 1], want), (mode, base, r)


def test_block_columns_grid_y_beyond_65535(q, oracle):
    """[2^20 + 3000, 1024] per column (block_dim=1, stride 1): the column
    plans need more than 65535 row chunks, so grid.y is capped and the kernels
    take the rest grid-stride (this used to fail the launch).
    Sampled rows vs the oracle with the device-reduced block maxima, plus the
    maxima themselves vs torch."""
    R, W = (1 << 20) + 3000, 1024
    x = q.random_uniform((R, W), 5, 0, -1.0, 1.0)
    x[R - 1] = torch.linspace(-3.0, 3.0, W, device="cuda")   # max in the last chunk
    for mode in (NEAREST_EVEN, STOCHASTIC):
        fmt = block_fmt(8, 1)
        spec = spec_of(q, fmt, mode, seed=9)
        y = q.quantize_fused_at(x, spec, 4)
        mx = x.abs().amax(dim=0)
        dmx = q.block_absmax(x, spec.format).view(torch.float32)
        assert torch.equal(dmx, mx)
        mxh = mx.cpu().numpy()
        for r in (0, 1, 16 * 65535 - 1, 16 * 65535, 16 * 65535 + 17, R - 2, R - 1):
            xr = x[r:r + 1].cpu().numpy()
            st, want = oracle.quantize_block_given_max(xr, fmt, mode, mxh, seed=9, call=4,
                                                       index_base=r * W)
            assert st == 0 and same_bits(y[r:r + 1], want), (mode, r)
    del x, y


def test_block_tiny_and_huge_maxima(q, oracle):
    rng = np.random.default_rng(3)
    for e in (-149, -140, -126, 0, 100, 126):
        x = (rng.uniform(-1, 1, (16, 256)) * 2.0**e).astype(np.float32)
        for mode in ALL_MODES:
            fmt = block_fmt(8, 0)
            st, want = oracle.quantize(x, fmt, mode, seed=1, call=e & 0xFF)
            got = q.quantize_fused_at(dev(x), spec_of(q, fmt, mode, seed=1), e & 0xFF)
            assert st == 0 and same_bits(got, want), (e, mode)


# ---- errors (errors.hpp taxonomy) ---------------------------------------------------
def test_errors(q):
    spec = q.QuantSpec(q.FixedFormat(8, 4))
    bad = np.array([1.0, np.inf, 2.0], np.float32)
    with pytest.raises(q.InvalidInputError):
        q.quantize_fused(dev(bad), spec)
    with pytest.raises(q.InvalidInputError):
        q.quantize_fused(bad, spec)
    with pytest.raises(q.InvalidInputError):
        q.quantize_fused(dev(np.array([np.nan, 1.0], np.float32)),
                         q.QuantSpec(q.FloatFormat(5, 2)))
    with pytest.raises(q.InvalidInputError):  # block max >= 2^127
        q.quantize_fused(dev(np.array([1.0, 2.0**127], np.float32)),
                         q.QuantSpec(q.BlockFloatFormat(8)))
    with pytest.raises(q.ShapeError):
        q.quantize_fused(dev(np.ones((4, 4), np.float32)),
                         q.QuantSpec(q.BlockFloatFormat(8, 3)))
    with pytest.raises(q.FormatError):
        q.quantize_fused(dev(np.ones(4, np.float32)), q.QuantSpec(q.FixedFormat(1, 0)))
    # the status word is cleared: a good call afterwards succeeds
    q.quantize_fused(dev(np.ones(4, np.float32)), spec)


def test_call_counter_and_replay(q):
    # quant_ops.cpp:179-183, test_quant_ops.cpp:96-117
    t = dev(np.random.default_rng(61).uniform(-2, 2, 100).astype(np.float32))
    a = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 5, 0)
    b = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 5, 0)
    assert same_bits(q.quantize_fused(t, a), q.quantize_fused(t, b).cpu().numpy())
    assert a.call_counter == 1
    assert same_bits(q.quantize_fused(t, a), q.quantize_fused(t, b).cpu().numpy())
    assert a.call_counter == 2
    n = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.NearestEven, 1, 0)
    q.quantize_fused(t, n)
    assert n.call_counter == 0


def test_pass_count_contract(q):
    # test_quant_ops.cpp:156-181: fused <= 2 data passes; ours counts the
    # HBM passes it actually makes (1, or 2 for the two-pass block plans)
    rng = np.random.default_rng(71)
    cases = [(q.FixedFormat(8, 4), (32, 32), 1), (q.FloatFormat(5, 2), (32, 32), 1),
             (q.BlockFloatFormat(8, 0), (16, 256), 1), (q.BlockFloatFormat(8), (32, 32), 1),
             (q.BlockFloatFormat(8), (8, 40000), 1), (q.BlockFloatFormat(8, 0), (300, 40000), 1),
             (q.BlockFloatFormat(8), (3, 999_999), 2),
             (q.BlockFloatFormat(8, 1), (32, 32), 2)]
    for fmt, shape, passes in cases:
        t = dev(rng.uniform(-4, 4, shape).astype(np.float32))
        q.reset_pass_count()
        q.quantize_fused_at(t, q.QuantSpec(fmt, q.RoundingMode.Stochastic), 0)
        assert q.pass_count() == passes <= 2, (fmt, shape)


def test_identity_format_and_quantized_op(q):
    t = dev(np.random.default_rng(41).uniform(-100, 100, (17, 9)).astype(np.float32))
    assert same_bits(q.quantize_fused(t, q.QuantSpec(q.FloatFormat(8, 23))), t.cpu().numpy())
    f31 = q.QuantSpec(q.FixedFormat(3, 1))
    qrelu = q.quantized_op(torch.relu, f31)
    r = qrelu(dev(np.array([-1.0, 0.74], np.float32))).cpu().numpy()
    assert list(r) == [0.0, 0.5]


def test_shards_equal_whole(q):
    # index_base makes a sharded quantization bit-identical to the whole
    x = q.random_uniform((1_000_000,), 2, 0, -10.0, 10.0)
    spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 0x15EED)
    whole = q.quantize_fused_at(x, spec, 0)
    parts = []
    for r in range(4):
        lo, hi = r * 250_000, (r + 1) * 250_000
        parts.append(q.quantize_fused_at(x[lo:hi], spec, 0, index_base=lo))
    assert torch.equal(torch.cat(parts).view(torch.int32), whole.view(torch.int32))


# ---- (c) BASELINE sizes --------------------------------------------------------------
def test_c1_float52_16M_full(q, oracle):
    n = 1 << 24
    x = q.random_uniform((n,), 7, 0, -4.0, 4.0)
    xh = x.cpu().numpy()
    for mode in (NEAREST_EVEN, STOCHASTIC):
        spec = q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode(mode), 0x15EED)
        got = q.quantize_fused_at(x, spec, 0).cpu().numpy()
        st, want = oracle.quantize(xh, float_fmt(5, 2), mode, seed=0x15EED, call=0)
        assert st == 0 and np.array_equal(bits(got), bits(want))


def test_c1_float52_16M_loguniform(q, oracle):
    """SURVEY 8(d) C1 variant: |x| log-uniform in [2^-20, 2^20], random sign --
    the underflow two-point grid, the saturation clamp and the bit-domain /
    scaled-form switch inside float4s all occur."""
    n = 1 << 24
    e = q.random_uniform((n,), 50, 0, -20.0, 20.0)
    s = q.random_uniform((n,), 60, 0, -1.0, 1.0)
    x = torch.copysign(torch.exp2(e), s)
    xh = x.cpu().numpy()
    for mode in (NEAREST_EVEN, STOCHASTIC):
        spec = q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode(mode), 0x15EED)
        got = q.quantize_fused_at(x, spec, 0).cpu().numpy()
        st, want = oracle.quantize(xh, float_fmt(5, 2), mode, seed=0x15EED, call=0)
        assert st == 0 and np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("shape,dim,shards", [
    ((8, 300, 5), None, 2), ((4, 7, 2048), None, 4), ((8, 300, 5), 1, 2),
    ((4, 7, 2048), 1, 4), ((6, 3, 4, 9), 2, 3), ((6, 3, 4, 9), 3, 2)], ids=str)
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_block_split_across_shards(q, shape, dim, shards, mode):
    """blocks spanning shards (whole tensor, or block_dim >= 1 of
    a tensor sharded along dim 0).  Per-shard lpq_block_absmax, the maxima
    combined by elementwise max (what all_reduce(MAX) does across ranks),
    then lpq_quantize_block_apply per shard with its index_base: bitwise the
    single-tensor quantize_fused_at."""
    from paper_1910_04540_b200.shard import quantize_block_split
    x = q.random_uniform(shape, 21, 0, -2.0, 2.0)
    x[0].view(-1)[3] = 40.0  # the global maximum lives in shard 0 only
    spec = q.QuantSpec(q.BlockFloatFormat(8, dim), q.RoundingMode(mode), 99)
    whole = q.quantize_fused_at(x, spec, 5)
    parts = list(torch.chunk(x, shards, dim=0))
    m = torch.stack([q.block_absmax(p, spec.format) for p in parts]).amax(0)
    ref_m = (x.abs().amax(dim=tuple(d for d in range(x.dim()) if d != dim))
             if dim is not None else x.abs().amax().reshape(1))
    assert torch.equal(m.view(torch.float32), ref_m.float().reshape(-1))
    got, base = [], 0
    for p in parts:
        got.append(q.quantize_block_apply(p, spec, 5, m, index_base=base))
        base += p.numel()
    assert torch.equal(torch.cat(got).view(torch.int32), whole.view(torch.int32))
    if dim != 0:  # one rank (no process group): the split path is the whole tensor
        one = quantize_block_split(q, x, spec, 5, 0)
        assert torch.equal(one.view(torch.int32), whole.view(torch.int32))


def test_block_split_whole_tensor_2p26(q):
    """The exchange path at scale: a 2^26-element whole-tensor block split
    into 4 flat shards equals the single-tensor quantization (both modes)."""
    n = 1 << 26
    x = q.random_uniform((n,), 33, 0, -8.0, 8.0)
    for mode in (NEAREST_EVEN, STOCHASTIC):
        spec = q.QuantSpec(q.BlockFloatFormat(8), q.RoundingMode(mode), 0x15EED)
        whole = q.quantize_fused_at(x, spec, 1)
        parts = list(torch.chunk(x, 4))
        m = torch.stack([q.block_absmax(p, spec.format) for p in parts]).amax(0)
        out = torch.empty_like(x)
        base = 0
        for p, o in zip(parts, torch.chunk(out, 4)):
            q.quantize_block_apply(p, spec, 1, m, out=o, index_base=base)
            base += p.numel()
        assert torch.equal(out.view(torch.int32), whole.view(torch.int32))


def test_block_split_errors(q):
    x = torch.ones(4, 8, device="cuda")
    spec = q.QuantSpec(q.BlockFloatFormat(8, 1), q.RoundingMode.NearestEven, 1)
    with pytest.raises(q.UnsupportedFormatError):
        q.block_absmax(x, q.FixedFormat(8, 4))
    with pytest.raises(ValueError):
        q.quantize_block_apply(x, spec, 0, torch.zeros(3, dtype=torch.int32, device="cuda"))
    with pytest.raises(TypeError):  # float maxima would be converted, not reinterpreted
        q.quantize_block_apply(x, spec, 0, torch.ones(8, device="cuda"))
    x[1, 2] = float("nan")
    m = q.block_absmax(x, spec.format)
    assert torch.equal(m.view(torch.float32), torch.ones(8, device="cuda"))  # NaN ignored
    with pytest.raises(q.InvalidInputError):
        q.quantize_block_apply(x, spec, 0, m)
    big = torch.full((8,), 0x7F000000, dtype=torch.int32, device="cuda")  # 2^127
    with pytest.raises(q.InvalidInputError):
        q.quantize_block_apply(torch.ones(4, 8, device="cuda"), spec, 0, big)


def test_c2_fixed84_1G_windows(q, oracle):
    n = 1 << 30
    x = q.random_uniform((n,), 2, 0, -10.0, 10.0)
    spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 0x15EED)
    y = q.quantize_fused_at(x, spec, 0)
    w = 1 << 20
    for lo in (0, n // 2 - 12345, n - w):
        xs = oracle.random_uniform(w, 2, 0, -10.0, 10.0, index_base=lo)
        assert np.array_equal(bits(xs), bits(x[lo:lo + w].cpu().numpy()))
        st, want = oracle.quantize(xs, fixed_fmt(8, 4), STOCHASTIC, seed=0x15EED,
                                   call=0, index_base=lo)
        assert np.array_equal(bits(y[lo:lo + w].cpu().numpy()), bits(want)), lo
    # properties over the whole 1G output: on the 1/16 grid and within range
    k = y * 16.0
    assert torch.equal(k, torch.round(k))
    assert float(y.min()) >= -8.0 and float(y.max()) <= 7.9375
    del x, y


def test_c3_block_rows_65536x4096(q, oracle):
    R, L = 65536, 4096
    base = q.random_uniform((R, L), 3, 0, -1.0, 1.0)
    scale = torch.exp2(torch.randint(-20, 21, (R, 1), device="cuda",
                                     generator=torch.Generator("cuda").manual_seed(0)).float())
    x = base * scale
    for mode in (NEAREST_EVEN, STOCHASTIC):
        spec = q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode(mode), 0x15EED)
        y = q.quantize_fused_at(x, spec, 0)
        rows = list(range(0, R, R // 32)) + [R - 1]
        for r in rows:
            st, want = oracle.quantize(x[r].cpu().numpy(), block_fmt(8),
                                       mode, seed=0x15EED, call=0, index_base=r * L)
            assert np.array_equal(bits(y[r].cpu().numpy()), bits(want)), (mode, r)
        # every one of the 2^28 outputs: an integer k in [-128, 127] times the
        # row's step 2^(E_r - 6), E_r = floor(log2 max|x_r|) (computed by torch)
        m = x.abs().amax(dim=1, keepdim=True)
        _, ex = torch.frexp(m)            # m = f * 2^ex, f in [0.5, 1)
        k = y / torch.exp2((ex - 1 - 6).float())
        assert torch.equal(k, torch.round(k))
        assert float(k.min()) >= -128 and float(k.max()) <= 127


# ---- grouped (multi-tensor) quantization --------------------------------------
@pytest.mark.parametrize("fmt_ctor,mode", [
    (lambda q: q.FixedFormat(8, 4), STOCHASTIC), (lambda q: q.FloatFormat(5, 2), NEAREST_EVEN),
    (lambda q: q.FloatFormat(8, 7), STOCHASTIC), (lambda q: q.BlockFloatFormat(8, 0), STOCHASTIC),
    (lambda q: q.BlockFloatFormat(6, 0), NEAREST_EVEN), (lambda q: q.BlockFloatFormat(8, 1), NEAREST_EVEN),
    (lambda q: q.BlockFloatFormat(8), STOCHASTIC)])
def test_grouped_equals_sequential(q, fmt_ctor, mode):
    fmt = fmt_ctor(q)
    rng = np.random.default_rng(99)
    shapes = [(64, 3, 7, 7), (256, 64, 1, 1), (10, 147), (1000, 2048), (3,), (7, 5),
              (128, 128, 3, 3)] * 12  # 84 tensors -> two launches of <= 64
    if getattr(fmt, "block_dim", None) == 1:
        shapes = [s for s in shapes if len(s) >= 2]
    ts = [dev(rng.uniform(-3, 3, s).astype(np.float32) * np.float32(2.0 ** rng.integers(-8, 8)))
          for s in shapes]
    spec_a = q.QuantSpec(fmt, q.RoundingMode(mode), 17, 4)
    spec_b = q.QuantSpec(fmt, q.RoundingMode(mode), 17, 4)
    got = q.quantize_fused_many(ts, spec_a)
    want = [q.quantize_fused(t, spec_b) for t in ts]
    assert spec_a.call_counter == spec_b.call_counter
    for g, w in zip(got, want):
        assert torch.equal(g.view(torch.int32), w.view(torch.int32))


# ---- full-size, every element: C2 (2^30) and C3 (2^28) against the oracle ------------
def _parallel_oracle_compare(oracle, fmt, mode, seed, n, chunk, gen, got_slice):
    """Compare got_slice(lo, hi) with the oracle over [0, n) in chunks, the
    oracle chunks in parallel (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(lo):
        hi = min(n, lo + chunk)
        x = gen(lo, hi)
        st, want = oracle.quantize(x, fmt, mode, seed=seed, call=0, index_base=lo)
        return lo, hi, st, want

    import os
    with ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2))) as ex:
        for lo, hi, st, want in ex.map(one, range(0, n, chunk)):
            assert st == 0
            assert np.array_equal(bits(got_slice(lo, hi)), bits(want.reshape(-1))), lo


def test_c2_full_tensor_every_element(q, oracle):
    n = 1 << 30
    x = q.random_uniform((n,), 2, 0, -10.0, 10.0)
    y = q.quantize_fused_at(x, q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic,
                                           0x15EED), 0)
    del x
    yh = y.cpu().numpy()
    del y
    _parallel_oracle_compare(
        oracle, fixed_fmt(8, 4), STOCHASTIC, 0x15EED, n, 1 << 25,
        lambda lo, hi: oracle.random_uniform(hi - lo, 2, 0, -10.0, 10.0, index_base=lo),
        lambda lo, hi: yh[lo:hi])


def test_c3_full_tensor_every_element(q, oracle):
    R, L = 65536, 4096
    x = q.random_uniform((R, L), 3, 0, -1.0, 1.0)
    x *= torch.exp2(torch.randint(-20, 21, (R, 1), device="cuda",
                                  generator=torch.Generator("cuda").manual_seed(1)).float())
    xh = x.cpu().numpy()
    for mode in (NEAREST_EVEN, STOCHASTIC):
        y = q.quantize_fused_at(x, q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode(mode),
                                               0x15EED), 0).cpu().numpy()
        rows = 1 << 11
        _parallel_oracle_compare(
            oracle, block_fmt(8, 0), mode, 0x15EED, R * L, rows * L,
            lambda lo, hi: xh.reshape(-1)[lo:hi].reshape(-1, L),
            lambda lo, hi: y.reshape(-1)[lo:hi])


# ---- `lpsim quantize` on the GPU: LPT1 -> quantize -> LPT1 ---------------------------
@pytest.mark.parametrize("fmt,mode,shape", [
    (fixed_fmt(8, 4), STOCHASTIC, (3, 1000, 7)), (float_fmt(5, 2), NEAREST_EVEN, (100001,)),
    (block_fmt(8, 0), STOCHASTIC, (64, 4096)), (block_fmt(8), NEAREST_EVEN, (5, 40001))])
def test_quantize_file_vs_oracle(q, oracle, tmp_path, fmt, mode, shape):
    from paper_1910_04540_b200 import io as lio
    rng = np.random.default_rng(sum(shape))
    x = (rng.standard_normal(shape) * 3).astype(np.float32)
    src, dst = str(tmp_path / "in.lpt"), str(tmp_path / "out.lpt")
    lio.write_tensor_file(src, x)
    spec = spec_of(q, fmt, mode, seed=0x15EED)
    spec.call_counter = 4
    lio.quantize_file(src, dst, spec)
    got = lio.read_tensor_file(dst)
    st, want = oracle.quantize(x, fmt, mode, seed=0x15EED, call=4)
    assert got.shape == x.shape and np.array_equal(bits(got), bits(want))
    assert spec.call_counter == (5 if mode == STOCHASTIC else 4)
    bad = x.copy()
    bad.reshape(-1)[3] = np.inf
    lio.write_tensor_file(src, bad)
    with pytest.raises(q.InvalidInputError):
        lio.quantize_file(src, dst, spec)
    with pytest.raises(q.FormatError):
        lio.quantize_file(str(tmp_path / "missing.lpt"), dst, spec)


NONFINITE_CASES = [((300, 4096), 0), ((77, 400), 0), ((7, 20000), 0), ((300, 40000), 0),
                   ((3, 802816), 0), ((1 << 20,), None),
                   ((5, 40000), 0), ((50, 70, 30), 1), ((1_000_003,), None), ((4096, 64), 0)]


@pytest.mark.parametrize("shape,dim", NONFINITE_CASES)
@pytest.mark.parametrize("mode", [0, 1])
def test_block_nonfinite_every_plan(q, shape, dim, mode):
    # fused_block (quant_ops.cpp:68-115): the block maxima and their range
    # check (scalar_quant.hpp:72-77) come before the element pass, so a block
    # holding inf (or >= 2^127) reports the range error even when another
    # element is NaN; NaN alone (ignored by reduce_max_abs) is the non-finite
    # input error of quant_pass (quant_ops.cpp:28-29)
    rng = np.random.default_rng(hash((shape, dim, mode)) % 2**32)
    x = rng.uniform(-1, 1, shape).astype(np.float32)
    n = x.size
    spec = q.QuantSpec(q.BlockFloatFormat(8, dim), q.RoundingMode(mode), 3, 0)
    i, j = (int(v) for v in rng.choice(n, 2, replace=False))
    for vals, msg in (({i: np.nan}, "non-finite"), ({i: np.inf}, "too large"),
                      ({i: -np.inf}, "too large"), ({i: np.nan, j: 2.0**127}, "too large"),
                      ({i: np.nan, j: -np.nan}, "non-finite")):
        xb = x.copy().reshape(-1)
        for k, v in vals.items():
            xb[k] = v
        with pytest.raises(q.InvalidInputError, match=msg):
            q.quantize_fused(dev(xb.reshape(shape)), spec)
    got = q.quantize_fused_at(dev(x), spec, 0)  # status cleared
    assert np.isfinite(got.cpu().numpy()).all()


def test_beyond_2p32_elements_windows(q, oracle):
    # 2^32 + 4100 elements (16 GiB in + out): flat indices past 2^32 feed the
    # RNG's high key word and every 64-bit index path; windows straddling
    # 2^31 and 2^32 are checked against the oracle with index_base
    n = (1 << 32) + 4100
    x = q.random_uniform((n,), 9, 0, -10.0, 10.0)
    for fmt, ofmt in ((q.FixedFormat(8, 4), fixed_fmt(8, 4)), (q.FloatFormat(5, 2), float_fmt(5, 2))):
        spec = q.QuantSpec(fmt, q.RoundingMode.Stochastic, 0x15EED)
        y = q.quantize_fused_at(x, spec, 7)
        w = 1 << 16
        for lo in ((1 << 31) - 999, (1 << 32) - 3 * w // 2, n - w):
            xs = x[lo:lo + w].cpu().numpy()
            st, want = oracle.quantize(xs, ofmt, STOCHASTIC, seed=0x15EED, call=7,
                                       index_base=lo)
            assert st == 0
            assert np.array_equal(bits(y[lo:lo + w].cpu().numpy()), bits(want)), (fmt, lo)
        del y
    # block rows: n // 4100 rows of 4100 floats (> 2^32 elements in total)
    rows = n // 4100
    xb = x[: rows * 4100].view(rows, 4100)
    spec = q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode.Stochastic, 3)
    yb = q.quantize_fused_at(xb, spec, 1)
    for r in (0, (1 << 19) + 7, rows - 2):
        rows = xb[r:r + 2].cpu().numpy()
        st, want = oracle.quantize(rows, block_fmt(8, 0), STOCHASTIC, seed=3, call=1,
                                   index_base=r * 4100)
        assert st == 0
        assert np.array_equal(bits(yb[r:r + 2].cpu().numpy()), bits(want)), r
    del x, xb, yb
    torch.cuda.empty_cache()


def test_out_argument_is_validated(q):
    x = torch.ones(64, device="cuda")
    spec = q.QuantSpec(q.FixedFormat(8, 4))
    for bad in (torch.empty(63, device="cuda"), torch.empty(64, device="cuda", dtype=torch.float16),
                torch.empty(128, device="cuda")[::2], torch.empty(64)):
        with pytest.raises(ValueError):
            q.quantize_fused_at(x, spec, 0, out=bad)
    out = torch.empty(8, 8, device="cuda")  # same element count, other shape: fine
    q.quantize_fused_at(x, spec, 0, out=out)
    assert torch.equal(out.view(-1), torch.ones(64, device="cuda"))


def test_concurrent_streams_do_not_share_workspace(q, oracle):
    # two two-pass block quantizations in flight on two streams at once
    rng = np.random.default_rng(4)
    xs = [rng.uniform(-1, 1, (5, 40000)).astype(np.float32) * s for s in (1.0, 1e-3)]
    spec = q.QuantSpec(q.BlockFloatFormat(8, 0), q.RoundingMode.Stochastic, 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for x, st in zip(xs, (s1, s2)):
        with torch.cuda.stream(st):
            outs.append(q.quantize_fused_at(dev(x), spec, 0, sync=False))
    torch.cuda.synchronize()
    for x, y in zip(xs, outs):
        st, want = oracle.quantize(x, block_fmt(8, 0), STOCHASTIC, seed=2, call=0)
        assert same_bits(y, want)


@pytest.mark.parametrize("fmt_name", ["fixed", "float", "block0"])
def test_grouped_index_bases(q, oracle, fmt_name):
    # lpq_quantize_grouped with per-tensor flat-index bases (aligned and not:
    # the float4-shared variates need base % 4 == 0) against the oracle
    import ctypes as C
    from paper_1910_04540_b200 import _lib
    fmt, ofmt = {"fixed": (q.FixedFormat(8, 4), fixed_fmt(8, 4)),
                 "float": (q.FloatFormat(5, 2), float_fmt(5, 2)),
                 "block0": (q.BlockFloatFormat(8, 0), block_fmt(8, 0))}[fmt_name]
    rng = np.random.default_rng(8)
    shapes = [(33, 100), (5000,), (64, 64), (7, 9)]
    if fmt_name == "block0":
        shapes = [(33, 100), (50, 8), (64, 64), (7, 12)]
    bases = [0, 3, 2**33 + 1, 4]
    xs = [rng.uniform(-3, 3, s).astype(np.float32) for s in shapes]
    dxs = [dev(x) for x in xs]
    ys = [torch.empty_like(d) for d in dxs]
    descs = (_lib.LpqTensorDesc * len(xs))()
    keep = []
    for i, (d, y, b) in enumerate(zip(dxs, ys, bases)):
        shp = _lib.shape_array(d.shape)
        keep.append(shp)
        descs[i] = _lib.LpqTensorDesc(d.data_ptr(), y.data_ptr(), shp, d.dim(), 0, b, 10 + i)
    status = q.quant._status_buf(torch.device("cuda", 0))
    st = _lib.lib.lpq_quantize_grouped(descs, len(xs), C.byref(fmt.c()), 0, 21, None, 0,
                                       C.c_void_p(status.data_ptr()),
                                       q.quant._stream_ptr(torch.device("cuda", 0)))
    assert st == 0
    q.fetch_status()
    for i, (x, y, b) in enumerate(zip(xs, ys, bases)):
        st, want = oracle.quantize(x, ofmt, STOCHASTIC, seed=21, call=10 + i, index_base=b)
        assert st == 0 and same_bits(y, want), (fmt_name, i)


@pytest.mark.parametrize("base", [1, 2, 3, 4, 2**40 + 3])
def test_index_base_device_path(q, oracle, base):
    # the variates follow the flat index index_base + i (shard offsets):
    # every alignment of the base, elementwise and block formats
    rng = np.random.default_rng(base % 1000)
    x = rng.uniform(-3, 3, (96, 130)).astype(np.float32)
    for fmt, ofmt in ((q.FixedFormat(8, 4), fixed_fmt(8, 4)), (q.FloatFormat(5, 2), float_fmt(5, 2)),
                      (q.BlockFloatFormat(8, 0), block_fmt(8, 0)), (q.BlockFloatFormat(8, 1), block_fmt(8, 1)),
                      (q.BlockFloatFormat(8), block_fmt(8))):
        got = q.quantize_fused_at(dev(x), q.QuantSpec(fmt, q.RoundingMode.Stochastic, 6), 2,
                                  index_base=base)
        st, want = oracle.quantize(x, ofmt, STOCHASTIC, seed=6, call=2, index_base=base)
        assert st == 0 and same_bits(got, want), (fmt, base)


@pytest.mark.parametrize("fmt_name", ["fixed84", "fixed41sym", "fixed8m3", "float52", "float43",
                                      "float21", "float34"])
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_host_path_byte_codes(q, fmt_name, mode):
    # tensors > 16 MB take the chunked host pipeline, which for these formats
    # copies one-byte codes device->host and decodes them on the host: the
    # result must equal the device path bit for bit (signed zeros, saturation,
    # the underflow grid, pageable and page-locked outputs)
    fmt = {"fixed84": q.FixedFormat(8, 4), "fixed41sym": q.FixedFormat(4, 1, True),
           "fixed8m3": q.FixedFormat(8, -3), "float52": q.FloatFormat(5, 2),
           "float43": q.FloatFormat(4, 3), "float21": q.FloatFormat(2, 1),
           "float34": q.FloatFormat(3, 4)}[fmt_name]
    rng = np.random.default_rng(len(fmt_name) * 7 + mode)
    n = 5_000_001
    x = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-30, 30, n)).astype(np.float32)
    x[:16] = [0.0, -0.0, 1e-30, -1e-30, 3.4e38, -3.4e38, 1.0, -1.0, 0.5, -0.5,
              114688.0, -114688.0, 2.0**-14, -2.0**-14, 2.0**-15, -2.0**-15]
    spec = q.QuantSpec(fmt, q.RoundingMode(mode), 11)
    want = q.quantize_fused_at(dev(x), spec, 4).cpu().numpy()
    got = q.quantize_fused_at(x, spec, 4)  # pageable numpy -> host path
    assert same_bits(got, want), (fmt_name, mode)
    xp = torch.from_numpy(x).pin_memory()
    got_p = q.quantize_fused_at(xp, spec, 4)
    assert same_bits(got_p.numpy(), want), (fmt_name, mode)


@pytest.mark.parametrize("case", ["fixed84", "float52", "block_whole", "block_dim1",
                                  "block_tiny", "block_wl4_cols", "block_rows"])
@pytest.mark.parametrize("mode", [NEAREST_EVEN, STOCHASTIC])
def test_direct_host_path_byte_codes(q, case, mode):
    """Tensors <= 16 MB take the direct host path; formats whose every value
    has a one-byte code copy codes device->host (fixed / float: ByteCode;
    block wl <= 8 on the two-pass plans: k plus the block maxima), decoded on
    the host.  Must equal the device path bit for bit, including blocks whose
    results fall in the fp32 subnormal range (the encoder flags them and the
    fp32 values are copied instead) and single-pass block plans (fp32)."""
    fmt, shape, scale = {
        "fixed84": (q.FixedFormat(8, 4), (1 << 20,), 8.0),
        "float52": (q.FloatFormat(5, 2), (16384, 64), 1e3),
        "block_whole": (q.BlockFloatFormat(8), (16384, 64), 4.0),   # criterion 7
        "block_dim1": (q.BlockFloatFormat(8, 1), (4096, 256), 1.0),
        "block_tiny": (q.BlockFloatFormat(8), (1 << 18,), 2.0 ** -140),
        "block_wl4_cols": (q.BlockFloatFormat(4, 1), (333, 77), 1.0),
        "block_rows": (q.BlockFloatFormat(8, 0), (512, 4096), 1.0),
    }[case]
    rng = np.random.default_rng(hash((case, mode)) % 2**32)
    x = (rng.uniform(-1, 1, shape) * scale).astype(np.float32)
    x.reshape(-1)[:4] = [0.0, -0.0, 1e-3 * scale, -1e-3 * scale]
    spec = q.QuantSpec(fmt, q.RoundingMode(mode), 21)
    want = q.quantize_fused_at(dev(x), spec, 2).cpu().numpy()
    for host in (x, torch.from_numpy(x.copy()).pin_memory()):
        got = q.quantize_fused_at(host, spec, 2)
        got = got.numpy() if isinstance(got, torch.Tensor) else got
        assert same_bits(got, want), (case, mode)


@pytest.mark.parametrize("n,base", [(300_001, 0), (1 << 20, 3), (262_144, 5),
                                    (4_000_003, 1), (2_097_155, 2),
                                    # sizes whose copy-pool parts used to drop a
                                    # remainder (count / 16 a multiple of 64)
                                    (1_048_577, 0), (4_194_305, 0)])
@pytest.mark.parametrize("fmt_name", ["fixed84", "float52", "float43_wrapless", "float8_10"])
@pytest.mark.parametrize("mode", [0, 1])
def test_direct_host_path_ragged_and_index_base(q, n, base, fmt_name, mode):
    """Pageable inputs take the direct host path up to 16 MB (staged copy in,
    one-byte codes back for byte-coded formats, fp32 otherwise) and the
    chunked stream beyond: ragged sizes, chunk boundaries that are not
    multiples of 4 and index bases that are not multiples of 4 (the
    variates' float4 grouping) must equal the device path bit for bit, and
    the call counts one data pass."""
    fmt = {"fixed84": q.FixedFormat(8, 4), "float52": q.FloatFormat(5, 2),
           "float43_wrapless": q.FloatFormat(4, 3),
           "float8_10": q.FloatFormat(8, 10)}[fmt_name]  # fp32 copy-back
    rng = np.random.default_rng(n + base)
    x = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-12, 12, n)).astype(np.float32)
    x[:3] = [0.0, -0.0, 3.0]
    spec = q.QuantSpec(fmt, q.RoundingMode(mode), 77)
    want = q.quantize_fused_at(dev(x), spec, 5, index_base=base).cpu().numpy()
    q.reset_pass_count()
    got = q.quantize_fused_at(x, spec, 5, index_base=base)
    assert q.pass_count() == 1
    assert same_bits(got, want), (n, base, fmt_name, mode)


def test_host_path_concurrent_callers(q):
    """Several host threads calling the host entry point at once (ctypes
    releases the GIL): the per-device context lock and the shared copy pool
    must keep every result bit-identical to the device path."""
    import threading
    cases = []
    for i, (fmt, n) in enumerate([(q.FixedFormat(8, 4), 1 << 20), (q.FloatFormat(5, 2), 300_001),
                                  (q.BlockFloatFormat(8), 1 << 21), (q.FloatFormat(8, 10), 5_000_003),
                                  (q.FixedFormat(6, 2), 4_194_305), (q.BlockFloatFormat(6), 777)]):
        rng = np.random.default_rng(40 + i)
        x = (rng.uniform(-1, 1, n) * 4).astype(np.float32)
        spec = q.QuantSpec(fmt, q.RoundingMode(i % 2), 90 + i)
        want = q.quantize_fused_at(dev(x), spec, 1).cpu().numpy()
        cases.append((x, spec, want))
    errors = []

    def worker(k):
        try:
            for r in range(3):
                x, spec, want = cases[(k + r) % len(cases)]
                got = q.quantize_fused_at(x, spec, 1)
                if not same_bits(got, want):
                    errors.append((k, r))
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("n", [1 << 20, (1 << 26) + 12, 300_001])
def test_dependent_launch_chains(q, n):
    """Back-to-back quantizations on one stream where each reads the previous
    one's output (and in place), launched under programmatic dependent
    launch with no host synchronisation between them: every result must
    equal the same chain run with a full synchronisation after each call
    (griddepcontrol.wait orders each kernel's loads after its predecessor)."""
    x = q.random_uniform((n,), 11, 0, -6.0, 6.0)
    specs = [q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode.Stochastic, 3),
             q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.NearestEven, 4),
             q.QuantSpec(q.FloatFormat(4, 3), q.RoundingMode.Stochastic, 5),
             q.QuantSpec(q.FixedFormat(6, 2), q.RoundingMode.Stochastic, 6)]
    want = []
    cur = x
    for i, sp in enumerate(specs):
        cur = q.quantize_fused_at(cur, sp, i)
        torch.cuda.synchronize()
        want.append(cur.clone())
    # the same chain, no synchronisation, alternating fresh and in-place outputs
    a = torch.empty_like(x)
    b = torch.empty_like(x)
    q.quantize_fused_at(x, specs[0], 0, out=a, sync=False)
    q.quantize_fused_at(a, specs[1], 1, out=b, sync=False)
    q.quantize_fused_at(b, specs[2], 2, out=b, sync=False)   # in place
    q.quantize_fused_at(b, specs[3], 3, out=a, sync=False)
    q.fetch_status()
    torch.cuda.synchronize()
    assert same_bits(a, want[3].cpu().numpy())


def test_dependent_launch_reads_the_predecessors_last_wave(q):
    """The sharpest case for programmatic dependent launch: the second kernel
    reads the LAST slice of the first one's output (which the first kernel's
    last wave writes while the second kernel's CTAs are already being
    scheduled).  Without griddepcontrol.wait this reads stale memory."""
    n, m = (1 << 26) + 4096, 1 << 20
    x = q.random_uniform((n,), 13, 0, -6.0, 6.0)
    s1 = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.NearestEven, 1)
    s2 = q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode.Stochastic, 2)
    want = q.quantize_fused_at(q.quantize_fused_at(x, s1, 0)[n - m:].contiguous(), s2, 0)
    torch.cuda.synchronize()
    for rep in range(20):
        a = torch.full_like(x, 1e3)            # stale contents that quantize differently
        b = torch.empty((m,), device="cuda")
        torch.cuda.synchronize()
        q.quantize_fused_at(x, s1, 0, out=a, sync=False)
        q.quantize_fused_at(a[n - m:], s2, 0, out=b, sync=False)
        q.fetch_status()
        torch.cuda.synchronize()
        assert same_bits(b, want.cpu().numpy()), rep
