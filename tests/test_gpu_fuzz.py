"""Randomised GPU parity sweep: random formats (every field over its valid
range), rounding modes, shapes (rank 1-4, ragged), block dimensions, index
bases, call ids, input distributions (log-uniform magnitudes over the whole
fp32 range, exact rounding ties, zeros and signed zeros) and buffer
misalignment, each quantized through the C ABI and compared bit for bit with
the C restatement of the reference (tests/oracle_lib.py).  Seeded: a failing
case prints its seed and reproduces."""
import numpy as np
import pytest

from oracle_lib import block_fmt, bits, fixed_fmt, float_fmt

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _random_case(seed):
    rng = np.random.default_rng(seed)
    kind = int(rng.integers(0, 3))
    if kind == 0:
        e = int(rng.integers(1, 9))
        m = int(rng.integers(0, 24))
        fmt = float_fmt(e, m)
        scale = 2.0 ** int(rng.integers(-20, 21))
    elif kind == 1:
        wl = int(rng.integers(2, 25))
        fl = int(rng.integers(-12, 30)) if rng.random() < 0.85 else \
            int(rng.choice([wl - 128, 126, -100, 100]))
        fmt = fixed_fmt(wl, fl, bool(rng.random() < 0.3), bool(rng.random() < 0.7))
        scale = 2.0 ** float(wl - 1 - fl + rng.integers(-3, 3))
    else:
        fmt = None  # block: needs the shape first
        scale = 2.0 ** int(rng.integers(-60, 60))
    rank = int(rng.integers(1, 5))
    shape = tuple(int(rng.integers(1, {1: 5000, 2: 300, 3: 40, 4: 16}[rank]))
                  for _ in range(rank))
    if kind == 2:
        dim = int(rng.integers(-1, rank))
        fmt = block_fmt(int(rng.integers(2, 25)), None if dim < 0 else dim)
    n = int(np.prod(shape))
    with np.errstate(over="ignore"):  # huge fixed-point ranges: inf, filtered below
        x = (rng.uniform(-1, 1, n) * scale).astype(np.float32)
    r = rng.random(n)
    wide = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-149, 127, n)).astype(np.float32)
    x = np.where(r < 0.15, wide, x)
    if kind == 1:  # exact ties of the fixed-point grid
        ties = ((rng.integers(-2 ** (fmt.wl - 1), 2 ** (fmt.wl - 1), n) + 0.5)
                * 2.0 ** -fmt.fl).astype(np.float32)
        x = np.where((r > 0.85) & (r < 0.95) & np.isfinite(ties), ties, x)
    x = np.where(r > 0.98, np.float32(0.0), x)
    x = np.where(r > 0.99, np.float32(-0.0), x).astype(np.float32)
    x = x[np.isfinite(x)] if kind != 2 else np.nan_to_num(x, posinf=1.0, neginf=-1.0)
    x = np.resize(x, n).astype(np.float32).reshape(shape)
    mode = int(rng.integers(0, 4))
    base = int(rng.choice([0, int(rng.integers(1, 2 ** 20)), 2 ** 40 + int(rng.integers(0, 4))]))
    call = int(rng.integers(0, 2 ** 31))
    offset = int(rng.integers(0, 4)) if rank == 1 else 0
    return fmt, mode, x, base, call, offset


@pytest.mark.parametrize("chunk", range(8))
def test_random_formats_shapes_modes(chunk):
    import paper_1910_04540_b200 as q
    from oracle_lib import Oracle
    o = Oracle()
    for seed in range(chunk * 60, (chunk + 1) * 60):
        fmt, mode, x, base, call, offset = _random_case(seed)
        if fmt.kind == 0:
            f = q.FloatFormat(fmt.exp_bits, fmt.man_bits)
        elif fmt.kind == 1:
            f = q.FixedFormat(fmt.wl, fmt.fl, bool(fmt.symmetric), bool(fmt.saturate))
        else:
            f = q.BlockFloatFormat(fmt.wl, None if fmt.block_dim < 0 else fmt.block_dim)
        spec = q.QuantSpec(f, q.RoundingMode(mode), 0xC0FFEE + seed, 0)
        st, want = o.quantize(x, fmt, mode, seed=0xC0FFEE + seed, call=call, index_base=base)
        buf = torch.empty(x.size + 4, device="cuda")
        xd = buf[offset:offset + x.size].view(x.shape)
        xd.copy_(torch.from_numpy(x))
        if st != 0:  # the reference raises (e.g. block maximum out of range)
            with pytest.raises(q.InvalidInputError):
                q.quantize_fused_at(xd, spec, call, index_base=base)
            continue
        got = q.quantize_fused_at(xd, spec, call, index_base=base).cpu().numpy()
        assert np.array_equal(bits(got), bits(want)), (seed, repr(fmt), mode, x.shape, base)


@pytest.fixture(scope="module")
def q():
    import paper_1910_04540_b200 as q
    return q


# ---- long block rows: the chunk-rendezvous and cluster plans --------------------
def _block_rows_case(seed):
    rng = np.random.default_rng(10_000 + seed)
    L = int(rng.integers(8193, 300_000)) * 4 if rng.random() < 0.8 else \
        int(rng.integers(32769, 1_200_000))          # some rows not a multiple of 4
    rows = int(rng.integers(1, max(2, 24_000_000 // L)))
    wl = int(rng.integers(2, 25))
    mode = int(rng.integers(0, 4))
    base = int(rng.choice([0, int(rng.integers(1, 2 ** 20))]))
    return L, rows, wl, mode, base


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_long_block_rows(q, oracle, seed):
    L, rows, wl, mode, base = _block_rows_case(seed)
    rng = np.random.default_rng(seed)
    x = q.random_uniform((rows, L), seed, 0, -1.0, 1.0)
    scale = torch.from_numpy((2.0 ** rng.integers(-40, 40, (rows, 1))).astype(np.float32)).cuda()
    x = x * scale
    x[rows // 2, (seed * 7919) % L] = 0.0
    spec = q.QuantSpec(q.BlockFloatFormat(wl, 0), q.RoundingMode(mode), seed)
    y = q.quantize_fused_at(x, spec, 5, index_base=base)
    for r in sorted({0, rows // 2, rows - 1}):
        xr = x[r:r + 1].cpu().numpy()
        st, want = oracle.quantize(xr, block_fmt(wl, 0), mode, seed=seed, call=5,
                                   index_base=base + r * L)
        assert st == 0
        assert np.array_equal(bits(y[r:r + 1].cpu().numpy()), bits(want)), (seed, L, rows, wl, mode, r)


# ---- the per-op GEMM: every kernel of the launch -----------------------------------
@pytest.mark.parametrize("seed", range(40))
def test_fuzz_quant_gemm(q, oracle, seed):
    rng = np.random.default_rng(20_000 + seed)
    M, N, K = (int(rng.integers(1, 70)) for _ in range(3))
    if rng.random() < 0.4:
        fm = fa = (8, 7)
    else:
        fm = (int(rng.integers(2, 9)), int(rng.integers(0, 24)))
        fa = (int(rng.integers(2, 9)), int(rng.integers(0, 24)))
    mode = int(rng.integers(0, 4))
    lo = float(2.0 ** rng.integers(-8, 1))
    a = (rng.uniform(lo, 2 * lo, (M, K)) * rng.choice([-1, 1], (M, K))).astype(np.float32)
    b = (rng.uniform(0.5, 1.5, (K, N)) * rng.choice([-1, 1], (K, N))).astype(np.float32)
    if rng.random() < 0.3:  # float(8,7)-exact operands (the exact-bf16 kernel's)
        _, a = oracle.quantize(a, float_fmt(8, 7), 1)
        _, b = oracle.quantize(b, float_fmt(8, 7), 1)
    if rng.random() < 0.2:
        a.reshape(-1)[:: 5] = 0.0
    got = q.quant_gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                       q.FloatFormat(*fm), q.FloatFormat(*fa), q.RoundingMode(mode), seed, 3,
                       row_base=_row_base_of(seed))
    st, want = oracle.quant_gemm(a, b, float_fmt(*fm), float_fmt(*fa), mode,
                                 seed=seed, call=3, row_base=_row_base_of(seed))
    assert st == 0
    assert np.array_equal(bits(got.cpu().numpy()), bits(want)), (seed, M, N, K, fm, fa, mode)


def _row_base_of(seed):
    return (seed * 37) % 100


_HOST_SIZES = [1, 3, 4097, 65_535, 65_536, 65_537, 300_001, 1 << 20, (1 << 20) + 1,
               (1 << 20) + 1025, 2_097_155, (1 << 22) - 1, 1 << 22, (1 << 22) + 1,
               4_194_305, 5_000_003, 9_000_011]


@pytest.mark.parametrize("chunk", range(4))
def test_fuzz_host_path_vs_device_path(chunk):
    """The host entry point (staged copies, byte-coded or fp32 copy-back, the
    direct path up to 16 MB and the chunked stream beyond, row-aligned chunks
    for per-row block formats) against the device path on the same input:
    random sizes around every threshold of the host runtime (the 256 KB
    staging cut, the 16 MB direct cut, the copy pool's part rounding), random
    formats, modes and index bases, pageable or pinned input.  Bit for bit."""
    import paper_1910_04540_b200 as q
    for seed in range(chunk * 12, (chunk + 1) * 12):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.choice(_HOST_SIZES)) + int(rng.integers(0, 3))
        kind = int(rng.integers(0, 4))
        if kind == 0:
            f = q.FixedFormat(int(rng.integers(4, 13)), int(rng.integers(0, 8)), False,
                              bool(rng.random() < 0.8))
        elif kind == 1:
            f = q.FloatFormat(int(rng.integers(2, 9)), int(rng.integers(0, 8)))
        elif kind == 2:  # per-row blocks: row-aligned stream chunks
            cols = int(rng.choice([64, 1000, 4096]))
            n = max(cols, (n // cols) * cols)
            f = q.BlockFloatFormat(int(rng.integers(4, 10)), 0)
        else:
            f = q.BlockFloatFormat(int(rng.integers(4, 10)))
        shape = (n // cols, cols) if kind == 2 else (n,)
        x = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-10, 10, n)).astype(np.float32)
        x = x.reshape(shape)
        mode = int(rng.integers(0, 4))
        base = int(rng.choice([0, 1, 2, 3, 1 << 33]))
        spec = q.QuantSpec(f, q.RoundingMode(mode), 0xF00D + seed)
        want = q.quantize_fused_at(torch.from_numpy(x).cuda(), spec, 3,
                                   index_base=base).cpu().numpy()
        xin = x if rng.random() < 0.6 else torch.from_numpy(x.copy()).pin_memory()
        got = q.quantize_fused_at(xin, spec, 3, index_base=base)
        got = got.numpy() if isinstance(got, torch.Tensor) else got
        assert np.array_equal(bits(got), bits(want)), (seed, n, f, mode, base, type(xin))
