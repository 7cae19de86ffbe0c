"""Generate golden fixtures from the reference library itself.

    make -C oracle && python tests/golden/make_golden.py

Runs the UNMODIFIED reference (oracle/_ref/liblpsim_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on seeded inputs and records
inputs and outputs in tests/golden/golden_v1.npz.  The fixtures travel with
the repo, so the GPU tests can check the kernels against the reference's own
outputs on a box where /root/reference does not exist.

Cases:
  * quantize_fused_at for float / fixed / block formats x 4 rounding modes on
    edge-case + random inputs (signed zeros, denormals, binade boundaries,
    midpoints, saturation, huge magnitudes), odd shapes, nonzero call ids;
  * block formats along every dimension of rank-3 tensors, tiny and huge
    block maxima, all-zero blocks;
  * random_uniform and uniform_variate (the input generator and the RNG);
  * matmul and quantized_matmul (the reference's only GEMM).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import (ALL_MODES, RefLib, block_fmt, f32_from_bits,  # noqa: E402
                        fixed_fmt, float_fmt)

OUT = os.path.join(HERE, "golden_v1.npz")

FLOAT_FMTS = [float_fmt(5, 2), float_fmt(8, 7), float_fmt(8, 23), float_fmt(4, 3),
              float_fmt(2, 1), float_fmt(1, 0), float_fmt(3, 2), float_fmt(8, 0),
              float_fmt(6, 9), float_fmt(1, 23)]
FIXED_FMTS = [fixed_fmt(8, 4), fixed_fmt(3, 1), fixed_fmt(8, 4, True),
              fixed_fmt(6, 2, False, False), fixed_fmt(5, 2, True, False),
              fixed_fmt(24, 126), fixed_fmt(2, -126), fixed_fmt(16, 12),
              fixed_fmt(24, -104, False, False), fixed_fmt(12, 60, True, False)]
BLOCK_FMTS = [block_fmt(8), block_fmt(4), block_fmt(8, 0), block_fmt(6, 1),
              block_fmt(8, 2), block_fmt(2, 0), block_fmt(24, 1)]


def edge_inputs(rng, n):
    specials = np.array([0.0, -0.0, 0.5, -0.5, 1.5, -1.5, 2.5, -2.5, 0.25, -0.25,
                         0.75, -0.75, 3.99, -3.99, 1e-45, -1e-45, 1.1754944e-38,
                         -1.1754944e-38, 3.4028235e38, -3.4028235e38, 114688.0,
                         -114688.0, 122880.0, 57344.0, 6.0, 7.9375, -8.0, -8.03125,
                         0.03125, 0.015625, 0.0078125],
                        dtype=np.float32)
    bits = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    rb = f32_from_bits(bits)
    rb = rb[np.isfinite(rb)]
    mags = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-150, 127, n)).astype(np.float32)
    unif = rng.uniform(-20, 20, n).astype(np.float32)
    x = np.concatenate([specials, rb[: n // 4], mags[: n // 4], unif[: n // 2]])
    return x[np.isfinite(x)][:n]


def main():
    ref = RefLib()
    rng = np.random.default_rng(20191010)
    arrays = {}
    meta = []

    def add(kind, fmt, mode, seed, call, x, y, st):
        i = len(meta)
        arrays[f"x{i}"] = x
        arrays[f"y{i}"] = y
        meta.append([kind, *[getattr(fmt, f) for f, _ in fmt._fields_], mode,
                     seed, call, st, x.ndim, *list(x.shape) + [0] * (4 - x.ndim)])

    x_flat = edge_inputs(rng, 3000).reshape(-1)
    x_odd = x_flat[:2999].copy()  # odd length
    for fmt in FLOAT_FMTS + FIXED_FMTS:
        for mode in ALL_MODES:
            seed, call = 77 + mode, 5 + mode
            for x in (x_flat, x_odd.reshape(1, 2999)):
                st, y = ref.quantize(x, fmt, mode, seed=seed, call=call)
                add(0, fmt, mode, seed, call, x, y, st)
    for fmt in BLOCK_FMTS:
        for mode in ALL_MODES:
            for scale_e in (0, -140, 100, -149, 126, -20):
                x = (rng.uniform(-1, 1, (6, 5, 9)) * 2.0 ** scale_e).astype(np.float32)
                if scale_e == -20:
                    x[1] = 0.0  # all-zero slices
                st, y = ref.quantize(x, fmt, mode, seed=3, call=1 + mode)
                add(0, fmt, mode, 3, 1 + mode, x, y, st)
    # generator and RNG
    u = ref.random_uniform((4097,), 7, 0, -4.0, 4.0)
    arrays["uniform_s7_m4_4"] = u
    arrays["uniform_s2_m10_10"] = ref.random_uniform((1000,), 2, 0, -10.0, 10.0)
    arrays["variates_15eed"] = np.array([ref.variate(0x15EED, 0, i) for i in range(1000)],
                                        dtype=np.float32)
    # matmul / quantized_matmul
    a = rng.uniform(-2, 2, (17, 33)).astype(np.float32)
    b = rng.uniform(-2, 2, (33, 29)).astype(np.float32)
    arrays["mm_a"], arrays["mm_b"] = a, b
    arrays["mm_c"] = ref.matmul(a, b)
    st, c, cc = ref.quantized_matmul(a, b, fixed_fmt(8, 4), 0, seed=11, call=3)
    arrays["qmm_fixed84_stoch_s11_c3"] = c
    st, c, cc = ref.quantized_matmul(a, b, float_fmt(5, 2), 1, seed=0, call=0)
    arrays["qmm_float52_even"] = c
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(meta)} quantize cases, "
          f"{os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
