"""Golden fixtures for the per-op-rounded GEMM, produced by the reference
library itself.

    make -C oracle && python tests/golden/make_golden_gemm.py

The per-op GEMM is not a reference API; SURVEY.md §8(c) defines it as the
reference's own tensor-op composition per k over M x N tensors:
mul -> quantize_fused_at(call + 2k) -> add -> quantize_fused_at(call + 2k + 1)
(tensor.cpp:140-156, quant_ops.cpp:154-164).  oracle/ref_capi.cpp
lpsr_quant_gemm_composed runs exactly those reference calls; this script
records inputs and outputs in tests/golden/golden_gemm_v1.npz so the GPU
tests check the kernels (k_qgemm_bf16 and k_qgemm_general) against the
reference's outputs on a box where /root/reference does not exist.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import ALL_MODES, NEAREST_EVEN, RefLib, float_fmt  # noqa: E402

OUT = os.path.join(HERE, "golden_gemm_v1.npz")

# (name, (e_mul, m_mul), (e_add, m_add), m, k, n, scale_a, scale_b, prequantize, modes)
CASES = [
    ("f87", (8, 7), (8, 7), 24, 96, 20, 1.0, 1.0, False, ALL_MODES),
    ("f87_pre", (8, 7), (8, 7), 64, 256, 80, 1.0, 1.0, True, ALL_MODES),   # bf16 path
    ("f87_pre_wide", (8, 7), (8, 7), 33, 130, 67, 8.0, 0.125, True, (NEAREST_EVEN,)),
    ("f52", (5, 2), (5, 2), 20, 77, 24, 1.0, 1.0, False, ALL_MODES),
    ("f43", (4, 3), (4, 3), 17, 64, 9, 2.0, 2.0, False, ALL_MODES),
    ("f52_f87", (5, 2), (8, 7), 12, 128, 16, 16.0, 16.0, False, ALL_MODES),
    ("f823_f510", (8, 23), (5, 10), 9, 50, 11, 1.0, 1.0, False, ALL_MODES),
]


def main():
    ref = RefLib()
    ref.set_num_threads(os.cpu_count() or 1)
    rng = np.random.default_rng(19100454)
    arrays, meta = {}, []
    for ci, (name, fm, fa, m, k, n, sa, sb, pre, modes) in enumerate(CASES):
        a = (rng.uniform(-1, 1, (m, k)) * sa).astype(np.float32)
        b = (rng.uniform(-1, 1, (k, n)) * sb).astype(np.float32)
        a.flat[::9] = 0.0
        b.flat[4::13] = np.float32(-0.0)
        if pre:  # inputs already float(8,7) (bf16-exact): the kernels' bf16 path
            _, a = ref.quantize(a, float_fmt(8, 7), NEAREST_EVEN)
            _, b = ref.quantize(b, float_fmt(8, 7), NEAREST_EVEN)
        arrays[f"a{ci}"], arrays[f"b{ci}"] = a, b
        for mode in modes:
            seed, call = 0x15EED + ci, 3 + mode
            st, c = ref.quant_gemm_composed(a, b, float_fmt(*fm), float_fmt(*fa), mode,
                                            seed=seed, call=call)
            assert st == 0, (name, mode)
            arrays[f"c{ci}_{mode}"] = c
            meta.append([ci, *fm, *fa, mode, seed, call])
    arrays["meta"] = np.array(meta, dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(meta)} GEMM cases, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
