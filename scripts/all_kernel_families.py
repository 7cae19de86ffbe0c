"""One small call of every kernel family, each checked against the oracle
(elementwise with scalar tail, rows in registers, short rows, cluster/DSMEM,
two-pass segments and columns, whole tensor, both GEMMs, the reference
matmul, composed chain, grouped launch, optimizer step, generators):

    python scripts/all_kernel_families.py

(Written for compute-sanitizer memcheck/racecheck/synccheck runs; the tool is
closed on this GPU pool, so it runs as a plain all-families check.)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402
from oracle_lib import Oracle, bits, block_fmt, fixed_fmt, float_fmt  # noqa: E402

o = Oracle()
rng = np.random.default_rng(5)
S, E = q.RoundingMode.Stochastic, q.RoundingMode.NearestEven


def check(x, fmt, ofmt, mode, base=0):
    got = q.quantize_fused_at(torch.from_numpy(x).cuda(), q.QuantSpec(fmt, mode, 9), 2,
                              index_base=base).cpu().numpy()
    st, want = o.quantize(x, ofmt, int(mode), seed=9, call=2, index_base=base)
    assert st == 0 and np.array_equal(bits(got), bits(want)), (fmt, mode, x.shape)


cases = [
    ((4099,), q.FixedFormat(8, 4), fixed_fmt(8, 4)),            # elementwise + tail
    ((1 << 16,), q.FloatFormat(5, 2), float_fmt(5, 2)),
    ((64, 4096), q.BlockFloatFormat(8, 0), block_fmt(8, 0)),   # rows in registers
    ((999, 12), q.BlockFloatFormat(8, 0), block_fmt(8, 0)),    # short rows
    ((300, 40000), q.BlockFloatFormat(8, 0), block_fmt(8, 0)), # cluster / DSMEM
    ((5, 40000), q.BlockFloatFormat(8, 0), block_fmt(8, 0)),   # two-pass segments
    ((50, 70, 30), q.BlockFloatFormat(8, 1), block_fmt(8, 1)), # two-pass columns
    ((100003,), q.BlockFloatFormat(8), block_fmt(8)),          # whole tensor
]
for shape, fmt, ofmt in cases:
    x = rng.uniform(-3, 3, shape).astype(np.float32)
    for mode in (E, S):
        check(x, fmt, ofmt, mode)
# per-op GEMM (bf16 path and general path) and the reference matmul
a = q.quantize_fused_at(torch.randn(70, 50, device="cuda"), q.QuantSpec(q.FloatFormat(8, 7)), 0)
b = q.quantize_fused_at(torch.randn(50, 90, device="cuda"), q.QuantSpec(q.FloatFormat(8, 7)), 0)
q.quant_gemm(a, b, q.FloatFormat(8, 7), q.FloatFormat(8, 7))
q.quant_gemm(a, b, q.FloatFormat(5, 2), q.FloatFormat(5, 2))
q.quantized_matmul_at(a, b, q.QuantSpec(q.FixedFormat(8, 4)), 0)
# composed chain, grouped launch, optimizer step, generators
x = torch.from_numpy(rng.uniform(-3, 3, (64, 300)).astype(np.float32)).cuda()
q.quantize_composed_at(x, q.QuantSpec(q.BlockFloatFormat(8, 0), S, 1), 0)
q.quantize_fused_many([x, x[:10]], q.QuantSpec(q.FixedFormat(8, 4), S, 1))
from paper_1910_04540_b200.optim import LowPrecisionOptimizer  # noqa: E402
p = torch.zeros(33, 17, device="cuda")
opt = LowPrecisionOptimizer([p], 0.1, 0.9, weight=q.QuantSpec(q.FixedFormat(8, 4)),
                            gradient=q.QuantSpec(q.FixedFormat(8, 6), S, 3))
opt.step([torch.randn(33, 17, device="cuda")])
q.random_uniform((1000,), 1, 0, -1.0, 1.0)
torch.cuda.synchronize()
q.fetch_status()
print("all kernel families ok")
