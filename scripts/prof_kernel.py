"""Run one quantizer config a few times (for ncu captures; not a benchmark).

    python scripts/prof_kernel.py c2 [n_log2] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nlog = int(sys.argv[2]) if len(sys.argv) > 2 else 28
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
S = q.RoundingMode.Stochastic
E = q.RoundingMode.NearestEven
specs = {
    "c1": (q.FloatFormat(5, 2), S, None), "c1n": (q.FloatFormat(5, 2), E, None),
    "c2": (q.FixedFormat(8, 4), S, None), "c2n": (q.FixedFormat(8, 4), E, None),
    "c3": (q.BlockFloatFormat(8, 0), E, 4096), "c3s": (q.BlockFloatFormat(8, 0), S, 4096),
    "whole": (q.BlockFloatFormat(8), E, None), "dim1": (q.BlockFloatFormat(8, 1), E, 64),
    "act": (q.BlockFloatFormat(8, 0), E, 802816),
    "acts": (q.BlockFloatFormat(8, 0), S, 802816),
    "short": (q.BlockFloatFormat(8, 0), S, 64),
}
fmt, mode, cols = specs[cfg]
n = 1 << nlog
if cfg in ("act", "acts"):
    n = 256 * 802816
shape = (n // cols, cols) if cols else (n,)
x = q.random_uniform(shape, 2, 0, -10.0, 10.0)
spec = q.QuantSpec(fmt, mode, 0x15EED)
y = torch.empty_like(x)
for _ in range(reps):
    q.quantize_fused_at(x, spec, 0, out=y, sync=False)
q.fetch_status()
torch.cuda.synchronize()
print("ok", cfg, shape)
