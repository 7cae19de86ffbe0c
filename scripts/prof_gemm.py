"""Run the per-op GEMM (C4) a few times (for ncu captures; not a benchmark).

    python scripts/prof_gemm.py [n] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
f87 = q.QuantSpec(q.FloatFormat(8, 7))
a = q.quantize_fused_at(q.random_uniform((n, n), 41, 0, -1.0, 1.0), f87, 0)
b = q.quantize_fused_at(q.random_uniform((n, n), 42, 0, -1.0, 1.0), f87, 0)
c = torch.empty((n, n), device="cuda")
fm = q.FloatFormat(8, 7)
for _ in range(reps):
    q.quant_gemm(a, b, fm, fm, out=c, sync=False)
q.fetch_status()
torch.cuda.synchronize()
print("ok", n)
