"""Per-op GEMM on the general path (formats other than float(8,7), or
stochastic rounding): TFLOP/s (2*M*N*K) with CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
c = torch.empty((n, n), device="cuda")
for fm, fa, mode in ((q.FloatFormat(5, 2), q.FloatFormat(5, 2), q.RoundingMode.NearestEven),
                     (q.FloatFormat(5, 2), q.FloatFormat(5, 2), q.RoundingMode.Stochastic),
                     (q.FloatFormat(8, 7), q.FloatFormat(8, 7), q.RoundingMode.Stochastic),
                     (q.FloatFormat(8, 23), q.FloatFormat(8, 23), q.RoundingMode.NearestEven)):
    for _ in range(2):
        q.quant_gemm(a, b, fm, fa, mode, 3, out=c, sync=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        q.quant_gemm(a, b, fm, fa, mode, 3, out=c, sync=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{fm} {mode.name}: {ms:.2f} ms {2 * n**3 / ms / 1e9:.2f} TFLOP/s")
q.fetch_status()
