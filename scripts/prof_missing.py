"""Drive one kernel family a few times for an ncu capture (not a benchmark).

    python scripts/prof_missing.py general|seg|col|group|encode8|c1|c1log [reps]

general : k_qgemm_general (per-op GEMM float(5,2) stochastic, 2048^3, raw fp32 inputs)
raw     : k_qgemm_bf16<raw> (per-op GEMM float(8,7) nearest, 4096^3, raw fp32 inputs)
exact   : k_qgemm_bf16<exact> (C4: float(8,7)-exact operands, nearest, 4096^3)
bits    : k_qgemm_bits (per-op GEMM float(8,7) stochastic, 2048^3, raw fp32 inputs)
seg     : k_seg_reduce + k_seg_apply (block(8) whole tensor, 2^28)
col     : k_col_reduce + k_col_apply (block(8) dim 1 on [2^22, 64])
group   : k_group_elementwise / k_group_block_rows (ResNet-50 weights, grouped)
encode8 : k_encode8 (host path, fixed(8,4) nearest, 2^26 pinned floats)
c1      : k_elementwise float(5,2) stochastic, 2^24 (BASELINE C1)
c1log   : the C1 log-uniform variant
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

what = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
S, E = q.RoundingMode.Stochastic, q.RoundingMode.NearestEven

if what == "general":
    n = 2048
    a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
    b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
    c = torch.empty((n, n), device="cuda")
    for _ in range(reps):
        q.quant_gemm(a, b, q.FloatFormat(5, 2), q.FloatFormat(5, 2), S, 3, out=c, sync=False)
elif what == "bits":
    n = 2048
    a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
    b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
    c = torch.empty((n, n), device="cuda")
    for _ in range(reps):
        q.quant_gemm(a, b, q.FloatFormat(8, 7), q.FloatFormat(8, 7), S, 3, out=c, sync=False)
elif what in ("raw", "exact"):
    n = 4096
    a = q.random_uniform((n, n), 41, 0, -1.0, 1.0)
    b = q.random_uniform((n, n), 42, 0, -1.0, 1.0)
    if what == "exact":  # operands pre-quantized to float(8,7) (BASELINE C4)
        a = q.quantize_fused_at(a, q.QuantSpec(q.FloatFormat(8, 7), E, 1), 0)
        b = q.quantize_fused_at(b, q.QuantSpec(q.FloatFormat(8, 7), E, 1), 0)
    c = torch.empty((n, n), device="cuda")
    for _ in range(reps):
        q.quant_gemm(a, b, q.FloatFormat(8, 7), q.FloatFormat(8, 7), E, out=c, sync=False)
elif what in ("seg", "col", "c1", "c1log"):
    if what == "seg":
        x, spec = q.random_uniform((1 << 28,), 2, 0, -10.0, 10.0), q.QuantSpec(q.BlockFloatFormat(8), E, 7)
    elif what == "col":
        x, spec = q.random_uniform((1 << 22, 64), 2, 0, -10.0, 10.0), q.QuantSpec(q.BlockFloatFormat(8, 1), E, 7)
    else:
        x = q.random_uniform((1 << 24,), 7, 0, -4.0, 4.0)
        if what == "c1log":
            u = q.random_uniform((1 << 24,), 8, 0, -20.0, 20.0)
            s = q.random_uniform((1 << 24,), 9, 0, -1.0, 1.0)
            x = torch.sign(s) * torch.exp2(u)
        spec = q.QuantSpec(q.FloatFormat(5, 2), S, 0x15EED)
    y = torch.empty_like(x)
    for _ in range(reps):
        q.quantize_fused_at(x, spec, 0, out=y, sync=False)
elif what == "group":
    from paper_1910_04540_b200.resnet50 import resnet50_layers
    ws = [q.random_uniform(w, 100 + i, 0, -0.1, 0.1) for i, (_, w, _) in enumerate(resnet50_layers(256))]
    for f in (q.FloatFormat(5, 2), q.FixedFormat(8, 4), q.BlockFloatFormat(8, 0)):
        for _ in range(reps):
            q.quantize_fused_many(ws, q.QuantSpec(f, E, 7), sync=False)
elif what == "encode8":
    xh = torch.empty(1 << 26, dtype=torch.float32).pin_memory()
    xh.copy_(q.random_uniform((1 << 26,), 2, 0, -10.0, 10.0).cpu())
    xn = xh.numpy()
    for _ in range(reps):
        q.quantize_fused_at(xn, q.QuantSpec(q.FixedFormat(8, 4), E, 7), 0)
else:
    raise SystemExit(f"unknown {what}")
q.fetch_status()
torch.cuda.synchronize()
print("ok", what)
