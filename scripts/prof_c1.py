"""One C1 launch (float(5,2) stochastic, 2^24 elements) for ncu."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
x = q.random_uniform((1 << 24,), 2, 0, -10.0, 10.0)
spec = q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode.Stochastic, 0x15EED)
for _ in range(3):
    y = q.quantize_fused_at(x, spec, 0)
torch.cuda.synchronize()
print("ok")
