"""Low-precision optimizer step over the ResNet-50 parameter set (54 weight
tensors, 25.5M elements): per-step time and algorithmic GB/s (24 B/element:
read g, vel, acc; write vel, acc, w).  Specs: gradient fixed(8,6) stochastic,
accumulator float(8,23)... see below."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402
from paper_1910_04540_b200.optim import LowPrecisionOptimizer  # noqa: E402
from paper_1910_04540_b200.resnet50 import resnet50_layers  # noqa: E402

S, E = q.RoundingMode.Stochastic, q.RoundingMode.NearestEven
params = [q.random_uniform(w, 100 + i, 0, -0.1, 0.1) for i, (_, w, _) in enumerate(resnet50_layers(256))]
grads = [q.random_uniform(w.shape, 200 + i, 0, -1e-3, 1e-3) for i, w in enumerate(params)]
n = sum(p.numel() for p in params)
opt = LowPrecisionOptimizer(params, 0.1, 0.9, weight=q.QuantSpec(q.FixedFormat(8, 6), E, 1),
                            accumulator=q.QuantSpec(q.FloatFormat(8, 7), S, 2),
                            gradient=q.QuantSpec(q.FixedFormat(8, 12), S, 3))
for _ in range(3):
    opt.step(grads)
torch.cuda.synchronize()
reps = 20
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    opt.step(grads)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
ms = e0.elapsed_time(e1) / reps
print(f"{len(params)} tensors, {n} params: {ms:.3f} ms/step (device), {wall:.3f} ms (wall), "
      f"{24 * n / ms / 1e6:.0f} GB/s algorithmic (step(sync=True): status read every step)")
e0.record()
for _ in range(reps):
    opt.step(grads, sync=False)
e1.record()
torch.cuda.synchronize()
q.fetch_status()
ms = e0.elapsed_time(e1) / reps
print(f"step(sync=False), back to back: {ms:.3f} ms/step, {24 * n / ms / 1e6:.0f} GB/s algorithmic")
