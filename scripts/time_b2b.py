"""Back-to-back quantize launches captured in one CUDA graph (no host
overhead, no events between kernels): the device-side cost of a stream of
small quantizations.

    python scripts/time_b2b.py [log2_elements] [format] [mode] [launches]

Measured on B200 (round 1): 2^24 float(5,2) nearest 21.8 us/launch (6145
GB/s), stochastic 31.6 us; 2^20 fixed(8,4) 3.0-3.2 us.  Programmatic
dependent launch (griddepcontrol) was tried on top of this and changed
nothing beyond noise (+-3 %), so the kernels use plain launches.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402
from paper_1910_04540_b200 import io as lio  # noqa: E402

nlog = int(sys.argv[1]) if len(sys.argv) > 1 else 24
fmt = lio.parse_format(sys.argv[2] if len(sys.argv) > 2 else "float:5:2")
mode = lio.parse_rounding(sys.argv[3] if len(sys.argv) > 3 else "nearest_even")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 200
n = 1 << nlog
shape = (n // 4096, 4096) if isinstance(fmt, q.BlockFloatFormat) and fmt.block_dim == 0 else (n,)
nbuf = max(2, (512 << 20) // (n * 8))
xs = [q.random_uniform(shape, 2 + i, 0, -10.0, 10.0, device="cuda") for i in range(nbuf)]
ys = [torch.empty_like(x) for x in xs]
spec = q.QuantSpec(fmt, mode, 5, 0)
for i in range(5):
    q.quantize_fused_at(xs[i % nbuf], spec, 0, out=ys[i % nbuf], sync=False)
torch.cuda.synchronize()
# capture the launches in a CUDA graph so host overhead cannot starve the GPU
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    with torch.cuda.graph(g, stream=side):
        for i in range(reps):
            q.quantize_fused_at(xs[i % nbuf], spec, 0, out=ys[i % nbuf], sync=False)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
print(f"2^{nlog} {sys.argv[2:4]} "
      f"{us:.2f} us/launch  {8 * n / us / 1e3:.0f} GB/s")
