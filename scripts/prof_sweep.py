"""Per-category timing of the C5 ResNet-50 sweep (diagnostic, not a bench):
each (tensor kind, format) group timed with CUDA events, achieved GB/s from
the library's own pass count."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402
from paper_1910_04540_b200.resnet50 import resnet50_layers  # noqa: E402

fmts = {"float52": q.FloatFormat(5, 2), "fixed84": q.FixedFormat(8, 4),
        "block8d0": q.BlockFloatFormat(8, 0)}
groups = defaultdict(list)
for i, (name, w, a) in enumerate(resnet50_layers(256)):
    groups["weight"].append((q.random_uniform(w, 100 + i, 0, -0.1, 0.1), q.RoundingMode.NearestEven))
    groups["grad"].append((q.random_uniform(w, 200 + i, 0, -1e-3, 1e-3), q.RoundingMode.Stochastic))
    groups["act"].append((q.random_uniform(a, 300 + i, 0, -4.0, 4.0), q.RoundingMode.NearestEven))
out = torch.empty(max(t.numel() for g in groups.values() for t, _ in g), device="cuda")
tot_ms = 0.0
for kind, ts in groups.items():
    for fname, f in fmts.items():
        def run():
            nbytes = 0
            for t, mode in ts:
                p0 = q.pass_count()
                q.quantize_fused_at(t, q.QuantSpec(f, mode, 7), 0, out=out[:t.numel()].view(t.shape), sync=False)
                nbytes += (8 if q.pass_count() - p0 == 1 else 12) * t.numel()
            return nbytes
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nb = run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tot_ms += ms
        print(f"{kind:7s} {fname:9s} {len(ts):3d} tensors {ms:8.3f} ms {nb / ms / 1e6:8.1f} GB/s")
q.fetch_status()
print(f"total {tot_ms:.3f} ms (eager, incl. launch gaps)")
