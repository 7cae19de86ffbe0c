import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
for n in (1 << 24, 1 << 28):
    x = q.random_uniform((n,), 5, 0, -4.0, 4.0)
    y = torch.empty_like(x)
    for mode in (q.RoundingMode.NearestEven, q.RoundingMode.Stochastic):
        spec = q.QuantSpec(q.BlockFloatFormat(8), mode, 3)
        for _ in range(2): q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"whole-tensor block 2^{n.bit_length()-1} {mode.name}: {ms:.3f} ms, {12 * n / ms / 1e6:.0f} GB/s of 12 B/elem traffic")
q.fetch_status()
