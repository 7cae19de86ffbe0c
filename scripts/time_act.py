"""Time block(8, dim0) on ResNet-50 activation shapes (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_04540_b200 as q
shapes = [(256, 64, 112, 112), (256, 256, 56, 56), (256, 512, 28, 28), (256, 1024, 14, 14), (256, 2048, 7, 7)]
for mode in (q.RoundingMode.NearestEven, q.RoundingMode.Stochastic):
    tot_b = tot_ms = 0.0
    for shp in shapes:
        x = q.random_uniform(shp, 5, 0, -4.0, 4.0)
        y = torch.empty_like(x)
        spec = q.QuantSpec(q.BlockFloatFormat(8, 0), mode, 3)
        for _ in range(2):
            q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tot_b += 8 * x.numel(); tot_ms += ms
    q.fetch_status()
    print(f"var={os.environ.get('LPQ_CL_VARIANT','0')} {mode.name:12s} {tot_ms:.3f} ms  {tot_b / tot_ms / 1e6:.0f} GB/s")
