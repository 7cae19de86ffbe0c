"""Per-shape block(8, dim 0) GB/s on the ResNet-50 activation row lengths
(diagnostic for the cluster size choice in csrc/block_cluster.cu)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
shapes = [(256, 64, 112, 112), (256, 512, 28, 28), (256, 1024, 14, 14), (256, 2048, 7, 7), (256, 256, 14, 14)]
res = []
for shp in shapes:
    x = q.random_uniform(shp, 5, 0, -4.0, 4.0)
    y = torch.empty_like(x)
    for mode in (q.RoundingMode.NearestEven, q.RoundingMode.Stochastic):
        spec = q.QuantSpec(q.BlockFloatFormat(8, 0), mode, 3)
        for _ in range(2):
            q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            q.quantize_fused_at(x, spec, 0, out=y, sync=False)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res.append(f"{shp[1]*shp[2]*shp[3]}/{mode.name[:5]}:{8 * x.numel() / ms / 1e6:.0f}")
q.fetch_status()
print(" ".join(res))
