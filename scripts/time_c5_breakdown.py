"""Where the C5 sweep's time goes: CUDA-event time and achieved GB/s (8 B per
element per single pass, 12 B two-pass) of each part of the ResNet-50 sweep
(weights / gradients grouped per format, activations per format)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
from paper_1910_04540_b200 import _lib
from paper_1910_04540_b200.resnet50 import resnet50_layers

dev = torch.device("cuda", 0)
layers = resnet50_layers(256)
fmts = {"float52": q.FloatFormat(5, 2), "fixed84": q.FixedFormat(8, 4),
        "block8d0": q.BlockFloatFormat(8, 0)}
acts = [q.random_uniform(a, 300 + i, 0, -4.0, 4.0, device=dev) for i, (_, _, a) in enumerate(layers)]
out = torch.empty(max(a.numel() for a in acts), device=dev)
ws = torch.empty(1 << 20, dtype=torch.uint8, device=dev)
status = q.quant._status_buf(dev)
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for name, f in fmts.items():
    fc = f.c()
    by_len = {}
    for a in acts:
        shp = _lib.shape_array(a.shape)

        def run(a=a, shp=shp):
            _lib.check(_lib.lib.lpq_quantize(C.c_void_p(a.data_ptr()), C.c_void_p(out.data_ptr()),
                                             shp, a.dim(), 0, C.byref(fc), 1, 7, 0,
                                             C.c_void_p(ws.data_ptr()), ws.numel(),
                                             C.c_void_p(status.data_ptr()), s), "q")
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        row = a.numel() // a.shape[0]
        k = (name, row)
        t, n = by_len.get(k, (0.0, 0))
        by_len[k] = (t + ms, n + a.numel())
    tot_ms = sum(v[0] for v in by_len.values())
    tot_n = sum(v[1] for v in by_len.values())
    print(f"{name}: {tot_ms:.3f} ms, {8 * tot_n / tot_ms / 1e6:.0f} GB/s")
    for (nm, row), (t, n) in sorted(by_len.items(), key=lambda kv: -kv[1][0])[:8]:
        print(f"   row {row:>7}: {t:.3f} ms {8 * n / t / 1e6:.0f} GB/s")
q.fetch_status()
