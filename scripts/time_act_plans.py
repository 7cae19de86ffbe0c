"""block(8, dim 0) GB/s on the ResNet-50 per-sample activation shapes
(batch 256): the chunk-rendezvous plan (lpq_quantize with a workspace) vs
the workspace-free cluster plan (ws = NULL), nearest and stochastic."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
from paper_1910_04540_b200 import _lib

shapes = [(256, 64, 112, 112), (256, 256, 56, 56), (256, 128, 56, 56), (256, 512, 28, 28),
          (256, 1024, 14, 14), (256, 2048, 7, 7), (256, 64, 56, 56), (256, 256, 14, 14)]
status = torch.zeros(1, dtype=torch.int32, device="cuda")
wsb = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for shp in shapes:
    x = q.random_uniform(shp, 5, 0, -4.0, 4.0)
    y = torch.empty_like(x)
    sa = _lib.shape_array(x.shape)
    line = [f"{shp[1] * shp[2] * shp[3]:>7}"]
    for mode in (1, 0):  # LPQ_NEAREST_EVEN = 1, LPQ_STOCHASTIC = 0 (include/lpq.h)
        fmt = q.BlockFloatFormat(8, 0).c()
        for plan, ws, nb in (("chunk", wsb.data_ptr(), wsb.numel()), ("cluster", 0, 0)):
            def run():
                rc = _lib.lib.lpq_quantize(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), sa,
                                           x.dim(), 0, C.byref(fmt), mode, 3, 0, C.c_void_p(ws),
                                           nb, C.c_void_p(status.data_ptr()), stream)
                assert rc == 0
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            # 10 launches captured in one CUDA graph (no host gaps)
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            with torch.cuda.graph(g, stream=side):
                sp = C.c_void_p(side.cuda_stream)
                for _ in range(10):
                    rc = _lib.lib.lpq_quantize(C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                               sa, x.dim(), 0, C.byref(fmt), mode, 3, 0,
                                               C.c_void_p(ws), nb, C.c_void_p(status.data_ptr()), sp)
                    assert rc == 0
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            line.append(f"{plan}/{'RN' if mode == 1 else 'SR'} {8 * x.numel() / ms / 1e6:6.0f}")
    print("  ".join(line), flush=True)
    del x, y
assert int(status.item()) == 0
