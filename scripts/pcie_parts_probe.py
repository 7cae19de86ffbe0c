"""H2D DMA of 1 MB parts from page-locked memory: per-part time alone and
back to back (CUDA events), the direct host path pipeline's copy leg."""
import torch

torch.cuda.init()
n = 1 << 20
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.uniform_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for parts in (1, 4, 16):
    m = n // parts
    for rep in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(parts + 1)]
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            ev[0].record()
            for k in range(parts):
                d[k * m:(k + 1) * m].copy_(h[k * m:(k + 1) * m], non_blocking=True)
                ev[k + 1].record()
        torch.cuda.synchronize()
    print(f"{parts} parts of {4 * m >> 10} KB:", " ".join(f"{ev[0].elapsed_time(e) * 1e3:.0f}" for e in ev[1:]), "us")
