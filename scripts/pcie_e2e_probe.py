"""Is the C2 e2e path (lpq_quantize_host, 2^30 pinned floats) H2D-bound?
Times, on one B200: the bare H2D of the 4 GiB input in 64 MiB chunks; the
same with a concurrent 16 MiB D2H per chunk (the byte codes); and the e2e
call itself."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04540_b200 as q
from paper_1910_04540_b200 import _lib

n = 1 << 30
chunk = 1 << 24
hx = torch.empty(n, dtype=torch.float32, pin_memory=True)
hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
hc = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)  # 1 B per element
d = [torch.empty(chunk, device="cuda") for _ in range(3)]
dc = torch.empty(chunk // 4, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def h2d_only():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s_in):
        for i in range(n // chunk):
            d[i % 3].copy_(hx[i * chunk:(i + 1) * chunk], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


def h2d_with_d2h():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n // chunk):
        with torch.cuda.stream(s_in):
            d[i % 3].copy_(hx[i * chunk:(i + 1) * chunk], non_blocking=True)
        with torch.cuda.stream(s_out):
            hc[i * (chunk // 4):(i + 1) * (chunk // 4)].copy_(dc, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


fmt = q.FixedFormat(8, 4).c()
shp = _lib.shape_array((n,))


def e2e():
    t0 = time.perf_counter()
    _lib.check(_lib.lib.lpq_quantize_host(C.c_void_p(hx.data_ptr()), C.c_void_p(hy.data_ptr()),
                                          shp, 1, 0, C.byref(fmt), 0, 7, 0, 0), "host")
    return time.perf_counter() - t0


for name, fn in (("h2d only", h2d_only), ("h2d + 1B d2h", h2d_with_d2h), ("e2e call", e2e)):
    fn()
    ts = [fn() for _ in range(3)]
    t = min(ts)
    print(f"{name:14s} {t * 1e3:7.1f} ms  H2D {4 * n / t / 1e9:5.1f} GB/s  "
          f"(e2e metric units {8 * n / t / 1e9:5.1f} GB/s)", flush=True)
