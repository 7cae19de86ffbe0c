"""The paper's fused-vs-many-kernel comparison (fused
fixed-point ~5x, fused block ~2.6x faster than the many-kernel approach) on
B200: lpq_quantize (fused) vs lpq_quantize_composed (one kernel per tensor op,
the reference's quantize_composed chain), CUDA events, device-resident data.

    python scripts/paper_compare.py [log2_elements ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


sizes = [int(a) for a in sys.argv[1:]] or [20, 24, 28]
rows = []
for lg in sizes:
    n = 1 << lg
    x = q.random_uniform((n // 64, 64), 7, 0, -4.0, 4.0)  # bench.cpp:58-60 shape
    for name, fmt in [("fixed:8:4", q.FixedFormat(8, 4)), ("block:8:tensor", q.BlockFloatFormat(8)),
                      ("block:8:dim0", q.BlockFloatFormat(8, 0))]:
        for mode in (q.RoundingMode.NearestEven, q.RoundingMode.Stochastic):
            spec = q.QuantSpec(fmt, mode, 0x15EED)
            fused = q.quantize_fused_at(x, spec, 0)
            comp = q.quantize_composed_at(x, spec, 0)
            assert torch.equal(fused.view(torch.int32), comp.view(torch.int32))
            tf = timeit(lambda: q.quantize_fused_at(x, spec, 0, sync=False))
            tc = timeit(lambda: q.quantize_composed_at(x, spec, 0, sync=False))
            rows.append({"elements": n, "format": name, "mode": mode.name,
                         "fused_ms": round(tf, 4), "composed_ms": round(tc, 4),
                         "speedup": round(tc / tf, 2)})
            print(json.dumps(rows[-1]), flush=True)
q.fetch_status()
