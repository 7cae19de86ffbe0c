"""Host-API timing (pageable numpy buffers, like the drop-in's std::vector):
lpq_quantize_host vs lpq_quantize_composed_host, the acceptance suite's
criterion 7 shape (2^20 elements, nearest, fixed(8,4) and block(8))."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
x = np.random.default_rng(1).uniform(-4, 4, n).astype(np.float32)
for fmt in (q.FixedFormat(8, 4), q.BlockFloatFormat(8)):
    spec = q.QuantSpec(fmt, q.RoundingMode.NearestEven, 3)
    res = {}
    for name, fn in (("fused", q.quantize_fused_at), ("composed", q.quantize_composed_at)):
        for _ in range(3):
            fn(x, spec, 0)
        ts = []
        for _ in range(9):
            t0 = time.perf_counter()
            fn(x, spec, 0)
            ts.append(time.perf_counter() - t0)
        res[name] = sorted(ts)[len(ts) // 2] * 1e3
    print(f"{fmt}: fused {res['fused']:.3f} ms composed {res['composed']:.3f} ms "
          f"ratio {res['fused'] / res['composed']:.3f}")
