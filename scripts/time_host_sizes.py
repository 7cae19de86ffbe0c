"""Host-API time of one fused quantize (fixed(8,4) stochastic, pageable and
pinned buffers) at sizes around the direct / streamed cut (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_04540_b200 as q  # noqa: E402

spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 3)
for n in (1 << 20, 1 << 21, 3 << 20, 1 << 22):
    x = np.random.default_rng(1).uniform(-6, 6, n).astype(np.float32)
    for kind in ("pageable", "pinned"):
        xin = x if kind == "pageable" else torch.from_numpy(x).pin_memory()
        for _ in range(3):
            q.quantize_fused_at(xin, spec, 0)
        ts = []
        for _ in range(11):
            t0 = time.perf_counter()
            q.quantize_fused_at(xin, spec, 0)
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(f"n={n} {kind}: {t * 1e6:.0f} us = {8 * n / t / 1e9:.1f} GB/s")
