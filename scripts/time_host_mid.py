import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1910_04540_b200 as q
spec = q.QuantSpec(q.FixedFormat(8, 4), q.RoundingMode.Stochastic, 3)
for n in (1 << 23, 1 << 24, 1 << 25):
    x = np.random.default_rng(1).uniform(-6, 6, n).astype(np.float32)
    for kind in ("pageable", "pinned"):
        xin = x if kind == "pageable" else torch.from_numpy(x).pin_memory()
        for _ in range(2): q.quantize_fused_at(xin, spec, 0)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter(); q.quantize_fused_at(xin, spec, 0); ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(f"mc={os.environ.get('LPQ_MIN_CHUNKS')} n={n} {kind}: {t*1e3:.2f} ms = {8*n/t/1e9:.1f} GB/s")
