"""GPU parity of the C5 sweep AS THE BENCH LAUNCHES IT (the
grouped + single launch plan had no end-to-end oracle check).

paper_1910_04540_b200.resnet50.ResNet50Sweep is the plan bench.py --config c5
replays: 6 grouped launches (54 weights / 54 gradients x 3 formats) and 162
single launches (54 activations x 3 formats).  Here every quantization gets
its own output and is compared with the oracle: weights and gradients in
full, activations on sampled per-sample blocks (rows of the [256, C*H*W]
view, with their global index base).  Bit-exact.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle_lib import NEAREST_EVEN, STOCHASTIC, bits, block_fmt, fixed_fmt, float_fmt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

OFMTS = (float_fmt(5, 2), fixed_fmt(8, 4), block_fmt(8, 0))


def test_c5_sweep_launch_plan_vs_oracle(oracle):
    import ctypes as C
    import os
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.resnet50 import SWEEP_SEED, ResNet50Sweep
    dev = torch.device("cuda", 0)
    plan = ResNet50Sweep(q, dev, separate_outputs=True)
    assert len(plan.groups) == 6 and len(plan.singles) == 162
    plan.launch(C.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    q.fetch_status(dev)
    jobs = []
    for (kind, i, fi), y in plan.outputs.items():
        x = plan.inputs[(kind, i)]
        if kind in (0, 1):  # weights / gradients: whole tensors
            mode = NEAREST_EVEN if kind == 0 else STOCHASTIC
            jobs.append(((kind, i, fi), x.cpu().numpy(), y.cpu().numpy(), mode, i, 0))
        else:  # activations: first, middle, last per-sample block
            B = x.shape[0]
            xr, yr = x.reshape(B, -1), y.reshape(B, -1)
            L = xr.shape[1]
            for s in (0, B // 2 + i % 7, B - 1):
                jobs.append(((kind, i, fi, s), xr[s:s + 1].cpu().numpy(),
                             yr[s:s + 1].cpu().numpy(), NEAREST_EVEN, 0, s * L))

    def check(job):
        key, xh, yh, mode, call, base = job
        st, want = oracle.quantize(xh, OFMTS[key[2]], mode, seed=SWEEP_SEED, call=call,
                                   index_base=base)
        return key, st == 0 and np.array_equal(bits(yh), bits(want))

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        res = list(ex.map(check, jobs))
    bad = [k for k, ok in res if not ok]
    assert len(res) == 2 * 54 * 3 + 54 * 3 * 3 and not bad, bad[:10]
