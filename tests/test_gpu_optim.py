"""Fused low-precision optimizer step (lpq_sgd_step) vs a restatement of
LowPrecisionOptimizer::step (proj/src/train.cpp:148-178) built from the
oracle's quantizer and numpy fp32 ops (IEEE RN, == float(double op double)).
"""
import numpy as np
import pytest

from oracle_lib import STOCHASTIC, bits, block_fmt, fixed_fmt, float_fmt

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def oracle_fmt(f):
    import paper_1910_04540_b200 as q
    if isinstance(f, q.FloatFormat):
        return float_fmt(f.exp_bits, f.man_bits)
    if isinstance(f, q.BlockFloatFormat):
        return block_fmt(f.wl, f.block_dim)
    return fixed_fmt(f.wl, f.fl, f.symmetric, f.saturate)


class RefOpt:
    """train.cpp:148-178, elementwise formats, numpy + oracle."""

    def __init__(self, oracle, params, lr, mom, w, a, g):
        self.o, self.lr, self.mom = oracle, np.float32(lr), np.float32(mom)
        self.specs = {"w": w, "a": a, "g": g}
        self.calls = {"w": w.call_counter if w else 0, "a": a.call_counter if a else 0,
                      "g": g.call_counter if g else 0}
        self.acc = [p.copy() for p in params]
        self.vel = [np.zeros_like(p) for p in params]

    def q(self, which, x):
        s = self.specs[which]
        if s is None:
            return x
        st, y = self.o.quantize(x, oracle_fmt(s.format), int(s.mode), seed=s.seed,
                                call=self.calls[which])
        assert st == 0
        if int(s.mode) == STOCHASTIC:
            self.calls[which] += 1
        return y

    def step(self, params, grads):
        out = []
        for i, (p, g) in enumerate(zip(params, grads)):
            g = self.q("g", g)
            v = (self.vel[i] * self.mom).astype(np.float32) + g
            v = self.q("a", v.astype(np.float32))
            self.vel[i] = v
            a = (self.acc[i] - (v * self.lr).astype(np.float32)).astype(np.float32)
            a = self.q("a", a)
            self.acc[i] = a
            out.append(self.q("w", a))
        return out


@pytest.mark.parametrize("cfg", ["wage_like", "float_all_stoch", "no_quant", "nearest_away",
                                 "block_all", "block_mixed"])
def test_sgd_step_matches_reference_semantics(oracle, cfg):
    run_cfg(oracle, cfg, [(64, 33), (33,), (10, 64), (10,)])


def test_sgd_step_many_tensors(oracle):
    # > 64 tensors: several grouped launches; empty and 1-element tensors;
    # per-tensor call ids continue across the launch boundary
    rng = np.random.default_rng(9)
    shapes = [(int(rng.integers(1, 700)),) for _ in range(66)] + [(0,), (1,), (3, 1025)]
    run_cfg(oracle, "float_all_stoch", shapes, steps=2)
    run_cfg(oracle, "wage_like", shapes, steps=2)


def run_cfg(oracle, cfg, shapes, steps=4):
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.optim import LowPrecisionOptimizer
    S, E = q.RoundingMode.Stochastic, q.RoundingMode.NearestEven
    specs = {
        "wage_like": dict(weight=q.QuantSpec(q.FixedFormat(8, 6), E),
                          accumulator=q.QuantSpec(q.FixedFormat(16, 12), S, 11),
                          gradient=q.QuantSpec(q.FixedFormat(8, 10), S, 12)),
        "float_all_stoch": dict(weight=q.QuantSpec(q.FloatFormat(5, 2), S, 1),
                                accumulator=q.QuantSpec(q.FloatFormat(8, 7), S, 2, 5),
                                gradient=q.QuantSpec(q.FloatFormat(4, 3), S, 3)),
        "no_quant": dict(),
        # block floating point (the paper's training formats): the unfused
        # per-parameter sequence (train.cpp:161-174) on the device
        "block_all": dict(weight=q.QuantSpec(q.BlockFloatFormat(8, 0), E),
                          accumulator=q.QuantSpec(q.BlockFloatFormat(16), S, 21),
                          gradient=q.QuantSpec(q.BlockFloatFormat(8), S, 22)),
        "block_mixed": dict(weight=q.QuantSpec(q.FixedFormat(8, 6), E),
                            accumulator=q.QuantSpec(q.FloatFormat(8, 7), S, 2),
                            gradient=q.QuantSpec(q.BlockFloatFormat(8, 0), S, 23)),
        "nearest_away": dict(weight=q.QuantSpec(q.FloatFormat(5, 2), q.RoundingMode.NearestAway),
                             gradient=q.QuantSpec(q.FixedFormat(6, 4, True, False),
                                                  q.RoundingMode.NearestTowardZero)),
    }[cfg]
    rng = np.random.default_rng(5)
    params = [rng.uniform(-0.5, 0.5, s).astype(np.float32) for s in shapes]
    dev_params = [torch.from_numpy(p.copy()).cuda() for p in params]
    opt = LowPrecisionOptimizer(dev_params, lr=0.05, momentum=0.9, **specs)
    import copy
    ref = RefOpt(oracle, params, 0.05, 0.9, copy.deepcopy(specs.get("weight")),
                 copy.deepcopy(specs.get("accumulator")), copy.deepcopy(specs.get("gradient")))
    host_params = params
    for step in range(steps):
        grads = [rng.normal(0, 0.1, s).astype(np.float32) for s in shapes]
        host_params = ref.step(host_params, grads)
        opt.step([torch.from_numpy(g).cuda() for g in grads])
        for hp, dp in zip(host_params, dev_params):
            assert np.array_equal(bits(hp), bits(dp.cpu().numpy())), (cfg, step)
        for ha, da in zip(ref.acc, opt.accumulators()):
            assert np.array_equal(bits(ha), bits(da.cpu().numpy()))
    for k, spec in (("w", opt.weight_spec), ("a", opt.acc_spec), ("g", opt.grad_spec)):
        if spec is not None:
            assert spec.call_counter == ref.calls[k]


def test_sgd_step_bad_args():
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.optim import LowPrecisionOptimizer
    p = [torch.zeros(8, device="cuda")]
    with pytest.raises(q.FormatError):
        LowPrecisionOptimizer(p, lr=-1.0, momentum=0.5)
    with pytest.raises(q.FormatError):
        LowPrecisionOptimizer(p, lr=0.1, momentum=1.0)
    with pytest.raises(q.ShapeError):
        LowPrecisionOptimizer(p, 0.1, 0.5).step([torch.ones(9, device="cuda")])
    # dtype / device: the kernel reads every pointer as n fp32 device values
    with pytest.raises(TypeError):
        LowPrecisionOptimizer([torch.zeros(8, device="cuda", dtype=torch.float16)], 0.1, 0.5)
    with pytest.raises(TypeError):
        LowPrecisionOptimizer([torch.zeros(8)], 0.1, 0.5)
    opt = LowPrecisionOptimizer(p, 0.1, 0.5)
    for g in (torch.ones(8, device="cuda", dtype=torch.bfloat16), torch.ones(8)):
        with pytest.raises(TypeError):
            opt.step([g])
    # a rejected launch leaves the call counters untouched
    bad = q.QuantSpec(q.FixedFormat(30, 4), q.RoundingMode.Stochastic, 1, 5)
    opt = LowPrecisionOptimizer(p, 0.1, 0.5, gradient=bad)
    with pytest.raises(q.FormatError):
        opt.step([torch.ones(8, device="cuda")])
    assert opt.grad_spec.call_counter == 5


def test_sgd_step_async_equals_sync_and_defers_errors():
    import paper_1910_04540_b200 as q
    from paper_1910_04540_b200.optim import LowPrecisionOptimizer
    S, E = q.RoundingMode.Stochastic, q.RoundingMode.NearestEven
    specs = dict(weight=q.QuantSpec(q.FixedFormat(8, 6), E),
                 accumulator=q.QuantSpec(q.FloatFormat(8, 7), S, 2),
                 gradient=q.QuantSpec(q.FixedFormat(8, 12), S, 3))
    import copy
    shapes = [(300,), (17, 33), (4096,)]
    rng = np.random.default_rng(3)
    init = [rng.uniform(-0.5, 0.5, s).astype(np.float32) for s in shapes]
    pa = [torch.from_numpy(p.copy()).cuda() for p in init]
    pb = [torch.from_numpy(p.copy()).cuda() for p in init]
    oa = LowPrecisionOptimizer(pa, lr=0.05, momentum=0.9, **copy.deepcopy(specs))
    ob = LowPrecisionOptimizer(pb, lr=0.05, momentum=0.9, **copy.deepcopy(specs))
    for _ in range(3):
        grads = [torch.from_numpy(rng.normal(0, 0.01, s).astype(np.float32)).cuda()
                 for s in shapes]
        oa.step(grads)
        ob.step(grads, sync=False)
    q.fetch_status()
    for a, b in zip(pa, pb):
        assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    bad = [torch.full(s, float("inf"), device="cuda") for s in shapes]
    ob.step(bad, sync=False)  # no exception yet: the launch is asynchronous
    with pytest.raises(q.InvalidInputError):
        q.fetch_status()
    q.fetch_status()  # the status word was cleared
