"""ActivationQuant / ErrorQuant / inject_quantizers (proj/src/train.cpp:54-128)
as torch modules: structure on CPU (the cases of proj/tests/test_train.cpp:
284-320), numerics on the GPU against the oracle quantizer."""
import numpy as np
import pytest

from oracle_lib import STOCHASTIC, bits, fixed_fmt

torch = pytest.importorskip("torch")


def mlp(dims, seed):
    torch.manual_seed(seed)
    mods = []
    for i in range(len(dims) - 1):
        mods.append(torch.nn.Linear(dims[i], dims[i + 1]))
        if i + 2 < len(dims):
            mods.append(torch.nn.ReLU())
    return torch.nn.Sequential(*mods)


def spec(wl, fl, mode=0, seed=3):
    import paper_1910_04540_b200 as q
    return q.QuantSpec(q.FixedFormat(wl, fl), q.RoundingMode(mode), seed, 0)


def test_inject_structure():
    from paper_1910_04540_b200 import layers as L
    from paper_1910_04540_b200.io import QuantConfig
    m = mlp([2, 16, 2], 51)
    assert len(m) == 3
    net = L.inject_quantizers(m, QuantConfig())
    assert len(net) == 3 and net._lpq_injected
    net = L.inject_quantizers(m, QuantConfig(activation=spec(8, 4), error=spec(8, 6)))
    kinds = [type(x).__name__ for x in net]
    assert kinds == ["Linear", "ErrorQuant", "ReLU", "ActivationQuant", "Linear",
                     "ErrorQuant", "ActivationQuant"]
    with pytest.raises(L.InjectionError):
        L.inject_quantizers(L.inject_quantizers(m, QuantConfig()), QuantConfig())
    with pytest.raises(L.InjectionError):
        L.inject_quantizers(torch.nn.Sequential(L.ActivationQuant(spec(8, 4))), QuantConfig())


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, STOCHASTIC])
def test_activation_and_error_quant_vs_oracle(oracle, mode):
    from paper_1910_04540_b200 import layers as L
    from paper_1910_04540_b200.io import QuantConfig
    m = mlp([2, 8, 2], 5).cuda()
    aspec, espec = spec(3, 1, mode, seed=11), spec(8, 6, mode, seed=12)
    net = L.inject_quantizers(m, QuantConfig(activation=aspec, error=espec))
    trace = []
    for layer in net:
        if isinstance(layer, L.ErrorQuant):
            layer.trace = trace
    x = torch.randn(32, 2, device="cuda")
    # forward: reproduce each stage with the oracle
    cur = x
    acts = []
    for layer in net:
        prev = cur
        cur = layer(cur)
        if isinstance(layer, L.ActivationQuant):
            # every layer owns a copy of the spec: its first call is 0
            st, want = oracle.quantize(prev.detach().cpu().numpy(), fixed_fmt(3, 1), mode,
                                       seed=11, call=0)
            assert st == 0
            assert np.array_equal(bits(cur.detach().cpu().numpy()), bits(want))
            acts.append(cur)
    assert all(layer.spec.call_counter == (1 if mode == STOCHASTIC else 0)
               for layer in net if isinstance(layer, L.ActivationQuant))
    # backward: error signals are the quantized incoming gradients
    grads = {}
    hooks = [layer.register_full_backward_hook(
        lambda mod, gin, gout, i=i: grads.__setitem__(i, gout[0].detach().clone()))
        for i, layer in enumerate(net) if isinstance(layer, L.ErrorQuant)]
    cur.sum().backward()
    for h in hooks:
        h.remove()
    assert len(trace) == 2
    for (i, g_in), sig in zip(sorted(grads.items(), reverse=True), trace):
        st, want = oracle.quantize(g_in.cpu().numpy(), fixed_fmt(8, 6), mode, seed=12, call=0)
        assert st == 0
        assert np.array_equal(bits(sig.cpu().numpy()), bits(want))
