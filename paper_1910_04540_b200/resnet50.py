"""ResNet-50 (torchvision v1.5 topology) tensor shapes for the C5 sweep
(BASELINE.json configs[4]: "training-step quantization sweep: ResNet-50-shaped
weight, activation and gradient tensors (batch 256) through all three
quantizers").

Weights: the 54 conv/fc weight tensors (25,502,912 elements); weight
gradients: the same 54 shapes; activations: the 54 conv/fc outputs at batch
256 (2,845,435,904 elements).  No network, no checkpoint: shapes only.
"""
from __future__ import annotations


def resnet50_layers(batch: int = 256):
    """[(name, weight_shape, activation_shape)] for the 54 conv/fc layers."""
    layers = []
    hw = 112
    layers.append(("conv1", (64, 3, 7, 7), (batch, 64, hw, hw)))
    hw = 56  # after the stride-2 max-pool
    cin = 64
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        cout = width * 4
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            hw_out = hw // stride
            p = f"layer{stage + 1}.{b}"
            layers.append((p + ".conv1", (width, cin, 1, 1), (batch, width, hw, hw)))
            layers.append((p + ".conv2", (width, width, 3, 3), (batch, width, hw_out, hw_out)))
            layers.append((p + ".conv3", (cout, width, 1, 1), (batch, cout, hw_out, hw_out)))
            if b == 0:
                layers.append((p + ".downsample", (cout, cin, 1, 1),
                               (batch, cout, hw_out, hw_out)))
            cin = cout
            hw = hw_out
    layers.append(("fc", (1000, 2048), (batch, 1000)))
    return layers


def numel(shape):
    n = 1
    for s in shape:
        n *= int(s)
    return n


SWEEP_SEED = 0x15EED  # proj/src/bench.cpp:56


class ResNet50Sweep:
    """The C5 training-step quantization sweep as a launch plan over the
    library's C ABI: every weight, weight gradient and activation tensor of
    ResNet-50 (batch 256) through float(5,2), fixed(8,4) and block(8, dim 0)
    (per out-channel for weights / gradients, per sample for activations);
    nearest-even for weights and activations, stochastic for gradients (call
    id = the tensor's position in its group, as a loop of quantize_fused calls
    over the 54 tensors would give).

    Work units (for multi-GPU bin-packing by bytes, shard.binpack):
      unit 0      the 54 weights      -> one lpq_quantize_grouped per format
      unit 1      the 54 gradients    -> one lpq_quantize_grouped per format
      unit 2 + i  activation i        -> one lpq_quantize per format
    Inputs are generated on the device with the reference generator
    (random_uniform: weights U(-0.1, 0.1) seed 100+i, gradients U(-1e-3, 1e-3)
    seed 200+i, activations U(-4, 4) seed 300+i).

    separate_outputs=False writes every activation's three outputs into one
    scratch buffer (the bench: outputs are not kept); True gives each
    quantization its own output tensor (parity tests)."""

    FORMAT_NAMES = ("float:5:2", "fixed:8:4", "block:8:0")

    def __init__(self, q, device, units=None, batch=256, separate_outputs=False):
        import ctypes as C
        import torch
        from . import _lib
        self.q, self.C, self._lib = q, C, _lib
        self.device = device
        self.layers = resnet50_layers(batch)
        self.fmts = [q.FloatFormat(5, 2), q.FixedFormat(8, 4), q.BlockFloatFormat(8, 0)]
        all_units = range(2 + len(self.layers))
        self.units = sorted(all_units if units is None else units)
        self.groups, self.singles, self._keep = [], [], []
        self.inputs = {}   # (kind, layer) -> tensor; kind 0 weight, 1 grad, 2 act
        self.outputs = {}  # (kind, layer, format index) -> tensor (when kept)
        E, S = q.RoundingMode.NearestEven, q.RoundingMode.Stochastic
        for kind in (0, 1):
            if kind not in self.units:
                continue
            seed0, half = (100, 0.1) if kind == 0 else (200, 1e-3)
            mode = E if kind == 0 else S
            ts = [q.random_uniform(w, seed0 + i, 0, -half, half, device=device)
                  for i, (_, w, _) in enumerate(self.layers)]
            for i, t in enumerate(ts):
                self.inputs[(kind, i)] = t
            for fi, f in enumerate(self.fmts):
                outs = [torch.empty_like(t) for t in ts]
                descs = (_lib.LpqTensorDesc * len(ts))()
                for j, (t, o) in enumerate(zip(ts, outs)):
                    shp = _lib.shape_array(t.shape)
                    self._keep.append(shp)
                    descs[j] = _lib.LpqTensorDesc(t.data_ptr(), o.data_ptr(), shp, t.dim(),
                                                  0, 0, j)
                    self.outputs[(kind, j, fi)] = o
                self.groups.append((descs, len(ts), f.c(), int(mode),
                                    sum(t.numel() for t in ts)))
        acts = [(i, q.random_uniform(a, 300 + i, 0, -4.0, 4.0, device=device))
                for i, (_, _, a) in enumerate(self.layers) if 2 + i in self.units]
        scratch = None
        if not separate_outputs and acts:
            scratch = torch.empty(max(t.numel() for _, t in acts), device=device)
        for i, t in acts:
            self.inputs[(2, i)] = t
            shp = _lib.shape_array(t.shape)
            self._keep.append(shp)
            for fi, f in enumerate(self.fmts):
                o = torch.empty_like(t) if separate_outputs else scratch
                if separate_outputs:
                    self.outputs[(2, i, fi)] = o
                self.singles.append((C.c_void_p(t.data_ptr()), C.c_void_p(o.data_ptr()), shp,
                                     t.dim(), f.c(), int(E), t.numel()))
        self._scratch = scratch
        self.ws = torch.empty(1 << 20, dtype=torch.uint8, device=device)
        self.status = q.quant._status_buf(device)
        self.nbytes = None
        self.launches = None

    @staticmethod
    def unit_bytes(batch=256):
        """Algorithmic bytes of each work unit (8 B per element per format)."""
        layers = resnet50_layers(batch)
        w = sum(numel(ws) for _, ws, _ in layers)
        return [24 * w, 24 * w] + [24 * numel(a) for _, _, a in layers]

    def launch(self, stream_ptr):
        """Every quantization of this plan on one stream (graph-capturable)."""
        C, L = self.C, self._lib
        for descs, cnt, fc, mode, _ in self.groups:
            L.check(L.lib.lpq_quantize_grouped(descs, cnt, C.byref(fc), mode, SWEEP_SEED,
                                               C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                               C.c_void_p(self.status.data_ptr()), stream_ptr),
                    "sweep")
        for xp, yp, shp, rank, fc, mode, _ in self.singles:
            L.check(L.lib.lpq_quantize(xp, yp, shp, rank, 0, C.byref(fc), mode, SWEEP_SEED, 0,
                                       C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                       C.c_void_p(self.status.data_ptr()), stream_ptr),
                    "sweep")

    def measure_once(self, stream_ptr):
        """Run the plan once eagerly; record the algorithmic bytes (8 B per
        element for single-pass plans, 12 for the two-pass block plans, from
        the library's pass counter) and the kernel launches."""
        q = self.q
        l0 = q.launch_count()
        nbytes = 8 * sum(g[4] for g in self.groups)
        C, L = self.C, self._lib
        for descs, cnt, fc, mode, _ in self.groups:
            L.check(L.lib.lpq_quantize_grouped(descs, cnt, C.byref(fc), mode, SWEEP_SEED,
                                               C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                               C.c_void_p(self.status.data_ptr()), stream_ptr),
                    "sweep")
        for xp, yp, shp, rank, fc, mode, n in self.singles:
            p0 = q.pass_count()
            L.check(L.lib.lpq_quantize(xp, yp, shp, rank, 0, C.byref(fc), mode, SWEEP_SEED, 0,
                                       C.c_void_p(self.ws.data_ptr()), self.ws.numel(),
                                       C.c_void_p(self.status.data_ptr()), stream_ptr),
                    "sweep")
            nbytes += (8 if q.pass_count() - p0 == 1 else 12) * n
        self.nbytes = nbytes
        self.launches = q.launch_count() - l0
        return nbytes
