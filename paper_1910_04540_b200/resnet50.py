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
