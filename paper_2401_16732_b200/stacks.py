"""Layer lists of the ResNet-shaped HE conv stacks of BASELINE configs 3-5.

The reference has no model format (SPEC's `model` module is absent), so the
stacks are written out here from BASELINE.json and SURVEY §8d:
  * strided convs run at the INPUT resolution and are subsampled at the next
    client repack (TileLayout.stride, conv.py:83,110,162-177);
  * stage transitions use 1x1 projection shortcuts (also stride 2);
  * config 5 reading (A): a 2x2 average pool after the 7x7 stride-2 stem.
Host-only metadata: the bench and the parity tests instantiate each layer's
K1 plan from it.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Layer:
    name: str
    kind: str  # "conv" | "pool" | "fc"
    H: int
    W: int
    f_w: int = 3
    c_i: int = 0
    c_o: int = 0
    stride: int = 1


def _resnet(stem, stages, blocks_per_stage, pool, fc_out):
    layers = [stem]
    H = stem.H // stem.stride
    c = stem.c_o
    if pool:
        layers.append(pool)
        H //= pool.f_w
    for si, width in enumerate(stages):
        for b in range(blocks_per_stage):
            first = b == 0 and si > 0
            s = 2 if first else 1
            cin = c if b == 0 else width
            layers.append(Layer(f"s{si + 1}b{b + 1}c1", "conv", H, H, 3, cin, width, s))
            Ho = H // s
            layers.append(Layer(f"s{si + 1}b{b + 1}c2", "conv", Ho, Ho, 3, width, width, 1))
            if first:
                layers.append(Layer(f"s{si + 1}b{b + 1}proj", "conv", H, H, 1, cin, width, 2))
            H = Ho
        c = width
    layers.append(Layer("avgpool", "pool", H, H, H, c, c))
    layers.append(Layer("fc", "fc", 1, 1, 1, c, fc_out))
    return layers


def config3():
    """ResNet-20 on 32x32x3: stem 3->16, 3 stages x 3 blocks at 16/32/64, pool 8, FC 64->100."""
    return _resnet(Layer("stem", "conv", 32, 32, 3, 3, 16), [16, 32, 64], 3, None, 100)


def config4():
    """ResNet-18 on 64x64x3: 3x3 stem 3->64, 4 stages x 2 blocks at 64..512, pool 8, FC 512->200."""
    return _resnet(Layer("stem", "conv", 64, 64, 3, 3, 64), [64, 128, 256, 512], 2, None, 200)


def config5():
    """ResNet-18 on 224x224x3: 7x7 s2 stem, 2x2 avg-pool (reading A), 4 stages, pool 7, FC 512->1000."""
    stem = Layer("stem", "conv", 224, 224, 7, 3, 64, 2)
    return _resnet(stem, [64, 128, 256, 512], 2, Layer("pool2", "pool", 112, 112, 2, 64, 64), 1000)


def config1():
    """The single config-1 layer: 3x3, 16->16 on 32x32."""
    return [Layer("conv", "conv", 32, 32, 3, 16, 16, 1)]


CONFIGS = {"config1": config1, "config3": config3, "config4": config4, "config5": config5}


def conv_layers(layers):
    return [l for l in layers if l.kind == "conv"]
