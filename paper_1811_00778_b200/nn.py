"""Network descriptions as data (the reference's NetworkSpec tables) and
synthetic quantised weights.

Mirror of nn_oracle.py:22-196 / 381-407 for use without the reference tree;
the GPU evaluator accepts either these objects or the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

import numpy as np


class LayerKind(Enum):
    CONV = "conv"
    SQUARE = "square"
    POOL = "pool"
    FC = "fc"


@dataclass(frozen=True)
class LayerSpec:
    kind: LayerKind
    name: str
    filters: int = 0
    kernel: tuple = (0, 0)
    stride: tuple = (1, 1)
    padded: bool = False
    groups: int = 1
    weight_scale: int = 1
    extent: int = 0
    recorded_mult_plain: int | None = None


def conv_layer(name, filters, kernel, stride, padded, weight_scale, groups=1, recorded=None):
    return LayerSpec(LayerKind.CONV, name, filters, tuple(kernel), tuple(stride), padded, groups,
                     weight_scale, recorded_mult_plain=recorded)


def square_layer_spec(name):
    return LayerSpec(LayerKind.SQUARE, name)


def pool_layer(name, extent, stride):
    return LayerSpec(LayerKind.POOL, name, extent=extent, stride=(stride, stride))


def fc_layer(name, outputs, weight_scale, recorded=None):
    return LayerSpec(LayerKind.FC, name, filters=outputs, weight_scale=weight_scale,
                     recorded_mult_plain=recorded)


def kind_of(layer) -> str:
    """'conv' | 'square' | 'pool' | 'fc' for either enum family."""
    k = layer.kind
    return k.value if hasattr(k, "value") else str(k)


@dataclass(frozen=True)
class NetworkSpec:
    name: str
    input_shape: tuple
    input_scale: int
    layers: tuple
    wide_values: bool = False

    def layer_shapes(self):
        return layer_shapes(self)


def layer_shapes(spec):
    """Shape after each layer (nn_oracle.py:83-105)."""
    h, w, c = spec.input_shape
    out = []
    for layer in spec.layers:
        k = kind_of(layer)
        if k == "conv":
            kh, kw = layer.kernel
            sh, sw = layer.stride
            ph = (kh - 1) // 2 if layer.padded else 0
            pw = (kw - 1) // 2 if layer.padded else 0
            h = (h + 2 * ph - kh) // sh + 1
            w = (w + 2 * pw - kw) // sw + 1
            c = layer.filters
        elif k == "pool":
            sh, sw = layer.stride
            h = (h - layer.extent) // sh + 1
            w = (w - layer.extent) // sw + 1
        elif k == "fc":
            h, w, c = 1, 1, layer.filters
        out.append((h, w, c))
    return out


def mnist_hcnn() -> NetworkSpec:
    """conv(5@5x5,s2) - square - conv(50@5x5,s2,groups=5) - square - fc(10)
    (nn_oracle.py:108-126)."""
    return NetworkSpec("mnist_hcnn", (28, 28, 1), 4, (
        conv_layer("conv1", 5, (5, 5), (2, 2), False, 15),
        square_layer_spec("square1"),
        conv_layer("conv2", 50, (5, 5), (2, 2), False, 15, groups=5),
        square_layer_spec("square2"),
        fc_layer("fc", 10, 15),
    ))


def cifar10_hcnn() -> NetworkSpec:
    """11-layer CIFAR-10 HCNN (nn_oracle.py:129-157)."""
    return NetworkSpec("cifar10_hcnn", (32, 32, 3), 255, (
        conv_layer("conv1", 32, (3, 3), (1, 1), True, 10000, recorded=589_824),
        square_layer_spec("square1"),
        pool_layer("pool1", 2, 2),
        conv_layer("conv2", 64, (3, 3), (1, 1), True, 4095, recorded=2_594_048),
        square_layer_spec("square2"),
        pool_layer("pool2", 2, 2),
        conv_layer("conv3", 128, (3, 3), (1, 1), True, 10000, recorded=3_308_544),
        square_layer_spec("square3"),
        pool_layer("pool3", 2, 2),
        fc_layer("fc1", 256, 1023, recorded=457_398),
        fc_layer("fc2", 10, 63, recorded=2_518),
    ), wide_values=True)


def toy_hcnn() -> NetworkSpec:
    """8x8 input, conv 2@3x3 s2, square, fc 3 (nn_oracle.py:160-171)."""
    return NetworkSpec("toy_hcnn", (8, 8, 1), 4, (
        conv_layer("conv1", 2, (3, 3), (2, 2), False, 15),
        square_layer_spec("square1"),
        fc_layer("fc", 3, 15),
    ))


NETWORKS = {"mnist_hcnn": mnist_hcnn, "cifar10_hcnn": cifar10_hcnn, "toy_hcnn": toy_hcnn}


@dataclass
class QuantizedModel:
    spec: object
    bit_width: int
    weights: list


def integerize(j: int, levels: int, weight_scale: int) -> int:
    """round(j/levels * scale), half away from zero (nn_oracle.py:203-219)."""
    f = Fraction(j, levels) * weight_scale
    num, den = f.numerator, f.denominator
    if num >= 0:
        return (2 * num + den) // (2 * den)
    return -((-2 * num + den) // (2 * den))


def random_model(spec, rng: np.random.Generator, bit_width: int = 4) -> QuantizedModel:
    """Dense random k-bit quantised weights at each layer's scale (every tap
    executes: the worst-case workload)."""
    levels = (1 << bit_width) - 1
    table = {}
    shapes = [spec.input_shape] + layer_shapes(spec)
    weights = []
    for i, layer in enumerate(spec.layers):
        k = kind_of(layer)
        if k not in ("conv", "fc"):
            weights.append(None)
            continue
        sc = layer.weight_scale
        if sc not in table:
            table[sc] = np.array([integerize(j, levels, sc) for j in range(-levels, levels + 1)],
                                 dtype=np.int64)
        if k == "conv":
            cg = shapes[i][2] // layer.groups
            shape = (layer.filters, *layer.kernel, cg)
        else:
            h, w, c = shapes[i]
            shape = (layer.filters, h * w * c)
        idx = rng.integers(0, 2 * levels + 1, shape)
        weights.append(table[sc][idx])
    return QuantizedModel(spec, bit_width, weights)
