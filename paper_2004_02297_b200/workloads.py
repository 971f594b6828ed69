"""The named synthetic weight sets of BASELINE.json configs.

Shapes are generated programmatically (torchvision is not needed at run
time); tests/test_host_logic.py checks them against torchvision's
meta-device parameter shapes in the build container.
"""

from __future__ import annotations

import math


def lenet():
    """Caffe LeNet weight tensors: 430,500 weights."""
    return [(20, 1, 5, 5), (50, 20, 5, 5), (500, 800), (10, 500)]


def alexnet():
    """torchvision AlexNet weight tensors (8 layers, 61,090,496 weights)."""
    return [(64, 3, 11, 11), (192, 64, 5, 5), (384, 192, 3, 3), (256, 384, 3, 3), (256, 256, 3, 3),
            (4096, 9216), (4096, 4096), (1000, 4096)]


ALEXNET_BITS = (8, 16, 24, 32, 8, 16, 24, 32)  # BASELINE.json configs[1]: widths by layer index


def vgg16():
    """torchvision VGG-16 weight tensors (16 layers, 138,344,128 weights)."""
    cfg = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512]
    shapes, cin = [], 3
    for c in cfg:
        shapes.append((c, cin, 3, 3))
        cin = c
    return shapes + [(4096, 512 * 7 * 7), (4096, 4096), (1000, 4096)]


def resnet50():
    """All 161 torchvision ResNet-50 parameter tensors (25,557,032 weights), in
    named_parameters() order: conv weights, BN weights/biases, fc weight/bias."""
    shapes = [(64, 3, 7, 7), (64,), (64,)]
    cin = 64
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        out = width * 4
        for b in range(blocks):
            shapes += [(width, cin, 1, 1), (width,), (width,),
                       (width, width, 3, 3), (width,), (width,),
                       (out, width, 1, 1), (out,), (out,)]
            if b == 0:
                shapes += [(out, cin, 1, 1), (out,), (out,)]
            cin = out
    return shapes + [(1000, 2048), (1000,)]


def synthetic_1b():
    """16 x 2^26 weights = 1,073,741,824."""
    return [(1 << 26,)] * 16


SETS = {"lenet": lenet, "alexnet": alexnet, "vgg16": vgg16, "resnet50": resnet50, "1b": synthetic_1b}


def shapes_of(name: str):
    return SETS[name]()


def counts_of(name: str):
    return [math.prod(s) for s in SETS[name]()]


def default_bits(name: str, bits: int | None = None):
    """Per-layer widths (bits) for a set: AlexNet's mixed widths unless `bits` given."""
    n = len(SETS[name]())
    if bits is not None:
        return [bits] * n
    if name == "alexnet":
        return list(ALEXNET_BITS)
    return [8] * n
