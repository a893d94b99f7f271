"""Seeded paper-shaped models and images ("same random-init binarized weights").

``export_synthetic_model`` reproduces `bnntuner/modelio.py:399-464` draw for
draw, because parity is defined on the reference's own synthetic weights:
one ``np.random.default_rng(seed)`` stream, consumed in layer order as
conv filter bits ``(K, C*9)`` u8, step thresholds
``integers(-wb, wb + 1, size=C)`` (wb = the preceding dot-product window),
fc rows ``(M, L)`` u8 and finally the logit rows ``(10, L)``.  All step
directions are POS.  tests/test_host.py checks the resulting
``model_digest`` against the digests the reference computes
(tests/golden/reference_digests.json).

``make_images`` is the reference tests' pixel convention
(`tests/test_layers.py:215-216`): default int64 ``integers(0, 256)`` draws.
"""

from __future__ import annotations

import numpy as np

from .model import InputSpec, LayerKind, LayerSpec, ModelSpec, StepDirection
from .tensors import BinaryTensor, IntTensor

ARCHITECTURES = ("fashion", "cifar10")

# (op, width) rows of the two paper networks (Tables I/II; modelio.py:383-396)
_STACKS = {
    "fashion": (
        (1, 28, 28),
        ["c64", "p", "s", "c64", "p", "s", "f", "d2048", "s", "o"],
    ),
    "cifar10": (
        (3, 32, 32),
        ["c64", "s", "c64", "p", "s", "c256", "s", "c256", "p", "s",
         "c512", "s", "c512", "p", "s", "f", "d1024", "s", "o"],
    ),
}


def _rows_as_tensors(bits: np.ndarray, dims) -> list:
    return [BinaryTensor.from_bits(row, dims) for row in bits]


def export_synthetic_model(arch: str, seed: int, num_classes: int = 10) -> ModelSpec:
    if arch not in _STACKS:
        raise ValueError(f"unknown architecture {arch!r}; choose from {ARCHITECTURES}")
    in_shape, ops = _STACKS[arch]
    rng = np.random.default_rng(seed)
    shape = tuple(in_shape)
    window = 0
    layers = []
    for idx, op in enumerate(ops):
        tag = op[0]
        if tag == "c":
            k = int(op[1:])
            c, h, w = shape
            bits = rng.integers(0, 2, size=(k, c * 9), dtype=np.uint8)
            kind = LayerKind.CONV_INT if idx == 0 else LayerKind.CONV_BIN
            layers.append(LayerSpec(kind, shape, (k, h, w), weights=_rows_as_tensors(bits, (c, 3, 3))))
            window, shape = c * 9, (k, h, w)
        elif tag == "p":
            c, h, w = shape
            layers.append(LayerSpec(LayerKind.MAXPOOL, shape, (c, h // 2, w // 2)))
            shape = (c, h // 2, w // 2)
        elif tag == "s":
            ch = shape[0]
            thr = rng.integers(-window, window + 1, size=ch)
            layers.append(LayerSpec(LayerKind.STEP, shape, shape, thresholds=IntTensor((ch,), thr),
                                    directions=[StepDirection.POS] * ch))
        elif tag == "f":
            length = int(np.prod(shape))
            layers.append(LayerSpec(LayerKind.FLATTEN, shape, (length,)))
            shape = (length,)
        elif tag == "d":
            m = int(op[1:])
            bits = rng.integers(0, 2, size=(m, shape[0]), dtype=np.uint8)
            layers.append(LayerSpec(LayerKind.FC_BIN, shape, (m,), weights=_rows_as_tensors(bits, (shape[0],))))
            window, shape = shape[0], (m,)
        else:
            bits = rng.integers(0, 2, size=(num_classes, shape[0]), dtype=np.uint8)
            layers.append(LayerSpec(LayerKind.FC_INT_OUT, shape, (num_classes,),
                                    weights=_rows_as_tensors(bits, (shape[0],))))
            shape = (num_classes,)
    return ModelSpec(name=f"{arch}-synthetic-seed{seed}", input=InputSpec(*in_shape),
                     layers=layers, num_classes=num_classes)


def make_images(model_or_shape, count: int, seed: int) -> np.ndarray:
    """(count, C, H, W) int64 pixels in 0..255 drawn like the reference tests."""
    shape = tuple(model_or_shape.input.shape) if hasattr(model_or_shape, "input") else tuple(model_or_shape)
    return np.random.default_rng(seed).integers(0, 256, size=(count,) + shape)
