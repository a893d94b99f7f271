"""Shared test helpers: rebuild golden cases / calibrated models in our own types."""

from __future__ import annotations

import numpy as np

from paper_2301_05126_b200.model import LayerKind, LayerSpec, StepDirection
from paper_2301_05126_b200.synthetic import export_synthetic_model
from paper_2301_05126_b200.tensors import BinaryTensor, IntTensor


def weights_from_bits(w01: np.ndarray, row_dims) -> list:
    rows = np.asarray(w01).reshape(w01.shape[0], -1)
    return [BinaryTensor.from_bits(r, row_dims) for r in rows]


def binary_from(bits, mask=None) -> BinaryTensor:
    return BinaryTensor.from_bits(bits, bits.shape, mask)


def model_with_steps(arch: str, seed: int, steps: dict):
    """Synthetic model with the step thresholds/directions recorded in golden.json."""
    m = export_synthetic_model(arch, seed)
    for key, rec in steps.items():
        i = int(key)
        old = m.layers[i]
        thr = np.asarray(rec["thr"], dtype=np.int64)
        dirs = [StepDirection.POS if p else StepDirection.NEG for p in rec["pos"]]
        m.layers[i] = LayerSpec(LayerKind.STEP, old.in_shape, old.out_shape,
                                thresholds=IntTensor((len(thr),), thr), directions=dirs)
    return m


def trace_images(model, img_seed: int, batch: int) -> np.ndarray:
    return np.random.default_rng(img_seed).integers(0, 256, size=(batch,) + tuple(model.input.shape))
