"""Deterministic single-layer parity cases shared by make_golden.py and the tests.

Each case is a plain dict of numpy arrays so that it can be turned into the
reference's objects (in make_golden.py, inside this container only) or into
ours (tests).  Shapes cover what the reference tests exercise
(`tests/conftest.py:24-51`, `tests/test_acceptance.py:132-214`): odd channel
counts (partial words), 1..11 spatial extents, masked inputs, mixed POS/NEG
step directions, v == T ties, and the real model layer shapes.
"""

from __future__ import annotations

import numpy as np


def _bits(rng, shape):
    return rng.integers(0, 2, size=shape, dtype=np.uint8)


def conv_bin_cases():
    rng = np.random.default_rng(9001)
    out = []
    shapes = [(1, 1, 1, 1, 3), (1, 2, 2, 3, 5), (2, 3, 4, 5, 7), (1, 5, 3, 11, 2),
              (2, 32, 8, 6, 6), (1, 33, 40, 5, 4), (2, 64, 64, 7, 7), (1, 70, 36, 9, 10),
              (1, 64, 32, 14, 14), (1, 128, 96, 4, 4), (1, 1, 2, 11, 11), (3, 96, 64, 3, 3)]
    for i, (B, C, K, H, W) in enumerate(shapes):
        masked = i % 3 == 1
        out.append(dict(name=f"conv_bin_{i}", B=B, C=C, K=K, H=H, W=W,
                        x=_bits(rng, (B, C, H, W)),
                        mask=_bits(rng, (B, C, H, W)) if masked else None,
                        w=_bits(rng, (K, C, 3, 3))))
    return out


def conv_int_cases():
    rng = np.random.default_rng(9002)
    out = []
    for i, (B, C, K, H, W) in enumerate([(1, 1, 8, 5, 5), (2, 3, 64, 7, 9), (1, 1, 64, 28, 28),
                                          (1, 3, 64, 32, 32), (2, 2, 33, 4, 3), (1, 4, 40, 6, 6)]):
        out.append(dict(name=f"conv_int_{i}", B=B, C=C, K=K, H=H, W=W,
                        x=rng.integers(0, 256, size=(B, C, H, W)),
                        w=_bits(rng, (K, C, 3, 3))))
    return out


def step_cases():
    rng = np.random.default_rng(9003)
    out = []
    for i, shape in enumerate([(2, 5, 3, 3), (1, 64, 14, 14), (3, 70, 2, 5), (4, 2048), (2, 33)]):
        C = shape[1]
        x = rng.integers(-40, 41, size=shape)
        thr = rng.integers(-8, 9, size=C)
        # force exact v == T ties on a few positions (strictness check)
        flat = x.reshape(shape[0], C, -1)
        flat[:, :, 0] = thr[None, :]
        out.append(dict(name=f"step_{i}", x=flat.reshape(shape), thr=thr,
                        pos=rng.integers(0, 2, size=C).astype(bool)))
    return out


def pool_cases():
    rng = np.random.default_rng(9004)
    out = []
    for i, shape in enumerate([(2, 3, 4, 6), (1, 64, 28, 28), (2, 70, 2, 2), (1, 512, 8, 8)]):
        out.append(dict(name=f"pool_int_{i}", x=rng.integers(-500, 500, size=shape)))
        out.append(dict(name=f"pool_bin_{i}", bits=_bits(rng, shape)))
    return out


def fc_cases():
    rng = np.random.default_rng(9005)
    out = []
    for i, (B, L, M) in enumerate([(1, 1, 3), (2, 63, 5), (3, 64, 64), (2, 65, 10), (1, 100, 33),
                                   (4, 3136, 70), (2, 8192, 40), (5, 2048, 10)]):
        masked = i % 3 == 2
        out.append(dict(name=f"fc_{i}", B=B, L=L, M=M, x=_bits(rng, (B, L)),
                        mask=_bits(rng, (B, L)) if masked else None, w=_bits(rng, (M, L))))
    return out


def all_cases():
    return conv_bin_cases() + conv_int_cases() + step_cases() + pool_cases() + fc_cases()


MODEL_TRACES = [
    # (arch, model seed, image seed, batch)
    ("fashion", 7, 123, 1),    # the reference golden image (tests/test_layers.py:214-220)
    ("fashion", 7, 2026, 3),
    ("cifar10", 1, 45, 1),
    ("cifar10", 1, 2026, 2),
]

CALIBRATED = [
    # (arch, model seed, calibration image seed, calib batch, calib seed, eval image seed, eval batch)
    ("fashion", 7, 77, 16, 5, 2027, 4),
    ("cifar10", 1, 78, 8, 6, 2028, 2),
]
