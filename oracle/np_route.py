"""numpy restatement of the reference's own CPU algorithm -- TEST/BASELINE INFRASTRUCTURE.

The reference computes every conv / FC as ONE float32 BLAS GEMM over
unpacked +-1 / 0 operands (`bnntuner/layers.py:70-88` im2col + ``@``,
`layers.py:164-175`), exact because all partial sums stay below 2**24.  This
module repeats that route (im2col into a (B*H*W, C*9) f32 patch matrix, one
sgemm per layer, int max-pool, strict step, first-max argmax) so that
``bench.py --impl reference`` times the same arithmetic the reference runs,
with numpy's OpenBLAS using every host core.  Binary activations go through
the same bit-packed carrier as the reference's ``BinaryTensor`` between layers
(``np.packbits`` after every step, ``np.unpackbits`` -> +-1 f32 before every
binary consumer; `tensors.py:29-52`, `layers.py:135-146`), so the per-layer
costs match too (tools/cpu_port_calibration.py times this port against
``bnntuner.reference_infer`` itself: profiles/r2_cpu_port_vs_reference.json).
It is cross-checked against ``oracle.py`` (C) and the reference golden
vectors in tests/test_oracle.py.  Only tests/ and bench.py may import it.
"""

from __future__ import annotations

import numpy as np


def _kind(layer) -> str:
    return layer.kind.value if hasattr(layer.kind, "value") else str(layer.kind)


def _dense_weights(layer) -> np.ndarray:
    """(rows, prod(row_dims)) float32 +-1 (the reference's w_dense, model.py:116-119)."""
    rows = []
    for t in layer.weights:
        n = int(np.prod(t.dims))
        by = np.ascontiguousarray(np.asarray(t.words, dtype="<u8")).view(np.uint8)
        rows.append(np.unpackbits(by, bitorder="little")[:n])
    return np.stack(rows).astype(np.float32) * 2.0 - 1.0


def _patches(x: np.ndarray) -> np.ndarray:
    """(B,C,H,W) f32 -> (B*H*W, C*9) with column order (c, dy, dx); zero halo (a strided 3x3 window
    view of the zero-padded input, materialised by the reshape -- the reference's im2col,
    layers.py:70-80)."""
    B, C, H, W = x.shape
    pad = np.zeros((B, C, H + 2, W + 2), dtype=np.float32)
    pad[:, :, 1:H + 1, 1:W + 1] = x
    win = np.lib.stride_tricks.sliding_window_view(pad, (3, 3), axis=(2, 3))  # (B, C, H, W, 3, 3)
    return win.transpose(0, 2, 3, 1, 4, 5).reshape(B * H * W, C * 9)


class PreparedModel:
    """Per-layer f32 weights computed once (the reference caches them on the spec)."""

    def __init__(self, model):
        self.model = model
        self.dense = [(_dense_weights(l) if l.weights is not None else None) for l in model.layers]
        self.thr = [
            (np.asarray(l.thresholds.values).reshape(-1),
             np.array([(d.value if hasattr(d, "value") else d) == "pos" for d in l.directions]))
            if l.thresholds is not None else None
            for l in model.layers
        ]

    def infer(self, images: np.ndarray):
        """-> (logits int32 (B,N), preds int64 (B,)) following layers.py:215-224."""
        x = np.ascontiguousarray(np.asarray(images, dtype=np.int32))  # IntTensor pixels; later int32 sums / +-1 f32
        packed = None  # a binary activation: (u64 words, dims) as the reference's BinaryTensor holds it
        for layer, wd, st in zip(self.model.layers, self.dense, self.thr):
            k = _kind(layer)
            if packed is not None and k != "flatten":  # BinaryTensor.unpack() -> +-1 (tensors.py:125-129)
                words, dims = packed
                n = int(np.prod(dims))
                bits = np.unpackbits(words.view(np.uint8), count=n, bitorder="little").reshape(dims)
                x = bits.astype(np.float32) * 2.0 - 1.0
                packed = None
            if k in ("conv_int", "conv_bin"):
                B, C, H, W = x.shape
                x = x.astype(np.float32)
                y = _patches(x) @ wd.T  # int32 sums held C-contiguous, as IntTensor does (tensors.py:203-209)
                x = np.ascontiguousarray(y.reshape(B, H, W, -1).transpose(0, 3, 1, 2).astype(np.int32))
            elif k == "maxpool":
                B, C, H, W = x.shape
                x = np.ascontiguousarray(x.reshape(B, C, H // 2, 2, W // 2, 2).max(axis=(3, 5)))
            elif k == "step":
                thr, pos = st
                shp = (1, -1) + (1,) * (x.ndim - 2)
                t, p = thr.reshape(shp), pos.reshape(shp)
                bits = np.where(p, x > t, x < t)
                # BinaryTensor.from_bits (tensors.py:97-113): little-endian bits in u64 words
                flat = np.zeros(-(-bits.size // 64) * 64, dtype=bool)
                flat[: bits.size] = bits.reshape(-1)
                packed = (np.packbits(flat, bitorder="little").view("<u8"), bits.shape)
            elif k == "flatten":
                if packed is not None:
                    packed = (packed[0], (packed[1][0], int(np.prod(packed[1][1:]))))
                else:
                    x = x.reshape(x.shape[0], -1)
            else:
                x = (x @ wd.T).astype(np.int32)
        logits = x.astype(np.int32)
        return logits, np.argmax(logits, axis=1)
