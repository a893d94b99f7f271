"""Host-side re-layout of reference layer parameters into the device formats.

Done once per model (``Engine.prepare``) or per layer-API call; never on the
timed path.  Every function takes reference-shaped specs (duck-typed
``LayerSpec``: ``weights`` = BinaryTensor rows, ``thresholds``, ``directions``)
and returns numpy arrays in the layouts documented in include/bnn.h:

* conv_bin filters   -> u32 (9, CW, K)  (the reference's tap-major w_cl,
  model.py:125-132, in 32-bit words, out-channel minor)
* conv_int filters   -> int8 +-1 (K, C*9) in (c, dy, dx) order (w_dense, model.py:116-119)
* fc rows            -> u32 (LW, M), columns permuted from the reference flatten
  order c*H*W + y*W + x (layers.py:149-161) to the device NHWC order
  (y*W + x)*CW*32 + c
* fc_int_out rows    -> u32 (M, LW), same permutation
* step               -> int32 thresholds (C,) and u32 direction bits
"""

from __future__ import annotations

import numpy as np

from .model import is_positive


def _row_bits(t) -> np.ndarray:
    n = int(np.prod(t.dims))
    by = np.ascontiguousarray(np.asarray(t.words, dtype="<u8")).view(np.uint8)
    return np.unpackbits(by, bitorder="little")[:n]


def weight_bits(layer) -> np.ndarray:
    """(rows, *row_dims) uint8 0/1."""
    return np.stack([_row_bits(t).reshape(t.dims) for t in layer.weights]).astype(np.uint8)


def pack_u32(bits: np.ndarray) -> np.ndarray:
    """0/1 along the last axis -> little-endian u32 words (bit i of word i//32)."""
    b = np.asarray(bits, dtype=bool)
    n = b.shape[-1]
    nw = (n + 31) // 32
    if nw * 32 != n:
        b = np.concatenate([b, np.zeros(b.shape[:-1] + (nw * 32 - n,), dtype=bool)], axis=-1)
    return np.ascontiguousarray(np.packbits(b, axis=-1, bitorder="little")).view("<u4").astype(np.uint32)


def conv_bin_weights(layer) -> np.ndarray:
    wb = weight_bits(layer)  # (K, C, 3, 3)
    K, C = wb.shape[:2]
    taps = wb.reshape(K, C, 9).transpose(2, 0, 1)  # (9, K, C)
    words = pack_u32(taps)  # (9, K, CW)
    return np.ascontiguousarray(words.transpose(0, 2, 1))  # (9, CW, K)


def conv_first_weights(layer) -> np.ndarray:
    wb = weight_bits(layer)  # (K, C, 3, 3)
    return np.ascontiguousarray((wb.reshape(wb.shape[0], -1).astype(np.int8) * 2 - 1))


def flatten_permutation(src_shape) -> tuple[np.ndarray, int]:
    """Reference flat column l -> device bit position, and the device words per row.

    ``src_shape`` = (C, H, W) of the NHWC activation being flattened, or (L,)
    for an already 1-D activation (identity order).
    """
    if len(src_shape) == 1:
        L = int(src_shape[0])
        return np.arange(L), (L + 31) // 32
    C, H, W = (int(d) for d in src_shape)
    cw = (C + 31) // 32
    l = np.arange(C * H * W)
    c, s = l // (H * W), l % (H * W)
    return s * (cw * 32) + c, H * W * cw


def fc_device_bits(layer, src_shape) -> tuple[np.ndarray, int, int]:
    """(M, LW*32) 0/1 rows in device order, real bit count L, words per row LW."""
    wb = weight_bits(layer)  # (M, L)
    M, L = wb.shape
    perm, lw = flatten_permutation(src_shape)
    dev = np.zeros((M, lw * 32), dtype=np.uint8)
    dev[:, perm] = wb
    return dev, L, lw


def fc_weights(layer, src_shape) -> tuple[np.ndarray, int, int]:
    dev, L, lw = fc_device_bits(layer, src_shape)
    return np.ascontiguousarray(pack_u32(dev).T), L, lw  # (LW, M)


def fc_out_weights(layer, src_shape) -> tuple[np.ndarray, int, int]:
    dev, L, lw = fc_device_bits(layer, src_shape)
    return pack_u32(dev), L, lw  # (M, LW)


def step_params(thresholds, directions) -> tuple[np.ndarray, np.ndarray]:
    thr = np.ascontiguousarray(np.asarray(thresholds.values if hasattr(thresholds, "values") else thresholds)
                               .reshape(-1).astype(np.int32))
    pos = np.array([is_positive(d) if not isinstance(d, (bool, np.bool_)) else bool(d) for d in directions])
    return thr, pack_u32(pos[None, :])[0]


def posbits_from_bool(pos) -> np.ndarray:
    return pack_u32(np.asarray(pos, dtype=bool)[None, :])[0]


# ----------------------------------------------------------------- tensor-engine (FP4 +-1) layouts
# The tensor engine's operands are E2M1 codes, +1 = 0x2, -1 = 0xA, two per byte, element 2i in the
# low nibble (include/bnn.h "NHWC f4"): a binary dot product is an exact block-scaled FP4 MMA.

F4_POS, F4_NEG = 0x2, 0xA


def pack_f4(bits01: np.ndarray) -> np.ndarray:
    """0/1 array (..., L), L even -> uint8 (..., L/2) of E2M1 +1/-1 nibbles (element 2i low)."""
    b = np.asarray(bits01, dtype=np.uint8)
    nib = np.where(b != 0, F4_POS, F4_NEG).astype(np.uint8)
    return np.ascontiguousarray(nib[..., 0::2] | (nib[..., 1::2] << 4))


def unpack_f4(packed: np.ndarray) -> np.ndarray:
    """uint8 (..., L/2) FP4 -> 0/1 (..., L): 1 where the nibble is +1 (0x2)."""
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty(p.shape[:-1] + (2 * p.shape[-1],), dtype=np.uint8)
    out[..., 0::2] = (p & 0xF) == F4_POS
    out[..., 1::2] = (p >> 4) == F4_POS
    return out


def fold_directions(packed: np.ndarray, flip) -> np.ndarray:
    """Direction folding for a fused step: negate (E2M1 sign flip) the filter rows of POS channels,
    so the accumulator is -v for POS and +v for NEG and the step is one add + sign (include/bnn.h)."""
    if flip is None:
        return packed
    out = packed.copy()
    out[np.asarray(flip, dtype=bool)] ^= 0x88
    return out


def conv_tc_weights(layer, flip=None) -> np.ndarray:
    """FP4 +-1 (K, 9*C/2 bytes), element t*C + c with t = dy*3 + dx (tap-major K for the TMA tap boxes);
    ``flip``: per-output-channel POS flags of the fused step (rows negated), or None."""
    wb = weight_bits(layer)  # (K, C, 3, 3)
    K, C = wb.shape[:2]
    taps = wb.reshape(K, C, 9).transpose(0, 2, 1).reshape(K, 9 * C)
    return fold_directions(pack_f4(taps), flip)


def flatten_permutation_i8(src_shape) -> np.ndarray:
    """Reference flat column l -> element position in the NHWC row ((y*W + x)*C + c)."""
    if len(src_shape) == 1:
        return np.arange(int(src_shape[0]))
    C, H, W = (int(d) for d in src_shape)
    l = np.arange(C * H * W)
    c, s = l // (H * W), l % (H * W)
    return s * C + c


def fc_tc_weights(layer, src_shape, flip=None) -> np.ndarray:
    """FP4 +-1 (M, L/2 bytes) with elements in the device NHWC order (``flip`` as conv_tc_weights)."""
    wb = weight_bits(layer)  # (M, L)
    dev = np.empty_like(wb, dtype=np.uint8)
    dev[:, flatten_permutation_i8(src_shape)] = wb
    return fold_directions(pack_f4(dev), flip)


# ----------------------------------------------------------------- step rows (the step as one MMA)
STEP_ROWS_MAX_KRED = 1600  # accumulated products per output for which every c_n is representable
# the constant A block of the step MMA: per 32-element half, 6.0 at elements 0-23, 0.5 at 24-31
STEP_A_VALUES = np.array(([6.0] * 24 + [0.5] * 8) * 2)
_E2M1 = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6, -0.0, -0.5, -1, -1.5, -2, -3, -4, -6])


def step_rows(thr: np.ndarray, posbits: np.ndarray, kred: int) -> np.ndarray:
    """(K, 32) uint8 FP4 step rows for bnn_tc_conv's step MMA (include/bnn.h bnn_step_rows): row n
    dotted with STEP_A_VALUES is c_n = T_n + 0.5 (POS) / 0.5 - T_n (NEG), T clamped to +-(kred+1)."""
    from . import native

    thr = np.ascontiguousarray(np.asarray(thr, dtype=np.int32).reshape(-1))
    pos = np.ascontiguousarray(np.asarray(posbits, dtype=np.uint32).reshape(-1))
    out = np.zeros((thr.size, 32), dtype=np.uint8)
    rc = native.load().bnn_step_rows(thr.ctypes.data, pos.ctypes.data, thr.size, int(kred), out.ctypes.data)
    if rc != 0:
        raise ValueError(f"step rows: constant not representable for kred={kred} (rc={rc}: {native.last_error()})")
    return out


def step_rows_values(rows: np.ndarray) -> np.ndarray:
    """Decode step rows to the c_n the tensor core adds: sum_k A_k * E2M1(row nibble k)."""
    r = np.asarray(rows, dtype=np.uint8)
    nib = np.empty(r.shape[:-1] + (2 * r.shape[-1],), dtype=np.uint8)
    nib[..., 0::2], nib[..., 1::2] = r & 0xF, r >> 4
    return (_E2M1[nib] * STEP_A_VALUES).sum(axis=-1)
