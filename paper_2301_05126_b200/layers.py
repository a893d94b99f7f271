"""The reference's single-layer API, executed on the GPU (drop-in for `bnntuner/layers.py`).

Same names, signatures, argument meaning, return types and exceptions as the
reference (`layers.py:23-224`); inputs may be the reference's own objects or
ours (duck-typed).  Each call uploads its operands, converts the reference
bit layout to the device NHWC layout with a libbnn kernel, runs the layer
kernel and converts back -- i.e. the unfused path.  Whole-model inference
should go through ``Engine`` (fused blocks, device-resident activations);
``reference_infer`` here does exactly that.

There is no CPU fallback: every function raises ``NativeUnavailable`` when
libbnn or the GPU is missing.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import native, prep
from .errors import OddSpatialDim, ShapeMismatch
from .model import LayerKind, kind_of
from .tensors import BinaryTensor, IntTensor, num_words


@dataclass(frozen=True, eq=False)
class Activation:
    """Exactly one of a binary or an integer tensor (layers.py:23-67)."""

    binary: object = None
    integer: object = None

    def __post_init__(self):
        if (self.binary is None) == (self.integer is None):
            raise ShapeMismatch("activation must hold exactly one of binary/integer")

    @classmethod
    def of_binary(cls, t) -> "Activation":
        return cls(binary=t)

    @classmethod
    def of_integer(cls, t) -> "Activation":
        return cls(integer=t)

    @property
    def is_binary(self) -> bool:
        return self.binary is not None

    @property
    def dims(self) -> tuple:
        return tuple((self.binary if self.is_binary else self.integer).dims)

    @property
    def batch(self) -> int:
        return self.dims[0]

    @property
    def sample_shape(self) -> tuple:
        return self.dims[1:]

    def __eq__(self, other) -> bool:
        if not hasattr(other, "is_binary") or self.is_binary != other.is_binary:
            return False
        mine = self.binary if self.is_binary else self.integer
        theirs = other.binary if other.is_binary else other.integer
        return mine == theirs

    __hash__ = None


class LayerTimer:
    """overhead = wall time of the call minus kernel time; compute = CUDA-event kernel time."""

    def __init__(self, torch):
        self.torch = torch
        self.overhead_ns = 0
        self.compute_ns = 0
        self._events = []
        self._t0 = None

    def start(self):
        self._t0 = time.perf_counter_ns()

    def kernel(self):
        t = self.torch
        a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        self._events.append((a, b))
        return a, b

    def stop(self):
        self.torch.cuda.synchronize()
        wall = time.perf_counter_ns() - self._t0
        comp = int(sum(a.elapsed_time(b) for a, b in self._events) * 1e6)
        self.compute_ns += comp
        self.overhead_ns += max(0, wall - comp)
        self._events.clear()


class _NoTimer:
    def start(self):
        pass

    def kernel(self):
        return None, None

    def stop(self):
        pass


def _torch():
    import torch

    native.device_ready()
    return torch


def _dev_words(torch, words) -> "torch.Tensor":
    a = np.ascontiguousarray(np.asarray(words, dtype=np.uint64)).view(np.int64)
    if a.size == 0:
        a = np.zeros(1, dtype=np.int64)
    return torch.from_numpy(a).cuda()


def _to_nhwc(torch, lib, words, B, C, H, W, st):
    out = torch.empty((B * H * W * ((C + 31) // 32) + 1,), dtype=torch.int32, device="cuda")
    native.check(lib.bnn_bits_ref_to_nhwc(native.ptr(_dev_words(torch, words)), B, C, H, W, native.ptr(out), st),
                 "ref_to_nhwc")
    return out


def _from_nhwc(torch, lib, nhwc, B, C, H, W, st) -> np.ndarray:
    nw = num_words(B * C * H * W)
    out = torch.empty((max(nw, 1),), dtype=torch.int64, device="cuda")
    native.check(lib.bnn_bits_nhwc_to_ref(native.ptr(nhwc), B, C, H, W, native.ptr(out), st), "nhwc_to_ref")
    return out.cpu().numpy().view(np.uint64)[:nw]


def _run(timer, fn):
    a, b = timer.kernel()
    if a is not None:
        a.record()
    fn()
    if b is not None:
        b.record()


class _Rows:
    """Minimal layer stand-in for prep.* (weights only)."""

    def __init__(self, weights):
        self.weights = weights


def _fully_valid(t) -> bool:
    return int(np.bitwise_count(np.asarray(t.valid_mask, np.uint64)).sum()) == math.prod(t.dims)


# --------------------------------------------------------------------------- layer functions


def conv_int_forward(inp, weights, out_channels: int, w_dense=None, *, timer=None, variant=None):
    """First-layer conv: integer pixels x +-1 filters (layers.py:91-101)."""
    if len(inp.dims) != 4:
        raise ShapeMismatch(f"conv input must be (B,C,H,W), got {tuple(inp.dims)}")
    B, C, H, W = inp.dims
    if len(weights) != out_channels or any(tuple(f.dims) != (C, 3, 3) for f in weights):
        raise ShapeMismatch(f"weights do not fit input {tuple(inp.dims)}")
    torch = _torch()
    lib = native.load()
    timer = timer or _NoTimer()
    timer.start()
    vals = np.asarray(inp.values)
    small = vals.size == 0 or (vals.min() >= 0 and vals.max() <= 255)
    x = torch.from_numpy(np.ascontiguousarray(vals.astype(np.uint8 if small else np.int32))).cuda()
    w = torch.from_numpy(prep.conv_first_weights(_Rows(weights))).cuda()
    out = torch.empty((B, out_channels, H, W), dtype=torch.int32, device="cuda")
    st = native.stream_handle()
    _run(timer, lambda: native.check(lib.bnn_conv_first(
        native.ptr(x), 1 if small else 0, B, C, H, W, native.ptr(w), out_channels, None, None, 0, native.OUT_BITS,
        None, native.ptr(out), st), "conv_int"))
    res = out.cpu().numpy()
    timer.stop()
    return IntTensor(res.shape, res)


def conv_bin_forward(inp, weights, out_channels: int, w_dense=None, *, timer=None, variant=None):
    """Binary conv with masked borders (layers.py:104-115): int32 pre-activations."""
    if len(inp.dims) != 4:
        raise ShapeMismatch(f"conv input must be (B,C,H,W), got {tuple(inp.dims)}")
    B, C, H, W = inp.dims
    if len(weights) != out_channels or any(tuple(f.dims) != (C, 3, 3) for f in weights):
        raise ShapeMismatch(f"weights do not fit input {tuple(inp.dims)}")
    torch = _torch()
    lib = native.load()
    timer = timer or _NoTimer()
    timer.start()
    st = native.stream_handle()
    x = _to_nhwc(torch, lib, inp.words, B, C, H, W, st)
    full = _fully_valid(inp)
    m = None if full else _to_nhwc(torch, lib, inp.valid_mask, B, C, H, W, st)
    out = torch.empty((B, out_channels, H, W), dtype=torch.int32, device="cuda")
    v = variant if isinstance(variant, native.Variant) else None
    if v is not None and v.engine == native.ENGINE_TC and full and C % 64 == 0 and W <= 128:
        xi = torch.empty((B * H * W * C // 2,), dtype=torch.uint8, device="cuda")
        native.check(lib.bnn_bits_to_f4(native.ptr(x), B * H * W, C, native.ptr(xi), st), "bits_to_f4")
        w = torch.from_numpy(prep.conv_tc_weights(_Rows(weights))).cuda()
        _run(timer, lambda: native.check(lib.bnn_tc_conv(
            native.ptr(xi), B, C, H, W, native.ptr(w), out_channels, None, None, 0, native.OUT_BITS, None,
            native.ptr(out), v, st), "tc_conv"))
    else:
        w = torch.from_numpy(prep.conv_bin_weights(_Rows(weights)).view(np.int32)).cuda()
        pv = v if (v is not None and v.engine == native.ENGINE_POPC) else None  # TC not applicable: popc default
        _run(timer, lambda: native.check(lib.bnn_conv_bin(
            native.ptr(x), native.ptr(m), B, C, H, W, native.ptr(w), out_channels, None, None, 0, native.OUT_BITS,
            None, native.ptr(out), pv, st), "conv_bin"))
    res = out.cpu().numpy()
    timer.stop()
    return IntTensor(res.shape, res)


def maxpool_forward(act, *, timer=None):
    """2x2 / stride-2 max; binary = OR of bits (layers.py:118-132)."""
    dims = tuple(act.dims)
    if len(dims) != 4:
        raise ShapeMismatch(f"maxpool input must be (B,C,H,W), got {dims}")
    B, C, H, W = dims
    if H % 2 or W % 2:
        raise OddSpatialDim(f"maxpool needs even spatial dims, got {H}x{W}")
    torch = _torch()
    lib = native.load()
    timer = timer or _NoTimer()
    timer.start()
    st = native.stream_handle()
    if act.is_binary:
        x = _to_nhwc(torch, lib, act.binary.words, B, C, H, W, st)
        out = torch.empty((B * (H // 2) * (W // 2) * ((C + 31) // 32) + 1,), dtype=torch.int32, device="cuda")
        _run(timer, lambda: native.check(lib.bnn_maxpool_bits_nhwc(native.ptr(x), B, C, H, W, native.ptr(out), st),
                                         "maxpool_bits"))
        words = _from_nhwc(torch, lib, out, B, C, H // 2, W // 2, st)
        timer.stop()
        shape = (B, C, H // 2, W // 2)
        from .tensors import full_mask

        return Activation.of_binary(BinaryTensor(shape, words, full_mask(math.prod(shape))))
    x = torch.from_numpy(np.ascontiguousarray(np.asarray(act.integer.values, dtype=np.int32))).cuda()
    out = torch.empty((B, C, H // 2, W // 2), dtype=torch.int32, device="cuda")
    _run(timer, lambda: native.check(lib.bnn_maxpool_int(native.ptr(x), B, C, H, W, native.ptr(out), st),
                                     "maxpool_int"))
    res = out.cpu().numpy()
    timer.stop()
    return Activation.of_integer(IntTensor(res.shape, res))


def step_forward(inp, thresholds, positive, *, timer=None):
    """Per-channel strict threshold (layers.py:135-146) -> BinaryTensor."""
    vals = np.asarray(inp.values)
    C = vals.shape[1]
    thr = np.asarray(thresholds.values if hasattr(thresholds, "values") else thresholds).reshape(-1)
    pos = np.asarray(positive).reshape(-1)
    if thr.shape[0] != C or pos.shape[0] != C:
        raise ShapeMismatch(f"{thr.shape[0]} thresholds / {pos.shape[0]} flags for {C} channels")
    torch = _torch()
    lib = native.load()
    timer = timer or _NoTimer()
    timer.start()
    B = vals.shape[0]
    S = int(np.prod(vals.shape[2:])) if vals.ndim > 2 else 1
    x = torch.from_numpy(np.ascontiguousarray(vals.astype(np.int32))).cuda()
    t = torch.from_numpy(np.ascontiguousarray(thr.astype(np.int32))).cuda()
    p = torch.from_numpy(prep.posbits_from_bool(pos.astype(bool)).view(np.int32)).cuda()
    nw = num_words(vals.size)
    out = torch.empty((max(nw, 1),), dtype=torch.int64, device="cuda")
    st = native.stream_handle()
    _run(timer, lambda: native.check(lib.bnn_step_ref(native.ptr(x), B, C, S, native.ptr(t), native.ptr(p),
                                                      native.ptr(out), st), "step"))
    words = out.cpu().numpy().view(np.uint64)[:nw]
    timer.stop()
    from .tensors import full_mask

    return BinaryTensor(vals.shape, words, full_mask(vals.size))


def flatten_forward(act, *, timer=None):
    """(B,C,H,W) -> (B, C*H*W), c-major; a relabelling of the same words (layers.py:149-161)."""
    b = act.batch
    length = math.prod(act.sample_shape)
    if act.is_binary:
        return Activation.of_binary(act.binary.with_dims((b, length)))
    return Activation.of_integer(act.integer.with_dims((b, length)))


def fc_forward(inp, weights, w_dense=None, *, timer=None, variant=None):
    """out[b, m] = masked +-1 dot of input row b with weight row m (layers.py:164-175)."""
    if len(inp.dims) != 2:
        raise ShapeMismatch(f"fc input must be (B, L), got {tuple(inp.dims)}")
    B, L = inp.dims
    if any(tuple(r.dims) != (L,) for r in weights):
        raise ShapeMismatch(f"fc weights expect L={weights[0].dims[0]}, input has L={L}")
    M = len(weights)
    torch = _torch()
    lib = native.load()
    timer = timer or _NoTimer()
    timer.start()
    st = native.stream_handle()
    x = _to_nhwc(torch, lib, inp.words, B, L, 1, 1, st)
    full = _fully_valid(inp)
    m = None if full else _to_nhwc(torch, lib, inp.valid_mask, B, L, 1, 1, st)
    out = torch.empty((B, M), dtype=torch.int32, device="cuda")
    v = variant if isinstance(variant, native.Variant) else None
    if v is not None and v.engine == native.ENGINE_TC and full and L % 64 == 0:
        xi = torch.empty((B * L // 2,), dtype=torch.uint8, device="cuda")
        native.check(lib.bnn_bits_to_f4(native.ptr(x), B, L, native.ptr(xi), st), "bits_to_f4")
        w = torch.from_numpy(prep.fc_tc_weights(_Rows(weights), (L,))).cuda()
        _run(timer, lambda: native.check(lib.bnn_tc_fc(
            native.ptr(xi), B, L, native.ptr(w), M, None, None, native.OUT_BITS, None, native.ptr(out), None, v, st),
            "tc_fc"))
    else:
        wt, L_, lw = prep.fc_weights(_Rows(weights), (L,))
        w = torch.from_numpy(wt.view(np.int32)).cuda()
        pv = v if (v is not None and v.engine == native.ENGINE_POPC) else None  # TC not applicable: popc default
        _run(timer, lambda: native.check(lib.bnn_fc_bin(
            native.ptr(x), native.ptr(m), B, L, lw, native.ptr(w), M, None, None, native.OUT_BITS, None,
            native.ptr(out), pv, st), "fc"))
    res = out.cpu().numpy()
    timer.stop()
    return IntTensor(res.shape, res)


def layer_forward(layer, act, *, timer=None, variant=None):
    """Apply one layer (layers.py:178-212), same carrier checks and errors."""
    if tuple(act.sample_shape) != tuple(layer.in_shape):
        raise ShapeMismatch(
            f"{kind_of(layer).value} expects sample shape {tuple(layer.in_shape)}, got {tuple(act.sample_shape)}")
    k = kind_of(layer)
    if k is LayerKind.CONV_INT:
        if act.is_binary:
            raise ShapeMismatch("conv_int expects an integer activation")
        return Activation.of_integer(conv_int_forward(act.integer, layer.weights, layer.out_shape[0], timer=timer))
    if k is LayerKind.CONV_BIN:
        if not act.is_binary:
            raise ShapeMismatch("conv_bin expects a binary activation")
        return Activation.of_integer(conv_bin_forward(act.binary, layer.weights, layer.out_shape[0], timer=timer,
                                                      variant=variant))
    if k is LayerKind.MAXPOOL:
        return maxpool_forward(act, timer=timer)
    if k is LayerKind.STEP:
        if act.is_binary:
            raise ShapeMismatch("step expects an integer activation")
        pos = np.array([(d.value if hasattr(d, "value") else d) == "pos" for d in layer.directions])
        return Activation.of_binary(step_forward(act.integer, layer.thresholds, pos, timer=timer))
    if k is LayerKind.FLATTEN:
        return flatten_forward(act)
    if not act.is_binary:
        raise ShapeMismatch(f"{k.value} expects a binary activation")
    return Activation.of_integer(fc_forward(act.binary, layer.weights, timer=timer, variant=variant))


_ENGINES: dict = {}


def reference_infer(model, batch):
    """Whole model on the GPU (fused plan); -> (IntTensor logits, list[int] preds) (layers.py:215-224)."""
    dims = tuple(batch.dims)
    if len(dims) != 4 or dims[1:] != tuple(model.input.shape):
        raise ShapeMismatch(f"batch dims {dims} do not match input {tuple(model.input.shape)}")
    from .engine import Engine

    torch = _torch()
    dev = torch.cuda.current_device()
    eng = _ENGINES.get(dev)
    if eng is None:
        eng = _ENGINES[dev] = Engine(device=dev)
    rep = eng.run_model(model, batch)
    return IntTensor(rep.logits.shape, rep.logits), list(rep.predictions)
