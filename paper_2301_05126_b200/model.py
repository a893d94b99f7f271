"""Model vocabulary of the drop-in surface (reference: `bnntuner/model.py`).

Seven layer kinds chained over {-1,+1} data; convolutions are 3x3 / stride 1
/ same padding, pools are 2x2 / stride 2.  ``LayerSpec`` / ``ModelSpec`` keep
the reference's field names so reference-built specs and ours are
interchangeable (all consumers duck-type on ``kind.value``, ``in_shape``,
``out_shape``, ``weights``, ``thresholds``, ``directions``).

The reference's ``ParallelConfig`` X/Y/Z thread-partition tags
(`model.py:38-67`) are kept as vocabulary only, so that a reference caller's
assignment vector (``run_model(model, images, [ParallelConfig...], bs)``) is
validated exactly as the reference validates it (length, applicability --
`backends.py:42-44`, `:514-518`).  On the GPU their role is played by kernel
variants (``tuner.Variant``): a validated tag vector runs
the engine's default (or tuned) variants -- every layer runs on the GPU.
"""

from __future__ import annotations

import enum
import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

KERNEL = 3
PAD = 1
POOL_WINDOW = 2
POOL_STRIDE = 2


class LayerKind(enum.Enum):
    """reference: model.py:28-35 (same string values, used in files and digests)."""

    CONV_INT = "conv_int"
    CONV_BIN = "conv_bin"
    MAXPOOL = "maxpool"
    STEP = "step"
    FLATTEN = "flatten"
    FC_BIN = "fc_bin"
    FC_INT_OUT = "fc_int_out"


class ParallelConfig(enum.Enum):
    """reference: model.py:38-60 -- the eight executor tags, in the reference's tie-break order."""

    CPU = "CPU"
    X = "X"
    Y = "Y"
    Z = "Z"
    XY = "XY"
    XZ = "XZ"
    YZ = "YZ"
    XYZ = "XYZ"

    @property
    def axes(self) -> frozenset:
        return frozenset() if self is ParallelConfig.CPU else frozenset(self.value)

    @property
    def tie_rank(self) -> int:
        return list(ParallelConfig).index(self)


def applicable_configs(kind) -> tuple:
    """reference: backends.py:42-44 -- flatten is CPU-only, every other kind takes all eight."""
    return (ParallelConfig.CPU,) if _kind_value(kind) == "flatten" else tuple(ParallelConfig)


def config_of(tag) -> "ParallelConfig":
    """Our ParallelConfig for a tag from either package (duck-typed on ``.value``) or a string."""
    return ParallelConfig(tag.value if hasattr(tag, "value") else str(tag))


class StepDirection(enum.Enum):
    """reference: model.py:70-74.  POS: +1 iff v > T; NEG: +1 iff v < T (strict)."""

    POS = "pos"
    NEG = "neg"


def _kind_value(kind) -> str:
    return kind.value if hasattr(kind, "value") else str(kind)


def kind_of(layer) -> LayerKind:
    """Our LayerKind for a layer built by either package (duck-typed on ``.kind.value``)."""
    return LayerKind(_kind_value(layer.kind))


def kind_is_conv(kind) -> bool:
    return _kind_value(kind) in ("conv_int", "conv_bin")


@dataclass(eq=False)
class LayerSpec:
    """One layer (reference: model.py:77-109).

    ``weights``: one BinaryTensor per output channel ((C,3,3) filters) or per
    output neuron ((L,) rows).  ``thresholds`` (IntTensor (C,)) and
    ``directions`` belong to step layers.
    """

    kind: LayerKind
    in_shape: tuple
    out_shape: tuple
    weights: list | None = None
    thresholds: object | None = None
    directions: list | None = None
    _prepared: dict | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.in_shape = tuple(int(d) for d in self.in_shape)
        self.out_shape = tuple(int(d) for d in self.out_shape)

    @property
    def out_channels(self) -> int:
        return self.out_shape[0]


@dataclass(frozen=True)
class InputSpec:
    """reference: model.py:145-155."""

    channels: int
    rows: int
    cols: int
    element: str = "u8"

    @property
    def shape(self) -> tuple:
        return (self.channels, self.rows, self.cols)


@dataclass(eq=False)
class ModelSpec:
    """reference: model.py:158-163."""

    name: str
    input: InputSpec
    layers: list
    num_classes: int


def layer_display_name(layer) -> str:
    """Paper shorthand C64 / MP14 / S / FLAT / FC2048 (reference: model.py:166-179)."""
    k = _kind_value(layer.kind)
    if k in ("conv_int", "conv_bin"):
        return f"C{layer.out_shape[0]}"
    if k == "maxpool":
        return f"MP{layer.out_shape[1]}"
    if k == "step":
        return "S"
    if k == "flatten":
        return "FLAT"
    if k == "fc_int_out":
        return f"FC{layer.in_shape[0]}"
    return f"FC{layer.out_shape[0]}"


# --------------------------------------------------------------------------- validation

_NEEDS_BINARY = ("conv_bin", "fc_bin", "fc_int_out")
_NEEDS_INTEGER = ("conv_int", "step")
_PRODUCES_INTEGER = ("conv_int", "conv_bin", "fc_bin", "fc_int_out")


def _fully_valid(t) -> bool:
    mask = np.asarray(t.valid_mask, dtype=np.uint64)
    return int(np.bitwise_count(mask).sum(dtype=np.int64)) == math.prod(t.dims)


def _layer_problems(layer, n: int) -> list:
    k = _kind_value(layer.kind)
    ins, outs = tuple(layer.in_shape), tuple(layer.out_shape)
    out: list = []
    if k in ("conv_int", "conv_bin"):
        if len(ins) != 3 or len(outs) != 3:
            return [f"layer {n}: conv shapes must be 3-D"]
        c, h, w = ins
        if outs[1:] != (h, w):
            out.append(f"layer {n}: same-padding conv must keep spatial dims ({h}x{w})")
        ws = layer.weights
        if not ws:
            out.append(f"layer {n}: conv has no weights")
            return out
        if len(ws) != outs[0]:
            out.append(f"layer {n}: {len(ws)} filters for {outs[0]} output channels")
        want = (c, KERNEL, KERNEL)
        for i, f in enumerate(ws):
            if tuple(f.dims) != want:
                out.append(f"layer {n}: filter {i} dims {tuple(f.dims)} != {want}")
                break
        if not _fully_valid(ws[0]):
            out.append(f"layer {n}: conv weights must be fully valid")
    elif k == "maxpool":
        if len(ins) != 3:
            return [f"layer {n}: maxpool shapes must be 3-D"]
        c, h, w = ins
        if h % 2 or w % 2:
            out.append(f"layer {n}: maxpool input spatial dims must be even, got {h}x{w}")
        if outs != (c, h // 2, w // 2):
            out.append(f"layer {n}: maxpool out_shape {outs} != {(c, h // 2, w // 2)}")
    elif k == "step":
        if outs != ins:
            out.append(f"layer {n}: step must preserve shape")
        ch = ins[0]
        thr = layer.thresholds
        if thr is None or math.prod(thr.dims) != ch:
            got = None if thr is None else math.prod(thr.dims)
            out.append(f"layer {n}: step needs {ch} thresholds, got {got}")
        if layer.directions is None or len(layer.directions) != ch:
            out.append(f"layer {n}: step needs {ch} direction flags")
    elif k == "flatten":
        if len(outs) != 1 or outs[0] != math.prod(ins):
            out.append(f"layer {n}: flatten out length must be {math.prod(ins)}")
    else:
        if len(ins) != 1 or len(outs) != 1:
            return [f"layer {n}: fc shapes must be 1-D"]
        length, m = ins[0], outs[0]
        ws = layer.weights
        if not ws:
            out.append(f"layer {n}: fc has no weights")
            return out
        if len(ws) != m:
            out.append(f"layer {n}: {len(ws)} weight rows for {m} outputs")
        if any(tuple(r.dims) != (length,) for r in ws):
            out.append(f"layer {n}: fc weight rows must have dims ({length},)")
        elif not _fully_valid(ws[0]):
            out.append(f"layer {n}: fc weights must be fully valid")
    return out


def validate_model(model) -> list:
    """Every structural violation, same messages as the reference (model.py:189-292)."""
    layers = list(model.layers)
    if not layers:
        return ["model has no layers"]
    problems: list = []
    first, last = layers[0], layers[-1]
    if _kind_value(first.kind) != "conv_int":
        problems.append(f"layer 1 must be conv_int, got {_kind_value(first.kind)}")
    if tuple(first.in_shape) != tuple(model.input.shape):
        problems.append(f"layer 1 in_shape {tuple(first.in_shape)} != input shape {tuple(model.input.shape)}")
    if _kind_value(last.kind) != "fc_int_out":
        problems.append(f"last layer must be fc_int_out, got {_kind_value(last.kind)}")
    elif tuple(last.out_shape) != (model.num_classes,):
        problems.append(f"last layer out length {tuple(last.out_shape)} != num_classes {model.num_classes}")
    for i in range(1, len(layers)):
        if tuple(layers[i - 1].out_shape) != tuple(layers[i].in_shape):
            problems.append(f"shape chain broken at layer {i + 1}")
    carrier = "int"
    for idx, layer in enumerate(layers):
        n = idx + 1
        k = _kind_value(layer.kind)
        problems.extend(_layer_problems(layer, n))
        if k == "conv_int" and idx != 0:
            problems.append(f"layer {n}: conv_int allowed only as layer 1")
        if k == "fc_int_out" and idx != len(layers) - 1:
            problems.append(f"layer {n}: fc_int_out allowed only as the last layer")
        if k in _NEEDS_BINARY and carrier != "bin":
            problems.append(f"layer {n}: {k} needs binary input but gets integer")
        if k in _NEEDS_INTEGER and carrier != "int":
            problems.append(f"layer {n}: {k} needs integer input but gets binary")
        if k in _PRODUCES_INTEGER:
            carrier = "int"
        elif k == "step":
            carrier = "bin"
    return problems


# --------------------------------------------------------------------------- digest

def model_digest(model) -> str:
    """SHA-256 over the canonical byte stream of `model.py:298-320`.

    Header tag, name, input shape + class count as <i8, then per layer: kind
    tag + NUL, shapes as <i8, raw <u8 weight words, <i4 thresholds and one
    direction letter per channel.  Plans bind to this value.
    """
    h = hashlib.sha256(b"bnntuner-model-v1\x00")
    h.update(str(model.name).encode())
    head = tuple(model.input.shape) + (int(model.num_classes),)
    h.update(np.asarray(head, dtype="<i8").tobytes())
    for layer in model.layers:
        h.update(_kind_value(layer.kind).encode() + b"\x00")
        h.update(np.asarray(layer.in_shape, dtype="<i8").tobytes())
        h.update(np.asarray(layer.out_shape, dtype="<i8").tobytes())
        if layer.weights is not None:
            for w in layer.weights:
                h.update(np.asarray(w.words, dtype=np.uint64).astype("<u8").tobytes())
        if layer.thresholds is not None:
            h.update(np.asarray(layer.thresholds.values).astype("<i4").tobytes())
            h.update("".join(_kind_value(d)[0] for d in layer.directions).encode())
    return h.hexdigest()


def is_positive(direction) -> bool:
    return _kind_value(direction) == "pos"
