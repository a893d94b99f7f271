"""Model and dataset files of the reference (format v1, docs/model-format.md of `bnntuner`).

* ``*.model.json`` -- trained or synthetic BNNs: canonical JSON (sorted keys, two-space indent,
  trailing newline; save(load(x)) is byte-stable), packed weights as base64 of little-endian u64
  words per output row (`bnntuner/modelio.py:60-177`).  Loading validates the structure with the
  same rules and messages as the reference (`model.validate_model`), so a model the reference
  accepts loads here unchanged -- including NEG step directions, which the synthetic models
  never contain -- and feeds ``Engine.prepare`` / ``reference_infer`` directly.
* ``*.csv`` datasets -- one row per image, label first, raw 0..255 pixels in row-major,
  channel-major order, no header (`bnntuner/modelio.py:187-240`).  Pixels are kept as read.

Plan files are the tuner's own format v2 (``tuner.save_plan`` / ``load_plan``): the reference's
v1 plans hold X/Y/Z thread-partition tags, which have no GPU meaning.
"""

from __future__ import annotations

import base64
import json
from pathlib import Path

import numpy as np

from .errors import LabelOutOfRange, ParseError, ShapeMismatch, UnsupportedVersion, ValidationFailed
from .model import InputSpec, LayerKind, LayerSpec, ModelSpec, StepDirection, kind_of, model_digest, validate_model
from .tensors import BinaryTensor, IntTensor, full_mask, num_words

FORMAT_VERSION = 1
ARCHITECTURES = ("fashion", "cifar10")


def _canonical(doc: dict) -> str:
    return json.dumps(doc, sort_keys=True, indent=2) + "\n"


def _read_json(path) -> dict:
    try:
        return json.loads(Path(path).read_text())
    except json.JSONDecodeError as e:
        raise ParseError(f"{path}: line {e.lineno}: {e.msg}") from e


def _require_version(doc: dict, source) -> None:
    if doc.get("format_version") != FORMAT_VERSION:
        raise UnsupportedVersion(f"{source}: format_version {doc.get('format_version')!r}, expected {FORMAT_VERSION}")


# ----------------------------------------------------------------------------- model


def _rows_b64(rows) -> str:
    """Concatenated little-endian u64 words of every weight row, base64."""
    return base64.b64encode(b"".join(np.asarray(r.words, dtype="<u8").tobytes() for r in rows)).decode("ascii")


def _rows_from_b64(rec: dict, n: int, rows: int, bits: int, dims: tuple) -> list:
    try:
        blob = base64.b64decode(rec["weights_b64"], validate=True)
    except Exception as e:  # binascii.Error, KeyError, TypeError
        raise ParseError(f"layer {n}: bad base64 weight blob: {e}") from e
    per_row = num_words(bits)
    if len(blob) != rows * per_row * 8:
        raise ValidationFailed([f"blob length mismatch layer {n}"])
    words = np.frombuffer(blob, dtype="<u8").astype(np.uint64).reshape(rows, per_row)
    mask = full_mask(bits)
    return [BinaryTensor(dims, words[r], mask) for r in range(rows)]


def model_to_doc(model) -> dict:
    layers = []
    for layer in model.layers:
        kind = kind_of(layer)
        rec = {"kind": kind.value, "in_shape": [int(d) for d in layer.in_shape],
               "out_shape": [int(d) for d in layer.out_shape]}
        if kind in (LayerKind.CONV_INT, LayerKind.CONV_BIN):
            rec.update(out_channels=int(layer.out_shape[0]), kernel=3, pad=1, weights_b64=_rows_b64(layer.weights))
        elif kind in (LayerKind.FC_BIN, LayerKind.FC_INT_OUT):
            rec["weights_b64"] = _rows_b64(layer.weights)
        elif kind is LayerKind.MAXPOOL:
            rec.update(window=2, stride=2)
        elif kind is LayerKind.STEP:
            rec["thresholds"] = [int(t) for t in np.asarray(layer.thresholds.values).reshape(-1)]
            rec["directions"] = [getattr(d, "value", d) for d in layer.directions]
        layers.append(rec)
    inp = model.input
    return {"format_version": FORMAT_VERSION, "name": model.name,
            "input": {"channels": int(inp.channels), "rows": int(inp.rows), "cols": int(inp.cols),
                      "element": getattr(inp, "element", "u8")},
            "num_classes": int(model.num_classes), "layers": layers}


def _layer_from_record(rec: dict, n: int) -> LayerSpec:
    try:
        kind = LayerKind(rec["kind"])
    except (KeyError, ValueError) as e:
        raise ParseError(f"layer {n}: unknown or missing kind {rec.get('kind')!r}") from e
    try:
        ins = tuple(int(d) for d in rec["in_shape"])
        outs = tuple(int(d) for d in rec["out_shape"])
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"layer {n}: bad shapes") from e
    if kind in (LayerKind.CONV_INT, LayerKind.CONV_BIN):
        if rec.get("kernel", 3) != 3 or rec.get("pad", 1) != 1:
            raise ParseError(f"layer {n}: only kernel=3 pad=1 convolutions are supported")
        if len(ins) != 3 or len(outs) != 3:
            raise ParseError(f"layer {n}: conv shapes must be 3-D")
        return LayerSpec(kind, ins, outs, weights=_rows_from_b64(rec, n, outs[0], ins[0] * 9, (ins[0], 3, 3)))
    if kind in (LayerKind.FC_BIN, LayerKind.FC_INT_OUT):
        if len(ins) != 1 or len(outs) != 1:
            raise ParseError(f"layer {n}: fc shapes must be 1-D")
        return LayerSpec(kind, ins, outs, weights=_rows_from_b64(rec, n, outs[0], ins[0], (ins[0],)))
    if kind is LayerKind.MAXPOOL:
        if rec.get("window", 2) != 2 or rec.get("stride", 2) != 2:
            raise ParseError(f"layer {n}: only window=2 stride=2 maxpool is supported")
        return LayerSpec(kind, ins, outs)
    if kind is LayerKind.STEP:
        try:
            thr = np.array(rec["thresholds"], dtype=np.int64)
            dirs = [StepDirection(d) for d in rec["directions"]]
        except (KeyError, TypeError, ValueError) as e:
            raise ParseError(f"layer {n}: bad step thresholds/directions") from e
        return LayerSpec(kind, ins, outs, thresholds=IntTensor((len(thr),), thr), directions=dirs)
    return LayerSpec(kind, ins, outs)


def model_from_doc(doc: dict, source: str = "<doc>") -> ModelSpec:
    _require_version(doc, source)
    try:
        inp = doc["input"]
        model = ModelSpec(str(doc["name"]),
                          InputSpec(int(inp["channels"]), int(inp["rows"]), int(inp["cols"]), str(inp.get("element", "u8"))),
                          [_layer_from_record(r, i + 1) for i, r in enumerate(doc["layers"])],
                          int(doc["num_classes"]))
    except (KeyError, TypeError) as e:
        raise ParseError(f"{source}: missing or malformed field: {e}") from e
    problems = validate_model(model)
    if problems:
        raise ValidationFailed(problems)
    return model


def save_model(model, path) -> None:
    Path(path).write_text(_canonical(model_to_doc(model)))


def load_model(path) -> ModelSpec:
    return model_from_doc(_read_json(path), source=str(path))


def model_hash(model) -> str:
    return model_digest(model)


# ----------------------------------------------------------------------------- dataset


def load_dataset(path, expected_shape, num_classes: int):
    """CSV ``label, pixel*`` rows -> (IntTensor images (N, C, H, W), labels list)."""
    c, h, w = (int(d) for d in expected_shape)
    npix = c * h * w
    images, labels = [], []
    with open(path) as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            fields = line.split(",")
            if len(fields) != 1 + npix:
                raise ParseError(f"{path}: row {lineno}: expected {1 + npix} fields, got {len(fields)}")
            try:
                vals = np.array(fields, dtype=np.int64)
            except ValueError as e:
                raise ParseError(f"{path}: row {lineno}: non-integer field: {e}") from e
            if not 0 <= vals[0] < num_classes:
                raise LabelOutOfRange(f"{path}: row {lineno}: label {int(vals[0])} outside 0..{num_classes - 1}")
            px = vals[1:]
            if px.size and (px.min() < 0 or px.max() > 255):
                raise ParseError(f"{path}: row {lineno}: pixel outside 0..255")
            labels.append(int(vals[0]))
            images.append(px)
    n = len(images)
    data = np.array(images, dtype=np.int32).reshape(n, c, h, w) if n else np.zeros((0, c, h, w), np.int32)
    return IntTensor((n, c, h, w), data), labels


def save_dataset(path, images, labels) -> None:
    vals = np.asarray(images.values if hasattr(images, "values") else images)
    n = vals.shape[0]
    if len(labels) != n:
        raise ShapeMismatch(f"{len(labels)} labels for {n} images")
    flat = vals.reshape(n, -1)
    with open(path, "w") as f:
        for i in range(n):
            f.write(",".join([str(int(labels[i]))] + [str(int(v)) for v in flat[i]]) + "\n")
