"""Model / dataset files (format v1 of the reference, docs/model-format.md): byte-exact writers
checked against digests of the reference's own output (tests/golden/make_modelio_golden.py),
loaders checked by round trips, NEG directions and the reference's error categories."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2301_05126_b200 import modelio
from paper_2301_05126_b200.errors import LabelOutOfRange, ParseError, UnsupportedVersion, ValidationFailed
from paper_2301_05126_b200.model import StepDirection, model_digest
from paper_2301_05126_b200.synthetic import export_synthetic_model
from paper_2301_05126_b200.tensors import IntTensor

GOLD = json.loads((Path(__file__).parent / "golden" / "modelio.json").read_text())


@pytest.mark.parametrize("arch,seed", [("fashion", 7), ("cifar10", 1)])
def test_save_model_bytes_match_reference(tmp_path, arch, seed):
    m = export_synthetic_model(arch, seed)
    p = tmp_path / "m.model.json"
    modelio.save_model(m, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == GOLD[f"{arch}_seed{seed}_model_sha256"]
    back = modelio.load_model(p)
    assert model_digest(back) == GOLD[f"{arch}_seed{seed}_digest"] == model_digest(m)
    p2 = tmp_path / "again.model.json"
    modelio.save_model(back, p2)
    assert p2.read_bytes() == p.read_bytes()  # save(load(x)) is byte-stable


def test_neg_directions_round_trip(tmp_path):
    m = export_synthetic_model("fashion", 7)
    doc = modelio.model_to_doc(m)
    step = next(r for r in doc["layers"] if r["kind"] == "step")
    step["directions"] = ["neg" if i % 3 == 0 else "pos" for i in range(len(step["directions"]))]
    step["thresholds"] = [int(t) - 5 for t in step["thresholds"]]
    m2 = modelio.model_from_doc(doc)
    layer = next(l for l in m2.layers if l.kind.value == "step")
    assert layer.directions[0] is StepDirection.NEG and layer.directions[1] is StepDirection.POS
    p = tmp_path / "neg.model.json"
    modelio.save_model(m2, p)
    assert modelio.model_to_doc(modelio.load_model(p)) == doc


def test_dataset_bytes_and_round_trip(tmp_path):
    imgs = np.random.default_rng(11).integers(0, 256, size=(3, 1, 28, 28))
    p = tmp_path / "d.csv"
    modelio.save_dataset(p, IntTensor(imgs.shape, imgs), [3, 1, 4])
    assert hashlib.sha256(p.read_bytes()).hexdigest() == GOLD["dataset_seed11_sha256"]
    got, labels = modelio.load_dataset(p, (1, 28, 28), 10)
    assert labels == [3, 1, 4] and np.array_equal(got.values, imgs)
    empty = tmp_path / "e.csv"
    empty.write_text("")
    e, el = modelio.load_dataset(empty, (1, 28, 28), 10)
    assert e.dims == (0, 1, 28, 28) and el == []


def test_error_categories(tmp_path):
    m = export_synthetic_model("fashion", 7)
    doc = modelio.model_to_doc(m)
    with pytest.raises(UnsupportedVersion):
        modelio.model_from_doc({**doc, "format_version": 2})
    bad = json.loads(json.dumps(doc))
    bad["layers"][0]["weights_b64"] = bad["layers"][0]["weights_b64"][:-8]
    with pytest.raises((ValidationFailed, ParseError)):
        modelio.model_from_doc(bad)
    bad = json.loads(json.dumps(doc))
    bad["layers"][0]["kind"] = "conv_magic"
    with pytest.raises(ParseError):
        modelio.model_from_doc(bad)
    p = tmp_path / "broken.json"
    p.write_text("{not json")
    with pytest.raises(ParseError):
        modelio.load_model(p)
    d = tmp_path / "d.csv"
    d.write_text("10," + ",".join(["0"] * 784) + "\n")
    with pytest.raises(LabelOutOfRange):
        modelio.load_dataset(d, (1, 28, 28), 10)
    d.write_text("1," + ",".join(["0"] * 783) + "\n")
    with pytest.raises(ParseError):
        modelio.load_dataset(d, (1, 28, 28), 10)
    d.write_text("1," + ",".join(["256"] * 784) + "\n")
    with pytest.raises(ParseError):
        modelio.load_dataset(d, (1, 28, 28), 10)
