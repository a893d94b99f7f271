"""Pin the CPU oracle (both C routes + the numpy f32 route) to the reference's outputs.

Every expected value here was produced by running the reference itself
(tests/golden/make_golden.py); nothing is re-derived from the oracle.
"""

import numpy as np
import pytest

from oracle import np_route
from oracle.oracle import Act, digest
from tests.golden import cases
from tests.helpers import model_with_steps, trace_images


def _case_act(oracle_mod, c, route):
    n = c["name"]
    if n.startswith("conv_bin"):
        a = Act("bin", bits=c["x"], mask=c["mask"])
        layer = type("L", (), {})()
        if route == "packed" and c["mask"] is None:
            return Act("int", vals=oracle_mod.conv3_packed(c["x"], c["w"]))
        x = c["x"].astype(np.int32) * 2 - 1
        if c["mask"] is not None:
            x = x * c["mask"]
        return Act("int", vals=oracle_mod.conv3(x, c["w"]))
    if n.startswith("conv_int"):
        return Act("int", vals=oracle_mod.conv3(c["x"], c["w"]))
    if n.startswith("step"):
        return Act("bin", bits=oracle_mod.step(c["x"], c["thr"], c["pos"]))
    if n.startswith("pool_int"):
        return Act("int", vals=oracle_mod.maxpool_int(c["x"]))
    if n.startswith("pool_bin"):
        return Act("bin", bits=oracle_mod.maxpool_bits(c["bits"]))
    if n.startswith("fc"):
        if route == "packed" and c["mask"] is None:
            return Act("int", vals=oracle_mod.fc_packed(c["x"], c["w"]))
        x = c["x"].astype(np.int8) * 2 - 1
        if c["mask"] is not None:
            x = x * c["mask"].astype(np.int8)
        return Act("int", vals=oracle_mod.fc(x, c["w"]))
    raise KeyError(n)


@pytest.mark.parametrize("route", ["direct", "packed"])
def test_oracle_layer_cases_match_reference(oracle_mod, golden, route):
    for c in cases.all_cases():
        got = digest(_case_act(oracle_mod, c, route))
        assert got == golden["cases"][c["name"]], c["name"]


def test_oracle_reference_golden_vector(oracle_mod, golden, fashion_model):
    """The reference's own golden file (pkg/tests/golden/fashion_seed7_logits.json)."""
    ref = golden["reference_golden_fashion_seed7"]
    images = np.random.default_rng(123).integers(0, 256, size=(1, 1, 28, 28))
    for route in ("direct", "packed"):
        logits, preds = oracle_mod.infer(fashion_model, images, route=route)
        assert logits.tolist() == [ref["logits"]]
        assert preds.tolist() == ref["predictions"]


@pytest.mark.parametrize("route", ["direct", "packed"])
def test_oracle_model_traces_match_reference(oracle_mod, golden, route):
    from paper_2301_05126_b200.synthetic import export_synthetic_model

    for tr in golden["traces"]:
        m = export_synthetic_model(tr["arch"], tr["seed"])
        imgs = trace_images(m, tr["img_seed"], tr["batch"])
        logits, preds, acts = oracle_mod.infer(m, imgs, route=route, keep=True)
        assert [digest(a) for a in acts] == tr["layer_digests"], (tr["arch"], tr["img_seed"])
        assert logits.tolist() == tr["logits"]
        assert preds.tolist() == tr["preds"]


def test_oracle_calibrated_models_match_reference(oracle_mod, golden):
    for cal in golden["calibrated"]:
        m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
        imgs = trace_images(m, cal["img_seed"], cal["batch"])
        logits, preds, acts = oracle_mod.infer(m, imgs, route="packed", keep=True)
        assert [digest(a) for a in acts] == cal["layer_digests"]
        assert logits.tolist() == cal["logits"]
        assert preds.tolist() == cal["preds"]


def test_calibration_is_reproducible(oracle_mod, golden):
    """Rebuilding the calibrated thresholds from seeds gives the recorded ones."""
    from paper_2301_05126_b200.synthetic import export_synthetic_model, make_images

    for (arch, seed, cimg, cb, cseed, _, _), cal in zip(cases.CALIBRATED, golden["calibrated"]):
        base = export_synthetic_model(arch, seed)
        m = oracle_mod.calibrated_model(base, make_images(base, cb, cimg), cseed)
        for key, rec in cal["steps"].items():
            layer = m.layers[int(key)]
            assert np.asarray(layer.thresholds.values).tolist() == rec["thr"]
            assert [d.value == "pos" for d in layer.directions] == rec["pos"]


def test_calibrated_models_are_input_dependent(oracle_mod, golden):
    """The stress models exist because the shipped ones saturate."""
    for cal in golden["calibrated"]:
        m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
        imgs = trace_images(m, 31337, 16)
        logits, _ = oracle_mod.infer(m, imgs, route="packed")
        assert len({tuple(r) for r in logits.tolist()}) > 8


def test_numpy_f32_route_matches_reference(golden):
    from paper_2301_05126_b200.synthetic import export_synthetic_model

    for tr in golden["traces"]:
        m = export_synthetic_model(tr["arch"], tr["seed"])
        logits, preds = np_route.PreparedModel(m).infer(trace_images(m, tr["img_seed"], tr["batch"]))
        assert logits.tolist() == tr["logits"]
        assert preds.tolist() == tr["preds"]
