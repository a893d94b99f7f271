"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run inside the build container only (the GPU box has no /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``bnntuner`` read-only from /root/reference/pkg/src and records,
for every case in cases.py and every model trace, a SHA-256 of the
reference's output in its own boundary format (IntTensor values / BinaryTensor
words + mask; hashing rule = oracle.oracle.digest), plus full logits and
predictions.  The oracle is pinned against these (tests/test_oracle.py) and
the GPU path is checked against the oracle and these (tests/test_gpu_*.py).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import bnntuner as R  # noqa: E402

from paper_2301_05126_b200 import synthetic  # noqa: E402
from oracle import oracle  # noqa: E402
from tests.golden import cases  # noqa: E402


def ref_digest(obj) -> str:
    if hasattr(obj, "is_binary"):
        obj = obj.binary if obj.is_binary else obj.integer
    h = hashlib.sha256()
    if hasattr(obj, "words"):
        h.update(b"bin\0" + np.asarray(obj.dims, "<i8").tobytes())
        h.update(np.asarray(obj.words).astype("<u8").tobytes())
        h.update(np.asarray(obj.valid_mask).astype("<u8").tobytes())
    else:
        h.update(b"int\0" + np.asarray(obj.dims, "<i8").tobytes())
        h.update(np.asarray(obj.values).astype("<i4").tobytes())
    return h.hexdigest()


def ref_weights(bits01, dims_per_row):
    return [R.BinaryTensor.from_bits(r, dims_per_row) for r in bits01]


def ref_binary(bits, mask):
    return R.BinaryTensor.from_bits(bits, bits.shape, mask)


def run_case(c):
    n = c["name"]
    if n.startswith("conv_bin"):
        x = ref_binary(c["x"], c["mask"])
        w = ref_weights(c["w"].reshape(c["K"], -1), (c["C"], 3, 3))
        return R.conv_bin_forward(x, w, c["K"])
    if n.startswith("conv_int"):
        x = R.IntTensor(c["x"].shape, c["x"])
        w = ref_weights(c["w"].reshape(c["K"], -1), (c["C"], 3, 3))
        return R.conv_int_forward(x, w, c["K"])
    if n.startswith("step"):
        return R.step_forward(R.IntTensor(c["x"].shape, c["x"]), R.IntTensor(c["thr"].shape, c["thr"]),
                              np.asarray(c["pos"], dtype=bool))
    if n.startswith("pool_int"):
        return R.maxpool_forward(R.Activation.of_integer(R.IntTensor(c["x"].shape, c["x"])))
    if n.startswith("pool_bin"):
        return R.maxpool_forward(R.Activation.of_binary(R.BinaryTensor.from_bits(c["bits"], c["bits"].shape)))
    if n.startswith("fc"):
        x = ref_binary(c["x"], c["mask"])
        return R.fc_forward(x, ref_weights(c["w"], (c["L"],)))
    raise KeyError(n)


def trace(model, images):
    act = R.Activation.of_integer(R.IntTensor(images.shape, images))
    digests = []
    for layer in model.layers:
        act = R.layer_forward(layer, act)
        digests.append(ref_digest(act))
    logits, preds = R.reference_infer(model, R.IntTensor(images.shape, images))
    return digests, logits.values.tolist(), list(preds)


def main():
    out = {"generator": "tests/golden/make_golden.py (reference bnntuner, /root/reference/pkg/src)"}
    out["digests"] = {f"{a}-{s}": R.model_digest(R.export_synthetic_model(a, s))
                      for a, s in (("fashion", 7), ("cifar10", 1))}
    ref_golden = json.loads(Path("/root/reference/pkg/tests/golden/fashion_seed7_logits.json").read_text())
    out["reference_golden_fashion_seed7"] = ref_golden
    out["cases"] = {c["name"]: ref_digest(run_case(c)) for c in cases.all_cases()}

    out["traces"] = []
    for arch, seed, img_seed, batch in cases.MODEL_TRACES:
        m = R.export_synthetic_model(arch, seed)
        images = np.random.default_rng(img_seed).integers(0, 256, size=(batch,) + m.input.shape)
        d, logits, preds = trace(m, images)
        out["traces"].append(dict(arch=arch, seed=seed, img_seed=img_seed, batch=batch,
                                  layer_digests=d, logits=logits, preds=preds))

    out["calibrated"] = []
    for arch, seed, cimg, cb, cseed, eimg, eb in cases.CALIBRATED:
        ours = synthetic.export_synthetic_model(arch, seed)
        calib = oracle.calibrated_model(ours, synthetic.make_images(ours, cb, cimg), cseed)
        steps = {}
        m = R.export_synthetic_model(arch, seed)
        for i, (lo, lr) in enumerate(zip(calib.layers, m.layers)):
            if lo.thresholds is not None:
                thr = [int(t) for t in np.asarray(lo.thresholds.values).reshape(-1)]
                pos = [d.value == "pos" for d in lo.directions]
                steps[str(i)] = {"thr": thr, "pos": pos}
                lr.thresholds = R.IntTensor((len(thr),), thr)
                lr.directions = [R.StepDirection.POS if p else R.StepDirection.NEG for p in pos]
                lr._prepared = None
        images = np.random.default_rng(eimg).integers(0, 256, size=(eb,) + m.input.shape)
        d, logits, preds = trace(m, images)
        out["calibrated"].append(dict(arch=arch, seed=seed, calib=[cimg, cb, cseed], img_seed=eimg,
                                      batch=eb, steps=steps, layer_digests=d, logits=logits, preds=preds))

    path = Path(__file__).with_name("golden.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
