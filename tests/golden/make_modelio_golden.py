"""Golden digests of the reference's file formats (run in the build container, where the
reference is importable read-only from /root/reference/pkg/src):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_modelio_golden.py

Writes tests/golden/modelio.json: SHA-256 of the bytes the reference's save_model writes for both
synthetic models, and of its save_dataset output for a seeded image set, so the restated
writers/readers (paper_2301_05126_b200/modelio.py) can be checked byte for byte without the
reference at test time.
"""
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import bnntuner  # noqa: E402
from bnntuner import modelio  # noqa: E402

out = {}
with tempfile.TemporaryDirectory() as d:
    for arch, seed in (("fashion", 7), ("cifar10", 1)):
        m = modelio.export_synthetic_model(arch, seed)
        p = Path(d) / f"{arch}.model.json"
        modelio.save_model(m, p)
        out[f"{arch}_seed{seed}_model_sha256"] = hashlib.sha256(p.read_bytes()).hexdigest()
        out[f"{arch}_seed{seed}_digest"] = bnntuner.model_digest(m)
    imgs = np.random.default_rng(11).integers(0, 256, size=(3, 1, 28, 28))
    p = Path(d) / "data.csv"
    modelio.save_dataset(p, bnntuner.IntTensor(imgs.shape, imgs), [3, 1, 4])
    out["dataset_seed11_sha256"] = hashlib.sha256(p.read_bytes()).hexdigest()
Path(__file__).with_name("modelio.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
print(out)
