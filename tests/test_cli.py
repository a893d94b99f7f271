"""The CLI (paper_2301_05126_b200/cli.py): same commands, files and exit codes as the reference's
`bnntuner` CLI (`bnntuner/cli.py`).  gen-model / validate / error paths run on CPU; tune / run /
compare need the GPU."""

import json

import numpy as np
import pytest

from paper_2301_05126_b200 import cli, modelio
from paper_2301_05126_b200.synthetic import export_synthetic_model
from paper_2301_05126_b200.tensors import IntTensor


def test_gen_model_and_validate(tmp_path, capsys):
    out = tmp_path / "f.model.json"
    assert cli.main(["gen-model", "--arch", "fashion", "--seed", "7", "--out", str(out), "--json"]) == cli.EXIT_OK
    rep = json.loads(capsys.readouterr().out)
    assert rep["model_hash"] == "104a74bf653e1d4696553918b01af18261d18b85a01f63954afea5417954bef7"
    assert cli.main(["gen-model", "--arch", "fashion", "--out", str(out)]) == cli.EXIT_IO  # exists, no --force
    capsys.readouterr()
    assert cli.main(["validate", "--model", str(out), "--json"]) == cli.EXIT_OK
    assert json.loads(capsys.readouterr().out)["valid"] is True


def test_exit_codes(tmp_path, capsys):
    good = tmp_path / "m.model.json"
    modelio.save_model(export_synthetic_model("fashion", 7), good)
    doc = json.loads(good.read_text())
    doc["format_version"] = 9
    bad = tmp_path / "v9.model.json"
    bad.write_text(json.dumps(doc))
    assert cli.main(["validate", "--model", str(bad)]) == cli.EXIT_PARSE
    doc["format_version"] = 1
    doc["layers"][1]["in_shape"] = [63, 28, 28]  # shapes no longer chain
    bad.write_text(json.dumps(doc))
    assert cli.main(["validate", "--model", str(bad)]) == cli.EXIT_VALIDATION
    assert cli.main(["validate", "--model", str(tmp_path / "missing.json")]) == cli.EXIT_IO
    with pytest.raises(SystemExit) as e:
        cli.main(["tune"])  # argparse usage error
    assert e.value.code == 2
    capsys.readouterr()


@pytest.mark.gpu
def test_tune_run_compare_on_gpu(tmp_path, capsys, golden, oracle_mod):
    """tune -> plan.json -> run on the CALIBRATED fashion model (mixed POS / NEG directions, written and
    re-read through the *.model.json format): the predictions file equals the CPU oracle's."""
    from paper_2301_05126_b200.errors import ModelHashMismatch  # noqa: F401
    from tests.helpers import model_with_steps

    cal = next(c for c in golden["calibrated"] if c["arch"] == "fashion")
    m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
    mp, dp = tmp_path / "m.model.json", tmp_path / "d.csv"
    modelio.save_model(m, mp)
    imgs = np.random.default_rng(5).integers(0, 256, size=(24, 1, 28, 28))
    labels = [int(x) for x in np.random.default_rng(6).integers(0, 10, 24)]
    modelio.save_dataset(dp, IntTensor(imgs.shape, imgs), labels)
    out = tmp_path / "out"
    args = ["--model", str(mp), "--data", str(dp), "--outpath", str(out), "--batch-lower", "0", "--batch-upper", "3",
            "--reps", "2", "--warmups", "1"]
    assert cli.main(["tune", *args, "--json"]) == cli.EXIT_OK
    rep = json.loads(capsys.readouterr().out)
    assert (out / "plan.json").exists() and (out / "profile.json").exists() and (out / "summary.md").exists()
    assert rep["chosen_batch_size"] in (1, 2, 4, 8)
    assert cli.main(["run", "--plan", str(out / "plan.json"), "--model", str(mp), "--data", str(dp),
                     "--outpath", str(out), "--json"]) == cli.EXIT_OK
    run = json.loads(capsys.readouterr().out)
    preds = [int(l.split(",")[2]) for l in (out / "predictions.csv").read_text().splitlines()[1:]]
    import paper_2301_05126_b200 as P

    _, want = oracle_mod.infer(m, imgs, route="packed")
    assert preds == [int(p) for p in want] and run["images"] == 24
    assert len(set(preds)) > 1  # informative model: the predictions depend on the image
    _, gpu_preds = P.reference_infer(m, IntTensor(imgs.shape, imgs))
    assert list(gpu_preds) == preds
    assert cli.main(["compare", *args, "--json"]) == cli.EXIT_OK
    cmp = json.loads(capsys.readouterr().out)
    assert set(cmp["measured_s"]) == {"popc-only", "tensor-only", "efficient"}
    other = tmp_path / "c.model.json"
    modelio.save_model(export_synthetic_model("fashion", 8), other)
    assert cli.main(["run", "--plan", str(out / "plan.json"), "--model", str(other), "--data", str(dp),
                     "--outpath", str(out)]) == cli.EXIT_HASH
