import json
import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: longer CPU-side test")


def pytest_collection_modifyitems(config, items):
    """``gpu`` tests are skipped (not failed) on a host without a CUDA device."""
    gpu_items = [it for it in items if it.get_closest_marker("gpu") is not None]
    if not gpu_items:
        return
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for it in gpu_items:
        it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return json.loads((REPO / "tests" / "golden" / "golden.json").read_text())


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def fashion_model():
    from paper_2301_05126_b200.synthetic import export_synthetic_model

    return export_synthetic_model("fashion", 7)


@pytest.fixture(scope="session")
def cifar_model():
    from paper_2301_05126_b200.synthetic import export_synthetic_model

    return export_synthetic_model("cifar10", 1)
