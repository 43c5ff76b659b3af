"""Shared fixtures: golden data from the reference, config builders, GPU gating."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running full-size parity runs (opt-in: FDR_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("FDR_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow full-length parity run; set FDR_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN_DIR, "acoustic_golden.json"), encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(os.path.join(GOLDEN_DIR, "acoustic_golden.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda_device():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
