"""bench.py's reference arm: the unmodified fdroof.kernel.step (baseline/_ref)
wrapped with the sponge, injection and receivers must equal the oracle (which
tests/test_oracle.py pins to the reference goldens) bit for bit, so the CPU
baseline times the same computation the GPU performs."""

import os

import numpy as np
import pytest

import bench
from oracle import acoustic as O
from paper_1608_03984_b200.synthetic import config2


@pytest.mark.parametrize("ref", [True, False])
def test_reference_stepper_matches_oracle(ref, monkeypatch):
    if ref and not os.path.isdir(os.path.join(bench.REF_DIR, "fdroof")):
        pytest.skip("baseline/_ref not installed")
    if not ref:
        monkeypatch.setattr(bench, "REF_DIR", "/nonexistent")
    cfg = config2(order=4, n_t=12, dims=(40, 36, 44))
    one, kind, _ = bench.reference_stepper(cfg, 4)
    assert kind == ("reference" if ref else "port")
    for _ in range(cfg.n_t):
        one()
    want = O.simulate(cfg)
    assert np.array_equal(one.latest(), want.latest())
