"""Failure paths on the GPU (failure detection).

* A multi-cluster neighbour wait that gives up is reported: the run's levels
  are NaN and the library returns FDR_ECUDA (DeviceError) from
  fdr_pending_error and from the next run on the device.
* Concurrent multi-cluster runs on different streams use separate step-flag
  slots (bit-exact results).
* The end-of-run NaN/inf check (fdr_count_nonfinite) on float32 and float64
  levels, and on a diverging (CFL-violating) run.
* In-place edits of a config's arrays after a run are refused (the cached
  device plan write-protects them; the reference re-reads cfg.m every step,
  kernel.py:188) and invalidate_plan() lets the next run see new values.
"""

import warnings

import numpy as np
import pytest

from cases import config1_case, random_levels, sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B(cuda_device):
    import paper_1608_03984_b200 as pkg
    from paper_1608_03984_b200 import _lib

    _lib.load()
    return pkg


def test_cluster_wait_timeout_is_reported(B, monkeypatch):
    import torch

    from paper_1608_03984_b200 import _lib

    lib = _lib.load()
    assert lib.fdr_pending_error() == 0
    cfg, _ = config1_case(True)
    # CTA 15 closes cluster 0 (4 clusters x 16 CTAs, one x-plane each): it
    # never publishes, so CTAs 16-17 wait ~1 ms and give up
    monkeypatch.setenv("B200FD_CLUSTERS", "4")
    monkeypatch.setenv("B200FD_TEST_STALL_CTA", "15")
    monkeypatch.setenv("B200FD_WAIT_CYCLES", "2000000")
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg, 3, variant="cluster")
    torch.cuda.synchronize()
    assert lib.fdr_pending_error() == _lib.FDR_ECUDA
    assert b"timed out" in lib.fdr_last_error()
    assert fld.nonfinite_count() > 0
    assert lib.fdr_pending_error() == 0  # reported once

    # a failure surfaces as the next run's error when nobody checked
    B.run(fld, cfg, 3, variant="cluster")
    torch.cuda.synchronize()
    monkeypatch.delenv("B200FD_TEST_STALL_CTA")
    with pytest.raises(B.DeviceError, match="timed out"):
        B.run(fld, cfg, 1, variant="cluster")
    # and the device is usable afterwards
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg, variant="cluster")
    torch.cuda.synchronize()
    assert fld.nonfinite_count() == 0


def test_concurrent_cluster_runs_on_two_streams(B, golden_meta, monkeypatch):
    """Several multi-cluster runs in flight at once on two streams, including
    graph replays: each needs its own step flags."""
    import torch

    monkeypatch.setenv("B200FD_CLUSTERS", "4")
    cfg, _ = config1_case(True)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    flds = []
    for rep in range(4):
        for s in streams:
            with torch.cuda.stream(s):
                f = B.Wavefield.allocate(cfg.dims, cfg.halo)
                B.run(f, cfg, variant="auto")
                flds.append(f)
    torch.cuda.synchronize()
    want = golden_meta["config1"]["final_sha256"]
    assert all(sha(f.numpy()) == want for f in flds)


def test_nonfinite_count(B):
    import torch

    dims = (20, 18, 17)
    for dtype in (torch.float32, torch.float64):
        fld = B.Wavefield.allocate(dims, 2, dtype=dtype)
        cur, prev = random_levels(dims, 3)
        fld.set_interior(2, cur)
        assert fld.nonfinite_count() == 0
        fld.grids[2][3, 4, 5] = float("nan")
        fld.grids[2][19, 17, 16] = float("inf")
        fld.grids[2][0, 0, 0] = -float("inf")
        fld.grids[2][0, 0, 19] = float("nan")  # row padding: not interior
        assert fld.nonfinite_count() == 3
        assert fld.nonfinite_count(1) == 0


def test_unstable_run_is_detected(B):
    """dt 1.5x the CFL bound: the StabilityWarning of kernel.py:85-93, then
    the final-field check finds the divergence."""
    dims = (24, 24, 24)
    dt = 1.5 * B.max_stable_dt(4, 1.0)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        cfg = B.KernelConfig(order=4, dims=dims, n_t=400, dt=dt)
    assert any(issubclass(x.category, B.StabilityWarning) for x in w)
    fld = B.Wavefield.allocate(dims, cfg.halo)
    cur, prev = random_levels(dims, 5)
    fld.set_interior(2, cur)
    B.run(fld, cfg)
    assert fld.nonfinite_count() > 0


def test_inplace_model_update_needs_invalidate(B):
    from oracle import acoustic as O
    from oracle import cref

    dims = (24, 20, 28)
    m = (1.0 + 0.5 * np.random.default_rng(2).random(dims)).astype(np.float32)
    dt = 0.5 * B.max_stable_dt(4, 1.0, m)
    cfg = B.KernelConfig(order=4, dims=dims, n_t=3, dt=dt, m=m)
    cur, prev = random_levels(dims, 9)

    def gpu():
        f = B.Wavefield.allocate(dims, 2)
        f.set_interior(2, cur)
        f.set_interior(1, prev)
        B.run(f, cfg)
        return f.numpy()

    def oracle():
        st = O.OracleState(dims, 2)
        O.interior(st.grids[2], 2)[...] = cur
        O.interior(st.grids[1], 2)[...] = prev
        cref.simulate(cfg, 3, state=st)
        return st.latest()

    assert sha(gpu()) == sha(oracle())
    with pytest.raises(ValueError):
        cfg.m[5, 5, 5] = 2.0  # frozen: a stale device copy is never used silently
    B.invalidate_plan(cfg)
    cfg.m[5:10, 5:10, 5:10] = 1.25
    got = gpu()
    assert sha(got) == sha(oracle())
    B.invalidate_plan(cfg)
    cfg.m = cfg.m * np.float32(1.1)  # a new array rebuilds the plan by itself
    assert sha(gpu()) == sha(oracle())
    assert sha(gpu()) != sha(got)
