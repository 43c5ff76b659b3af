"""Off-grid (trilinear) receivers and source (receivers are on
grid in the BASELINE configs, trilinear off grid with a fixed op order).
GPU results are bit-exact against the numpy oracle's restatement."""

import numpy as np
import pytest

from cases import sha
from oracle import acoustic as O
import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker


def offgrid_case(dims=(28, 26, 30), order=8, n_t=10, integer=False):
    rng = np.random.default_rng(21)
    m = (1.0 + 0.5 * rng.random(dims)).astype(np.float32)
    dt = 0.5 * B.max_stable_dt(order, 1.0, m)
    pos = np.stack([rng.uniform(0, dims[0] - 1, 40), rng.uniform(0, dims[1] - 1, 40),
                    rng.uniform(0, dims[2] - 1, 40)], 1)
    pos[0] = [d - 1 for d in dims]            # the far corner: 7 corners outside
    pos[1] = [0.0, 0.0, 0.0]
    src = (13.37, 12.5, 14.81)
    if integer:
        pos = np.floor(pos)
        src = (13.0, 12.0, 14.0)
    return B.KernelConfig(order=order, dims=dims, n_t=n_t, dt=dt, m=m,
                          source=B.OffGridSource(src, 100.0 * ricker(0.2, dt, n_t)),
                          receivers=B.OffGridReceivers(pos), sponge=cerjan_sponge(dims, 4, 0.1))


def test_trilinear_weights_match_oracle_restatement():
    pos = np.random.default_rng(3).uniform(0, 40, (500, 3))
    b1, w1 = B.trilinear_weights(pos)
    b2, w2 = O.trilinear(pos)
    assert (b1 == b2).all() and (w1 == w2).all()
    assert np.allclose(w1.astype(np.float64).sum(1), 1.0, atol=1e-6)
    b, w = B.trilinear_weights([[3.0, 4.0, 5.0]])
    assert (b == [[3, 4, 5]]).all() and w[0, 0] == 1.0 and not w[0, 1:].any()


def test_integer_positions_reduce_to_on_grid_oracle():
    cfg = offgrid_case(integer=True)
    on = B.KernelConfig(order=cfg.order, dims=cfg.dims, n_t=cfg.n_t, dt=cfg.dt, m=cfg.m,
                        source=B.Source((13, 12, 14), cfg.source.series),
                        receivers=B.Receivers(cfg.receivers.positions.astype(np.int32)),
                        sponge=cfg.sponge)
    a, b = O.simulate(cfg), O.simulate(on)
    assert (a.latest() == b.latest()).all() and (a.traces == b.traces).all()


def test_validation():
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=4, dims=(10, 10, 10), n_t=1, dt=0.1,
                       source=B.OffGridSource((9.5, 1.0, 1.0), np.ones(1)))
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=4, dims=(10, 10, 10), n_t=1, dt=0.1,
                       receivers=B.OffGridReceivers([[1.0, 1.0, -0.1]]))


# ------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["auto", "queue", "queue2", "tma", "direct"])
def test_gpu_offgrid_bitexact_vs_oracle(cuda_device, variant):
    cfg = offgrid_case()
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg, variant=variant)
    st = O.simulate(cfg)
    assert sha(fld.numpy()) == sha(st.latest())
    assert (fld.traces.cpu().numpy()[: cfg.n_t] == st.traces[: cfg.n_t]).all()
    assert np.abs(st.traces).max() > 0


@pytest.mark.gpu
def test_gpu_offgrid_small_grid_and_stepwise(cuda_device):
    """A config-1-sized grid (AUTO's small-grid path must not take the
    persistent kernel with an off-grid source) and step-by-step == one run."""
    cfg = offgrid_case(dims=(40, 36, 44), order=4, n_t=12)
    a = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(a, cfg)
    b = B.Wavefield.allocate(cfg.dims, cfg.halo)
    for _ in range(cfg.n_t):
        B.step(b, cfg)
    st = O.simulate(cfg)
    assert sha(a.numpy()) == sha(st.latest()) == sha(b.numpy())
    assert (a.traces.cpu().numpy() == st.traces).all()
    with pytest.raises(B.ValidationError):
        B.run(B.Wavefield.allocate(cfg.dims, cfg.halo), cfg, variant="persistent")
    with pytest.raises(B.ValidationError, match="on-grid"):
        B.run(B.Wavefield.allocate(cfg.dims, cfg.halo), cfg, variant="cluster")


@pytest.mark.gpu
def test_gpu_offgrid_rejected_where_unsupported(cuda_device):
    import torch

    cfg = offgrid_case(n_t=2)
    with pytest.raises(B.ValidationError):
        B.HostSimulation(cfg)
    with pytest.raises(B.ValidationError):
        B.run(B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64), cfg)
