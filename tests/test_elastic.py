"""Elastic velocity-stress system (BASELINE config 5): oracles and GPU parity.

No reference implementation exists (SURVEY.md §8(a')); the float32 sequence is
defined by oracle/elastic_ref.c (the bit-exact bar for the GPU) and checked for
accuracy against the independent float64 oracle.
"""

import numpy as np
import pytest

from cases import rel_l2, sha
from oracle import elastic as E
from paper_1608_03984_b200 import Receivers, Source
from paper_1608_03984_b200.elastic import (FIELDS, ElasticConfig, elastic_max_stable_dt,
                                           elastic_weights_f32)
from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker, smooth_random_field


def small_cfg(order=8, dims=(24, 22, 20), n_t=30, seed=0, sponge=True, h=10.0):
    def smooth(lo, hi, s):
        f = smooth_random_field(dims, 3.0, seed + s)
        f = (f - f.min()) / (f.max() - f.min())
        return (lo + (hi - lo) * f).astype(np.float32)

    vp = smooth(1500.0, 4500.0, 0)
    vs = (vp.astype(np.float64) / 1.8).astype(np.float32)
    rho = smooth(1000.0, 2500.0, 1)
    dt = 0.4 * h / 4500.0
    rec = np.stack([np.arange(dims[0]), np.full(dims[0], dims[1] // 2), np.full(dims[0], 2)], 1)
    src = (dims[0] // 2, dims[1] // 2 - 1, dims[2] // 2 + 1)
    return ElasticConfig(order=order, dims=dims, n_t=n_t, dt=dt, h=h, vp=vp, vs=vs, rho=rho,
                         source=Source(src, 1e6 * ricker(30.0, dt, n_t)), receivers=Receivers(rec),
                         sponge=cerjan_sponge(dims, 4, 0.1) if sponge else None)


def test_staggered_weights_and_cfl():
    c = elastic_weights_f32(8)
    assert c[1] == np.float32(1225 / 1024)
    assert 0.4 * 10 / 4500 < elastic_max_stable_dt(8, 10.0, 4500.0)


@pytest.mark.parametrize("order", [4, 8])
def test_f32_oracle_accuracy_vs_f64(order):
    cfg = small_cfg(order=order, n_t=40)
    st = E.simulate_c(cfg, cfg.params(), elastic_weights_f32(order), threads=4)
    f64, tr64 = E.simulate_f64(cfg)
    assert np.abs(f64["vz"]).max() > 1e-6
    for k in FIELDS:
        assert rel_l2(st.interior(k), f64[k]) < 1e-5, k  # north_star tolerance (measured <= 2.4e-7)
    assert rel_l2(st.traces, tr64) < 1e-5


def test_c_oracle_threads_bitexact():
    cfg = small_cfg(n_t=6)
    c = elastic_weights_f32(8)
    a = E.simulate_c(cfg, cfg.params(), c, threads=1)
    b = E.simulate_c(cfg, cfg.params(), c, threads=5)
    for k in FIELDS:
        assert sha(a.interior(k)) == sha(b.interior(k))


def test_explosive_source_symmetry():
    """Homogeneous medium, centred explosive source, no sponge: vz is
    antisymmetric in z about the source (to float64 rounding)."""
    dims = (31, 31, 31)  # two steps spread 16 points: the boundaries are never reached
    cfg = ElasticConfig(order=8, dims=dims, n_t=2, dt=0.4 * 10 / 3000, h=10.0, vp=3000.0,
                        vs=3000.0 / 1.8, rho=2000.0, source=Source((15, 15, 15), 1e6 * np.ones(2)))
    f64, _ = E.simulate_f64(cfg)
    vz = f64["vz"]  # vz[k] sits at z = k + 1/2: mirror about z = 15 maps k -> 29 - k
    assert np.abs(vz).max() > 0
    assert np.allclose(vz[:, :, :30], -vz[:, :, 29::-1], rtol=0, atol=1e-12 * np.abs(vz).max())
    sxx = f64["sxx"]
    assert np.allclose(sxx, sxx[::-1], rtol=0, atol=1e-12 * np.abs(sxx).max())


# ------------------------------------------------------------------- GPU


@pytest.fixture(scope="module")
def el_mod(cuda_device):
    from paper_1608_03984_b200 import _lib, elastic

    _lib.load()
    return elastic


GPU_VARIANTS = ["queue", "stream", "direct"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", GPU_VARIANTS)
@pytest.mark.parametrize("order,dims", [(2, (11, 12, 13)), (4, (17, 16, 15)), (6, (19, 18, 21)),
                                        (8, (24, 22, 20)), (8, (33, 30, 37))])
def test_gpu_elastic_bitexact_vs_c_oracle(el_mod, variant, order, dims):
    cfg = small_cfg(order=order, dims=dims, n_t=12)
    fld = el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    el_mod.elastic_run(fld, cfg, variant=variant)
    st = E.simulate_c(cfg, cfg.params(), elastic_weights_f32(order))
    for k in FIELDS:
        assert sha(fld.numpy(k)) == sha(st.interior(k)), k
    assert (fld.traces.cpu().numpy() == st.traces).all()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [12, 16])
def test_gpu_elastic_high_orders_bitexact(el_mod, order):
    """Orders above 8 run the direct kernel (AUTO); the streaming variants
    reject them with the reference's ValidationError."""
    from paper_1608_03984_b200.errors import ValidationError

    cfg = small_cfg(order=order, dims=(order + 3, order + 2, order + 5), n_t=8)
    fld = el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    el_mod.elastic_run(fld, cfg, variant="auto")
    st = E.simulate_c(cfg, cfg.params(), elastic_weights_f32(order))
    for k in FIELDS:
        assert sha(fld.numpy(k)) == sha(st.interior(k)), k
    assert (fld.traces.cpu().numpy() == st.traces).all()
    assert np.abs(st.interior("vz")).max() > 0
    with pytest.raises(ValidationError):
        el_mod.elastic_run(el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo), cfg, variant="queue")


@pytest.mark.gpu
def test_gpu_elastic_config5_grid_vs_c_oracle(el_mod):
    """BASELINE config 5 (320^3, order 8, smooth vp/vs/rho, sponge, explosive
    source, 320 vz receivers) for 3 steps from random fields, bit-exact."""
    cfg = el_mod.config5(n_t=3)
    rng = np.random.default_rng(5)
    st = E.ElasticState(cfg.dims, cfg.halo)
    fld = el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    for k in FIELDS:
        v = rng.standard_normal(cfg.dims, dtype=np.float32)
        st.interior(k)[...] = v
        fld.set_interior(k, v)
    el_mod.elastic_run(fld, cfg)
    E.simulate_c(cfg, cfg.params(), elastic_weights_f32(8), state=st)
    for k in FIELDS:
        assert sha(fld.numpy(k)) == sha(st.interior(k)), k
    assert (fld.traces.cpu().numpy() == st.traces).all()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [4, 8])
def test_gpu_elastic_float64_path_vs_f64_oracle(order, cuda_device):
    """fdr_elastic64_run (the direct kernels in double) against the independent
    numpy float64 oracle."""
    import torch

    from paper_1608_03984_b200 import elastic
    from paper_1608_03984_b200.errors import ValidationError

    cfg = small_cfg(order=order, n_t=40)
    fld = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    elastic.elastic_run(fld, cfg)
    f64, tr64 = E.simulate_f64(cfg)
    for k in FIELDS:
        assert rel_l2(fld.numpy(k), f64[k]) < 1e-10, k
    assert rel_l2(fld.traces.cpu().numpy()[: cfg.n_t], tr64) < 1e-10
    with pytest.raises(ValidationError):
        elastic.elastic_run(fld, cfg, 1, variant="queue")


# The experimental L2-window schedules of the queue path: the
# library re-reads their knobs at every run, so one process can flip them.
SCHEDULES = [{"B200FD_EL_WINDOW": "4"}, {"B200FD_EL_WINDOW": "5", "B200FD_EL_WINDOW_STREAMS": "2"},
             {"B200FD_EL_WINDOW": "8", "B200FD_EL_WINDOW_SUB": "2"}, {"B200FD_EL_FUSE": "4"},
             {"B200FD_EL_FUSE": "6", "B200FD_EL_FUSE_LAG": "3"}]


@pytest.mark.gpu
@pytest.mark.parametrize("knobs", SCHEDULES, ids=lambda k: "-".join(f"{a[10:]}{b}" for a, b in k.items()))
@pytest.mark.parametrize("order,dims", [(4, (17, 16, 15)), (8, (33, 30, 37)), (8, (41, 70, 100))])
def test_gpu_elastic_window_schedules_bitexact(el_mod, monkeypatch, knobs, order, dims):
    """V(k+1) before S(k) on windows of x-planes (separate launches, or items of
    the persistent el_fused kernel): same bits as the two full passes."""
    cfg = small_cfg(order=order, dims=dims, n_t=7)
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    fld = el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    el_mod.elastic_run(fld, cfg, variant="queue")
    from paper_1608_03984_b200 import _lib

    assert _lib.load().fdr_pending_error() == 0
    st = E.simulate_c(cfg, cfg.params(), elastic_weights_f32(order))
    for k in FIELDS:
        assert sha(fld.numpy(k)) == sha(st.interior(k)), k
    assert (fld.traces.cpu().numpy() == st.traces).all()


@pytest.mark.gpu
def test_gpu_elastic_fused_config5_grid_equals_two_pass(el_mod, monkeypatch):
    """el_fused on the 320^3 config-5 grid (16000 items per pass and step handed
    out by tickets over 296 CTAs): 4 steps, bit-identical to the two passes."""
    cfg = el_mod.config5(n_t=4)
    rng = np.random.default_rng(7)
    start = {k: rng.standard_normal(cfg.dims, dtype=np.float32) for k in FIELDS}

    def run():
        fld = el_mod.ElasticWavefield.allocate(cfg.dims, cfg.halo)
        for k in FIELDS:
            fld.set_interior(k, start[k])
        el_mod.elastic_run(fld, cfg, variant="queue")
        return {k: sha(fld.numpy(k)) for k in FIELDS}, sha(fld.traces.cpu().numpy())

    ref = run()
    monkeypatch.setenv("B200FD_EL_FUSE", "4")
    got = run()
    from paper_1608_03984_b200 import _lib

    assert _lib.load().fdr_pending_error() == 0
    assert got == ref
