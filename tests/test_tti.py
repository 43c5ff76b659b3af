"""TTI pseudo-acoustic system (BASELINE config 4): oracles and GPU parity.

No reference implementation exists (SURVEY.md §8(a')): the exact float32
sequence is defined by oracle/tti_ref.c (parity oracle, bit-exact bar for the
GPU), and its accuracy is checked against the independent float64 oracle
built from the paper's operators.
"""

import math

import numpy as np
import pytest

from cases import rel_l2, sha
from oracle import tti as T
from paper_1608_03984_b200 import Receivers, Source
from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker, smooth_random_field
from paper_1608_03984_b200.tti import TTIConfig, tti_flops_per_point, tti_weights_f32


def small_cfg(order=8, dims=(24, 22, 20), n_t=30, seed=0, sponge=True, h=10.0):
    rng = np.random.default_rng(seed)

    def smooth(lo, hi, s):
        f = smooth_random_field(dims, 3.0, seed + s)
        f = (f - f.min()) / (f.max() - f.min())
        return (lo + (hi - lo) * f).astype(np.float32)

    v = smooth(1500.0, 4500.0, 0)
    m = (1.0 / np.square(v.astype(np.float64))).astype(np.float32)
    eps = smooth(0.0, 0.3, 1)
    delta = np.minimum(smooth(0.0, 0.15, 2), eps)
    theta = smooth(0.0, math.pi / 4, 3)
    phi = smooth(0.0, math.pi / 4, 4)
    dt = 0.4 * h / (4500.0 * math.sqrt(1.0 + 2.0 * float(eps.max())))
    rec = np.stack([np.arange(dims[0]), np.full(dims[0], dims[1] // 2), np.full(dims[0], 2)], 1)
    src = (dims[0] // 2, dims[1] // 2 + 1, dims[2] // 2 - 1)
    del rng
    return TTIConfig(order=order, dims=dims, n_t=n_t, dt=dt, h=h, m=m, epsilon=eps, delta=delta,
                     theta=theta, phi=phi, source=Source(src, 1e3 * ricker(25.0, dt, n_t)),
                     receivers=Receivers(rec), sponge=cerjan_sponge(dims, 4, 0.1) if sponge else None)


def test_catalog_flops():
    # equations.py:144-155 with k = 9: the catalogue's 964 FLOPs per point
    assert tti_flops_per_point(8) == 964


def test_paper_operators_sum_to_laplacian():
    """G_xx + G_yy + G_zz = lap (with the G_yy sign fix of SURVEY.md App. B)."""
    rng = np.random.default_rng(1)
    u = rng.standard_normal((14, 13, 12))
    th = rng.uniform(0, math.pi / 4, u.shape)
    ph = rng.uniform(0, math.pi / 4, u.shape)
    d = T.derivatives_f64(u, 8)
    gxx, gyy, gzz = T.paper_operators(d, th, ph)
    lap = d["xx"] + d["yy"] + d["zz"]
    assert np.allclose(gxx + gyy + gzz, lap, rtol=0, atol=1e-12 * np.abs(lap).max())


def test_gzz_coefficients_match_paper():
    cfg = small_cfg(n_t=1)
    prm = cfg.params()
    th, ph = cfg.theta.astype(np.float64), cfg.phi.astype(np.float64)
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    assert np.allclose(prm["cxx"], cp * cp * st * st, atol=1e-7)
    assert np.allclose(prm["cxy"], np.sin(2 * ph) * st * st, atol=1e-7)
    assert np.allclose(prm["cyz"], sp * np.sin(2 * th), atol=1e-7)
    assert np.allclose(prm["cxz"], cp * np.sin(2 * th), atol=1e-7)


@pytest.mark.parametrize("order", [4, 8])
def test_f32_oracle_accuracy_vs_f64(order):
    """The float32 parity sequence against the float64 paper-operator oracle."""
    cfg = small_cfg(order=order, n_t=40)
    w2, w1 = tti_weights_f32(order)
    st = T.simulate_c(cfg, cfg.params(), w2, w1, threads=4)
    p64, r64, tr64 = T.simulate_f64(cfg)
    assert np.isfinite(st.interior()).all()
    assert np.abs(p64).max() > 1e-3  # the wavefield is non-trivial
    assert rel_l2(st.interior("p"), p64) < 1e-5  # north_star tolerance (measured 3e-7 .. 5e-7)
    assert rel_l2(st.interior("r"), r64) < 1e-5
    assert rel_l2(st.traces, tr64) < 1e-5


def test_c_oracle_threads_bitexact():
    cfg = small_cfg(n_t=6)
    w2, w1 = tti_weights_f32(8)
    a = T.simulate_c(cfg, cfg.params(), w2, w1, threads=1)
    b = T.simulate_c(cfg, cfg.params(), w2, w1, threads=5)
    assert sha(a.interior()) == sha(b.interior()) and sha(a.interior("r")) == sha(b.interior("r"))


def test_isotropic_limit_is_acoustic():
    """eps = delta = 0: p and r both follow m u_tt = lap u (to float32 rounding)."""
    cfg = small_cfg(n_t=25, sponge=False)
    cfg.epsilon = np.zeros(cfg.dims, np.float32)
    cfg.delta = np.zeros(cfg.dims, np.float32)
    w2, w1 = tti_weights_f32(8)
    st = T.simulate_c(cfg, cfg.params(), w2, w1)
    assert rel_l2(st.interior("p"), st.interior("r")) < 1e-5


# ------------------------------------------------------------------- GPU


@pytest.fixture(scope="module")
def tti_mod(cuda_device):
    from paper_1608_03984_b200 import _lib, tti

    _lib.load()
    return tti


def _gpu(tti_mod, cfg, variant, n=None, interleaved=None):
    # the TMA variant (tti_stream) takes separate p/r levels; the others run
    # on the default interleaved (p, r) pairs, "queue_sep" on separate levels
    il = variant not in ("stream", "queue_sep") if interleaved is None else interleaved
    fld = tti_mod.TTIWavefield.allocate(cfg.dims, cfg.halo, interleaved=il)
    tti_mod.tti_run(fld, cfg, n, variant="queue" if variant == "queue_sep" else variant)
    return fld


GPU_VARIANTS = ["queue", "queue_sep", "stream", "direct"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant", GPU_VARIANTS)
@pytest.mark.parametrize("order,dims", [(2, (11, 12, 13)), (4, (17, 16, 15)), (6, (19, 18, 21)),
                                        (8, (24, 22, 20)), (8, (33, 30, 37))])
def test_gpu_tti_bitexact_vs_c_oracle(tti_mod, variant, order, dims):
    cfg = small_cfg(order=order, dims=dims, n_t=12)
    fld = _gpu(tti_mod, cfg, variant)
    w2, w1 = tti_weights_f32(order)
    st = T.simulate_c(cfg, cfg.params(), w2, w1)
    assert sha(fld.numpy("p")) == sha(st.interior("p"))
    assert sha(fld.numpy("r")) == sha(st.interior("r"))
    assert sha(fld.numpy("p", 1)) == sha(st.interior("p", 1))
    assert (fld.traces.cpu().numpy() == st.traces).all()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [12, 16])
def test_gpu_tti_high_orders_bitexact(tti_mod, order):
    """Orders above 8 run the direct kernel (AUTO); the streaming variants
    reject them with the reference's ValidationError."""
    from paper_1608_03984_b200.errors import ValidationError

    cfg = small_cfg(order=order, dims=(order + 3, order + 2, order + 5), n_t=8)
    fld = _gpu(tti_mod, cfg, "auto")
    w2, w1 = tti_weights_f32(order)
    st = T.simulate_c(cfg, cfg.params(), w2, w1)
    assert sha(fld.numpy("p")) == sha(st.interior("p"))
    assert sha(fld.numpy("r")) == sha(st.interior("r"))
    assert (fld.traces.cpu().numpy() == st.traces).all()
    assert np.abs(st.interior("p")).max() > 0
    with pytest.raises(ValidationError):
        _gpu(tti_mod, cfg, "queue")


@pytest.mark.gpu
def test_gpu_tti_config4_grid_vs_c_oracle(tti_mod):
    """BASELINE config 4 (384^3, order 8, smooth eps/delta/tilt/azimuth,
    sponge, source, receivers) for 3 steps from random levels, bit-exact."""
    cfg = tti_mod.config4(n_t=3)
    rng = np.random.default_rng(4)
    st = T.TTIState(cfg.dims, cfg.halo)
    fld = tti_mod.TTIWavefield.allocate(cfg.dims, cfg.halo)
    for f in ("p", "r"):
        for lvl in (1, 2):
            v = rng.standard_normal(cfg.dims, dtype=np.float32)
            st.interior(f, lvl)[...] = v
            fld.set_interior(f, lvl, v)
    tti_mod.tti_run(fld, cfg)
    w2, w1 = tti_weights_f32(8)
    T.simulate_c(cfg, cfg.params(), w2, w1, state=st)
    assert sha(fld.numpy("p")) == sha(st.interior("p"))
    assert sha(fld.numpy("r")) == sha(st.interior("r"))
    assert (fld.traces.cpu().numpy() == st.traces).all()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [4, 8])
def test_gpu_tti_float64_path_vs_f64_oracle(tti_mod, order):
    """fdr_tti64_run (the direct kernel in double) against the independent
    numpy float64 paper-operator oracle: the same system to double precision."""
    import torch

    from paper_1608_03984_b200.errors import ValidationError

    cfg = small_cfg(order=order, n_t=40)
    fld = tti_mod.TTIWavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    tti_mod.tti_run(fld, cfg)
    p64, r64, tr64 = T.simulate_f64(cfg)
    assert fld.p[0].dtype == torch.float64 and fld.traces.dtype == torch.float64
    assert rel_l2(fld.numpy("p"), p64) < 1e-10
    assert rel_l2(fld.numpy("r"), r64) < 1e-10
    assert rel_l2(fld.traces.cpu().numpy()[: cfg.n_t], tr64) < 1e-10
    with pytest.raises(ValidationError):
        tti_mod.tti_run(fld, cfg, 1, variant="queue")
