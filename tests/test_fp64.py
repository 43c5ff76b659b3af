"""The float64 path: the reference step's sequence in IEEE
double on the GPU (fdr_acoustic64_run), bit-exact against the numpy float64
restatement (oracle/acoustic.py: simulate_f64), and the float32 path's
rounding error measured against it."""

import hashlib

import numpy as np
import pytest

from cases import RAGGED, config1_case, medium_o8_case, ragged_case, random_case, rel_l2, scalarm_case, varm_case
from oracle import acoustic as O


def sha64(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def _f64_state(cfg, levels):
    st = O.OracleState(cfg.dims, cfg.halo, dtype=np.float64)
    if levels is not None:
        cur, prev = levels
        O.interior(st.grids[2], st.halo)[...] = cur
        O.interior(st.grids[1], st.halo)[...] = prev
    return st


def test_f64_oracle_constants_and_precision():
    centre, taps, coef = O.kernel_constants_f64(8, 1e-3, 10.0)
    c32, t32, k32 = O.kernel_constants(8, 1e-3, 10.0)
    assert isinstance(centre, float) and np.float32(centre) == c32
    assert [np.float32(t) for t in taps] == list(t32) and np.float32(coef) == k32
    cfg, levels = random_case(8)
    st64 = O.simulate_f64(cfg, state=_f64_state(cfg, levels))
    assert st64.latest().dtype == np.float64
    st32 = O.OracleState(cfg.dims, cfg.halo)
    O.interior(st32.grids[2], cfg.halo)[...] = levels[0]
    O.interior(st32.grids[1], cfg.halo)[...] = levels[1]
    O.simulate(cfg, state=st32)
    err = rel_l2(st32.latest(), st64.latest())
    assert 1e-9 < err < 1e-5  # float32 rounding, not a different scheme


def test_f64_oracle_matches_exact_convolution():
    """One float64 step vs the same update with the Laplacian accumulated in
    exact rational arithmetic on a tiny grid: double rounding only."""
    from fractions import Fraction

    cfg, (cur, prev) = random_case(4)
    st = O.simulate_f64(cfg, n_steps=1, state=_f64_state(cfg, (cur, prev)))
    r = cfg.halo
    w = O.fornberg_weights(2, 4)
    pad = np.zeros(tuple(d + 2 * r for d in cfg.dims))
    pad[r:-r, r:-r, r:-r] = cur
    x, y, z = 7, 9, 11
    lap = 3 * w[r] * Fraction(float(cur[x, y, z]))
    for j in range(1, r + 1):
        for d in ((j, 0, 0), (0, j, 0), (0, 0, j)):
            a = pad[x + r + d[0], y + r + d[1], z + r + d[2]]
            b = pad[x + r - d[0], y + r - d[1], z + r - d[2]]
            lap += w[r + j] * (Fraction(float(a)) + Fraction(float(b)))
    exact = 2 * Fraction(float(cur[x, y, z])) - Fraction(float(prev[x, y, z])) + \
        Fraction(cfg.dt * cfg.dt / (cfg.h * cfg.h)) * lap
    assert abs(st.latest()[x, y, z] - float(exact)) <= 1e-13 * max(1.0, abs(float(exact)))


# ------------------------------------------------------------------- GPU


@pytest.fixture(scope="module")
def B(cuda_device):
    import paper_1608_03984_b200 as pkg
    from paper_1608_03984_b200 import _lib

    _lib.load()
    return pkg


def _gpu_f64(B, cfg, levels, variant, n=None):
    import torch

    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    if levels is not None:
        fld.set_interior(2, levels[0])
        fld.set_interior(1, levels[1])
    B.run(fld, cfg, n, variant=variant)
    return fld


CASES = {
    "random_o2": lambda: random_case(2),
    "random_o8": lambda: random_case(8),
    "random_o16": lambda: random_case(16),
    "varm_o4": varm_case,
    "scalarm_o6": scalarm_case,
    **{f"ragged_o{o}": (lambda o=o, d=d, s=s: ragged_case(o, d, s)) for o, d, s in RAGGED},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["queue", "tma", "direct"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_gpu_f64_bitexact_vs_oracle(B, case, variant):
    cfg, levels = CASES[case]()
    fld = _gpu_f64(B, cfg, levels, variant)
    st = O.simulate_f64(cfg, state=_f64_state(cfg, levels))
    assert fld.numpy().dtype == np.float64
    assert sha64(fld.numpy()) == sha64(st.latest())
    assert sha64(fld.numpy(1)) == sha64(O.interior(st.grids[1], st.halo))
    assert fld.halo_is_zero()


@pytest.mark.gpu
@pytest.mark.parametrize("order", [20, 32])
def test_gpu_f64_high_order_direct(B, order):
    from paper_1608_03984_b200 import KernelConfig, max_stable_dt

    dims = (order + 3, order + 5, order + 2)
    cfg = KernelConfig(order=order, dims=dims, n_t=2, dt=0.5 * max_stable_dt(order, 1.0))
    rng = np.random.default_rng(order)
    levels = (rng.standard_normal(dims), rng.standard_normal(dims))
    fld = _gpu_f64(B, cfg, levels, "auto")
    st = O.simulate_f64(cfg, state=_f64_state(cfg, levels))
    assert sha64(fld.numpy()) == sha64(st.latest())


@pytest.mark.gpu
def test_gpu_f64_config1_sponge_source_receivers(B):
    """BASELINE config 1 (m grid, sponge, Ricker, 64 receivers) in float64, 30
    steps, bit-exact incl. traces; and the float32 path's error against it."""
    cfg, _ = config1_case()
    cfg.n_t = 30
    fld = _gpu_f64(B, cfg, None, "auto")
    st = O.simulate_f64(cfg)
    assert sha64(fld.numpy()) == sha64(st.latest())
    assert sha64(fld.traces.cpu().numpy()[:30]) == sha64(st.traces[:30])
    f32 = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(f32, cfg)
    err = rel_l2(f32.numpy(), fld.numpy())
    assert 1e-9 < err < 1e-4


@pytest.mark.gpu
def test_gpu_f64_stream_equals_direct_medium(B):
    """96x80x72 order 8 with every extension, 40 steps: both streaming
    kernels == direct."""
    cfg, _ = medium_o8_case()
    b = _gpu_f64(B, cfg, None, "direct")
    for v in ("queue", "tma"):
        a = _gpu_f64(B, cfg, None, v)
        assert sha64(a.numpy()) == sha64(b.numpy()), v
        assert sha64(a.traces.cpu().numpy()) == sha64(b.traces.cpu().numpy()), v
    assert np.abs(b.numpy()).max() > 0


@pytest.mark.gpu
def test_gpu_f64_rejects_persistent_variant(B):
    import torch

    cfg, levels = random_case(4)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    with pytest.raises(B.ValidationError):
        B.run(fld, cfg, variant="persistent")


@pytest.mark.gpu
@pytest.mark.parametrize("m_lo,m_hi", [(4.9e-8, 4.5e-7), (0.5, 2.0), (1e-150, 1e-140),
                                       (2.0 ** -500, 2.0 ** 500), (1e-200, 1e200)])
def test_gpu_f64_scaled_division_matches_ieee(B, m_lo, m_hi):
    """The a64_queue kernel's scaled exact division (fast path + __ddiv_rn
    fallback) against IEEE __ddiv_rn bit for bit, over dividends from
    subnormals to 2^520 and wide divisor ranges."""
    from paper_1608_03984_b200.kernel import selftest_division64

    n = 1 << 25
    bad, n_fast = selftest_division64(n, m_lo, m_hi, seed=7)
    assert bad == 0
    assert n_fast > n // 8


@pytest.mark.gpu
@pytest.mark.parametrize("m_lo,m_hi", [(4.9e-8, 4.5e-7), (0.5, 2.0), (2.0 ** -60, 2.0 ** 40)])
def test_gpu_f64_division_subnormal_midpoints(B, m_lo, m_hi):
    """Subnormal quotients stay on the fast path; the double-rounding hazard
    (the scaled quotient exactly on a midpoint of the subnormal grid) is
    resolved by the remainder sign.  Constructed midpoint candidates (seed
    bit 31) against __ddiv_rn bit for bit, with the correction branch taken."""
    from paper_1608_03984_b200.kernel import selftest_division64

    n = 1 << 24
    bad, n_mid = selftest_division64(n, m_lo, m_hi, seed=0x80000000 | 11)
    assert bad == 0
    assert n_mid > n // 64
