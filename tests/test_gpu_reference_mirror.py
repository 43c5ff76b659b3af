"""The reference's own kernel tests (/root/reference/pkg/tests/test_kernel.py
and the kernel criterion 09 of test_acceptance.py), restated one for one
against the GPU path: same configs, seeds, tolerances and assertions, with
the float64 convolution oracle (oracle/acoustic.py::conv_step_f64, the
restatement of kernel.py:225-254) standing in for `oracle_step`."""

import numpy as np
import pytest

from oracle import acoustic as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B(cuda_device):
    import paper_1608_03984_b200 as pkg
    from paper_1608_03984_b200 import _lib

    _lib.load()
    return pkg


def make_config(B, order, dims, n_t=1, dt_frac=0.5, **kw):  # test_kernel.py:20-22
    dt = dt_frac * B.max_stable_dt(order, kw.get("h", 1.0), kw.get("m", 1.0))
    return B.KernelConfig(order=order, dims=dims, n_t=n_t, dt=dt, **kw)


def random_levels(cfg, seed=0):  # test_kernel.py:25-30
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(cfg.dims).astype(np.float32),
            rng.standard_normal(cfg.dims).astype(np.float32))


def gpu_field(B, cfg, levels=None):
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    if levels is not None:
        fld.set_interior(2, levels[0])
        fld.set_interior(1, levels[1])
    return fld


def oracle_field(cfg, levels):
    st = O.OracleState(cfg.dims, cfg.halo)
    O.interior(st.grids[2], cfg.halo)[...] = levels[0]
    O.interior(st.grids[1], cfg.halo)[...] = levels[1]
    return st


@pytest.mark.parametrize("order", [2, 4, 8, 16])
def test_step_matches_convolution_oracle(B, order):  # test_kernel.py:67-77
    cfg = make_config(B, order, (20, 20, 20))
    lv = random_levels(cfg, seed=order)
    a, b = gpu_field(B, cfg, lv), oracle_field(cfg, lv)
    for _ in range(3):
        B.step(a, cfg)
        O.conv_step_f64(b, cfg)
        u = a.numpy()
        scale = float(np.abs(u).max())
        diff = float(np.abs(u - b.latest()).max())
        assert diff <= 1e-6 * scale


def test_oracle_matches_with_varying_slowness(B):  # test_kernel.py:80-88
    m = 1.0 + 0.5 * np.random.default_rng(3).random((16, 16, 16)).astype(np.float32)
    cfg = make_config(B, 4, (16, 16, 16), m=m)
    lv = random_levels(cfg, seed=11)
    a, b = gpu_field(B, cfg, lv), oracle_field(cfg, lv)
    B.step(a, cfg)
    O.conv_step_f64(b, cfg)
    u = a.numpy()
    assert float(np.abs(u - b.latest()).max()) <= 1e-6 * float(np.abs(u).max())


def test_halo_stays_zero_across_orders(B):  # test_kernel.py:98-104
    for order in (2, 8):
        cfg = make_config(B, order, (15, 15, 15))
        fld = gpu_field(B, cfg, random_levels(cfg, seed=1))
        for _ in range(10):
            B.step(fld, cfg)
        assert fld.halo_is_zero()
        host = fld.host_grids()  # the reference layout: padded, halo exactly zero
        r = cfg.halo
        for g in host:
            inner = g[r:-r, r:-r, r:-r].copy()
            g[r:-r, r:-r, r:-r] = 0
            assert not g.any()
            g[r:-r, r:-r, r:-r] = inner


def test_slab_decomposition_bitexact(B):  # test_kernel.py:137-144
    cfg = make_config(B, 8, (24, 20, 18))
    ref = gpu_field(B, cfg, random_levels(cfg, seed=5))
    B.step(ref, cfg, slabs=1)
    for slabs in (2, 3, 7):
        fld = gpu_field(B, cfg, random_levels(cfg, seed=5))
        B.step(fld, cfg, slabs=slabs)
        assert (fld.numpy() == ref.numpy()).all(), slabs


def test_repeated_runs_bit_identical(B):  # test_kernel.py:147-152
    cfg = make_config(B, 4, (16, 16, 16), n_t=4)
    r1 = B.run_benchmark(cfg)
    r2 = B.run_benchmark(cfg)
    assert (r1.wavefield.numpy() == r2.wavefield.numpy()).all()
    assert r1.total_flops == r2.total_flops


def test_benchmark_oi_independent_of_grid(B):  # test_kernel.py:155-160
    small = B.run_benchmark(make_config(B, 8, (12, 12, 12), n_t=2))
    large = B.run_benchmark(make_config(B, 8, (24, 24, 24), n_t=2))
    assert small.point.oi == large.point.oi == 3.625  # 3*9/8 + 1/4
    assert small.measured_gflops > 0 and np.isfinite(small.measured_gflops)
    assert small.point.measured_gflops == small.measured_gflops


def test_benchmark_flop_accounting(B):  # test_kernel.py:163-167
    cfg = make_config(B, 2, (10, 10, 10), n_t=3)
    res = B.run_benchmark(cfg)
    assert res.total_flops == 10 ** 3 * 22 * 3  # N * kernel_flops(k=3) * steps
    assert res.measured_gflops == pytest.approx(res.total_flops / res.wall_time_s / 1e9)


def test_source_injection_matches_series(B):  # test_kernel.py:186-195
    cfg = make_config(B, 2, (9, 9, 9))
    cfg.source = B.Source(location=(4, 4, 4), series=np.array([2.0, 3.0], dtype=np.float32))
    fld = gpu_field(B, cfg)
    B.step(fld, cfg)
    assert fld.numpy()[4, 4, 4] == 2.0
    B.step(fld, cfg)
    assert fld.it == 2
    # 2*u(t-1) - 0 + lap contribution at the centre + q[1], in the reference's order
    st = O.simulate(cfg, 2)
    assert (fld.numpy() == st.latest()).all()


def test_acceptance_criterion_09_kernel_checks(B):  # test_acceptance.py:152-223
    for order in (2, 4, 8, 16):
        dt = 0.5 * B.max_stable_dt(order, 1.0)
        cfg = B.KernelConfig(order=order, dims=(20, 20, 20), n_t=1, dt=dt)
        rng = np.random.default_rng(order)
        lv = (rng.standard_normal(cfg.dims).astype(np.float32),
              rng.standard_normal(cfg.dims).astype(np.float32))
        a, b = gpu_field(B, cfg, lv), oracle_field(cfg, lv)
        B.step(a, cfg)
        O.conv_step_f64(b, cfg)
        u = a.numpy()
        assert float(np.abs(u - b.latest()).max()) <= 1e-6 * float(np.abs(u).max()), order
    cfg = B.KernelConfig(order=4, dims=(16, 16, 16), n_t=1, dt=0.5 * B.max_stable_dt(4, 1.0))
    zero = gpu_field(B, cfg)
    for _ in range(10):
        B.step(zero, cfg)
    assert not zero.numpy().any() and zero.halo_is_zero()
    cfg = B.KernelConfig(order=2, dims=(15, 15, 15), n_t=1, dt=0.5 * B.max_stable_dt(2, 1.0))
    sym = gpu_field(B, cfg)
    sym.grids[2][7, 7, 7] = 1.0
    for _ in range(8):
        B.step(sym, cfg)
        u = sym.numpy()
        for axis in range(3):
            assert (u == np.flip(u, axis=axis)).all()
