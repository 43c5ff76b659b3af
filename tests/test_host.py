"""Host-side logic and the C-ABI library, without a GPU."""

import ctypes
import os
import re
import warnings

import numpy as np
import pytest

import paper_1608_03984_b200 as B
from paper_1608_03984_b200 import _lib, roofline, synthetic
from paper_1608_03984_b200.stencils import (acoustic_weights_f32, second_derivative_weights,
                                            staggered_first_derivative_weights, taylor_weights)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "b200fd.h"), encoding="utf-8").read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(fdr_\w+)\s*\(", header, re.M))
    assert declared == {name for name, _, _ in _lib.EXPORTS}
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fdr_abi_version() == _lib.ABI_VERSION
    assert lib.fdr_acoustic_args_size() == ctypes.sizeof(_lib.AcousticArgs)


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_invalid_args_rejected_without_gpu():
    args = _lib.AcousticArgs()
    args.abi_version = _lib.ABI_VERSION
    args.order = 8
    args.nx = args.ny = args.nz = 5  # too small for halo 4
    args.pitch_y = 8
    args.pitch_x = 40
    with pytest.raises(B.ValidationError, match="too small"):
        _lib.check(_lib.load().fdr_acoustic_run(ctypes.byref(args), None))
    args.abi_version = 99
    with pytest.raises(B.ValidationError, match="abi_version"):
        _lib.check(_lib.load().fdr_acoustic_run(ctypes.byref(args), None))
    assert _lib.load().fdr_acoustic_workspace_bytes(ctypes.byref(args)) == 0


def test_workspace_size():
    args = _lib.AcousticArgs()
    args.abi_version = _lib.ABI_VERSION
    args.order = 4
    args.nx, args.ny, args.nz = 64, 64, 64
    args.pitch_y, args.pitch_x = 64, 64 * 64
    args.m_mode = _lib.M_GRID
    args.n_steps, args.n_rec, args.n_series = 100, 64, 100
    n = _lib.load().fdr_acoustic_workspace_bytes(ctypes.byref(args))
    assert n >= 4 * 64 ** 3 * 4 + 100 * 64 * 4


def test_config_validation_mirrors_reference():
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=3, dims=(9, 9, 9), n_t=1, dt=0.1)
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=8, dims=(5, 9, 9), n_t=1, dt=0.1)
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.1, source=B.Source((9, 0, 0), np.ones(1)))
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.1, m=np.ones((9, 9, 8)))
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.1,
                       receivers=B.Receivers(np.array([[0, 0, 9]])))
    with pytest.raises(B.ValidationError):
        B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.1,
                       sponge=B.Sponge(np.ones(9), np.ones(9), np.ones(8)))
    assert issubclass(B.ValidationError, ValueError)


def test_cfl_warning_semantics(recwarn):
    bound = B.max_stable_dt(2, 1.0)
    with pytest.warns(B.StabilityWarning):
        B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=2 * bound)
    B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=bound)
    assert not [w for w in recwarn if issubclass(w.category, B.StabilityWarning)]


def test_max_stable_dt_values():
    # 0.5774 / 0.5 / 0.4529 / 0.4342 / 0.4237 for orders 2..16
    got = [B.max_stable_dt(o, 1.0) for o in (2, 4, 8, 12, 16)]
    assert got == pytest.approx([0.57735, 0.5, 0.45290, 0.43422, 0.42373], abs=5e-5)
    assert B.max_stable_dt(2, 1.0, m=0.25) == pytest.approx(B.max_stable_dt(2, 1.0) / 2)
    bounds = [B.max_stable_dt(o, 1.0) for o in (2, 4, 8, 16, 24)]
    assert bounds == sorted(bounds, reverse=True)


def test_centre_weight_rounding_matches_reference_rule():
    # f32(3*w0) differs from 3*f32(w0) at orders 20, 30, 32
    differs = []
    for order in range(2, 34, 2):
        w = acoustic_weights_f32(order)
        w0 = float(second_derivative_weights(order)[order // 2])
        assert w[0] == np.float32(3.0 * w0)
        if np.float32(3.0 * w0) != np.float32(3) * np.float32(w0):
            differs.append(order)
    assert differs == [20, 30, 32]


def test_staggered_weights_exact():
    assert staggered_first_derivative_weights(2) == (1,)
    c = staggered_first_derivative_weights(8)
    assert [str(x) for x in c] == ["1225/1024", "-245/3072", "49/5120", "-5/7168"]
    assert taylor_weights([-1, 0, 1], 1) == (-0.5, 0, 0.5)


def test_roofline_model_matches_reference_catalog():
    assert roofline.acoustic_flops_per_point(2) == 22
    assert roofline.acoustic_flops_per_point(8) == 58
    m = roofline.MachineSpec("t", 1000.0, 100.0)
    p = roofline.roofline_point(m, 8)
    assert p.oi == 3.625 and p.bound == "memory" and p.attainable_gflops == 362.5


def test_synthetic_inputs():
    r = synthetic.ricker(10.0, 1e-3, 300)
    assert abs(r.max() - 1.0) < 1e-6 and np.argmax(r) == 100
    g = synthetic.cerjan_profile(64)
    assert g.dtype == np.float32 and g[0] < g[9] < g[10] == 1.0 and g[-1] == g[0]
    v = synthetic.smooth_random_velocity((32, 32, 32), sigma=4.0, seed=1)
    assert v.min() == 1500.0 and v.max() == 4500.0
    lay = synthetic.layered_velocity((4, 4, 64), 8, seed=2)
    assert len(np.unique(lay[0, 0])) <= 8
    cfg = synthetic.config1(n_t=10)
    assert cfg.dims == (64, 64, 64) and cfg.order == 4 and cfg.receivers.count == 64
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        synthetic.config1(n_t=10)  # dt = 0.4 h/vmax is below the CFL bound


def test_step_requires_cuda_tensors():
    if B.kernel._torch().cuda.is_available():
        pytest.skip("CPU-only check")
    cfg = B.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.1)
    import torch

    fld = B.Wavefield(1, [torch.zeros((9, 9, 12)) for _ in range(3)], (9, 9, 9))
    with pytest.raises(B.ValidationError):
        B.step(fld, cfg)


def test_dump_wavefield_layout(tmp_path):
    import torch

    fld = B.Wavefield(1, [torch.zeros((3, 4, 8)) for _ in range(3)], (3, 4, 5))
    fld.grids[2][:, :, :5] = torch.arange(60, dtype=torch.float32).reshape(3, 4, 5)
    path = tmp_path / "field.bin"
    B.dump_wavefield(fld, path)
    assert (tmp_path / "field.bin.dims").read_text() == "3 4 5\n"
    raw = np.fromfile(path, dtype="<f4")
    u = fld.numpy(2)
    assert raw.shape == (60,) and raw[1] == u[1, 0, 0] and raw[3] == u[0, 1, 0]


def test_b200_machine_uses_measured_peaks():
    m = roofline.b200_machine()
    assert m.peak_bw_achievable > 5000
    assert m.ridge_point > 5


def test_wavefield_and_trace_files_round_trip(tmp_path):
    import torch

    fld = B.Wavefield(1, [torch.zeros((3, 4, 8)) for _ in range(3)], (3, 4, 5))
    fld.grids[2][:, :, :5] = torch.arange(60, dtype=torch.float32).reshape(3, 4, 5)
    fld.traces = torch.arange(12, dtype=torch.float32).reshape(4, 3)
    fld.it = 3
    B.dump_wavefield(fld, tmp_path / "u.bin")
    assert np.array_equal(B.load_wavefield(tmp_path / "u.bin"), fld.numpy(2))
    B.dump_traces(fld, tmp_path / "t.bin")
    assert (tmp_path / "t.bin.dims").read_text() == "3 3\n"
    assert np.array_equal(B.load_traces(tmp_path / "t.bin"), fld.traces[:3].numpy())
    (tmp_path / "t.bin.dims").write_text("4 4\n")
    with pytest.raises(B.ValidationError):
        B.load_traces(tmp_path / "t.bin")


def test_oracle_cache_keys_and_reuse(tmp_path, monkeypatch):
    from oracle import cache

    monkeypatch.setattr(cache, "CACHE_DIR", str(tmp_path))
    cfg = synthetic.config1(n_t=5)
    k1 = cache.key("tag", cfg, 5)
    assert k1 == cache.key("tag", synthetic.config1(n_t=5), 5)
    assert k1 != cache.key("tag", cfg, 6)
    m2 = np.array(cfg.m, copy=True)
    m2[0, 0, 0] *= 2
    assert k1 != cache.key("tag", B.KernelConfig(order=4, dims=cfg.dims, n_t=5, dt=cfg.dt, h=cfg.h, m=m2), 5)
    calls = []

    def compute():
        calls.append(1)
        return {"a": np.arange(4.0)}

    assert np.array_equal(cache.cached(k1, compute)["a"], np.arange(4.0))
    assert np.array_equal(cache.cached(k1, compute)["a"], np.arange(4.0))
    assert len(calls) == 1


def test_tti_interleaved_layout_validated_without_gpu():
    """ABI 4's fdr_tti_args.interleaved: r[i] must be p[i] + 1 float, the flag
    0 or 1, and the TMA (tti_stream) variant takes separate levels only."""
    from paper_1608_03984_b200 import tti

    lib = _lib.load()
    assert lib.fdr_tti_args_size() == ctypes.sizeof(tti._TTIArgs)
    a = tti._TTIArgs()
    a.abi_version = _lib.ABI_VERSION
    a.order = 8
    a.nx = a.ny = a.nz = 24
    a.pitch_y, a.pitch_x = 24, 24 * 24
    base = 1 << 20  # fake device addresses: validation runs before any CUDA call
    for i in range(3):
        a.p[i] = base + i * 4096
        a.r[i] = base + i * 4096 + 4
    for i in range(9):
        a.params[i] = base + 65536 + i * 4096
    a.n_steps = 1
    a.interleaved = 1
    a.r[2] = base + 2 * 4096 + 8  # not p + 1 float
    with pytest.raises(B.ValidationError, match="r\\[i\\] == p\\[i\\] \\+ 1"):
        _lib.check(lib.fdr_tti_run(ctypes.byref(a), None))
    a.r[2] = base + 2 * 4096 + 4
    a.interleaved = 2
    with pytest.raises(B.ValidationError, match="interleaved must be 0 or 1"):
        _lib.check(lib.fdr_tti_run(ctypes.byref(a), None))
    a.interleaved = 1
    a.variant = _lib.VARIANT_TMA
    with pytest.raises(B.ValidationError, match="separate p/r levels"):
        _lib.check(lib.fdr_tti_run(ctypes.byref(a), None))


def test_tb2_variant_is_known_to_the_library():
    args = _lib.AcousticArgs()
    args.abi_version = _lib.ABI_VERSION
    args.order = 8
    args.nx = args.ny = args.nz = 5  # rejected for its size, not for the variant
    args.pitch_y, args.pitch_x = 8, 40
    args.variant = _lib.VARIANT_TB2
    with pytest.raises(B.ValidationError, match="too small"):
        _lib.check(_lib.load().fdr_acoustic_run(ctypes.byref(args), None))
    args.nx = args.ny = args.nz = 16
    args.pitch_y, args.pitch_x = 16, 256
    args.variant = _lib.VARIANT_QUEUE2 + 1
    with pytest.raises(B.ValidationError, match="unknown variant"):
        _lib.check(_lib.load().fdr_acoustic_run(ctypes.byref(args), None))
