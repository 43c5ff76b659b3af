"""Full-length parity on BASELINE configs 2-5 (north_star: "the final wavefield
and receiver traces must match the reference after the same number of steps
on the same seeded inputs").

Each test builds the config's seeded inputs, checks their sha256 against the
ones the goldens were generated from (input drift on this host fails loudly
instead of comparing unrelated runs), runs the complete simulation from zero
levels through the public API (`run` / `tti_run` / `elastic_run`, AUTO
variant, i.e. the production kernels) and compares the sha256 of the final
fields and the traces with tests/golden/full_length.json.  That file is made
on the CPU by tests/golden/make_full_goldens.py from the exact C oracles
(oracle/acoustic_ref.c is pinned bit for bit to the unmodified reference
step, /root/reference/pkg/src/fdroof/kernel.py:176-222, by tests/test_oracle.py;
the run loop is the reference's kernel.py:281-284).

The bar is bit-exact.  A mismatch also reports the relative L2 on the
committed strided sample so that the size of a failure is visible.  For the
acoustic configs the float64 path (fdr_acoustic64_run) runs the same
simulation and the float32 result's relative L2 against it is recorded (the
"fp64 error is reported too" clause); set FDR_PARITY_REPORT=<path> to write
those numbers as JSON.
"""

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "full_length.json")
SAMPLES = os.path.join(HERE, "golden", "full_length_samples.npz")
ACOUSTIC = [f"config2_o{o}" for o in (2, 4, 8, 12, 16)] + ["config3"]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d > 0 else float(np.linalg.norm(a - b))


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN, encoding="utf-8") as fh:
        meta = json.load(fh)
    with np.load(SAMPLES) as z:
        samples = {k: z[k] for k in z.files}
    return meta, samples


@pytest.fixture(scope="module")
def B(cuda_device):
    import paper_1608_03984_b200 as pkg
    from paper_1608_03984_b200 import _lib

    _lib.load()
    return pkg


_REPORT = {}


def _record(name, **kw):
    _REPORT.setdefault(name, {}).update(kw)
    path = os.environ.get("FDR_PARITY_REPORT")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(_REPORT, fh, indent=1, sort_keys=True)


def _check_inputs(name, want, got):
    drift = {k: (got[k], want[k]) for k in want if k in got and got[k] != want[k]}
    assert not drift, (f"{name}: generated inputs differ from the ones the goldens were made "
                       f"from (host-dependent input generation?): {sorted(drift)}")


def _compare(name, label, arr, ref_stats, sample, stride):
    if sha(arr) == ref_stats["sha256"]:
        return
    err = rel_l2(arr[::stride, ::stride, ::stride], sample) if arr.ndim == 3 else float("nan")
    pytest.fail(f"{name}: {label} differs from the C oracle's full-length run "
                f"(rel L2 on the strided sample {err:.3e})")


@pytest.mark.parametrize("name", ACOUSTIC)
def test_acoustic_full_length(B, golden, name):
    import torch

    from paper_1608_03984_b200.synthetic import config2, config3

    meta, samples = golden
    g = meta[name]
    cfg = config2(order=g["order"]) if name.startswith("config2") else config3()
    assert cfg.n_t == g["n_t"] and list(cfg.dims) == g["dims"]
    inputs = {"m": sha(np.asarray(cfg.m, np.float32)),
              "series": sha(np.asarray(cfg.source.series).astype(np.float32)),
              "receivers": sha(np.asarray(cfg.receivers.locations, np.int32)),
              "sponge": sha(np.concatenate([np.asarray(p, np.float32) for p in
                                            (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
              "dt": float(cfg.dt)}
    _check_inputs(name, g["inputs"], inputs)

    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg)
    torch.cuda.synchronize()
    assert fld.it == cfg.n_t
    final = fld.numpy(2)
    assert np.isfinite(final).all(), f"{name}: non-finite values in the final wavefield"
    traces = fld.traces.cpu().numpy()[: cfg.n_t]
    _compare(name, "final wavefield", final, g["final"], samples[f"{name}/final"],
             g["field_stride"])
    assert sha(fld.numpy(1)) == g["prev"]["sha256"], f"{name}: previous level differs"
    if sha(traces) != g["traces"]["sha256"]:
        err = rel_l2(traces[:, ::g["trace_stride"]], samples[f"{name}/traces"])
        pytest.fail(f"{name}: traces differ from the C oracle's (rel L2 on the sample {err:.3e})")

    # the float64 path on the same inputs: the float32 error, reported
    f64 = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    B.run(f64, cfg)
    torch.cuda.synchronize()
    ref = f64.numpy(2)
    tr64 = f64.traces.cpu().numpy()[: cfg.n_t]
    e_field = rel_l2(final, ref)
    # at config 2 the 512 receivers at z = 2 lie ~250 points from the source:
    # after 500 steps only the numerical precursor reaches them, which the
    # float64 path resolves (|u| ~ 1e-40 and below) and float32 flushes to
    # zero; a relative error of such traces says nothing, so it is reported
    # only where the float64 traces are within float32's normal range
    t_scale = float(np.abs(tr64).max())
    e_traces = rel_l2(traces, tr64) if t_scale > 1e-30 else None
    _record(name, bitexact_vs_oracle=True, n_t=cfg.n_t, order=cfg.order, dims=list(cfg.dims),
            f32_rel_l2_vs_f64_field=e_field, f32_rel_l2_vs_f64_traces=e_traces,
            f64_traces_maxabs=t_scale, f32_traces_maxabs=float(np.abs(traces).max()))
    del f64, fld
    torch.cuda.empty_cache()
    assert e_field < 1e-3
    assert e_traces is None or e_traces < 1e-3


def test_tti_config4_full_length(B, golden):
    import torch

    from paper_1608_03984_b200 import tti

    meta, samples = golden
    g = meta["config4"]
    cfg = tti.config4()
    prm = cfg.params()
    inputs = {f"param_{k}": sha(prm[k]) for k in tti.PARAM_NAMES}
    inputs.update(series=sha(np.asarray(cfg.source.series).astype(np.float32)),
                  receivers=sha(np.asarray(cfg.receivers.locations, np.int32)),
                  sponge=sha(np.concatenate([np.asarray(p, np.float32) for p in
                                             (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
                  dt=float(cfg.dt))
    _check_inputs("config4", g["inputs"], inputs)
    del prm
    f = tti.TTIWavefield.allocate(cfg.dims, cfg.halo)
    tti.tti_run(f, cfg)
    torch.cuda.synchronize()
    for fld in ("p", "r"):
        arr = f.numpy(fld)
        assert np.isfinite(arr).all()
        _compare("config4", f"final {fld}", arr, g[f"{fld}_final"], samples[f"config4/{fld}"],
                 g["field_stride"])
    traces = f.traces.cpu().numpy()[: cfg.n_t]
    if sha(traces) != g["traces"]["sha256"]:
        err = rel_l2(traces[:, ::g["trace_stride"]], samples["config4/traces"])
        pytest.fail(f"config4: traces differ (rel L2 on the sample {err:.3e})")
    # the float64 path (fdr_tti64_run) on the same model: the float32 error
    p32, r32 = f.numpy("p"), f.numpy("r")
    del f
    torch.cuda.empty_cache()
    f64 = tti.TTIWavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    tti.tti_run(f64, cfg)
    e_p, e_r = rel_l2(p32, f64.numpy("p")), rel_l2(r32, f64.numpy("r"))
    tr64 = f64.traces.cpu().numpy()[: cfg.n_t]
    t_scale = float(np.abs(tr64).max())
    e_tr = rel_l2(traces, tr64) if t_scale > 1e-30 else None
    _record("config4", bitexact_vs_oracle=True, n_t=cfg.n_t, f32_rel_l2_vs_f64_p=e_p,
            f32_rel_l2_vs_f64_r=e_r, f32_rel_l2_vs_f64_traces=e_tr, f64_traces_maxabs=t_scale)
    del f64
    torch.cuda.empty_cache()
    assert e_p < 1e-3 and e_r < 1e-3
    assert e_tr is None or e_tr < 1e-3


def test_elastic_config5_full_length(B, golden):
    import torch

    from paper_1608_03984_b200 import elastic

    meta, samples = golden
    g = meta["config5"]
    cfg = elastic.config5()
    prm = cfg.params()
    inputs = {f"param_{k}": sha(prm[k]) for k in ("bs", "lam", "mu")}
    inputs.update(series=sha(np.asarray(cfg.source.series).astype(np.float32)),
                  receivers=sha(np.asarray(cfg.receivers.locations, np.int32)),
                  sponge=sha(np.concatenate([np.asarray(p, np.float32) for p in
                                             (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
                  dt=float(cfg.dt))
    _check_inputs("config5", g["inputs"], inputs)
    f = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    elastic.elastic_run(f, cfg)
    torch.cuda.synchronize()
    for k in elastic.FIELDS:
        arr = f.numpy(k)
        assert np.isfinite(arr).all()
        _compare("config5", f"final {k}", arr, g[k], samples[f"config5/{k}"], g["field_stride"])
    traces = f.traces.cpu().numpy()[: cfg.n_t]
    if sha(traces) != g["traces"]["sha256"]:
        err = rel_l2(traces[:, ::g["trace_stride"]], samples["config5/traces"])
        pytest.fail(f"config5: traces differ (rel L2 on the sample {err:.3e})")
    # the float64 path (fdr_elastic64_run) on the same model: the float32 error
    f32 = {k: f.numpy(k) for k in elastic.FIELDS}
    del f
    torch.cuda.empty_cache()
    f64 = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    elastic.elastic_run(f64, cfg)
    errs = {k: rel_l2(f32[k], f64.numpy(k)) for k in elastic.FIELDS}
    tr64 = f64.traces.cpu().numpy()[: cfg.n_t]
    t_scale = float(np.abs(tr64).max())
    e_tr = rel_l2(traces, tr64) if t_scale > 1e-30 else None
    _record("config5", bitexact_vs_oracle=True, n_t=cfg.n_t,
            f32_rel_l2_vs_f64_fields=errs, f32_rel_l2_vs_f64_traces=e_tr, f64_traces_maxabs=t_scale)
    del f64
    torch.cuda.empty_cache()
    assert max(errs.values()) < 1e-3
    assert e_tr is None or e_tr < 1e-3


@pytest.mark.parametrize("order", [12, 16])
def test_fma_variant_drift_within_north_star_tolerance(B, order):
    """The opt-in FMA variant (taps contracted, two roundings instead of three;
    not bit-exact) against the exact kernel over the full config-2 run (512^3,
    500 steps): relative L2 of the final level <= 1e-5, the north_star
    tolerance.  At order 8 the same run drifts to 1.4e-5
    (profiles/r02_fma_variant_drift.jsonl), so AUTO and the headline keep the
    bit-exact kernel at every order."""
    import torch

    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=order)
    res = {}
    for variant in ("queue", "fma"):
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
        B.run(fld, cfg, variant=variant)
        res[variant] = fld.numpy(2)
        del fld
        torch.cuda.empty_cache()
    err = rel_l2(res["fma"], res["queue"])
    _record(f"config2_o{order}", fma_rel_l2_vs_exact_field=err)
    assert 0.0 < err <= 1e-5
