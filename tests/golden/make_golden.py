"""Generate the golden fixtures from the REAL reference (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified `fdroof` package (/root/reference/pkg/src) and records
outputs of `fdroof.kernel.step` (kernel.py:176-222) and `oracle_step`
(kernel.py:225-254) on seeded inputs.  Cases mirror the reference's own
kernel tests (tests/test_kernel.py:33-195, tests/test_acceptance.py:152-223)
plus BASELINE config 1 (64^3, order 4, 100 steps).  The sponge / receiver
extension (SURVEY.md §8(a')) is driven here around the unmodified reference
`step`: the step runs with a source-free config, then the new level is
multiplied by the taper, then series[it] is injected and receivers sampled.

Outputs: acoustic_golden.npz (small arrays) and acoustic_golden.json
(sha256 of every final level / trace array, for large cases).  Nothing here
runs on the GPU box; the fixtures travel, the reference does not.
"""

import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from fdroof import kernel as K  # noqa: E402  (the unmodified reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return hashlib.sha256(a.tobytes()).hexdigest()


def random_levels(fld, dims, seed):
    rng = np.random.default_rng(seed)
    fld.interior(2)[...] = rng.standard_normal(dims).astype(np.float32)
    fld.interior(1)[...] = rng.standard_normal(dims).astype(np.float32)


def ricker(f0, dt, nt):
    tau = np.arange(nt, dtype=np.float64) * dt - 1.0 / f0
    a = (math.pi * f0 * tau) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def cerjan(n, width=10, alpha=0.03):
    i = np.arange(n)
    d = np.minimum(i, n - 1 - i).astype(np.float64)
    return np.where(d < width, np.exp(-(alpha * (width - d)) ** 2), 1.0).astype(np.float32)


def run_extended(cfg_nosrc, series, loc, rec, taper, n_steps):
    """Reference step + sponge taper + injection + receivers (§8(a'))."""
    fld = K.Wavefield.allocate(cfg_nosrc.dims, cfg_nosrc.halo)
    r = fld.halo
    traces = np.zeros((n_steps, len(rec)), dtype=np.float32)
    for _ in range(n_steps):
        it = fld.it
        K.step(fld, cfg_nosrc)
        new = fld.interior(2)
        if taper is not None:
            new *= taper
        if it < len(series):
            x, y, z = (c + r for c in loc)
            fld.grids[2][x, y, z] += np.float32(series[it])
        traces[it] = new[rec[:, 0], rec[:, 1], rec[:, 2]]
    return fld, traces


def main():
    arrays, meta = {}, {}

    # impulse known answer (test_kernel.py:42-52)
    cfg = K.KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.3)
    fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
    fld.interior(2)[4, 4, 4] = 1.0
    K.step(fld, cfg)
    arrays["impulse_o2"] = fld.interior(2).copy()

    # step vs random levels, orders 2..16, 20^3, 3 steps (test_kernel.py:67-77)
    for order in (2, 4, 6, 8, 12, 16):
        dt = 0.5 * K.max_stable_dt(order, 1.0)
        cfg = K.KernelConfig(order=order, dims=(20, 20, 20), n_t=3, dt=dt)
        fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
        random_levels(fld, cfg.dims, order)
        for _ in range(3):
            K.step(fld, cfg)
        # reference fp64 oracle on the same start, for the fp64-error report
        ob = K.Wavefield.allocate(cfg.dims, cfg.halo)
        random_levels(ob, cfg.dims, order)
        for _ in range(3):
            K.oracle_step(ob, cfg)
        diff = np.abs(fld.interior(2).astype(np.float64) - ob.interior(2))
        meta[f"random_o{order}"] = {"order": order, "dims": [20, 20, 20], "dt": dt, "seed": order,
                                    "steps": 3, "final_sha256": sha(fld.interior(2)),
                                    "prev_sha256": sha(fld.interior(1)),
                                    "f64oracle_sha256": sha(ob.interior(2)),
                                    "f64oracle_maxabs": float(diff.max()),
                                    "f64oracle_rel_l2": float(np.linalg.norm(diff) / np.linalg.norm(ob.interior(2).astype(np.float64)))}

    # varying slowness (test_kernel.py:80-88), plus scalar m != 1
    m = 1.0 + 0.5 * np.random.default_rng(3).random((16, 16, 16)).astype(np.float32)
    dt = 0.5 * K.max_stable_dt(4, 1.0, m)
    cfg = K.KernelConfig(order=4, dims=(16, 16, 16), n_t=1, dt=dt, m=m)
    fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
    random_levels(fld, cfg.dims, 11)
    for _ in range(2):
        K.step(fld, cfg)
    meta["varm_o4"] = {"order": 4, "dims": [16, 16, 16], "dt": dt, "seed": 11, "steps": 2,
                       "final_sha256": sha(fld.interior(2))}

    dt = 0.5 * K.max_stable_dt(6, 1.0, 1.7)
    cfg = K.KernelConfig(order=6, dims=(14, 15, 17), n_t=1, dt=dt, m=1.7)
    fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
    random_levels(fld, cfg.dims, 21)
    for _ in range(2):
        K.step(fld, cfg)
    meta["scalarm_o6"] = {"order": 6, "dims": [14, 15, 17], "dt": dt, "seed": 21, "steps": 2,
                          "m": 1.7, "final_sha256": sha(fld.interior(2))}

    # mirror symmetry with a centred source (test_kernel.py:55-64)
    dt = 0.5 * K.max_stable_dt(8, 1.0)
    series = np.array([1.0, 0.5, -0.25, 0.1], dtype=np.float32)
    cfg = K.KernelConfig(order=8, dims=(17, 17, 17), n_t=4, dt=dt,
                         source=K.Source((8, 8, 8), series))
    fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
    for _ in range(4):
        K.step(fld, cfg)
    arrays["mirror_o8"] = fld.interior(2).copy()
    meta["mirror_o8"] = {"order": 8, "dims": [17, 17, 17], "dt": dt, "steps": 4}

    # ragged dims, odd nz (device row padding), sources off-centre
    for order, dims, seed in ((2, (13, 11, 9), 31), (10, (23, 21, 22), 32), (16, (33, 34, 35), 33)):
        dt = 0.5 * K.max_stable_dt(order, 1.0)
        series = np.random.default_rng(seed).standard_normal(6)
        loc = (dims[0] // 3, dims[1] - 2, 1)
        cfg = K.KernelConfig(order=order, dims=dims, n_t=6, dt=dt,
                             source=K.Source(loc, series))
        fld = K.Wavefield.allocate(cfg.dims, cfg.halo)
        random_levels(fld, cfg.dims, seed)
        for _ in range(6):
            K.step(fld, cfg)
        key = f"ragged_o{order}"
        meta[key] = {"order": order, "dims": list(dims), "dt": dt, "seed": seed, "steps": 6,
                     "source": list(loc), "final_sha256": sha(fld.interior(2)),
                     "prev_sha256": sha(fld.interior(1))}

    # BASELINE config 1 (64^3, order 4, h=10, two-layer, 100 steps)
    dims, h, order, nt = (64, 64, 64), 10.0, 4, 100
    v = np.empty(dims)
    v[:, :, :32] = 1500.0
    v[:, :, 32:] = 2500.0
    m = (1.0 / np.square(v)).astype(np.float32)
    dt = 0.4 * h / 2500.0
    series = ricker(10.0, dt, nt)
    loc = (32, 32, 32)
    rec = np.stack([np.arange(64), np.full(64, 32), np.full(64, 2)], axis=1).astype(np.int32)
    cfg_nosrc = K.KernelConfig(order=order, dims=dims, n_t=nt, dt=dt, h=h, m=m)
    # (a) plain reference path: no sponge -> exactly repeated fdroof step
    cfg_src = K.KernelConfig(order=order, dims=dims, n_t=nt, dt=dt, h=h, m=m,
                             source=K.Source(loc, series))
    fld = K.Wavefield.allocate(dims, 2)
    tr = np.zeros((nt, 64), dtype=np.float32)
    for _ in range(nt):
        it = fld.it
        K.step(fld, cfg_src)
        tr[it] = fld.interior(2)[rec[:, 0], rec[:, 1], rec[:, 2]]
    meta["config1_nosponge"] = {"final_sha256": sha(fld.interior(2)), "traces_sha256": sha(tr),
                                "final_l2": float(np.linalg.norm(fld.interior(2).astype(np.float64)))}
    arrays["config1_nosponge_traces"] = tr
    # (b) with the 10-point sponge extension
    taper = (cerjan(64)[:, None, None] * cerjan(64)[None, :, None]) * cerjan(64)[None, None, :]
    fld2, tr2 = run_extended(cfg_nosrc, series, loc, rec, taper, nt)
    assert fld2.halo_is_zero()
    meta["config1"] = {"final_sha256": sha(fld2.interior(2)), "traces_sha256": sha(tr2),
                       "final_l2": float(np.linalg.norm(fld2.interior(2).astype(np.float64))),
                       "dt": dt}
    arrays["config1_traces"] = tr2
    arrays["config1_final_slice"] = fld2.interior(2)[:, 32, :].copy()

    # a larger order-8 smooth-model case for the GPU parity tests
    dims, order, nt = (96, 80, 72), 8, 40
    rng = np.random.default_rng(5)
    v = 1500.0 + 3000.0 * rng.random(dims)
    m = (1.0 / np.square(v)).astype(np.float32)
    dt = 0.4 * 10.0 / float(v.max())
    series = ricker(15.0, dt, nt)
    rec = np.stack([np.arange(96), np.full(96, 40), np.full(96, 2)], axis=1).astype(np.int32)
    cfg_nosrc = K.KernelConfig(order=order, dims=dims, n_t=nt, dt=dt, h=10.0, m=m)
    taper = (cerjan(96)[:, None, None] * cerjan(80)[None, :, None]) * cerjan(72)[None, None, :]
    fld3, tr3 = run_extended(cfg_nosrc, series, (48, 40, 36), rec, taper, nt)
    meta["medium_o8"] = {"final_sha256": sha(fld3.interior(2)), "traces_sha256": sha(tr3),
                         "dims": list(dims), "dt": dt, "steps": nt, "seed": 5}

    meta["_generator"] = "tests/golden/make_golden.py with fdroof from /root/reference/pkg/src"
    meta["_numpy"] = np.__version__
    np.savez_compressed(os.path.join(HERE, "acoustic_golden.npz"), **arrays)
    with open(os.path.join(HERE, "acoustic_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays and", len(meta), "meta entries")


if __name__ == "__main__":
    main()
