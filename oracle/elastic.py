"""Elastic velocity-stress oracles -- TEST INFRASTRUCTURE ONLY.

* `simulate_c` runs oracle/elastic_ref.c, the exact float32 sequence the CUDA
  kernels must reproduce bit for bit (parity oracle);
* `simulate_f64` is an independent float64 numpy implementation of the same
  staggered-grid system (Virieux 1986) from exact staggered weights, used for
  the accuracy check (no reference implementation exists, SURVEY.md §8(a')).
"""

import ctypes
import os

import numpy as np

from .cref import load as _load_c

FIELDS = ("vx", "vy", "vz", "sxx", "syy", "szz", "sxy", "sxz", "syz")


def _p(a):
    return None if a is None else a.ctypes.data


class ElasticState:
    def __init__(self, dims, halo):
        self.dims = tuple(dims)
        self.halo = halo
        shape = tuple(d + 2 * halo for d in dims)
        self.f = {k: np.zeros(shape, np.float32) for k in FIELDS}
        self.it = 0
        self.traces = None

    def interior(self, name):
        h = self.halo
        return self.f[name][h:-h, h:-h, h:-h]


def simulate_c(cfg, params, c, n_steps=None, state=None, threads=None):
    lib = _load_c()
    fn = lib.fdo_elastic_run
    P, I = ctypes.c_void_p, ctypes.c_int
    fn.restype = I
    fn.argtypes = [I, I, I, I, P, P, P, P, P, P, P, P, P, I, I, I, I, I, P, P, I, I, I, I]
    n = cfg.n_t if n_steps is None else n_steps
    st = state or ElasticState(cfg.dims, cfg.order // 2)
    bs, lam, mu = (np.ascontiguousarray(params[k], np.float32) for k in ("bs", "lam", "mu"))
    fptr = (ctypes.c_void_p * 9)(*[st.f[k].ctypes.data for k in FIELDS])
    sp = cfg.sponge
    gx = gy = gz = None
    if sp is not None:
        gx, gy, gz = (np.ascontiguousarray(v, np.float32) for v in (sp.x, sp.y, sp.z))
    series, n_series, loc = None, 0, (-1, 0, 0)
    if cfg.source is not None:
        series = np.ascontiguousarray(np.asarray(cfg.source.series).astype(np.float32).reshape(-1))
        n_series = series.size
        loc = tuple(int(v) for v in cfg.source.location)
    rec, n_rec = None, 0
    if cfg.receivers is not None:
        rec = np.ascontiguousarray(cfg.receivers.locations, np.int32)
        n_rec = rec.shape[0]
        if st.traces is None:
            st.traces = np.zeros((max(cfg.n_t, st.it + n), n_rec), np.float32)
    threads = threads or len(os.sched_getaffinity(0))
    c = np.ascontiguousarray(c, np.float32)
    fn(cfg.order, *cfg.dims, _p(c), _p(bs), _p(lam), _p(mu), ctypes.cast(fptr, ctypes.c_void_p),
       _p(gx), _p(gy), _p(gz), _p(series), n_series, *loc, n_rec, _p(rec), _p(st.traces),
       0 if st.traces is None else st.traces.shape[0], st.it, n, threads)
    st.it += n
    return st


def _shift(u, axis, s):
    out = np.zeros_like(u)
    n = u.shape[axis]
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if s >= 0:
        src[axis], dst[axis] = slice(s, n), slice(0, n - s)
    else:
        src[axis], dst[axis] = slice(0, n + s), slice(-s, n)
    out[tuple(dst)] = u[tuple(src)]
    return out


def simulate_f64(cfg, n_steps=None):
    """float64 staggered velocity-stress stepping; returns (fields dict, vz traces)."""
    from paper_1608_03984_b200.stencils import staggered_first_derivative_weights

    n = cfg.n_t if n_steps is None else n_steps
    r = cfg.order // 2
    c = [0.0] + [float(v) for v in staggered_first_derivative_weights(cfg.order)]
    shape = tuple(cfg.dims)

    def grid(v):
        return np.broadcast_to(np.asarray(v, dtype=np.float64), shape)

    vp, vs, rho = grid(cfg.vp), grid(cfg.vs), grid(cfg.rho)
    muv = rho * vs * vs
    lamv = rho * vp * vp - 2.0 * muv
    f = cfg.dt / cfg.h
    bs, lam, mu = f / rho, f * lamv, f * muv

    def F(u, ax):
        return sum(c[k] * (_shift(u, ax, k) - _shift(u, ax, 1 - k)) for k in range(1, r + 1))

    def B(u, ax):
        return sum(c[k] * (_shift(u, ax, k - 1) - _shift(u, ax, -k)) for k in range(1, r + 1))

    taper = 1.0
    if cfg.sponge is not None:
        gx, gy, gz = (np.asarray(v, np.float64) for v in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
        taper = gx[:, None, None] * gy[None, :, None] * gz[None, None, :]
    fld = {k: np.zeros(shape) for k in FIELDS}
    traces = None if cfg.receivers is None else np.zeros((n, cfg.receivers.count))
    for it in range(n):
        s = fld
        s["vx"] = (s["vx"] + bs * (B(s["sxy"], 1) + B(s["sxz"], 2) + F(s["sxx"], 0))) * taper
        s["vy"] = (s["vy"] + bs * (F(s["syy"], 1) + B(s["syz"], 2) + B(s["sxy"], 0))) * taper
        s["vz"] = (s["vz"] + bs * (B(s["syz"], 1) + F(s["szz"], 2) + B(s["sxz"], 0))) * taper
        ex, ey, ez = B(s["vx"], 0), B(s["vy"], 1), B(s["vz"], 2)
        l2m = lam + 2.0 * mu
        sxx = s["sxx"] + l2m * ex + lam * (ey + ez)
        syy = s["syy"] + l2m * ey + lam * (ex + ez)
        szz = s["szz"] + l2m * ez + lam * (ex + ey)
        sxy = s["sxy"] + mu * (F(s["vx"], 1) + F(s["vy"], 0))
        sxz = s["sxz"] + mu * (F(s["vx"], 2) + F(s["vz"], 0))
        syz = s["syz"] + mu * (F(s["vy"], 2) + F(s["vz"], 1))
        for k, v in (("sxx", sxx), ("syy", syy), ("szz", szz), ("sxy", sxy), ("sxz", sxz),
                     ("syz", syz)):
            s[k] = v * taper
        if cfg.source is not None and it < len(cfg.source.series):
            x, y, z = cfg.source.location
            q = float(np.float32(cfg.source.series[it]))
            for k in ("sxx", "syy", "szz"):
                s[k][x, y, z] += q
        if traces is not None:
            loc = cfg.receivers.locations
            traces[it] = s["vz"][loc[:, 0], loc[:, 1], loc[:, 2]]
    return fld, traces
