"""TTI oracles -- TEST INFRASTRUCTURE ONLY.

Two independent restatements of the TTI pseudo-acoustic system of
PAPER.md:804-829 (no reference implementation exists, SURVEY.md §8(a')):

* `simulate_c` runs oracle/tti_ref.c, the exact float32 operation sequence the
  CUDA kernels must match bit for bit (the parity oracle);
* `simulate_f64` is a float64 numpy implementation written from the paper's
  operator definitions: G_zz, G_xx + G_yy assembled from the paper's rotated
  operators (with the sign of the G_yy cross term corrected, SURVEY.md
  App. B) using float64 derivative stencils.  It is used to check the
  float32 path's accuracy ("the fp64 error is reported too") and the operator
  identity G_xx + G_yy + G_zz = laplacian.
"""

import ctypes
import os

import numpy as np

from .acoustic import fornberg_weights
from .cref import load as _load_c

# ----------------------------------------------------------------- C oracle


def _p(a):
    return None if a is None else a.ctypes.data


class TTIState:
    """Zero-padded float32 levels of p and r ([scratch, prev, cur]) + it + traces."""

    def __init__(self, dims, halo):
        self.dims = tuple(dims)
        self.halo = halo
        shape = tuple(d + 2 * halo for d in dims)
        self.p = [np.zeros(shape, np.float32) for _ in range(3)]
        self.r = [np.zeros(shape, np.float32) for _ in range(3)]
        self.it = 0
        self.traces = None

    def interior(self, field="p", level=2):
        h = self.halo
        g = (self.p if field == "p" else self.r)[level]
        return g[h:-h, h:-h, h:-h]


def simulate_c(cfg, params, w2, w1, n_steps=None, state=None, threads=None):
    """Run the exact float32 C oracle; `params` = the 9 float32 grids of
    TTIConfig.params(), (w2, w1) = tti_weights_f32(order)."""
    lib = _load_c()
    fn = lib.fdo_tti_run
    P, I = ctypes.c_void_p, ctypes.c_int
    fn.restype = I
    fn.argtypes = [I, I, I, I, P, P, P] + [P] * 6 + [P] * 3 + [P, I, I, I, I, I, P, P, I, I, I, I]
    n = cfg.n_t if n_steps is None else n_steps
    st = state or TTIState(cfg.dims, cfg.order // 2)
    names = ("k", "a", "b", "cxx", "cyy", "czz", "cxy", "cyz", "cxz")
    prm = [np.ascontiguousarray(params[k], dtype=np.float32) for k in names]
    prm_ptrs = (ctypes.c_void_p * 9)(*[a.ctypes.data for a in prm])
    sp = getattr(cfg, "sponge", None)
    gx = gy = gz = None
    if sp is not None:
        gx, gy, gz = (np.ascontiguousarray(v, dtype=np.float32) for v in (sp.x, sp.y, sp.z))
    series, n_series, loc = None, 0, (-1, 0, 0)
    if cfg.source is not None:
        series = np.ascontiguousarray(np.asarray(cfg.source.series).astype(np.float32).reshape(-1))
        n_series = series.size
        loc = tuple(int(c) for c in cfg.source.location)
    rec, n_rec = None, 0
    if cfg.receivers is not None:
        rec = np.ascontiguousarray(cfg.receivers.locations, dtype=np.int32)
        n_rec = rec.shape[0]
        if st.traces is None:
            st.traces = np.zeros((max(cfg.n_t, st.it + n), n_rec), np.float32)
    threads = threads or len(os.sched_getaffinity(0))
    w2 = np.ascontiguousarray(w2, np.float32)
    w1 = np.ascontiguousarray(w1, np.float32)
    newest = fn(cfg.order, *cfg.dims, _p(w2), _p(w1), ctypes.cast(prm_ptrs, ctypes.c_void_p),
                *(_p(g) for g in st.p), *(_p(g) for g in st.r), _p(gx), _p(gy), _p(gz),
                _p(series), n_series, *loc, n_rec, _p(rec), _p(st.traces),
                0 if st.traces is None else st.traces.shape[0], st.it, n, threads)
    for lv in (st.p, st.r):
        g = list(lv)
        lv[:] = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]
    assert newest == (2 + n) % 3
    st.it += n
    return st


# ------------------------------------------------------------- fp64 oracle


def _shift(u, axis, s):
    """u shifted by s along axis with zero fill (u(x+s))."""
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


def derivatives_f64(u, order):
    """Undivided float64 derivatives of an interior-shaped field with a zero
    halo: second derivatives along x, y, z and the mixed ones, from exact
    Fornberg weights."""
    r = order // 2
    w2 = [float(w) for w in fornberg_weights(2, order)]
    w1 = [float(w) for w in fornberg_weights(1, order)]

    def d2(v, ax):
        acc = w2[r] * v
        for j in range(1, r + 1):
            acc = acc + w2[r + j] * (_shift(v, ax, j) + _shift(v, ax, -j))
        return acc

    def d1(v, ax):
        acc = np.zeros_like(v)
        for j in range(1, r + 1):
            acc = acc + w1[r + j] * (_shift(v, ax, j) - _shift(v, ax, -j))
        return acc

    dx, dy, dz = d1(u, 0), d1(u, 1), d1(u, 2)
    return {"xx": d2(u, 0), "yy": d2(u, 1), "zz": d2(u, 2),
            "xy": d1(dy, 0), "xz": d1(dz, 0), "yz": d1(dz, 1)}


def paper_operators(d, theta, phi):
    """G_xx, G_yy, G_zz of PAPER.md:820-829 with the G_yy cross term corrected
    to -sin(2 phi) (the paper prints sin(2 phi)^2)."""
    st, ct, sp, cp = np.sin(theta), np.cos(theta), np.sin(phi), np.cos(phi)
    s2p, s2t = np.sin(2 * phi), np.sin(2 * theta)
    gxx = (cp * cp * ct * ct * d["xx"] + sp * sp * ct * ct * d["yy"] + st * st * d["zz"]
           + s2p * ct * ct * d["xy"] - sp * s2t * d["yz"] - cp * s2t * d["xz"])
    gyy = sp * sp * d["xx"] + cp * cp * d["yy"] - s2p * d["xy"]
    gzz = (cp * cp * st * st * d["xx"] + sp * sp * st * st * d["yy"] + ct * ct * d["zz"]
           + s2p * st * st * d["xy"] + sp * s2t * d["yz"] + cp * s2t * d["xz"])
    return gxx, gyy, gzz


def simulate_f64(cfg, n_steps=None):
    """float64 time stepping of the paper's TTI system (paper operators,
    float64 parameters from the config's physical grids).  Returns
    (p, r, traces) after n_steps, interior-shaped."""
    n = cfg.n_t if n_steps is None else n_steps
    shape = tuple(cfg.dims)

    def grid(v):
        return np.broadcast_to(np.asarray(v, dtype=np.float64), shape)

    m = grid(np.asarray(cfg.m, dtype=np.float32).astype(np.float64))
    eps, dl, th, ph = (grid(getattr(cfg, k)) for k in ("epsilon", "delta", "theta", "phi"))
    k = cfg.dt * cfg.dt / (cfg.h * cfg.h * m)
    a, b = 1.0 + 2.0 * eps, np.sqrt(1.0 + 2.0 * dl)
    taper = None
    if cfg.sponge is not None:
        gx, gy, gz = (np.asarray(v, np.float64) for v in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
        taper = gx[:, None, None] * gy[None, :, None] * gz[None, None, :]
    p0, p1 = np.zeros(shape), np.zeros(shape)
    r0, r1 = np.zeros(shape), np.zeros(shape)
    traces = None
    if cfg.receivers is not None:
        traces = np.zeros((n, cfg.receivers.count))
    for it in range(n):
        dp = derivatives_f64(p1, cfg.order)
        dr = derivatives_f64(r1, cfg.order)
        gxx, gyy, _ = paper_operators(dp, th, ph)
        _, _, gzz_r = paper_operators(dr, th, ph)
        hp = gxx + gyy
        pn = 2 * p1 - p0 + k * (a * hp + b * gzz_r)
        rn = 2 * r1 - r0 + k * (b * hp + gzz_r)
        if taper is not None:
            pn *= taper
            rn *= taper
        if cfg.source is not None and it < len(cfg.source.series):
            x, y, z = cfg.source.location
            pn[x, y, z] += float(np.float32(cfg.source.series[it]))
            rn[x, y, z] += float(np.float32(cfg.source.series[it]))
        if traces is not None:
            loc = cfg.receivers.locations
            traces[it] = pn[loc[:, 0], loc[:, 1], loc[:, 2]]
        p0, p1 = p1, pn
        r0, r1 = r1, rn
    return p1, r1, traces
