"""ctypes wrapper of oracle/libfdoracle.so -- TEST INFRASTRUCTURE ONLY.

Runs the C restatement (acoustic_ref.c) on an `oracle.acoustic.OracleState`
with the same semantics as `oracle.acoustic.simulate`, multi-threaded.
"""

import ctypes
import os

import numpy as np

from .acoustic import OracleState, kernel_constants, _m_args

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfdoracle.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle`")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int
        F = ctypes.c_float
        lib.fdo_acoustic_run.restype = I
        lib.fdo_acoustic_run.argtypes = [I, I, I, I, P, F, I, F, P, P, P, P, P, P, P, P, I, I, I,
                                         I, I, P, P, I, I, I, I]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def simulate(cfg, n_steps=None, threads=None, state: OracleState = None):
    lib = load()
    n = cfg.n_t if n_steps is None else n_steps
    r = cfg.order // 2
    st = state or OracleState(cfg.dims, r)
    centre, taps, coef = kernel_constants(cfg.order, cfg.dt, cfg.h)
    w = np.array([centre] + taps, dtype=np.float32)
    m_grid, m_scalar = _m_args(cfg.m)
    m_mode = 2 if m_grid is not None else (1 if m_scalar is not None else 0)
    if m_grid is not None:
        m_grid = np.ascontiguousarray(m_grid)
    sp = getattr(cfg, "sponge", None)
    gx = gy = gz = None
    if sp is not None:
        gx, gy, gz = (np.ascontiguousarray(np.asarray(p, dtype=np.float32)) for p in (sp.x, sp.y, sp.z))
    src = getattr(cfg, "source", None)
    series, n_series, loc = None, 0, (-1, 0, 0)
    if src is not None:
        series = np.ascontiguousarray(np.asarray(src.series).astype(np.float32).reshape(-1))
        n_series = series.size
        loc = tuple(int(c) for c in src.location)
    rec = getattr(cfg, "receivers", None)
    rec_arr, n_rec = None, 0
    if rec is not None:
        rec_arr = np.ascontiguousarray(np.asarray(rec.locations, dtype=np.int32))
        n_rec = rec_arr.shape[0]
        if st.traces is None:
            st.traces = np.zeros((max(cfg.n_t, st.it + n), n_rec), dtype=np.float32)
    for g in st.grids:
        assert g.flags.c_contiguous and g.dtype == np.float32
    threads = threads or len(os.sched_getaffinity(0))
    newest = lib.fdo_acoustic_run(
        cfg.order, *st.dims, _p(w), float(coef), m_mode,
        float(m_scalar) if m_scalar is not None else 1.0, _p(m_grid),
        *(_p(g) for g in st.grids), _p(gx), _p(gy), _p(gz), _p(series), n_series, *loc,
        n_rec, _p(rec_arr), _p(st.traces), 0 if st.traces is None else st.traces.shape[0],
        st.it, n, threads)
    g = st.grids
    st.grids = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]
    assert st.grids[2] is g[newest]
    st.it += n
    return st
