"""Isotropic elastic velocity-stress time stepping on B200 (BASELINE config 5).

The reference has no velocity-stress kernel: its elastic catalogue entries are
a displacement-form anisotropic kernel (/root/reference/pkg/src/fdroof/
equations.py:156-177), so this system is new (SURVEY.md
§8(a')).  Virieux staggered grid, order-2r staggered first derivatives (exact
Taylor weights on offsets +-(k-1/2), stencils.staggered_first_derivative_weights),
3 velocities + 6 stresses updated in place, one velocity pass and one stress
pass per time step.  The float32 operation sequence is defined by the parity
oracle oracle/elastic_ref.c; accuracy is checked against a float64 oracle.
Parameters: bs = dt/(h rho), lam = dt lambda/h, mu = dt mu/h (float32, from
float64), lambda = rho (vp^2 - 2 vs^2), mu = rho vs^2.
"""

import ctypes
import math
import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._inputs import InputGuard, cached_plan, config_inputs, grow_traces, host_tensor, to_host
from .errors import ValidationError
from .kernel import Receivers, Source, Sponge, StabilityWarning, row_pitch
from .stencils import staggered_first_derivative_weights

FIELDS = ("vx", "vy", "vz", "sxx", "syy", "szz", "sxy", "sxz", "syz")
ELASTIC_BYTES_PER_POINT = 84  # 9 fields read + 9 written + 3 parameters


def elastic_flops_per_point(order: int) -> int:
    """FLOPs of the defined update with FMA counted as 2: 15 staggered
    derivatives of 2r taps (r subtractions + r-1 FMAs + 1 multiply = 3r FLOPs
    ... counted as 2 per tap pair) plus the combination terms."""
    r = order // 2
    deriv = 15 * (4 * r - 1)            # c1*(a-b) (2) + (r-1) x [sub + fma] (3 each) ~ 4r-1
    combine = 3 * (2 + 2) + 3 * (2 + 2 + 2) + 3 * (1 + 2) + 2  # vel + normal + shear + l2m
    return deriv + combine


def elastic_weights_f32(order: int) -> np.ndarray:
    """c[0..r] float32 (c[0] unused): staggered d/dx weights on +-(k-1/2)."""
    c = staggered_first_derivative_weights(order)
    return np.array([0.0] + [float(v) for v in c], dtype=np.float32)


def elastic_weights_f64(order: int) -> np.ndarray:
    """c[0..r] float64 of the exact rationals (the float64 path)."""
    c = staggered_first_derivative_weights(order)
    return np.array([0.0] + [float(v) for v in c], dtype=np.float64)


def elastic_max_stable_dt(order: int, h: float, vp_max: float) -> float:
    """Staggered leapfrog bound dt <= h / (sqrt(3) vp_max sum|c_k|)."""
    s = float(sum(abs(v) for v in staggered_first_derivative_weights(order)))
    return h / (math.sqrt(3.0) * vp_max * s)


@dataclass
class ElasticConfig:
    order: int
    dims: tuple
    n_t: int
    dt: float
    h: float
    vp: object
    vs: object
    rho: object
    source: Optional[Source] = None
    receivers: Optional[Receivers] = None
    sponge: Optional[Sponge] = None

    def __post_init__(self):
        if self.order < 2 or self.order % 2 != 0 or self.order > 16:
            raise ValidationError(f"order must be even and within [2, 16], got {self.order}")
        if len(self.dims) != 3 or any(d < self.order + 1 for d in self.dims):
            raise ValidationError(f"interior dims {self.dims} too small for order {self.order}")
        if self.n_t < 0 or self.dt <= 0 or self.h <= 0:
            raise ValidationError("n_t must be >= 0 and dt, h positive")
        for name in ("vp", "vs", "rho"):
            v = getattr(self, name)
            if not np.isscalar(v) and np.shape(v) != tuple(self.dims):
                raise ValidationError(f"{name} grid must match interior dims")
            if np.min(v) <= 0:
                raise ValidationError(f"{name} must be positive")
        if np.any(np.asarray(self.vs, dtype=np.float64) * math.sqrt(2.0) >=
                  np.asarray(self.vp, dtype=np.float64)):
            raise ValidationError("needs vp > sqrt(2) vs (positive lambda)")
        if self.source is not None:
            loc = self.source.location
            if len(loc) != 3 or any(not 0 <= c < d for c, d in zip(loc, self.dims)):
                raise ValidationError(f"source location {loc} outside interior")
        if self.receivers is not None:
            loc = self.receivers.locations
            if (loc < 0).any() or (loc >= np.asarray(self.dims)).any():
                raise ValidationError("receiver location outside interior")
        if self.sponge is not None and tuple(
                len(p) for p in (self.sponge.x, self.sponge.y, self.sponge.z)) != tuple(self.dims):
            raise ValidationError("sponge profile lengths must match interior dims")
        bound = elastic_max_stable_dt(self.order, self.h, float(np.max(self.vp)))
        if self.dt > bound * (1.0 + 1e-12):
            warnings.warn(f"dt={self.dt:g} exceeds the staggered CFL bound {bound:g}",
                          StabilityWarning, stacklevel=2)

    @property
    def halo(self) -> int:
        return self.order // 2

    def params(self, precision: int = 4) -> dict:
        """bs, lam, mu computed in float64; rounded once to float32 unless
        precision == 8 (the float64 path, fdr_elastic64_run)."""
        shape = tuple(self.dims)

        def grid(v):
            return np.broadcast_to(np.asarray(v, dtype=np.float64), shape)

        vp, vs, rho = grid(self.vp), grid(self.vs), grid(self.rho)
        mu = rho * vs * vs
        lam = rho * vp * vp - 2.0 * mu
        f = self.dt / self.h
        out = {"bs": f / rho, "lam": f * lam, "mu": f * mu}
        dt = np.float64 if precision == 8 else np.float32
        return {k: np.ascontiguousarray(v, dtype=dt) for k, v in out.items()}


def _torch():
    import torch

    return torch


class ElasticWavefield:
    """The 9 velocity/stress fields in HBM (one level each: updated in place)."""

    def __init__(self, halo, fields, dims, it=0):
        self.halo = int(halo)
        self.fields = list(fields)
        self._dims = tuple(int(d) for d in dims)
        self.it = int(it)
        self.traces = None

    @classmethod
    def allocate(cls, dims, halo, device=None, dtype=None):
        """float32 fields (default), or dtype=torch.float64 for the float64
        path (fdr_elastic64_run, the direct kernel in double)."""
        torch = _torch()
        _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dtype = torch.float32 if dtype is None else dtype
        if dtype not in (torch.float32, torch.float64):
            raise ValidationError("elastic fields are float32 or float64")
        nx, ny, nz = (int(d) for d in dims)
        shape = (nx, ny, row_pitch(nz))
        return cls(halo, [torch.zeros(shape, dtype=dtype, device=dev) for _ in FIELDS],
                   (nx, ny, nz))

    @property
    def dims(self):
        return self._dims

    @property
    def device(self):
        return self.fields[0].device

    def numpy(self, name: str) -> np.ndarray:
        return to_host(self.fields[FIELDS.index(name)][:, :, : self._dims[2]])

    def nonfinite_count(self, name: str = "vz") -> int:
        """NaN/inf values of one field, counted on the device."""
        from .kernel import count_nonfinite

        return count_nonfinite(self.fields[FIELDS.index(name)], self._dims)

    def set_interior(self, name: str, values) -> None:
        torch = _torch()
        f64 = self.fields[0].dtype == torch.float64
        arr = np.ascontiguousarray(np.asarray(values, dtype=np.float64 if f64 else np.float32))
        if arr.shape != self._dims:
            raise ValidationError("interior values do not match dims")
        self.fields[FIELDS.index(name)][:, :, : self._dims[2]].copy_(host_tensor(arr))


class _ElArgs(ctypes.Structure):
    """Mirror of fdr_elastic_args (include/b200fd.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32), ("order", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
        ("pitch_y", ctypes.c_int32), ("pitch_x", ctypes.c_int64),
        ("c", ctypes.c_float * (_lib.MAX_RADIUS + 1)),
        ("params", ctypes.c_void_p * 3), ("fields", ctypes.c_void_p * 9),
        ("sponge_x", ctypes.c_void_p), ("sponge_y", ctypes.c_void_p), ("sponge_z", ctypes.c_void_p),
        ("series", ctypes.c_void_p), ("n_series", ctypes.c_int32),
        ("src_x", ctypes.c_int32), ("src_y", ctypes.c_int32), ("src_z", ctypes.c_int32),
        ("n_rec", ctypes.c_int32), ("rec_xyz", ctypes.c_void_p), ("traces", ctypes.c_void_p),
        ("trace_rows", ctypes.c_int32), ("it0", ctypes.c_int32), ("n_steps", ctypes.c_int32),
        ("variant", ctypes.c_int32),
    ]


class _ElArgs64(ctypes.Structure):
    """Mirror of fdr_elastic64_args (include/b200fd.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32), ("order", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
        ("pitch_y", ctypes.c_int32), ("pitch_x", ctypes.c_int64),
        ("c", ctypes.c_double * (_lib.MAX_RADIUS + 1)),
        ("params", ctypes.c_void_p * 3), ("fields", ctypes.c_void_p * 9),
        ("sponge_x", ctypes.c_void_p), ("sponge_y", ctypes.c_void_p), ("sponge_z", ctypes.c_void_p),
        ("series", ctypes.c_void_p), ("n_series", ctypes.c_int32),
        ("src_x", ctypes.c_int32), ("src_y", ctypes.c_int32), ("src_z", ctypes.c_int32),
        ("n_rec", ctypes.c_int32), ("rec_xyz", ctypes.c_void_p), ("traces", ctypes.c_void_p),
        ("trace_rows", ctypes.c_int32), ("it0", ctypes.c_int32), ("n_steps", ctypes.c_int32),
    ]


class _ElPlan:
    """Device copies of a config's inputs; precision 8: everything in double
    (parameters unrounded, exact float64 weights, float64 sponge and series)."""

    def __init__(self, cfg: ElasticConfig, device, pitch: int, precision: int = 4):
        torch = _torch()
        self.key = _el_key(cfg, device, pitch)
        self.guard = InputGuard(config_inputs(cfg, _EL_FIELDS))  # frozen while cached
        nx, ny, nz = cfg.dims
        f64 = precision == 8
        tdt, ndt = (torch.float64, np.float64) if f64 else (torch.float32, np.float32)
        self.c = elastic_weights_f64(cfg.order) if f64 else elastic_weights_f32(cfg.order)
        self.params = []
        for host in cfg.params(precision).values():
            t = torch.zeros((nx, ny, pitch), dtype=tdt, device=device)
            t[:, :, :nz].copy_(host_tensor(host))
            self.params.append(t)
        self.sponge = None if cfg.sponge is None else tuple(
            host_tensor(np.asarray(v, dtype=ndt)).to(device)
            for v in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
        self.series, self.src, self.n_series = None, (-1, 0, 0), 0
        if cfg.source is not None:
            # float32 samples (what the float32 path injects), converted exactly
            # to double on the float64 path, as the acoustic float64 path does
            s = np.ascontiguousarray(np.asarray(cfg.source.series).astype(np.float32)
                                     .astype(ndt).reshape(-1))
            self.series = host_tensor(s).to(device)
            self.src = tuple(int(v) for v in cfg.source.location)
            self.n_series = int(s.size)
        self.rec = None
        if cfg.receivers is not None:
            self.rec = host_tensor(cfg.receivers.locations.reshape(-1).copy()).to(device)


_EL_FIELDS = ("vp", "vs", "rho")


def _el_key(cfg, device, pitch):
    return (cfg.order, tuple(cfg.dims), float(cfg.dt), float(cfg.h),
            tuple(id(o) for o in config_inputs(cfg, _EL_FIELDS)), str(device), int(pitch))


_VARIANTS = {"auto": 0, "direct": 1, "stream": 2, "queue": 3}


def elastic_run(fld: ElasticWavefield, cfg: ElasticConfig, n_steps: Optional[int] = None,
                variant: str = "auto") -> ElasticWavefield:
    """Advance n_steps (default cfg.n_t) velocity+stress steps in one library call."""
    if fld.halo != cfg.halo or fld.dims != tuple(cfg.dims):
        raise ValidationError(
            f"wavefield (dims {fld.dims}, halo {fld.halo}) does not match "
            f"config (dims {tuple(cfg.dims)}, halo {cfg.halo})")
    n = cfg.n_t if n_steps is None else int(n_steps)
    if n < 0:
        raise ValidationError("n_steps must be >= 0")
    if variant not in _VARIANTS:
        raise ValidationError(f"unknown variant {variant!r}")
    if n == 0:
        return fld
    torch = _torch()
    lib = _lib.load()
    dev = fld.device
    pitch_y = int(fld.fields[0].shape[2])
    f64 = fld.fields[0].dtype == torch.float64
    if f64 and variant not in ("auto", "direct"):
        raise ValidationError("the float64 elastic path is the direct kernel (variant auto or direct)")
    prec = 8 if f64 else 4
    plan = cached_plan(cfg, "_device_plan64" if f64 else "_device_plan", _el_key(cfg, dev, pitch_y),
                       lambda: _ElPlan(cfg, dev, pitch_y, prec))
    a = _ElArgs64() if f64 else _ElArgs()
    a.abi_version = _lib.ABI_VERSION
    a.order = cfg.order
    a.nx, a.ny, a.nz = fld.dims
    a.pitch_y = pitch_y
    a.pitch_x = int(fld.fields[0].shape[1]) * pitch_y
    for j, v in enumerate(plan.c):
        a.c[j] = float(v)
    for i, t in enumerate(plan.params):
        a.params[i] = t.data_ptr()
    for i, t in enumerate(fld.fields):
        a.fields[i] = t.data_ptr()
    if plan.sponge is not None:
        a.sponge_x, a.sponge_y, a.sponge_z = (t.data_ptr() for t in plan.sponge)
    if plan.series is not None:
        a.series = plan.series.data_ptr()
    a.n_series = plan.n_series
    a.src_x, a.src_y, a.src_z = plan.src
    if plan.rec is not None:
        rows = max(cfg.n_t, fld.it + n)
        n_rec = cfg.receivers.count
        tdt = torch.float64 if f64 else torch.float32
        if (fld.traces is None or fld.traces.shape[0] < rows or fld.traces.shape[1] != n_rec
                or fld.traces.dtype != tdt):
            fld.traces = grow_traces(fld, rows, n_rec, tdt, dev)
        a.n_rec = n_rec
        a.rec_xyz = plan.rec.data_ptr()
        a.traces = fld.traces.data_ptr()
        a.trace_rows = int(fld.traces.shape[0])
    a.it0 = fld.it
    a.n_steps = n
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        if f64:
            _lib.check(lib.fdr_elastic64_run(ctypes.byref(a), ctypes.c_void_p(stream)))
        else:
            a.variant = _VARIANTS[variant]
            _lib.check(lib.fdr_elastic_run(ctypes.byref(a), ctypes.c_void_p(stream)))
    fld.it += n
    return fld


def config5(n_t: int = 300, dims=(320, 320, 320), seed: int = 0) -> ElasticConfig:
    """BASELINE config 5: order 8, 320^3 at 10 m, smooth vp in [1.5, 4.5] km/s,
    vs = vp/1.8, rho in [1.0, 2.5] g/cc, explosive 12 Hz Ricker in the normal
    stresses at the centre, 320 receivers recording vz, 300 steps."""
    from .synthetic import cerjan_sponge, receiver_line, ricker, smooth_random_field

    def smooth(lo, hi, s):
        f = smooth_random_field(dims, 20.0, seed + s)
        f = (f - f.min()) / (f.max() - f.min())
        return (lo + (hi - lo) * f.astype(np.float64)).astype(np.float32)

    vp = smooth(1500.0, 4500.0, 10)
    vs = (vp.astype(np.float64) / 1.8).astype(np.float32)
    rho = smooth(1000.0, 2500.0, 11)
    h = 10.0
    dt = 0.4 * h / 4500.0
    nx, ny, nz = dims
    return ElasticConfig(order=8, dims=tuple(dims), n_t=n_t, dt=dt, h=h, vp=vp, vs=vs, rho=rho,
                         source=Source((nx // 2, ny // 2, nz // 2), 1e6 * ricker(12.0, dt, n_t)),
                         receivers=receiver_line(nx, ny // 2, 2), sponge=cerjan_sponge(dims))
