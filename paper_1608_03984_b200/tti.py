"""TTI pseudo-acoustic (coupled p/r) time stepping on B200 (BASELINE config 4).

The reference has no TTI time stepping (SURVEY.md §8(a')): its cost catalog
describes the kernel (/root/reference/pkg/src/fdroof/equations.py:144-155,
15 fields, factor 2, 3 second + 3 cross derivatives) and PAPER.md:804-829
states the system (Liu 2009):

    m p_tt = (1+2 eps) (Gxx+Gyy) p + sqrt(1+2 delta) Gzz r + q
    m r_tt = sqrt(1+2 delta) (Gxx+Gyy) p + Gzz r + q

with Gzz = (c . grad)^2 along the tilted symmetry axis
c = (cos phi sin theta, sin phi sin theta, cos theta) and Gxx + Gyy = lap - Gzz
(the paper's Gyy cross term carries a sign typo).  The
float32 operation sequence the kernels follow is defined in
oracle/tti_ref.c (the parity oracle); accuracy is checked against a float64
oracle (oracle/tti.py).  The per-point parameters are the 9 float32 grids the
catalogue counts (m-derived k, the two Thomsen factors and the 6 Gzz
coefficients), prepared on the host in float64.
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
from .stencils import first_derivative_weights, second_derivative_weights

PARAM_NAMES = ("k", "a", "b", "cxx", "cyy", "czz", "cxy", "cyz", "cxz")
TTI_BYTES_PER_POINT = 60        # 15 fields x 4 B (equations.py:144-155)


def tti_flops_per_point(order: int) -> int:
    """Reference catalogue count (equations.py:55-71 with the tti entry):
    2 * (3*2k + 3*(2k^2-4k-1) + 44 + 17 - 8), k = order+1."""
    k = order + 1
    return 2 * (3 * 2 * k + 3 * (2 * k * k - 4 * k - 1) + 44 + 17 - 8)


def tti_weights_f32(order: int):
    """(w2[0..r], w1[0..r]) float32: second-derivative centre/taps and the
    first-derivative taps (w1[0] = 0), float32 of the exact rationals."""
    r = order // 2
    w2 = second_derivative_weights(order)
    w1 = first_derivative_weights(order)
    a2 = np.array([float(w2[r])] + [float(w2[r + j]) for j in range(1, r + 1)], dtype=np.float32)
    a1 = np.array([0.0] + [float(w1[r + j]) for j in range(1, r + 1)], dtype=np.float32)
    return a2, a1


def tti_weights_f64(order: int):
    """(w2[0..r], w1[0..r]) float64 of the exact rationals (the float64 path)."""
    r = order // 2
    w2 = second_derivative_weights(order)
    w1 = first_derivative_weights(order)
    a2 = np.array([float(w2[r])] + [float(w2[r + j]) for j in range(1, r + 1)], dtype=np.float64)
    a1 = np.array([0.0] + [float(w1[r + j]) for j in range(1, r + 1)], dtype=np.float64)
    return a2, a1


def tti_max_stable_dt(order: int, h: float, m, epsilon) -> float:
    """CFL-style bound h*sqrt(4/a2)/(v_max*sqrt(1+2 eps_max)) (cf. kernel.py:35-46)."""
    a2 = 3.0 * float(sum(abs(w) for w in second_derivative_weights(order)))
    m_min = float(np.min(m))
    if m_min <= 0:
        raise ValidationError("squared slowness must be positive")
    v_eff = math.sqrt(1.0 + 2.0 * max(0.0, float(np.max(epsilon)))) / math.sqrt(m_min)
    return h * math.sqrt(4.0 / a2) / v_eff


@dataclass
class TTIConfig:
    """TTI run configuration; m, epsilon, delta, theta, phi are interior-shaped
    grids or scalars (theta = tilt, phi = azimuth, radians)."""

    order: int
    dims: tuple
    n_t: int
    dt: float
    h: float
    m: object
    epsilon: object = 0.0
    delta: object = 0.0
    theta: object = 0.0
    phi: object = 0.0
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
        for name in ("m", "epsilon", "delta", "theta", "phi"):
            v = getattr(self, name)
            if not np.isscalar(v) and np.shape(v) != tuple(self.dims):
                raise ValidationError(f"{name} grid must match interior dims")
        if np.any(np.asarray(self.delta) > np.asarray(self.epsilon)):
            raise ValidationError("TTI pseudo-acoustic needs delta <= epsilon")
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
        bound = tti_max_stable_dt(self.order, self.h, self.m, self.epsilon)
        if self.dt > bound * (1.0 + 1e-12):
            warnings.warn(f"dt={self.dt:g} exceeds the TTI CFL bound {bound:g}",
                          StabilityWarning, stacklevel=2)

    @property
    def halo(self) -> int:
        return self.order // 2

    def params(self, precision: int = 4) -> dict:
        """The 9 parameter grids (host, float64; rounded once to float32 unless
        precision == 8, the float64 path)."""
        shape = tuple(self.dims)

        def grid(v):
            return np.broadcast_to(np.asarray(v, dtype=np.float64), shape)

        m = grid(np.asarray(self.m, dtype=np.float32).astype(np.float64))
        eps, dl, th, ph = (grid(getattr(self, n)) for n in ("epsilon", "delta", "theta", "phi"))
        st, ct = np.sin(th), np.cos(th)
        sp, cp = np.sin(ph), np.cos(ph)
        out = {
            "k": self.dt * self.dt / (self.h * self.h * m),
            "a": 1.0 + 2.0 * eps,
            "b": np.sqrt(1.0 + 2.0 * dl),
            "cxx": (cp * st) ** 2,
            "cyy": (sp * st) ** 2,
            "czz": ct ** 2,
            "cxy": np.sin(2.0 * ph) * st * st,
            "cyz": sp * np.sin(2.0 * th),
            "cxz": cp * np.sin(2.0 * th),
        }
        dt = np.float64 if precision == 8 else np.float32
        return {k: np.ascontiguousarray(v, dtype=dt) for k, v in out.items()}


def _torch():
    import torch

    return torch


class TTIWavefield:
    """p and r, three HBM levels each ([scratch, prev, cur] like kernel.py:104-116).

    `interleaved` (the default) stores each level as (p, r) pairs per point
    in one (nx, ny, pitch, 2) tensor; `p[i]` / `r[i]` are strided views of
    it, so the packed streaming kernel reads both fields of a tap with one
    8-byte shared load (fdr_tti_args.interleaved, include/b200fd.h).
    interleaved=False keeps two separate arrays (the layout tti_stream needs)."""

    def __init__(self, halo, p, r, dims, it=0, interleaved=False):
        self.halo = int(halo)
        self.p = list(p)
        self.r = list(r)
        self._dims = tuple(int(d) for d in dims)
        self.it = int(it)
        self.traces = None
        self.interleaved = bool(interleaved)

    @classmethod
    def allocate(cls, dims, halo, device=None, interleaved=True, dtype=None):
        """dtype=torch.float64 allocates separate float64 levels for the
        float64 path (fdr_tti64_run, the direct kernel in double)."""
        torch = _torch()
        _lib.load()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nx, ny, nz = (int(d) for d in dims)
        shape = (nx, ny, row_pitch(nz))
        if dtype is not None and dtype != torch.float32:
            if dtype != torch.float64:
                raise ValidationError("TTI levels are float32 or float64")
            mk64 = lambda: [torch.zeros(shape, dtype=torch.float64, device=dev) for _ in range(3)]  # noqa: E731
            return cls(halo, mk64(), mk64(), (nx, ny, nz))
        if interleaved:
            levels = [torch.zeros(shape + (2,), dtype=torch.float32, device=dev) for _ in range(3)]
            return cls(halo, [t[..., 0] for t in levels], [t[..., 1] for t in levels], (nx, ny, nz),
                       interleaved=True)
        mk = lambda: [torch.zeros(shape, dtype=torch.float32, device=dev) for _ in range(3)]  # noqa: E731
        return cls(halo, mk(), mk(), (nx, ny, nz))

    @property
    def dims(self):
        return self._dims

    @property
    def device(self):
        return self.p[0].device

    def numpy(self, field: str = "p", level: int = 2) -> np.ndarray:
        t = (self.p if field == "p" else self.r)[level]
        return to_host(t[:, :, : self._dims[2]])

    def nonfinite_count(self, field: str = "p", level: int = 2) -> int:
        """NaN/inf values of a field's level, counted on the device.
        Interleaved levels are counted as (p, r) pairs: both fields together."""
        from .kernel import count_nonfinite

        t = (self.p if field == "p" else self.r)[level]
        if self.interleaved:
            nx, ny, nz = self._dims
            pair = t.as_strided((nx, ny, 2 * t.shape[2]), (t.stride(0), t.stride(1), 1),
                                t.storage_offset() - (0 if field == "p" else 1))
            return count_nonfinite(pair, (nx, ny, 2 * nz))
        return count_nonfinite(t, self._dims)

    def set_interior(self, field: str, level: int, values) -> None:
        torch = _torch()
        f64 = self.p[0].dtype == torch.float64
        arr = np.ascontiguousarray(np.asarray(values, dtype=np.float64 if f64 else np.float32))
        if arr.shape != self._dims:
            raise ValidationError("interior values do not match dims")
        (self.p if field == "p" else self.r)[level][:, :, : self._dims[2]].copy_(host_tensor(arr))


class _TTIArgs(ctypes.Structure):
    """Mirror of fdr_tti_args (include/b200fd.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32), ("order", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
        ("pitch_y", ctypes.c_int32), ("pitch_x", ctypes.c_int64),
        ("w2", ctypes.c_float * (_lib.MAX_RADIUS + 1)), ("w1", ctypes.c_float * (_lib.MAX_RADIUS + 1)),
        ("params", ctypes.c_void_p * 9), ("p", ctypes.c_void_p * 3), ("r", ctypes.c_void_p * 3),
        ("sponge_x", ctypes.c_void_p), ("sponge_y", ctypes.c_void_p), ("sponge_z", ctypes.c_void_p),
        ("series", ctypes.c_void_p), ("n_series", ctypes.c_int32),
        ("src_x", ctypes.c_int32), ("src_y", ctypes.c_int32), ("src_z", ctypes.c_int32),
        ("n_rec", ctypes.c_int32), ("rec_xyz", ctypes.c_void_p), ("traces", ctypes.c_void_p),
        ("trace_rows", ctypes.c_int32), ("it0", ctypes.c_int32), ("n_steps", ctypes.c_int32),
        ("variant", ctypes.c_int32), ("interleaved", ctypes.c_int32),
    ]


class _TTIArgs64(ctypes.Structure):
    """Mirror of fdr_tti64_args (include/b200fd.h)."""

    _fields_ = [
        ("abi_version", ctypes.c_int32), ("order", ctypes.c_int32),
        ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
        ("pitch_y", ctypes.c_int32), ("pitch_x", ctypes.c_int64),
        ("w2", ctypes.c_double * (_lib.MAX_RADIUS + 1)), ("w1", ctypes.c_double * (_lib.MAX_RADIUS + 1)),
        ("params", ctypes.c_void_p * 9), ("p", ctypes.c_void_p * 3), ("r", ctypes.c_void_p * 3),
        ("sponge_x", ctypes.c_void_p), ("sponge_y", ctypes.c_void_p), ("sponge_z", ctypes.c_void_p),
        ("series", ctypes.c_void_p), ("n_series", ctypes.c_int32),
        ("src_x", ctypes.c_int32), ("src_y", ctypes.c_int32), ("src_z", ctypes.c_int32),
        ("n_rec", ctypes.c_int32), ("rec_xyz", ctypes.c_void_p), ("traces", ctypes.c_void_p),
        ("trace_rows", ctypes.c_int32), ("it0", ctypes.c_int32), ("n_steps", ctypes.c_int32),
    ]


class _TTIPlan:
    """Device copies of a config's inputs; precision 8: everything in double
    (parameters unrounded, exact float64 weights, float64 sponge and series)."""

    def __init__(self, cfg: TTIConfig, device, pitch: int, precision: int = 4):
        torch = _torch()
        self.key = _tti_key(cfg, device, pitch)
        self.guard = InputGuard(config_inputs(cfg, _TTI_FIELDS))  # frozen while cached
        nx, ny, nz = cfg.dims
        f64 = precision == 8
        tdt, ndt = (torch.float64, np.float64) if f64 else (torch.float32, np.float32)
        self.w2, self.w1 = tti_weights_f64(cfg.order) if f64 else tti_weights_f32(cfg.order)
        self.params = []
        for name, host in cfg.params(precision).items():
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
            self.src = tuple(int(c) for c in cfg.source.location)
            self.n_series = int(s.size)
        self.rec = None
        if cfg.receivers is not None:
            self.rec = host_tensor(cfg.receivers.locations.reshape(-1).copy()).to(device)


_TTI_FIELDS = ("m", "epsilon", "delta", "theta", "phi")


def _tti_key(cfg, device, pitch):
    return (cfg.order, tuple(cfg.dims), float(cfg.dt), float(cfg.h),
            tuple(id(o) for o in config_inputs(cfg, _TTI_FIELDS)), str(device), int(pitch))


_VARIANTS = {"auto": 0, "direct": 1, "stream": 2, "queue": 3}


def tti_run(fld: TTIWavefield, cfg: TTIConfig, n_steps: Optional[int] = None,
            variant: str = "auto") -> TTIWavefield:
    """Advance n_steps (default cfg.n_t) TTI steps in one library call."""
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
    pitch_y = int(fld.p[0].shape[2])
    f64 = fld.p[0].dtype == torch.float64
    if f64 and variant not in ("auto", "direct"):
        raise ValidationError("the float64 TTI path is the direct kernel (variant auto or direct)")
    prec = 8 if f64 else 4
    plan = cached_plan(cfg, "_device_plan64" if f64 else "_device_plan", _tti_key(cfg, dev, pitch_y),
                       lambda: _TTIPlan(cfg, dev, pitch_y, prec))
    a = _TTIArgs64() if f64 else _TTIArgs()
    a.abi_version = _lib.ABI_VERSION
    a.order = cfg.order
    a.nx, a.ny, a.nz = fld.dims
    a.pitch_y = pitch_y
    a.pitch_x = int(fld.p[0].shape[1]) * pitch_y
    for j in range(len(plan.w2)):
        a.w2[j] = float(plan.w2[j])
        a.w1[j] = float(plan.w1[j])
    for i, t in enumerate(plan.params):
        a.params[i] = t.data_ptr()
    for i in range(3):
        a.p[i] = fld.p[i].data_ptr()
        a.r[i] = fld.r[i].data_ptr()
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
            _lib.check(lib.fdr_tti64_run(ctypes.byref(a), ctypes.c_void_p(stream)))
        else:
            a.variant = _VARIANTS[variant]
            a.interleaved = 1 if fld.interleaved else 0
            _lib.check(lib.fdr_tti_run(ctypes.byref(a), ctypes.c_void_p(stream)))
    for lv in (fld.p, fld.r):
        g = list(lv)
        lv[:] = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]
    fld.it += n
    return fld


def config4(n_t: int = 300, dims=(384, 384, 384), seed: int = 0) -> TTIConfig:
    """BASELINE config 4: order 8, 384^3 at 12.5 m, smooth seeded v in
    [1.5, 4.5] km/s, eps in [0, 0.3], delta in [0, 0.15] with delta <= eps,
    tilt and azimuth in [0, pi/4], 12 Hz Ricker at the centre, 300 steps."""
    from .synthetic import cerjan_sponge, receiver_line, ricker, smooth_random_field, squared_slowness

    def smooth(lo, hi, s):
        f = smooth_random_field(dims, 20.0, seed + s)
        f = (f - f.min()) / (f.max() - f.min())
        return lo + (hi - lo) * f.astype(np.float64)

    v = smooth(1500.0, 4500.0, 0)
    m = squared_slowness(v)
    del v
    eps = smooth(0.0, 0.3, 1)
    delta = np.minimum(smooth(0.0, 0.15, 2), eps)
    theta = smooth(0.0, math.pi / 4, 3)
    phi = smooth(0.0, math.pi / 4, 4)
    h = 12.5
    dt = 0.4 * h / (4500.0 * math.sqrt(1.0 + 2.0 * float(eps.max())))
    nx, ny, nz = dims
    return TTIConfig(order=8, dims=tuple(dims), n_t=n_t, dt=dt, h=h, m=m,
                     epsilon=eps.astype(np.float32), delta=delta.astype(np.float32),
                     theta=theta.astype(np.float32), phi=phi.astype(np.float32),
                     source=Source((nx // 2, ny // 2, nz // 2), ricker(12.0, dt, n_t)),
                     receivers=receiver_line(nx, ny // 2, 2), sponge=cerjan_sponge(dims))
