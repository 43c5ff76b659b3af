"""Acoustic leapfrog time stepping on one B200, behind the reference's kernel API.

Drop-in for /root/reference/pkg/src/fdroof/kernel.py: the same `KernelConfig`,
`Source`, `Wavefield`, `step`, `run_benchmark`, `max_stable_dt`,
`dump_wavefield` and `StabilityWarning` names, argument meanings and error
behaviour, but the wavefield lives in HBM and every step is one launch of the
sm_100a kernel in libb200fd.so (ctypes, include/b200fd.h).  Extensions the
BASELINE configs need and the reference lacks (SURVEY.md §8(a')): an
absorbing `Sponge`, `Receivers` with recorded traces, and `run` for many steps
per library call.

Results are bit-identical to the reference's numpy float32 path: the kernel
performs the reference's operations in the reference's order with one IEEE
rounding each (kernel.py:199-211).  There is no CPU fallback.
"""

import ctypes
import math
import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._inputs import (InputGuard, cached_plan, config_inputs, grow_traces, host_tensor,  # noqa: F401
                      invalidate_plan, to_host)
from .errors import ValidationError
from .roofline import (
    ACOUSTIC_BYTES_PER_POINT,
    MachineSpec,
    RooflinePoint,
    acoustic_flops_per_point,
    b200_machine,
    roofline_point,
)
from .stencils import abs_sum, acoustic_weights_f32, second_derivative_weights

_VARIANTS = {"auto": _lib.VARIANT_AUTO, "direct": _lib.VARIANT_DIRECT, "tma": _lib.VARIANT_TMA,
             "queue": _lib.VARIANT_QUEUE, "persistent": _lib.VARIANT_PERSISTENT,
             "cluster": _lib.VARIANT_CLUSTER, "tb2": _lib.VARIANT_TB2,
             "fma": _lib.VARIANT_FMA,  # fma: contracted taps, opt-in, NOT bit-exact
             "queue2": _lib.VARIANT_QUEUE2}  # queue kernel, two y rows per thread


def _torch():
    import torch

    return torch


class StabilityWarning(UserWarning):
    """Configured time step exceeds the CFL bound (kernel.py:31-32)."""


def max_stable_dt(order: int, h: float, m=1.0) -> float:
    """CFL bound h*sqrt(4/a2)/v_max with a2 = 3*sum|w| (kernel.py:35-46)."""
    a2 = float(3 * abs_sum(second_derivative_weights(order)))
    m_min = float(np.min(m))
    if m_min <= 0:
        raise ValidationError("squared slowness must be positive")
    return h * math.sqrt(4.0 / a2) / (1.0 / math.sqrt(m_min))


@dataclass(frozen=True)
class Source:
    """Point source: additive time series injected at one interior point (kernel.py:49-54)."""

    location: tuple
    series: np.ndarray


@dataclass(frozen=True)
class Receivers:
    """On-grid receivers: traces[it, i] = u_new[locations[i]] after injection."""

    locations: np.ndarray

    def __post_init__(self):
        loc = np.asarray(self.locations)
        if loc.ndim != 2 or loc.shape[1] != 3 or loc.shape[0] < 1:
            raise ValidationError("receiver locations must have shape (n, 3), n >= 1")
        object.__setattr__(self, "locations", np.ascontiguousarray(loc, dtype=np.int32))

    @property
    def count(self) -> int:
        return int(self.locations.shape[0])


def trilinear_weights(positions):
    """Base corners (floor, int32, shape (n, 3)) and float32 weights (n, 8)
    of off-grid positions in grid units; corner c = 4 dx + 2 dy + dz, weight
    f32(wx * wy * wz) formed in float64."""
    pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    base = np.floor(pos)
    t = pos - base
    w = np.empty((pos.shape[0], 8), dtype=np.float64)
    for c in range(8):
        dx, dy, dz = c >> 2, (c >> 1) & 1, c & 1
        w[:, c] = ((t[:, 0] if dx else 1.0 - t[:, 0]) * (t[:, 1] if dy else 1.0 - t[:, 1])
                   * (t[:, 2] if dz else 1.0 - t[:, 2]))
    return base.astype(np.int32), w.astype(np.float32)


@dataclass(frozen=True)
class OffGridSource:
    """Point source at a fractional grid position: each step adds
    f32(w_c) * f32(series[it]) to the 8 surrounding points (trilinear)."""

    position: tuple
    series: np.ndarray


@dataclass(frozen=True)
class OffGridReceivers:
    """Receivers at fractional grid positions (n, 3), sampled trilinearly:
    trace = w0 u0, then trace + w_c u_c for c = 1..7, in float32."""

    positions: np.ndarray

    def __post_init__(self):
        pos = np.asarray(self.positions, dtype=np.float64)
        if pos.ndim != 2 or pos.shape[1] != 3 or pos.shape[0] < 1:
            raise ValidationError("receiver positions must have shape (n, 3), n >= 1")
        object.__setattr__(self, "positions", np.ascontiguousarray(pos))

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


@dataclass(frozen=True)
class Sponge:
    """Separable absorbing taper G = (gx[x]*gy[y])*gz[z] applied to the new level.

    The reference keeps a zero-Dirichlet halo with no absorbing layer
    (kernel.py:5-6); this extension multiplies the freshly updated level by G
    before the source is injected (SURVEY.md §8(a')).  Profiles are float32
    and equal 1 away from the faces, where the update is bit-identical to the
    reference.
    """

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray

    def __post_init__(self):
        for name in ("x", "y", "z"):
            arr = np.ascontiguousarray(np.asarray(getattr(self, name), dtype=np.float32))
            if arr.ndim != 1:
                raise ValidationError("sponge profiles must be 1-D")
            object.__setattr__(self, name, arr)


@dataclass
class KernelConfig:
    """Mirror of fdroof.kernel.KernelConfig (kernel.py:57-101) plus extensions."""

    order: int
    dims: tuple
    n_t: int
    dt: float
    h: float = 1.0
    m: object = 1.0
    source: Optional[Source] = None
    receivers: Optional[Receivers] = None
    sponge: Optional[Sponge] = None

    def __post_init__(self):
        if self.order < 2 or self.order % 2 != 0:
            raise ValidationError(f"order must be even and >= 2, got {self.order}")
        if self.order > 32:
            raise ValidationError(f"order must be <= 32, got {self.order}")
        if len(self.dims) != 3 or any(d < 1 for d in self.dims):
            raise ValidationError(f"dims must be three positive extents, got {self.dims}")
        if self.n_t < 0 or self.dt <= 0 or self.h <= 0:
            raise ValidationError("n_t must be >= 0 and dt, h positive")
        halo = self.order // 2
        if any(d < 2 * halo + 1 for d in self.dims):
            raise ValidationError(f"interior dims {self.dims} too small for halo width {halo}")
        if not np.isscalar(self.m) and np.shape(self.m) != tuple(self.dims):
            raise ValidationError("squared-slowness grid must match interior dims")
        if isinstance(self.source, OffGridSource):
            pos = self.source.position
            if len(pos) != 3 or any(not 0 <= c <= d - 1 for c, d in zip(pos, self.dims)):
                raise ValidationError(f"source position {pos} outside interior")
        elif self.source is not None:
            loc = self.source.location
            if len(loc) != 3 or any(not 0 <= c < d for c, d in zip(loc, self.dims)):
                raise ValidationError(f"source location {loc} outside interior")
        if isinstance(self.receivers, OffGridReceivers):
            pos = self.receivers.positions
            if (pos < 0).any() or (pos > np.asarray(self.dims) - 1).any():
                raise ValidationError("receiver position outside interior")
        elif self.receivers is not None:
            loc = self.receivers.locations
            if (loc < 0).any() or (loc >= np.asarray(self.dims)).any():
                raise ValidationError("receiver location outside interior")
        if self.sponge is not None:
            if tuple(len(p) for p in (self.sponge.x, self.sponge.y, self.sponge.z)) != tuple(self.dims):
                raise ValidationError("sponge profile lengths must match interior dims")
        bound = max_stable_dt(self.order, self.h, self.m)
        if self.dt > bound * (1.0 + 1e-12):
            warnings.warn(
                f"dt={self.dt:g} exceeds the CFL bound {bound:g}; the scheme will be unstable",
                StabilityWarning,
                stacklevel=2,
            )

    @property
    def halo(self) -> int:
        return self.order // 2

    @property
    def k(self) -> int:
        return self.order + 1


def row_pitch(nz: int) -> int:
    """Device z-row pitch in floats: a multiple of 4 (16-byte rows for TMA/float4)."""
    return (nz + 3) // 4 * 4


class Wavefield:
    """Three time levels in HBM, rotated by reference between steps (kernel.py:104-142).

    grids[2] is the latest level u(t-1), grids[1] is u(t-2) and grids[0] the
    scratch level that receives u(t), exactly as in the reference.  Each grid
    is a CUDA float32 tensor of shape (nx, ny, pitch) holding the interior only
    (z contiguous, pitch = row_pitch(nz)); the reference's zero halo is implied
    (the kernels read zeros outside the interior), so `halo` records the
    width a host copy is padded with.  `traces` holds receiver samples,
    shape (rows, n_rec), when the config has receivers.

    Levels allocated with dtype=torch.float64 select the float64 path
    (fdr_acoustic64_run): the same update sequence in IEEE
    double, for measuring the float32 path's rounding error.
    """

    def __init__(self, halo: int, grids: list, dims: tuple, it: int = 0):
        self.halo = int(halo)
        self.grids = list(grids)
        self._dims = tuple(int(d) for d in dims)
        self.it = int(it)
        self.traces = None

    @classmethod
    def allocate(cls, dims, halo: int, device=None, dtype=None) -> "Wavefield":
        if len(dims) != 3 or any(d < 2 * halo + 1 for d in dims):
            raise ValidationError(f"dims {tuple(dims)} too small for halo width {halo}")
        torch = _torch()
        _lib.load()
        dtype = torch.float32 if dtype is None else dtype
        if dtype not in (torch.float32, torch.float64):
            raise ValidationError(f"wavefield dtype must be float32 or float64, got {dtype}")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nx, ny, nz = (int(d) for d in dims)
        shape = (nx, ny, row_pitch(nz))
        grids = [torch.zeros(shape, dtype=dtype, device=dev) for _ in range(3)]
        return cls(halo, grids, (nx, ny, nz))

    @property
    def dtype(self):
        return self.grids[0].dtype

    @property
    def _np_dtype(self):
        return np.float64 if self.dtype == _torch().float64 else np.float32

    @property
    def dims(self):
        return self._dims

    @property
    def device(self):
        return self.grids[0].device

    def interior(self, level: int = 2):
        """Device view of a level's interior, shape dims (kernel.py:130-133)."""
        return self.grids[level][:, :, : self._dims[2]]

    def numpy(self, level: int = 2) -> np.ndarray:
        """Host copy of a level's interior (float32, or float64 levels), C order."""
        return to_host(self.interior(level))

    def set_interior(self, level: int, values) -> None:
        torch = _torch()
        arr = np.ascontiguousarray(np.asarray(values, dtype=self._np_dtype))
        if arr.shape != self._dims:
            raise ValidationError(f"interior values of shape {arr.shape} do not match dims {self._dims}")
        self.interior(level).copy_(host_tensor(arr))

    def nonfinite_count(self, level: int = 2) -> int:
        """NaN/inf values in a level, counted on the device (the end-of-run
        failure check; fdr_count_nonfinite)."""
        return count_nonfinite(self.grids[level], self._dims)

    def halo_is_zero(self) -> bool:
        """The halo is not stored; row-padding columns must stay zero."""
        nz = self._dims[2]
        return all(not bool(g[:, :, nz:].any()) for g in self.grids)

    def host_grids(self) -> list:
        """The three levels as the reference lays them out: zero-padded
        (nx+2r, ny+2r, nz+2r) float32 numpy arrays (kernel.py:119-123)."""
        r = self.halo
        out = []
        for lvl in range(3):
            padded = np.zeros(tuple(d + 2 * r for d in self._dims), dtype=self._np_dtype)
            padded[r : r + self._dims[0], r : r + self._dims[1], r : r + self._dims[2]] = self.numpy(lvl)
            out.append(padded)
        return out

    @classmethod
    def from_host_grids(cls, grids, halo: int, it: int = 0, device=None) -> "Wavefield":
        """Upload a reference-layout Wavefield (three padded numpy levels)."""
        r = int(halo)
        dims = tuple(s - 2 * r for s in np.shape(grids[0]))
        torch = _torch()
        f64 = np.asarray(grids[0]).dtype == np.float64
        fld = cls.allocate(dims, r, device, torch.float64 if f64 else torch.float32)
        for lvl in range(3):
            g = np.asarray(grids[lvl], dtype=fld._np_dtype)
            fld.set_interior(lvl, g[r : r + dims[0], r : r + dims[1], r : r + dims[2]])
        fld.it = int(it)
        return fld


def count_nonfinite(t, dims) -> int:
    """Number of NaN/inf interior values of one (nx, ny, pitch) device level."""
    torch = _torch()
    if not t.is_cuda or t.dtype not in (torch.float32, torch.float64) or not t.is_contiguous():
        raise ValidationError("count_nonfinite takes a contiguous float32/float64 CUDA level")
    lib = _lib.load()
    n = ctypes.c_int64(0)
    pitch_y = int(t.shape[2])
    with torch.cuda.device(t.device):
        stream = torch.cuda.current_stream(t.device).cuda_stream
        _lib.check(lib.fdr_count_nonfinite(ctypes.c_void_p(t.data_ptr()), t.element_size(),
                                           *(int(d) for d in dims), pitch_y,
                                           int(t.shape[1]) * pitch_y, ctypes.byref(n),
                                           ctypes.c_void_p(stream)))
    return int(n.value)


def _check_match(fld: Wavefield, cfg: KernelConfig):
    if fld.halo != cfg.halo or fld.dims != tuple(cfg.dims):
        raise ValidationError(
            f"wavefield (dims {fld.dims}, halo {fld.halo}) does not match "
            f"config (dims {tuple(cfg.dims)}, halo {cfg.halo})"
        )


class _DevicePlan:
    """Device-resident per-config constants: weights, m grid, sponge, series, receivers."""

    def __init__(self, cfg: KernelConfig, device, pitch: int):
        torch = _torch()
        self.key = _plan_key(cfg, device, pitch)
        self.guard = InputGuard(config_inputs(cfg, ("m",)))  # frozen while cached
        nx, ny, nz = cfg.dims
        self.weights = acoustic_weights_f32(cfg.order)
        self.coef = np.float32(cfg.dt * cfg.dt / (cfg.h * cfg.h))  # kernel.py:187
        self.m_grid = None
        self.m_scalar = np.float32(1.0)
        self.m_bounds = (0.0, 0.0)
        if np.isscalar(cfg.m):
            self.m_scalar = np.float32(cfg.m)  # kernel.py:189
            self.m_mode = _lib.M_NONE if self.m_scalar == np.float32(1.0) else _lib.M_SCALAR
        else:
            self.m_mode = _lib.M_GRID
            host = np.asarray(cfg.m, dtype=np.float32)  # kernel.py:188
            self.m_grid = torch.zeros((nx, ny, pitch), dtype=torch.float32, device=device)
            self.m_grid[:, :, :nz].copy_(host_tensor(np.ascontiguousarray(host)))
            # bounds of m for the division window, reduced on the device (two
            # host passes over a 512^3 grid cost ~70 ms of the plan build; NaN
            # propagates through amin / amax as through numpy's min / max)
            inner = self.m_grid[:, :, :nz]
            self.m_bounds = (float(inner.amin().item()), float(inner.amax().item()))
        self.sponge = None
        if cfg.sponge is not None:
            self.sponge = tuple(
                host_tensor(p).to(device) for p in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)
            )
        self.series = None
        self.src = (-1, 0, 0)
        self.src_w = None
        if cfg.source is not None:
            series = np.asarray(cfg.source.series).astype(np.float32)  # kernel.py:173
            self.series = host_tensor(np.ascontiguousarray(series.reshape(-1))).to(device)
            if isinstance(cfg.source, OffGridSource):
                base, w = trilinear_weights([cfg.source.position])
                self.src = tuple(int(c) for c in base[0])
                self.src_w = host_tensor(np.ascontiguousarray(w[0])).to(device)
            else:
                self.src = tuple(int(c) for c in cfg.source.location)
        self.n_series = 0 if self.series is None else int(self.series.numel())
        self.rec = None
        self.rec_w = None
        if isinstance(cfg.receivers, OffGridReceivers):
            base, w = trilinear_weights(cfg.receivers.positions)
            self.rec = host_tensor(base.reshape(-1).copy()).to(device)
            self.rec_w = host_tensor(np.ascontiguousarray(w.reshape(-1))).to(device)
        elif cfg.receivers is not None:
            self.rec = host_tensor(cfg.receivers.locations.reshape(-1).copy()).to(device)


def _plan_key(cfg: KernelConfig, device, pitch: int = 0):
    """Plan identity: the scalars plus the identities of the input arrays
    (which the plan holds and write-protects, see _inputs.py)."""
    return (cfg.order, tuple(cfg.dims), float(cfg.dt), float(cfg.h),
            tuple(id(o) for o in config_inputs(cfg, ("m",))), str(device), int(pitch))


def _plan(cfg: KernelConfig, device, pitch: int) -> _DevicePlan:
    return cached_plan(cfg, "_device_plan", _plan_key(cfg, device, pitch),
                       lambda: _DevicePlan(cfg, device, pitch))


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _fill_args(args: _lib.AcousticArgs, cfg: KernelConfig, plan: _DevicePlan, dims, pitch_y,
               pitch_x, it0: int, n_steps: int, variant: int):
    args.abi_version = _lib.ABI_VERSION
    args.order = cfg.order
    args.nx, args.ny, args.nz = dims
    args.pitch_y = pitch_y
    args.pitch_x = pitch_x
    for j, w in enumerate(plan.weights):
        args.weights[j] = float(w)
    args.coef = float(plan.coef)
    args.m_mode = plan.m_mode
    args.m_scalar = float(plan.m_scalar)
    # grid bounds feed the exact division's fast-path window; NaN/inf/<=0
    # entries make the library fall back to IEEE division everywhere
    lo, hi = plan.m_bounds
    ok = np.isfinite(lo) and np.isfinite(hi) and lo > 0
    args.m_lo, args.m_hi = (lo, hi) if ok else (0.0, 0.0)
    args.src_x, args.src_y, args.src_z = plan.src
    args.n_series = plan.n_series
    args.n_rec = 0 if cfg.receivers is None else cfg.receivers.count
    args.it0 = it0
    args.n_steps = n_steps
    args.variant = variant


def device_args(fld: Wavefield, cfg: KernelConfig, n: int, variant: str = "auto") -> "_lib.AcousticArgs":
    """The fdr_acoustic_args of n float32 steps of `fld` under `cfg` (device
    plan built or reused, trace buffer grown); the caller launches them."""
    torch = _torch()
    dev = fld.device
    pitch_y = int(fld.grids[0].shape[2])
    pitch_x = int(fld.grids[0].shape[1]) * pitch_y
    plan = _plan(cfg, dev, pitch_y)
    args = _lib.AcousticArgs()
    _fill_args(args, cfg, plan, fld.dims, pitch_y, pitch_x, fld.it, n, _VARIANTS[variant])
    args.m = _ptr(plan.m_grid)
    args.rec_w = _ptr(plan.rec_w)
    args.src_w = _ptr(plan.src_w)
    for i in range(3):
        args.levels[i] = fld.grids[i].data_ptr()
    if plan.sponge is not None:
        args.sponge_x, args.sponge_y, args.sponge_z = (p.data_ptr() for p in plan.sponge)
    args.series = _ptr(plan.series)
    if plan.rec is not None:
        rows = max(cfg.n_t, fld.it + n)
        n_rec = cfg.receivers.count
        if fld.traces is None or fld.traces.shape[1] != n_rec or fld.traces.shape[0] < rows:
            fld.traces = grow_traces(fld, rows, n_rec, torch.float32, dev)
        args.rec_xyz = plan.rec.data_ptr()
        args.traces = fld.traces.data_ptr()
        args.trace_rows = int(fld.traces.shape[0])
    args._keep = plan  # the plan's device buffers outlive the call
    return args


def run(fld: Wavefield, cfg: KernelConfig, n_steps: Optional[int] = None,
        variant: str = "auto") -> Wavefield:
    """Advance `n_steps` (default cfg.n_t) steps in one library call.

    Equivalent to calling the reference's `step` n_steps times (kernel.py:176-222):
    levels rotate by reference, the source injects series[it] after each
    update and `it` advances.  Work is queued on the current torch stream.
    """
    _check_match(fld, cfg)
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
    dt0 = fld.grids[0].dtype
    for g in fld.grids:
        if (g.dtype != dt0 or dt0 not in (torch.float32, torch.float64) or not g.is_cuda
                or not g.is_contiguous() or g.shape != fld.grids[0].shape):
            raise ValidationError("wavefield levels must be contiguous float32 (or float64) CUDA "
                                  "tensors of one shape and dtype")
    if dt0 == torch.float64:
        return _run_f64(fld, cfg, n, variant)
    args = device_args(fld, cfg, n, variant)
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _lib.check(lib.fdr_acoustic_run(ctypes.byref(args), ctypes.c_void_p(stream)))
    g = fld.grids
    fld.grids = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]  # kernel.py:219, n times
    fld.it += n
    return fld


class _DevicePlan64:
    """Device-resident float64 constants of a config for the float64 path:
    weights 3 w0 and w_j in double, coef = dt*dt/(h*h) in double, m, sponge
    and series converted exactly to double."""

    def __init__(self, cfg: KernelConfig, device, pitch: int):
        torch = _torch()
        self.key = _plan_key(cfg, device, pitch)
        self.guard = InputGuard(config_inputs(cfg, ("m",)))
        nx, ny, nz = cfg.dims
        r = cfg.order // 2
        w = [float(x) for x in second_derivative_weights(cfg.order)]
        self.weights = [3.0 * w[r]] + [w[r + j] for j in range(1, r + 1)]
        self.coef = cfg.dt * cfg.dt / (cfg.h * cfg.h)
        self.m_grid = None
        self.m_scalar = 1.0
        if np.isscalar(cfg.m):
            self.m_scalar = float(cfg.m)
            self.m_mode = _lib.M_NONE if self.m_scalar == 1.0 else _lib.M_SCALAR
        else:
            self.m_mode = _lib.M_GRID
            host = np.ascontiguousarray(np.asarray(cfg.m, dtype=np.float64))
            self.m_grid = torch.zeros((nx, ny, pitch), dtype=torch.float64, device=device)
            self.m_grid[:, :, :nz].copy_(host_tensor(host))
        self.sponge = None
        if cfg.sponge is not None:
            self.sponge = tuple(host_tensor(np.asarray(p, dtype=np.float64)).to(device)
                                for p in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
        self.series = None
        self.src = (-1, 0, 0)
        if cfg.source is not None:
            series = np.ascontiguousarray(np.asarray(cfg.source.series, dtype=np.float64).reshape(-1))
            self.series = host_tensor(series).to(device)
            self.src = tuple(int(c) for c in cfg.source.location)
        self.n_series = 0 if self.series is None else int(self.series.numel())
        self.rec = None
        if cfg.receivers is not None:
            self.rec = host_tensor(cfg.receivers.locations.reshape(-1).copy()).to(device)


def _run_f64(fld: Wavefield, cfg: KernelConfig, n: int, variant: str) -> Wavefield:
    """The float64 path of `run` (fdr_acoustic64_run)."""
    torch = _torch()
    lib = _lib.load()
    dev = fld.device
    if variant in ("persistent", "cluster", "tb2", "fma"):
        raise ValidationError("the float64 path has variants auto, queue, tma and direct")
    if isinstance(cfg.source, OffGridSource) or isinstance(cfg.receivers, OffGridReceivers):
        raise ValidationError("the float64 path takes on-grid sources and receivers")
    pitch_y = int(fld.grids[0].shape[2])
    pitch_x = int(fld.grids[0].shape[1]) * pitch_y
    plan = cached_plan(cfg, "_device_plan64", _plan_key(cfg, dev, pitch_y),
                       lambda: _DevicePlan64(cfg, dev, pitch_y))
    a = _lib.Acoustic64Args()
    a.abi_version = _lib.ABI_VERSION
    a.order = cfg.order
    a.nx, a.ny, a.nz = fld.dims
    a.pitch_y, a.pitch_x = pitch_y, pitch_x
    for j, w in enumerate(plan.weights):
        a.weights[j] = w
    a.coef = plan.coef
    a.m_mode = plan.m_mode
    a.m_scalar = plan.m_scalar
    a.m = _ptr(plan.m_grid)
    for i in range(3):
        a.levels[i] = fld.grids[i].data_ptr()
    if plan.sponge is not None:
        a.sponge_x, a.sponge_y, a.sponge_z = (p.data_ptr() for p in plan.sponge)
    a.series = _ptr(plan.series)
    a.n_series = plan.n_series
    a.src_x, a.src_y, a.src_z = plan.src
    a.n_rec = 0 if cfg.receivers is None else cfg.receivers.count
    if plan.rec is not None:
        rows = max(cfg.n_t, fld.it + n)
        if fld.traces is None or fld.traces.dtype != torch.float64 or fld.traces.shape[0] < rows \
                or fld.traces.shape[1] != a.n_rec:
            if fld.traces is not None and fld.traces.dtype != torch.float64:
                fld.traces = None
            fld.traces = grow_traces(fld, rows, a.n_rec, torch.float64, dev)
        a.rec_xyz = plan.rec.data_ptr()
        a.traces = fld.traces.data_ptr()
        a.trace_rows = int(fld.traces.shape[0])
    a.it0 = fld.it
    a.n_steps = n
    a.variant = _VARIANTS[variant]
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _lib.check(lib.fdr_acoustic64_run(ctypes.byref(a), ctypes.c_void_p(stream)))
    g = fld.grids
    fld.grids = [g[n % 3], g[(1 + n) % 3], g[(2 + n) % 3]]
    fld.it += n
    return fld


def selftest_division(n: int = 1 << 26, m_lo: float = 4.9e-8, m_hi: float = 4.5e-7,
                      seed: int = 1):
    """Compare the kernels' branch-free division with IEEE __fdiv_rn on the
    GPU over n hashed operand pairs; returns (mismatches, fast_path_pairs)."""
    lib = _lib.load()
    n_fast = ctypes.c_int64(0)
    bad = lib.fdr_selftest_division(int(n), float(m_lo), float(m_hi), int(seed) & 0xffffffff,
                                    ctypes.byref(n_fast))
    _lib.check(int(bad) if bad < 0 else 0)
    return int(bad), int(n_fast.value)


def selftest_division64(n: int = 1 << 26, m_lo: float = 4.9e-8, m_hi: float = 4.5e-7,
                        seed: int = 1):
    """The float64 kernels' scaled exact division against IEEE __ddiv_rn on
    the GPU over n hashed operand pairs; returns (mismatches, fast_path_pairs)."""
    lib = _lib.load()
    n_fast = ctypes.c_int64(0)
    bad = lib.fdr_selftest_division64(int(n), float(m_lo), float(m_hi), int(seed) & 0xffffffff,
                                      ctypes.byref(n_fast))
    _lib.check(int(bad) if bad < 0 else 0)
    return int(bad), int(n_fast.value)


def step(fld: Wavefield, cfg: KernelConfig, slabs: int = 1) -> Wavefield:
    """Advance one time step in place; returns the same Wavefield (kernel.py:176).

    `slabs` is accepted for signature compatibility: the GPU's thread-block
    decomposition replaces the reference's x-slab threads, and results are
    independent of it exactly as in the reference (test_kernel.py:137-144).
    """
    return run(fld, cfg, 1)


def oracle_step(fld: Wavefield, cfg: KernelConfig) -> Wavefield:
    """Mirror of fdroof.kernel.oracle_step (kernel.py:225-254) on the GPU.

    The reference's independent check of `step`: the star-stencil convolution
    accumulated in float64 in stencil_geometry("star") order (stencils.py:
    161-179), the update (2c - prev) + (coef acc)/m in float64, one rounding
    to float32, then the rotation and the source (kernel.py:219-221).  The
    reference caps the grid at 32^3 for CPU time; this one takes any grid.
    Like the reference it knows no sponge, receivers or off-grid source.
    """
    _check_match(fld, cfg)
    if (cfg.sponge is not None or cfg.receivers is not None
            or isinstance(cfg.source, OffGridSource)):
        raise ValidationError("oracle_step mirrors the reference: on-grid source only, "
                              "no sponge or receivers")
    torch = _torch()
    if fld.grids[0].dtype != torch.float32:
        raise ValidationError("oracle_step takes a float32 wavefield")
    lib = _lib.load()
    dev = fld.device
    pitch_y = int(fld.grids[0].shape[2])
    pitch_x = int(fld.grids[0].shape[1]) * pitch_y
    plan = _plan(cfg, dev, pitch_y)
    args = _lib.AcousticArgs()
    _fill_args(args, cfg, plan, fld.dims, pitch_y, pitch_x, fld.it, 1, _lib.VARIANT_AUTO)
    args.m = _ptr(plan.m_grid)
    args.series = _ptr(plan.series)
    for i in range(3):
        args.levels[i] = fld.grids[i].data_ptr()
    r = cfg.order // 2
    w = second_derivative_weights(cfg.order)  # exact rationals, as fd_weights
    w64 = (ctypes.c_double * (r + 1))(float(3 * w[r]), *(float(w[r + j]) for j in range(1, r + 1)))
    coef = float(cfg.dt) ** 2 / float(cfg.h) ** 2  # kernel.py:246
    # the reference divides by cfg.m itself (kernel.py:247): a scalar even when
    # it is 1, a grid as float64 (a float64 grid must not be rounded to float32)
    m_scalar = float(cfg.m) if np.isscalar(cfg.m) else 1.0
    m64 = None
    if not np.isscalar(cfg.m) and np.asarray(cfg.m).dtype != np.float32:
        host = np.ascontiguousarray(np.asarray(cfg.m, dtype=np.float64))
        m64 = torch.zeros(tuple(fld.grids[0].shape), dtype=torch.float64, device=dev)
        m64[:, :, : fld.dims[2]].copy_(host_tensor(host))
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _lib.check(lib.fdr_acoustic_oracle_step(ctypes.byref(args), w64, coef, m_scalar,
                                                _ptr(m64), ctypes.c_void_p(stream)))
    scratch, prev, cur = fld.grids
    fld.grids = [prev, cur, scratch]
    fld.it += 1
    return fld


@dataclass(frozen=True)
class BenchResult:
    """Mirror of fdroof.kernel.BenchResult (kernel.py:257-263) plus GPts/s."""

    measured_gflops: float
    point: RooflinePoint
    wall_time_s: float
    total_flops: float
    wavefield: Wavefield

    @property
    def gpts_per_s(self) -> float:
        n = float(np.prod(self.wavefield.dims))
        steps = self.total_flops / (n * (self.point.k * 6 + 4))
        return n * steps / self.wall_time_s / 1e9

    @property
    def achieved_gbs(self) -> float:
        return self.gpts_per_s * ACOUSTIC_BYTES_PER_POINT


def run_benchmark(cfg: KernelConfig, machine: Optional[MachineSpec] = None, slabs: int = 1,
                  seed: int = 0, variant: str = "auto") -> BenchResult:
    """Run n_t steps, time them on the device and pin the result on the roofline.

    Mirrors kernel.py:266-290: the same seeded start when there is no source
    (level 2 = standard_normal*1e-3), GFLOPS = points x kernel_flops x n_t /
    time, with the time taken by CUDA events around the n_t launches.
    """
    if cfg.n_t < 1:
        raise ValidationError("benchmark needs n_t >= 1")
    torch = _torch()
    fld = Wavefield.allocate(cfg.dims, cfg.halo)
    if cfg.source is None:
        rng = np.random.default_rng(seed)
        fld.set_interior(2, rng.standard_normal(cfg.dims).astype(np.float32) * 1e-3)
    _plan(cfg, fld.device, int(fld.grids[0].shape[2]))
    stream = torch.cuda.current_stream(fld.device)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(fld.device)
    start.record(stream)
    run(fld, cfg, cfg.n_t, variant=variant)
    end.record(stream)
    end.synchronize()
    wall = start.elapsed_time(end) / 1e3
    n_interior = float(np.prod(cfg.dims))
    total = n_interior * acoustic_flops_per_point(cfg.order) * cfg.n_t
    measured = total / wall / 1e9
    point = roofline_point(machine or b200_machine(), cfg.order, measured_gflops=measured)
    return BenchResult(measured, point, wall, total, fld)


def dump_wavefield(fld: Wavefield, path) -> None:
    """Write the current level as little-endian float32, x-fastest order, with a
    one-line `nx ny nz` sidecar at <path>.dims (kernel.py:293-301)."""
    data = np.asarray(fld.numpy(2), dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(data.tobytes(order="F"))
    nx, ny, nz = fld.dims
    with open(f"{path}.dims", "w", encoding="utf-8") as fh:
        fh.write(f"{nx} {ny} {nz}\n")


def load_wavefield(path) -> np.ndarray:
    """Read a `dump_wavefield` file back: (nx, ny, nz) float32 from the
    x-fastest little-endian data and the `nx ny nz` sidecar (kernel.py:293-301)."""
    with open(f"{path}.dims", encoding="utf-8") as fh:
        dims = tuple(int(v) for v in fh.read().split())
    if len(dims) != 3:
        raise ValidationError(f"{path}.dims: expected 'nx ny nz'")
    data = np.fromfile(path, dtype="<f4")
    if data.size != int(np.prod(dims)):
        raise ValidationError(f"{path}: {data.size} values, sidecar says {dims}")
    return data.reshape(dims, order="F").astype(np.float32)


def dump_traces(fld: Wavefield, path) -> None:
    """Write the recorded receiver traces next to a wavefield dump: the fld.it
    recorded rows (one per step, receivers in config order) as little-endian
    float32, row-major, with a one-line `n_t n_rec` sidecar at <path>.dims --
    the trace-file counterpart of `dump_wavefield`."""
    if fld.traces is None:
        raise ValidationError("wavefield has no traces (config without receivers)")
    rows = min(int(fld.it), int(fld.traces.shape[0]))
    data = np.asarray(fld.traces[:rows].cpu().numpy(), dtype="<f4")
    with open(path, "wb") as fh:
        fh.write(data.tobytes(order="C"))
    with open(f"{path}.dims", "w", encoding="utf-8") as fh:
        fh.write(f"{data.shape[0]} {data.shape[1]}\n")


def load_traces(path) -> np.ndarray:
    """Read a `dump_traces` file back: (n_t, n_rec) float32."""
    with open(f"{path}.dims", encoding="utf-8") as fh:
        shape = tuple(int(v) for v in fh.read().split())
    if len(shape) != 2:
        raise ValidationError(f"{path}.dims: expected 'n_t n_rec'")
    data = np.fromfile(path, dtype="<f4")
    if data.size != shape[0] * shape[1]:
        raise ValidationError(f"{path}: {data.size} values, sidecar says {shape}")
    return data.reshape(shape).astype(np.float32)


class HostSimulation:
    """End-to-end simulation from host buffers through `fdr_acoustic_run_host`.

    Prepares pinned host copies of the inputs, a device workspace and pinned
    output buffers once; every `run()` then uploads m / sponge / series /
    receivers, zeroes the levels, advances cfg.n_t steps on the GPU and
    downloads the final interior and the traces (the whole job a user of the
    reference's `run_benchmark` + `dump_wavefield` performs).
    """

    def __init__(self, cfg: KernelConfig, variant: str = "auto", device=None):
        if isinstance(cfg.source, OffGridSource) or isinstance(cfg.receivers, OffGridReceivers):
            raise ValidationError("HostSimulation takes on-grid sources and receivers")
        torch = _torch()
        self.lib = _lib.load()
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nx, ny, nz = cfg.dims
        self.pitch_y = row_pitch(nz)
        self.pitch_x = ny * self.pitch_y
        self.args = _lib.AcousticArgs()
        # host-side constants (same derivation as _DevicePlan)
        plan = _HostPlan(cfg)
        _fill_args(self.args, cfg, plan, cfg.dims, self.pitch_y, self.pitch_x, 0, cfg.n_t,
                   _VARIANTS[variant])

        def pinned(arr):
            if arr is None:
                return None
            t = host_tensor(np.ascontiguousarray(arr)).pin_memory()
            return t

        self.h_m = pinned(plan.m_host)
        self.h_sponge = None if cfg.sponge is None else tuple(pinned(p) for p in (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
        self.h_series = pinned(plan.series_host)
        self.h_rec = pinned(None if cfg.receivers is None else cfg.receivers.locations.reshape(-1))
        self.h_final = torch.empty(tuple(cfg.dims), dtype=torch.float32).pin_memory()
        n_rec = 0 if cfg.receivers is None else cfg.receivers.count
        self.h_traces = torch.empty((max(cfg.n_t, 1), max(n_rec, 1)), dtype=torch.float32).pin_memory()
        self.ws_bytes = int(self.lib.fdr_acoustic_workspace_bytes(ctypes.byref(self.args)))
        if self.ws_bytes == 0:
            _lib.check(_lib.FDR_EINVAL)
        self.workspace = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        self.ws_ptr = (base + 255) // 256 * 256

    @property
    def h2d_bytes(self) -> int:
        tensors = [self.h_m, self.h_series, self.h_rec] + list(self.h_sponge or ())
        return int(sum(t.numel() * t.element_size() for t in tensors if t is not None))

    @property
    def d2h_bytes(self) -> int:
        n_rec = 0 if self.cfg.receivers is None else self.cfg.receivers.count
        return int(self.h_final.numel() * 4 + n_rec * self.cfg.n_t * 4)

    def run(self):
        torch = _torch()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        sx, sy, sz = (None, None, None) if self.h_sponge is None else tuple(p(t) for t in self.h_sponge)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.fdr_acoustic_run_host(
                ctypes.byref(self.args), p(self.h_m), sx, sy, sz, p(self.h_series), p(self.h_rec),
                p(self.h_final), p(self.h_traces) if self.cfg.receivers is not None else None,
                ctypes.c_void_p(self.ws_ptr), self.ws_bytes, ctypes.c_void_p(stream)))
        traces = None
        if self.cfg.receivers is not None:
            traces = self.h_traces.numpy()[: self.cfg.n_t, : self.cfg.receivers.count]
        return self.h_final.numpy(), traces


    def _slot(self, k: int):
        """(workspace pointer, pinned final, pinned traces) of pipeline slot k;
        slot 0 reuses the synchronous `run`'s buffers."""
        torch = _torch()
        if not hasattr(self, "_slots"):
            self._slots = []
            self._streams = tuple(torch.cuda.Stream(self.device) for _ in range(3))
        while len(self._slots) <= k:
            if not self._slots:
                keep, ws, hf, ht = None, self.ws_ptr, self.h_final, self.h_traces
            else:
                keep = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
                ws = (keep.data_ptr() + 255) // 256 * 256
                hf = torch.empty_like(self.h_final).pin_memory()
                ht = torch.empty_like(self.h_traces).pin_memory()
            self._slots.append((ws, hf, ht, keep))
        return self._slots[k][:3]

    def run_pipelined(self, n_sims: int, depth: int = 2, on_result=None):
        """`n_sims` back-to-back simulations (shots), each uploading all its
        inputs and downloading its final level and traces, with `depth`
        workspaces: the time steps run in order on one compute stream while
        shot i+1's upload and shot i's download run on two copy streams
        (fdr_acoustic_host_upload / _run_ws / _download), so the copies hide
        behind the steps.  Ordered after the caller's current stream, which
        waits for all of it: CUDA events on that stream time the whole batch.
        on_result(i, final, traces) receives each shot's host results (copies).
        Returns the last shot's (final, traces) as views of the pinned output
        buffers, valid until the next run (as `run` does).
        """
        torch = _torch()
        if n_sims < 1 or depth < 1:
            raise ValidationError("need n_sims >= 1 and depth >= 1")
        lib = self.lib
        cur = torch.cuda.current_stream(self.device)
        self._slot(depth - 1)
        up, comp, down = self._streams
        start = torch.cuda.Event()
        start.record(cur)
        for st in (up, comp, down):
            st.wait_event(start)
        p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        sx, sy, sz = (None, None, None) if self.h_sponge is None else tuple(p(t) for t in self.h_sponge)
        has_rec = self.cfg.receivers is not None
        args = ctypes.byref(self.args)
        comp_done, down_done = [None] * n_sims, [None] * n_sims
        delivered = set()

        def deliver(i):
            if on_result is not None and i not in delivered:
                down_done[i].synchronize()
                on_result(i, *self._host_results(*self._slot(i % depth)[1:]))
                delivered.add(i)

        with torch.cuda.device(self.device):
            for i in range(n_sims):
                ws, hf, ht = self._slot(i % depth)
                if i >= depth:
                    up.wait_event(comp_done[i - depth])  # slot inputs no longer read
                _lib.check(lib.fdr_acoustic_host_upload(args, p(self.h_m), sx, sy, sz, p(self.h_series),
                                                        p(self.h_rec), ctypes.c_void_p(ws), self.ws_bytes,
                                                        ctypes.c_void_p(up.cuda_stream)))
                ev = torch.cuda.Event()
                ev.record(up)
                comp.wait_event(ev)
                if i >= depth:
                    comp.wait_event(down_done[i - depth])  # slot levels downloaded
                newest = _lib.check(lib.fdr_acoustic_host_run_ws(args, int(self.h_sponge is not None),
                                                                 ctypes.c_void_p(ws), self.ws_bytes,
                                                                 ctypes.c_void_p(comp.cuda_stream)))
                comp_done[i] = torch.cuda.Event()
                comp_done[i].record(comp)
                down.wait_event(comp_done[i])
                if i >= depth:
                    deliver(i - depth)  # before its pinned buffers are overwritten
                _lib.check(lib.fdr_acoustic_host_download(args, newest, p(hf), p(ht) if has_rec else None,
                                                          ctypes.c_void_p(ws), self.ws_bytes,
                                                          ctypes.c_void_p(down.cuda_stream)))
                down_done[i] = torch.cuda.Event()
                down_done[i].record(down)
        cur.wait_event(down_done[-1])
        for i in range(max(0, n_sims - depth), n_sims):
            deliver(i)
        down_done[-1].synchronize()
        hf, ht = self._slot((n_sims - 1) % depth)[1:]
        traces = None
        if has_rec:
            traces = ht.numpy()[: self.cfg.n_t, : self.cfg.receivers.count]
        return hf.numpy(), traces  # views of the pinned buffers, like run()

    def _host_results(self, hf, ht):
        traces = None
        if self.cfg.receivers is not None:
            traces = ht.numpy()[: self.cfg.n_t, : self.cfg.receivers.count].copy()
        return hf.numpy().copy(), traces


class _HostPlan:
    """Host-side float32 constants of a config (same casts as _DevicePlan)."""

    def __init__(self, cfg: KernelConfig):
        self.weights = acoustic_weights_f32(cfg.order)
        self.coef = np.float32(cfg.dt * cfg.dt / (cfg.h * cfg.h))
        self.m_host = None
        self.m_scalar = np.float32(1.0)
        self.m_bounds = (0.0, 0.0)
        if np.isscalar(cfg.m):
            self.m_scalar = np.float32(cfg.m)
            self.m_mode = _lib.M_NONE if self.m_scalar == np.float32(1.0) else _lib.M_SCALAR
        else:
            self.m_mode = _lib.M_GRID
            self.m_host = np.ascontiguousarray(np.asarray(cfg.m, dtype=np.float32))
            self.m_bounds = (float(self.m_host.min()), float(self.m_host.max()))
        self.series_host = None
        self.series = None
        self.src = (-1, 0, 0)
        if cfg.source is not None:
            self.series_host = np.ascontiguousarray(np.asarray(cfg.source.series).astype(np.float32).reshape(-1))
            self.series = self.series_host
            self.src = tuple(int(c) for c in cfg.source.location)
        self.n_series = 0 if self.series is None else int(self.series.size)
        self.rec = None if cfg.receivers is None else cfg.receivers.locations
