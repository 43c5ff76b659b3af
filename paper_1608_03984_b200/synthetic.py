"""Seeded synthetic inputs for the BASELINE configurations.

The reference ships no velocity models, wavelets, sponge or receivers
(SURVEY.md §0.4, §8(a')); BASELINE.json names seeded synthetic models, which
this module defines once so that the GPU path and the CPU oracle consume the
same float32 bits:

* `ricker(f0, dt, nt)`: (1 - 2 pi^2 f^2 tau^2) exp(-pi^2 f^2 tau^2), tau = it*dt - 1/f,
  evaluated in float64; injected raw like kernel.py:173.
* `cerjan_profile(n, width, alpha)`: 1-D taper g(d) = exp(-(alpha (W - d))^2)
  for a point at distance d < W from the nearest face, else 1 (Cerjan et
  al. 1985 style), float64 then rounded to float32.
* velocity models (m/s): two-layer (config 1), smooth random field (config 2;
  uniform noise low-passed by a Gaussian of sigma 20 points, applied in the
  Fourier domain with periodic wrap, then min-max scaled to [1500, 4500]) and
  an 8-layer model (config 3).  m = f32(1 / v^2) in s^2/m^2.
* dt = 0.4 h / v_max ("CFL 0.4 of vmax" in BASELINE.json).
"""

import math

import numpy as np

from .errors import ValidationError
from .kernel import KernelConfig, Receivers, Source, Sponge

SPONGE_WIDTH = 10
SPONGE_ALPHA = 0.03  # edge factor exp(-(0.03*10)^2) = 0.914


def ricker(f0: float, dt: float, nt: int, t0: float = None) -> np.ndarray:
    """Ricker wavelet samples at t = it*dt (float64)."""
    if f0 <= 0 or dt <= 0 or nt < 0:
        raise ValidationError("ricker needs f0 > 0, dt > 0, nt >= 0")
    t0 = 1.0 / f0 if t0 is None else t0
    tau = np.arange(nt, dtype=np.float64) * dt - t0
    a = (math.pi * f0 * tau) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def cerjan_profile(n: int, width: int = SPONGE_WIDTH, alpha: float = SPONGE_ALPHA) -> np.ndarray:
    """float32 taper along one axis of n interior points."""
    i = np.arange(n)
    d = np.minimum(i, n - 1 - i).astype(np.float64)
    g = np.where(d < width, np.exp(-(alpha * (width - d)) ** 2), 1.0)
    return g.astype(np.float32)


def cerjan_sponge(dims, width: int = SPONGE_WIDTH, alpha: float = SPONGE_ALPHA) -> Sponge:
    return Sponge(*(cerjan_profile(n, width, alpha) for n in dims))


def squared_slowness(v: np.ndarray) -> np.ndarray:
    """m = f32(1/v^2) computed in float64."""
    return (1.0 / np.square(np.asarray(v, dtype=np.float64))).astype(np.float32)


def two_layer_velocity(dims, interface_z: int, v_top: float = 1500.0,
                       v_bottom: float = 2500.0) -> np.ndarray:
    """v = v_top for z < interface_z, v_bottom below (z = axis 2, depth)."""
    v = np.empty(dims, dtype=np.float64)
    v[:, :, :interface_z] = v_top
    v[:, :, interface_z:] = v_bottom
    return v


def smooth_random_field(dims, sigma: float, seed: int) -> np.ndarray:
    """Uniform noise (default_rng(seed)) low-passed by a Gaussian of `sigma`
    grid points via FFT (periodic), float32."""
    rng = np.random.default_rng(seed)
    noise = rng.random(dims, dtype=np.float32)
    try:
        import scipy.fft as sfft

        fwd = lambda a: sfft.rfftn(a, workers=-1)  # noqa: E731
        inv = lambda a, s: sfft.irfftn(a, s=s, workers=-1)  # noqa: E731
    except ImportError:  # pragma: no cover
        fwd = np.fft.rfftn
        inv = lambda a, s: np.fft.irfftn(a, s=s)  # noqa: E731
    spec = fwd(noise)
    del noise
    for ax, n in enumerate(dims):
        k = np.fft.rfftfreq(n) if ax == len(dims) - 1 else np.fft.fftfreq(n)
        shape = [1] * len(dims)
        shape[ax] = k.size
        spec *= np.exp(-2.0 * (math.pi * sigma * k) ** 2).astype(np.float32).reshape(shape)
    return np.asarray(inv(spec, dims), dtype=np.float32)


def smooth_random_velocity(dims, sigma: float = 20.0, seed: int = 0, vmin: float = 1500.0,
                           vmax: float = 4500.0) -> np.ndarray:
    f = smooth_random_field(dims, sigma, seed)
    lo, hi = float(f.min()), float(f.max())
    scaled = (f - np.float32(lo)) * np.float32((vmax - vmin) / (hi - lo)) + np.float32(vmin)
    return np.clip(scaled, vmin, vmax)


def layered_velocity(dims, n_layers: int = 8, seed: int = 0, vmin: float = 1500.0,
                     vmax: float = 4500.0) -> np.ndarray:
    """n_layers with speeds ~ U[vmin, vmax] and sorted interface depths ~ U(0, nz)."""
    rng = np.random.default_rng(seed)
    speeds = rng.uniform(vmin, vmax, n_layers)
    nz = dims[2]
    depths = np.sort(rng.uniform(0, nz, n_layers - 1))
    layer_of_z = np.searchsorted(depths, np.arange(nz) + 0.5)
    prof = speeds[layer_of_z]
    return np.broadcast_to(prof, dims)


def layered_slowness(dims, n_layers: int = 8, seed: int = 0) -> np.ndarray:
    """m for the layered model built plane-by-plane (avoids a float64 full grid)."""
    v = layered_velocity((1, 1, dims[2]), n_layers, seed)[0, 0]
    prof = squared_slowness(v)
    return np.ascontiguousarray(np.broadcast_to(prof, dims))


def cfl_dt(h: float, v_max: float, cfl: float = 0.4) -> float:
    return cfl * h / v_max


def receiver_line(nx: int, y: int, z: int) -> Receivers:
    """Receivers at (i, y, z), i = 0..nx-1 (a surface line at depth z)."""
    loc = np.stack([np.arange(nx), np.full(nx, y), np.full(nx, z)], axis=1)
    return Receivers(loc)


def config1(n_t: int = 100, dims=(64, 64, 64)) -> KernelConfig:
    """BASELINE config 1: order 4, 64^3, h=10 m, two-layer 1500/2500 m/s split at
    z=32, 10-point sponge, 10 Hz Ricker at the centre, 64 receivers at z=2."""
    nx, ny, nz = dims
    h = 10.0
    v = two_layer_velocity(dims, nz // 2)
    dt = cfl_dt(h, float(v.max()))
    src = Source((nx // 2, ny // 2, nz // 2), ricker(10.0, dt, n_t))
    return KernelConfig(order=4, dims=tuple(dims), n_t=n_t, dt=dt, h=h, m=squared_slowness(v),
                        source=src, receivers=receiver_line(nx, ny // 2, 2),
                        sponge=cerjan_sponge(dims))


def config2(order: int = 8, n_t: int = 500, dims=(512, 512, 512), seed: int = 0) -> KernelConfig:
    """BASELINE config 2: smooth random 1.5-4.5 km/s model (sigma 20), h=10 m,
    CFL-limited dt, 15 Hz Ricker at the centre, a surface line of receivers."""
    nx, ny, nz = dims
    h = 10.0
    v = smooth_random_velocity(dims, 20.0, seed)
    m = squared_slowness(v)
    del v
    dt = cfl_dt(h, 4500.0)
    src = Source((nx // 2, ny // 2, nz // 2), ricker(15.0, dt, n_t))
    return KernelConfig(order=order, dims=tuple(dims), n_t=n_t, dt=dt, h=h, m=m, source=src,
                        receivers=receiver_line(nx, ny // 2, 2), sponge=cerjan_sponge(dims))


def config3(n_t: int = 200, dims=(1024, 1024, 768), seed: int = 0) -> KernelConfig:
    """BASELINE config 3: order 8, 1024x1024x768, 8-layer model, 200 steps,
    one source at the centre and 1024 receivers at z=2."""
    nx, ny, nz = dims
    h = 10.0
    m = layered_slowness(dims, 8, seed)
    v_max = float(1.0 / math.sqrt(float(m.min())))
    dt = cfl_dt(h, v_max)
    src = Source((nx // 2, ny // 2, nz // 2), ricker(15.0, dt, n_t))
    return KernelConfig(order=8, dims=tuple(dims), n_t=n_t, dt=dt, h=h, m=m, source=src,
                        receivers=receiver_line(nx, ny // 2, 2), sponge=cerjan_sponge(dims))
