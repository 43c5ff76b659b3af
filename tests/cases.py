"""Golden-case builders shared by the oracle and GPU tests.

Each builder reproduces the exact inputs tests/golden/make_golden.py fed to
the reference (same seeds, same float32 casts) as a
paper_1608_03984_b200.KernelConfig plus the initial interior levels.
"""

import hashlib
import math

import numpy as np

from paper_1608_03984_b200 import KernelConfig, Receivers, Source, max_stable_dt
from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def random_levels(dims, seed):
    rng = np.random.default_rng(seed)
    cur = rng.standard_normal(dims).astype(np.float32)
    prev = rng.standard_normal(dims).astype(np.float32)
    return cur, prev


def random_case(order):
    dt = 0.5 * max_stable_dt(order, 1.0)
    cfg = KernelConfig(order=order, dims=(20, 20, 20), n_t=3, dt=dt)
    return cfg, random_levels(cfg.dims, order)


def varm_case():
    m = 1.0 + 0.5 * np.random.default_rng(3).random((16, 16, 16)).astype(np.float32)
    dt = 0.5 * max_stable_dt(4, 1.0, m)
    cfg = KernelConfig(order=4, dims=(16, 16, 16), n_t=2, dt=dt, m=m)
    return cfg, random_levels(cfg.dims, 11)


def scalarm_case():
    dt = 0.5 * max_stable_dt(6, 1.0, 1.7)
    cfg = KernelConfig(order=6, dims=(14, 15, 17), n_t=2, dt=dt, m=1.7)
    return cfg, random_levels(cfg.dims, 21)


def mirror_case():
    dt = 0.5 * max_stable_dt(8, 1.0)
    series = np.array([1.0, 0.5, -0.25, 0.1], dtype=np.float32)
    cfg = KernelConfig(order=8, dims=(17, 17, 17), n_t=4, dt=dt, source=Source((8, 8, 8), series))
    return cfg, None


RAGGED = ((2, (13, 11, 9), 31), (10, (23, 21, 22), 32), (16, (33, 34, 35), 33))


def ragged_case(order, dims, seed):
    dt = 0.5 * max_stable_dt(order, 1.0)
    series = np.random.default_rng(seed).standard_normal(6)
    loc = (dims[0] // 3, dims[1] - 2, 1)
    cfg = KernelConfig(order=order, dims=dims, n_t=6, dt=dt, source=Source(loc, series))
    return cfg, random_levels(dims, seed)


def config1_case(sponge=True):
    dims, h, nt = (64, 64, 64), 10.0, 100
    v = np.empty(dims)
    v[:, :, :32] = 1500.0
    v[:, :, 32:] = 2500.0
    m = (1.0 / np.square(v)).astype(np.float32)
    dt = 0.4 * h / 2500.0
    rec = np.stack([np.arange(64), np.full(64, 32), np.full(64, 2)], axis=1)
    cfg = KernelConfig(order=4, dims=dims, n_t=nt, dt=dt, h=h, m=m,
                       source=Source((32, 32, 32), ricker(10.0, dt, nt)),
                       receivers=Receivers(rec), sponge=cerjan_sponge(dims) if sponge else None)
    return cfg, None


def medium_o8_case():
    dims, nt = (96, 80, 72), 40
    rng = np.random.default_rng(5)
    v = 1500.0 + 3000.0 * rng.random(dims)
    m = (1.0 / np.square(v)).astype(np.float32)
    dt = 0.4 * 10.0 / float(v.max())
    rec = np.stack([np.arange(96), np.full(96, 40), np.full(96, 2)], axis=1)
    cfg = KernelConfig(order=8, dims=dims, n_t=nt, dt=dt, h=10.0, m=m,
                       source=Source((48, 40, 36), ricker(15.0, dt, nt)),
                       receivers=Receivers(rec), sponge=cerjan_sponge(dims))
    return cfg, None


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))


__all__ = ["sha", "random_case", "varm_case", "scalarm_case", "mirror_case", "RAGGED",
           "ragged_case", "config1_case", "medium_o8_case", "rel_l2", "math"]
