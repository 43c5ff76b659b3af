"""Configs for the slab-decomposition tests: the source sits next to a slab
boundary and receivers span every slab."""
import numpy as np

from paper_1608_03984_b200 import (KernelConfig, OffGridReceivers, OffGridSource, Receivers,
                                   Source, max_stable_dt)
from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker


def slab_case():
    out = {}
    for order, dims, src_x in ((4, (24, 14, 12), 11), (8, (30, 13, 15), 16)):
        rng = np.random.default_rng(order)
        m = (1.0 + rng.random(dims)).astype(np.float32)
        dt = 0.5 * max_stable_dt(order, 1.0, m)
        rec = np.stack([np.arange(dims[0]), np.full(dims[0], dims[1] // 2), np.full(dims[0], 2)], 1)
        cfg = KernelConfig(order=order, dims=dims, n_t=14, dt=dt, m=m,
                           source=Source((src_x, dims[1] // 2, dims[2] // 2), 50.0 * ricker(0.1, dt, 14)),
                           receivers=Receivers(rec), sponge=cerjan_sponge(dims, 3, 0.1))
        out[f"o{order}"] = (cfg, 14)
    # off-grid: the source straddles the 2-slab (x 14|15) or the 3-slab (x 9|10)
    # boundary; receivers on base planes next to every boundary of 2 and 3 slabs
    for order, src_x in ((8, 14.37), (4, 9.71)):
        dims = (30, 13, 15)
        rng = np.random.default_rng(100 + order)
        m = (1.0 + rng.random(dims)).astype(np.float32)
        dt = 0.5 * max_stable_dt(order, 1.0, m)
        xs = np.array([0.0, 9.4, 9.0, 10.2, 14.6, 14.0, 15.5, 19.5, 20.1, 29.0, 3.3, 24.8])
        pos = np.stack([xs, rng.uniform(0, dims[1] - 1, xs.size), rng.uniform(0, dims[2] - 1, xs.size)], 1)
        cfg = KernelConfig(order=order, dims=dims, n_t=40, dt=dt, m=m,
                           source=OffGridSource((src_x, 6.25, 7.6), 50.0 * ricker(0.1, dt, 40)),
                           receivers=OffGridReceivers(pos), sponge=cerjan_sponge(dims, 3, 0.1))
        out[f"off{order}"] = (cfg, 40)
    return out
