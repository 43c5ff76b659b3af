"""Configs for the slab-decomposition tests: the source sits next to a slab
boundary and receivers span every slab."""
import numpy as np

from paper_1608_03984_b200 import KernelConfig, Receivers, Source, max_stable_dt
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
    return out
