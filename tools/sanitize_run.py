"""Small-grid runs of every production kernel for compute-sanitizer
(racecheck / synccheck / memcheck / initcheck on small grids).
Each case is checked bit for bit against its C oracle so a sanitizer run also
confirms the result.  Usage: python tools/sanitize_run.py [case ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def acoustic(variant, order=8, dims=(40, 36, 44), steps=3):
    import paper_1608_03984_b200 as B
    from cases import random_levels
    from oracle import acoustic as O
    from oracle import cref
    from paper_1608_03984_b200.synthetic import cerjan_sponge, ricker

    dt = 0.4 * B.max_stable_dt(order, 10.0, 1.0 / 3000.0 ** 2)
    rec = np.stack([np.arange(dims[0]), np.full(dims[0], dims[1] // 2), np.full(dims[0], 2)], 1)
    cfg = B.KernelConfig(order=order, dims=dims, n_t=steps, dt=dt, h=10.0,
                         m=np.full(dims, 1.0 / 3000.0 ** 2, np.float32),
                         source=B.Source((dims[0] // 2, dims[1] // 2, dims[2] // 2),
                                         1e3 * ricker(20.0, dt, steps)),
                         receivers=B.Receivers(rec), sponge=cerjan_sponge(dims, 4, 0.1))
    cur, prev = random_levels(dims, 7)
    f = B.Wavefield.allocate(dims, cfg.halo)
    f.set_interior(2, cur)
    f.set_interior(1, prev)
    B.run(f, cfg, steps, variant=variant)
    st = O.OracleState(dims, cfg.halo)
    O.interior(st.grids[2], st.halo)[...] = cur
    O.interior(st.grids[1], st.halo)[...] = prev
    cref.simulate(cfg, steps, state=st)
    assert np.array_equal(f.numpy(), st.latest()), f"acoustic {variant} differs"
    assert np.array_equal(f.traces.cpu().numpy()[:steps], st.traces[:steps])


def acoustic64():
    import torch

    import paper_1608_03984_b200 as B

    dims = (24, 20, 28)
    cfg = B.KernelConfig(order=8, dims=dims, n_t=3, dt=0.5 * B.max_stable_dt(8, 1.0))
    f = B.Wavefield.allocate(dims, cfg.halo, dtype=torch.float64)
    f.set_interior(2, np.random.default_rng(1).standard_normal(dims))
    B.run(f, cfg)
    torch.cuda.synchronize()


def tti():
    from oracle import tti as T
    from paper_1608_03984_b200 import Receivers, Source, tti as TT
    from paper_1608_03984_b200.synthetic import ricker

    dims = (24, 22, 20)
    rec = Receivers(np.stack([np.arange(24), np.full(24, 11), np.full(24, 2)], 1))
    cfg = TT.TTIConfig(order=8, dims=dims, n_t=3, dt=1e-3, h=10.0, m=1.0 / 3000.0 ** 2,
                       epsilon=0.2, delta=0.1, theta=0.4, phi=0.3,
                       source=Source((12, 11, 10), 1e3 * ricker(25.0, 1e-3, 3)), receivers=rec)
    f = TT.TTIWavefield.allocate(dims, cfg.halo)
    TT.tti_run(f, cfg)
    w2, w1 = TT.tti_weights_f32(8)
    st = T.simulate_c(cfg, cfg.params(), w2, w1)
    assert np.array_equal(f.numpy("p"), st.interior("p")), "tti differs"


def elastic():
    from oracle import elastic as E
    from paper_1608_03984_b200 import Receivers, Source, elastic as EL
    from paper_1608_03984_b200.synthetic import ricker

    dims = (24, 22, 20)
    rec = Receivers(np.stack([np.arange(24), np.full(24, 11), np.full(24, 2)], 1))
    cfg = EL.ElasticConfig(order=8, dims=dims, n_t=3, dt=8e-4, h=10.0, vp=3000.0,
                           vs=3000.0 / 1.8, rho=2000.0, receivers=rec,
                           source=Source((12, 11, 10), 1e6 * ricker(25.0, 8e-4, 3)))
    f = EL.ElasticWavefield.allocate(dims, cfg.halo)
    EL.elastic_run(f, cfg)
    st = E.simulate_c(cfg, cfg.params(), EL.elastic_weights_f32(8))
    for k in EL.FIELDS:
        assert np.array_equal(f.numpy(k), st.interior(k)), f"elastic {k} differs"


CASES = {
    "queue": lambda: acoustic("queue"),
    "queue_o16": lambda: acoustic("queue", order=16, dims=(40, 36, 44)),
    "persistent": lambda: acoustic("persistent", order=4),
    "cluster": lambda: acoustic("cluster", order=4, dims=(64, 64, 64)),
    "direct": lambda: acoustic("direct", order=4),
    "fp64": acoustic64,
    "tti": tti,
    "elastic": elastic,
}

if __name__ == "__main__":
    import torch

    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        torch.cuda.synchronize()
        print(f"{name}: ok", flush=True)
