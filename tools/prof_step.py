"""Short run of the acoustic step for profiling (ncu launch lists / full captures).

    python tools/prof_step.py --order 8 --grid 512 --nt 6 [--variant tma]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--order", type=int, default=8)
    p.add_argument("--grid", type=int, default=512)
    p.add_argument("--nt", type=int, default=6)
    p.add_argument("--variant", default="auto")
    p.add_argument("--random", action="store_true", help="random initial levels (no zeros)")
    a = p.parse_args()
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=a.order, n_t=a.nt, dims=(a.grid,) * 3)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    if a.random:
        import numpy as np

        rng = np.random.default_rng(a.order)
        fld.set_interior(2, rng.standard_normal(cfg.dims, dtype=np.float32))
        fld.set_interior(1, rng.standard_normal(cfg.dims, dtype=np.float32))
    B.run(fld, cfg, variant=a.variant)
    torch.cuda.synchronize()
    print("ok", a.order, a.grid, a.nt, float(fld.interior().abs().max()))


if __name__ == "__main__":
    main()
