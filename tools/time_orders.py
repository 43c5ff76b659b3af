"""Time the acoustic step per order on a config-2 style grid (device events).

    python tools/time_orders.py [--grid 512] [--nt 50] [--orders 2,4,8,12,16]
Prints one JSON line per (order, variant) with ms/step and GPts/s.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--grid", type=int, default=512)
    p.add_argument("--nt", type=int, default=50)
    p.add_argument("--orders", default="2,4,6,8,10,12,14,16")
    p.add_argument("--variants", default="auto")
    p.add_argument("--tag", default=os.environ.get("B200FD_LIB", "default"))
    a = p.parse_args()
    import numpy as np
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    base = config2(order=8, n_t=a.nt, dims=(a.grid,) * 3)
    npts = float(np.prod(base.dims))
    for order in [int(o) for o in a.orders.split(",")]:
        cfg = B.KernelConfig(order=order, dims=base.dims, n_t=a.nt, dt=base.dt, h=base.h, m=base.m,
                             source=base.source, receivers=base.receivers, sponge=base.sponge)
        for variant in a.variants.split(","):
            fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
            # warm + random-ish start so the field is non-zero everywhere
            rng = np.random.default_rng(order)
            fld.set_interior(2, rng.standard_normal(cfg.dims, dtype=np.float32))
            fld.set_interior(1, rng.standard_normal(cfg.dims, dtype=np.float32))
            B.run(fld, cfg, 2, variant=variant)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            B.run(fld, cfg, a.nt, variant=variant)
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / a.nt
            print(json.dumps({"tag": a.tag, "order": order, "variant": variant,
                              "ms_per_step": round(ms, 4), "gpts": round(npts / ms / 1e6, 2),
                              "frac_hbm": round(npts * 16 / ms / 1e6 / 6557.4, 4)}), flush=True)
            del fld


if __name__ == "__main__":
    main()
