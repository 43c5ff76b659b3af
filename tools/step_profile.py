"""Per-segment step time and field statistics over a config-2 simulation.

    python tools/step_profile.py [--order 8] [--nt 500] [--seg 50] [--random]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--order", type=int, default=8)
    p.add_argument("--grid", type=int, default=512)
    p.add_argument("--nt", type=int, default=500)
    p.add_argument("--seg", type=int, default=50)
    p.add_argument("--nosponge", action="store_true")
    p.add_argument("--random", action="store_true")
    p.add_argument("--m1", action="store_true", help="scalar m = 1 (no division)")
    p.add_argument("--count", action="store_true", help="report slow-path quads (instrumented lib)")
    p.add_argument("--f64", action="store_true", help="float64 levels (a64 kernels)")
    a = p.parse_args()
    import numpy as np
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=a.order, n_t=a.nt, dims=(a.grid,) * 3)
    if a.nosponge:
        cfg.sponge = None
    if a.m1:
        cfg = B.KernelConfig(order=cfg.order, dims=cfg.dims, n_t=cfg.n_t, dt=0.4 * cfg.h, h=cfg.h,
                             m=1.0, source=cfg.source, receivers=cfg.receivers, sponge=cfg.sponge)
    slow = None
    if a.count:
        import ctypes

        from paper_1608_03984_b200 import _lib

        slow = _lib.load().fdr_debug_slow_quads
        slow.restype = ctypes.c_ulonglong
        slow.argtypes = [ctypes.c_int]
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64 if a.f64 else torch.float32)
    npts = float(np.prod(cfg.dims))
    B.run(fld, cfg, 1)
    fld.it = 0
    for g in fld.grids:
        g.zero_()
    if a.random:
        rng = np.random.default_rng(1)
        dt = np.float64 if a.f64 else np.float32
        fld.set_interior(2, rng.standard_normal(cfg.dims).astype(dt))
        fld.set_interior(1, rng.standard_normal(cfg.dims).astype(dt))
    done = 0
    while done < a.nt:
        n = min(a.seg, a.nt - done)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if slow is not None:
            slow(1)
        B.run(fld, cfg, n)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / n
        u = fld.interior().abs()
        tiny = 2.0 ** (-900 if a.f64 else -100)
        sub = 2.0 ** (-1022 if a.f64 else -126)
        st = {"steps": f"{done}-{done + n}", "ms_per_step": round(ms, 4),
              "gpts": round(npts / ms / 1e6, 1),
              "zero": round(float((u == 0).float().mean()), 4),
              "subnormal": round(float(((u > 0) & (u < sub)).float().mean()), 4),
              "lt_2m100": round(float(((u > 0) & (u < tiny)).float().mean()), 4),
              "max": float(u.max())}
        if slow is not None:
            st["slow_frac"] = round(slow(1) / n / (npts / 4), 5)
        print(json.dumps(st), flush=True)
        done += n


if __name__ == "__main__":
    main()
