"""The opt-in FMA variant against the exact kernel on the config-2 workload
(512^3, smooth model, sponge, Ricker, receivers, 500 steps from zero): device
time of each and the FMA result's relative L2 drift (final level and traces)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config2


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / n) if n > 0 else float(np.linalg.norm(a - b))


orders = [int(o) for o in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,12,16").split(",")]
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 500
for order in orders:
    cfg = config2(order=order, n_t=nt)
    out = {}
    for variant in ("queue", "fma"):
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
        B.run(fld, cfg, 20, variant=variant)  # warm (plan, maps)
        for g in fld.grids:
            g.zero_()
        fld.it = 0
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        B.run(fld, cfg, variant=variant)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        out[variant] = (ms, fld.numpy(2), fld.traces.cpu().numpy()[:nt].copy())
        del fld
        torch.cuda.empty_cache()
    npts = float(np.prod(cfg.dims)) * nt
    q, f = out["queue"], out["fma"]
    print(json.dumps({"order": order, "n_t": nt,
                      "exact_gpts": round(npts / q[0] / 1e6, 2), "fma_gpts": round(npts / f[0] / 1e6, 2),
                      "fma_rel_l2_field": rel_l2(f[1], q[1]),
                      "fma_rel_l2_traces": rel_l2(f[2], q[2]) if np.abs(q[2]).max() > 1e-30 else None,
                      "exact_field_l2": float(np.linalg.norm(q[1].astype(np.float64)))}), flush=True)
