"""Time the TTI step on BASELINE config 4 (384^3, order 8); device events."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1608_03984_b200 import tti

    nt = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    cfg = tti.config4(n_t=nt)
    npts = float(np.prod(cfg.dims))
    for variant, il in (("queue", True), ("queue", False), ("stream", False)):
        fld = tti.TTIWavefield.allocate(cfg.dims, cfg.halo, interleaved=il)
        tti.tti_run(fld, cfg, 2, variant=variant)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        tti.tti_run(fld, cfg, nt, variant=variant)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / nt
        g = npts / ms / 1e6
        print(json.dumps({"variant": variant, "interleaved": il, "ms_per_step": round(ms, 4), "gpts": round(g, 2),
                          "gflops_catalog": round(g * tti.tti_flops_per_point(8), 1),
                          "gbs_60B": round(g * 60, 1)}), flush=True)


if __name__ == "__main__":
    main()
