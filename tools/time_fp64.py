"""Time the float64 acoustic step (512^3 random levels, device events):
GPts/s and the fraction of the measured HBM bandwidth at 32 B/pt."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import roofline as RL

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    nt = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    hbm = RL.measured_peaks().get("hbm_gbs", RL.FALLBACK_HBM_GBS)
    for order in (2, 4, 8, 12, 16):
        dims = (n, n, n)
        rng = np.random.default_rng(order)
        m = (1.0 / np.square(1500.0 + 3000.0 * rng.random(dims, dtype=np.float32))).astype(np.float32)
        cfg = B.KernelConfig(order=order, dims=dims, n_t=nt, dt=0.4 * 10 / 4500.0, h=10.0, m=m)
        fld = B.Wavefield.allocate(dims, cfg.halo, dtype=torch.float64)
        fld.grids[2].normal_()
        fld.grids[1].normal_()
        nz = dims[2]
        for g in fld.grids:
            g[:, :, nz:] = 0
        for variant in ("queue", "tma", "direct") if order <= 8 else ("queue", "tma"):
            B.run(fld, cfg, 2, variant=variant)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            B.run(fld, cfg, nt, variant=variant)
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / nt
            g = n ** 3 / ms / 1e6
            print(json.dumps({"order": order, "variant": variant, "ms_per_step": round(ms, 4),
                              "gpts": round(g, 2), "gbs_32B": round(g * 32, 1),
                              "frac_hbm": round(g * 32 / hbm, 4)}), flush=True)


if __name__ == "__main__":
    main()
