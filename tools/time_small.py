"""Config-1 sized runs: queue vs direct kernel (device time per 100-step run)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config1

    for dims in ((64, 64, 64), (96, 96, 96), (128, 128, 128), (192, 192, 192)):
        cfg = config1(dims=dims)
        for variant in ("queue", "direct", "persistent"):
            fld = B.Wavefield.allocate(cfg.dims, cfg.halo)

            def sim():
                for g in fld.grids:
                    g.zero_()
                fld.it = 0
                B.run(fld, cfg, variant=variant)

            sim(); sim(); sim()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                sim()
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b) / 5
            n = dims[0] * dims[1] * dims[2] * cfg.n_t
            print(json.dumps({"dims": dims, "variant": variant, "ms_per_sim": round(ms, 4),
                              "gpts": round(n / ms / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    main()
