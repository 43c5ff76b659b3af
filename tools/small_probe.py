"""Per-size probe of the small-grid paths (device time per 100-step run)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config1

    sizes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
    variants = sys.argv[2].split(",")
    nt = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    for dims in sizes:
        cfg = config1(dims=dims, n_t=nt)
        for variant in variants:
            fld = B.Wavefield.allocate(cfg.dims, cfg.halo)

            def sim():
                for g in fld.grids:
                    g.zero_()
                fld.it = 0
                B.run(fld, cfg, variant=variant)

            for _ in range(3):
                sim()
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                sim()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            print(json.dumps({"dims": dims, "variant": variant, "ms": [round(t, 3) for t in ts],
                              "us_per_step": round(min(ts) * 1e3 / nt, 2)}), flush=True)


if __name__ == "__main__":
    main()
