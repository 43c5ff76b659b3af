"""float64 config-2 simulation (512^3 order 8, 500 steps from zero levels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=int(sys.argv[1]) if len(sys.argv) > 1 else 500)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    for rep in range(2):
        for g in fld.grids:
            g.zero_()
        fld.it = 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        B.run(fld, cfg)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        print(f"rep {rep}: {ms:.1f} ms, {512 ** 3 * cfg.n_t / ms / 1e6:.2f} GPts/s")


if __name__ == "__main__":
    main()
