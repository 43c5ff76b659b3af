"""float64 config-2 step time early in the run (mostly-zero wavefield) and on
random levels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=500)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    B.run(fld, cfg, 20)
    torch.cuda.synchronize()
    for label in ("early (steps 20-40)", "random levels"):
        if label.startswith("random"):
            fld.grids[2].normal_()
            fld.grids[1].normal_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        B.run(fld, cfg, 20)
        b.record()
        b.synchronize()
        print(f"{label}: {a.elapsed_time(b) / 20:.3f} ms/step")


if __name__ == "__main__":
    main()
