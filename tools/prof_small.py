"""One config-1 style run on a given variant (ncu target for the small-grid kernels).

    python tools/prof_small.py [variant] [nt] [n]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config1

    variant = sys.argv[1] if len(sys.argv) > 1 else "cluster"
    nt = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    cfg = config1(dims=(n, n, n), n_t=nt)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg, variant=variant)
    torch.cuda.synchronize()
    print("ok", variant, nt, float(fld.interior().abs().max()))


if __name__ == "__main__":
    main()
