"""config-2 order-8 simulation from zero for profiling (ncu -s N -c 1 picks step N)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    nt = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    cfg = config2(order=8, n_t=nt)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg)
    torch.cuda.synchronize()
    print("ok", nt)
