"""Does the headline rate depend on where the levels sit in HBM?  Times the
config-2 order-8 simulation on two Wavefields allocated one after the other,
alternating, several simulations each (device events).

    python tools/alloc_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = config2(order=8, n_t=500, dims=(512, 512, 512))
    npts = float(np.prod(cfg.dims))
    flds = [B.Wavefield.allocate(cfg.dims, cfg.halo) for _ in range(2)]
    st = torch.cuda.current_stream()

    def sim(f):
        for g in f.grids:
            g.zero_()
        f.it = 0
        B.run(f, cfg)

    for f in flds:
        sim(f)
    torch.cuda.synchronize()
    for rnd in range(2):
        for i, f in enumerate(flds):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(reps):
                sim(f)
            b.record(st)
            b.synchronize()
            ms = a.elapsed_time(b) / reps
            print(f"round {rnd} field {i}: {ms:.2f} ms/sim, {npts * cfg.n_t / ms / 1e6:.1f} GPts/s, "
                  f"levels at {[hex(g.data_ptr()) for g in f.grids]}", flush=True)


if __name__ == "__main__":
    main()
