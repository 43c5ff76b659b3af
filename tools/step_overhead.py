"""Host cost of the reference's calling pattern (one step() per time step,
kernel.py:281-284) against one run(): per-call wall time on a small grid
(GPU time per step ~ tens of microseconds) and a cProfile of the step loop."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=400, dims=(128, 128, 128))
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg, 4)
    torch.cuda.synchronize()
    t = time.perf_counter()
    B.run(fld, cfg, 400)
    torch.cuda.synchronize()
    run_us = (time.perf_counter() - t) / 400 * 1e6
    t = time.perf_counter()
    for _ in range(400):
        B.step(fld, cfg)
    torch.cuda.synchronize()
    step_us = (time.perf_counter() - t) / 400 * 1e6
    print(f"run(): {run_us:.1f} us/step   step(): {step_us:.1f} us/call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(400):
        B.step(fld, cfg)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
