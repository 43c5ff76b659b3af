"""Where the step()-loop e2e leg spends its time (bench.py step_loop_leg): plan build (uploads),
n_t step() calls, numpy() of the final level, traces to the host."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=500)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)

    def sync():
        torch.cuda.synchronize()
        return time.perf_counter()

    for rep in range(2):
        t0 = sync()
        B.invalidate_plan(cfg)
        for g in fld.grids:
            g.zero_()
        fld.it = 0
        B.step(fld, cfg)
        t1 = sync()
        for _ in range(cfg.n_t - 1):
            B.step(fld, cfg)
        t2 = sync()
        out = fld.numpy(2)
        t3 = sync()
        tr = fld.traces.cpu().numpy()
        t4 = sync()
        print(json.dumps({"rep": rep, "plan_and_first_step_ms": round((t1 - t0) * 1e3, 1),
                          "steps_ms": round((t2 - t1) * 1e3, 1), "numpy_ms": round((t3 - t2) * 1e3, 1),
                          "traces_ms": round((t4 - t3) * 1e3, 1), "out_mb": out.nbytes / 1e6,
                          "traces_shape": list(tr.shape)}), flush=True)


if __name__ == "__main__":
    main()
