"""GPU determinism stress: the BASELINE config-2 grid from seeded random levels,
run `reps` times per order; every run must match the first bit for bit (on the
device), and the first must match the C oracle.  Prints one line per order.

usage: python tools/determinism.py [reps] [orders...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))

import paper_1608_03984_b200 as B  # noqa: E402
from paper_1608_03984_b200.synthetic import config2  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    orders = [int(a) for a in sys.argv[2:]] or [2, 4, 8, 12, 16]
    bad_total = 0
    for order in orders:
        cfg = config2(order=order, n_t=3, dims=(512, 512, 512))
        rng = np.random.default_rng(order)
        cur = rng.standard_normal(cfg.dims, dtype=np.float32)
        prev = rng.standard_normal(cfg.dims, dtype=np.float32)
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
        cur_d = torch.from_numpy(cur).cuda()
        prev_d = torch.from_numpy(prev).cuda()
        first = None
        bad = []
        t0 = time.time()
        for i in range(reps):
            for g in fld.grids:
                g.zero_()
            fld.interior(2).copy_(cur_d)
            fld.interior(1).copy_(prev_d)
            fld.it = 0
            B.run(fld, cfg)
            out = fld.interior(2).clone()
            if first is None:
                first = out
            else:
                ne = (out.view(torch.int32) != first.view(torch.int32))
                n = int(ne.sum())
                if n:
                    idx = ne.nonzero()[:4].tolist()
                    bad.append((i, n, idx))
        torch.cuda.synchronize()
        dt = time.time() - t0
        # oracle check of the first run
        from oracle import acoustic as O
        from oracle import cref
        st = O.OracleState(cfg.dims, cfg.halo)
        O.interior(st.grids[2], st.halo)[...] = cur
        O.interior(st.grids[1], st.halo)[...] = prev
        cref.simulate(cfg, cfg.n_t, state=st)
        ref = np.ascontiguousarray(st.latest())
        got = first.cpu().numpy()
        nbad = int((got.view(np.int32) != ref.view(np.int32)).sum())
        where = np.argwhere(got.view(np.int32) != ref.view(np.int32))[:4].tolist() if nbad else []
        print(f"order {order}: reps {reps} ({dt:.1f}s) gpu-vs-gpu mismatching runs {len(bad)} {bad[:3]} "
              f"gpu-vs-oracle mismatches {nbad} {where}", flush=True)
        bad_total += len(bad) + (nbad > 0)
    print("DETERMINISM", "FAIL" if bad_total else "OK")


if __name__ == "__main__":
    main()
