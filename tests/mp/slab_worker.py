"""One rank of the world-size-2 gloo test of the x-slab decomposition
(tests/test_slab.py): the numpy oracle steps this rank's slab and the real
torch.distributed halo exchange refreshes its ghost planes after every step;
rank 0 checks the gathered field and traces against the full-grid oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import acoustic as O
    from paper_1608_03984_b200.slab import SlabPlan, exchange, slab_config, slab_halo
    from slab_cases import slab_case

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    results = {}
    for name, (cfg, nsteps) in slab_case().items():
        plan = SlabPlan(cfg.dims[0], world, slab_halo(cfg))
        local, rec_index = slab_config(cfg, plan, rank)
        st = O.OracleState(local.dims, local.halo)
        if local.receivers is not None:
            st.traces = np.zeros((cfg.n_t, local.receivers.count), np.float32)
        taper = O.sponge_taper(local)
        r, nxl = local.halo, local.dims[0]
        for _ in range(nsteps):
            O.step(st, local, taper=taper)
            exchange(torch.from_numpy(st.grids[2])[r: r + nxl], plan, rank)
        own = O.interior(st.grids[2], r)[plan.owned_local(rank)]
        parts = [None] * world
        dist.all_gather_object(parts, (plan.span(rank), own, rec_index,
                                       None if st.traces is None else st.traces))
        if rank == 0:
            full = O.simulate(cfg, nsteps)
            got = np.zeros(cfg.dims, np.float32)
            traces = np.zeros_like(full.traces) if full.traces is not None else None
            for (x0, x1), block, idx, tr in parts:
                got[x0:x1] = block
                if tr is not None and len(idx):
                    traces[:, idx] = tr
            results[name] = {
                "field_equal": bool(np.array_equal(got, full.latest())),
                "traces_equal": traces is None or bool(np.array_equal(traces, full.traces)),
                "nonzero": bool(np.abs(got).max() > 0),
            }
    if rank == 0:
        with open(os.environ["FDR_MP_OUT"], "w", encoding="utf-8") as fh:
            json.dump(results, fh)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
