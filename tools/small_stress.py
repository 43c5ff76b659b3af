"""Repeatability of the small-grid kernels (cluster, persistent) on config 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config1

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = config1()
rng = np.random.default_rng(3)
cur = rng.standard_normal(cfg.dims, dtype=np.float32)
prev = rng.standard_normal(cfg.dims, dtype=np.float32)
for variant in ("cluster", "persistent", "queue", "auto"):
    f = B.Wavefield.allocate(cfg.dims, cfg.halo)
    outs = []
    for i in range(reps):
        f.it = 0
        for g in f.grids:
            g.zero_()
        f.set_interior(2, cur)
        f.set_interior(1, prev)
        B.run(f, cfg, variant=variant)
        torch.cuda.synchronize()
        outs.append(f.numpy(2).tobytes() + f.traces.cpu().numpy().tobytes())
    print(f"config1 {variant}: {sum(o != outs[0] for o in outs)} of {reps - 1} differ", flush=True)
