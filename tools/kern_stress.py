"""Run-to-run determinism of the TTI, elastic and float64 streaming kernels on
their BASELINE-size grids (repeated short runs from the same random levels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1608_03984_b200 as B
from paper_1608_03984_b200 import elastic, tti
from paper_1608_03984_b200.synthetic import config2

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(7)

cfg = tti.config4(n_t=4)
lv = {(f, l): rng.standard_normal(cfg.dims, dtype=np.float32) for f in "pr" for l in (1, 2)}
f = tti.TTIWavefield.allocate(cfg.dims, cfg.halo)
outs = []
for i in range(reps):
    f.it = 0
    for g in f.p + f.r:
        g.zero_()
    for (fl, l), v in lv.items():
        f.set_interior(fl, l, v)
    tti.tti_run(f, cfg)
    torch.cuda.synchronize()
    outs.append(f.numpy("p").tobytes() + f.numpy("r").tobytes())
print("tti config4:", sum(o != outs[0] for o in outs), "of", reps - 1, "differ", flush=True)
del f

cfg = elastic.config5(n_t=4)
lv = {k: rng.standard_normal(cfg.dims, dtype=np.float32) * 1e-3 for k in elastic.FIELDS}
f = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo)
outs = []
for i in range(reps):
    f.it = 0
    for k, v in lv.items():
        f.set_interior(k, v)
    elastic.elastic_run(f, cfg)
    torch.cuda.synchronize()
    outs.append(b"".join(f.numpy(k).tobytes() for k in elastic.FIELDS))
print("elastic config5:", sum(o != outs[0] for o in outs), "of", reps - 1, "differ", flush=True)
del f

for order in (2, 8):
    cfg = config2(order=order, n_t=9, dims=(512, 512, 512))
    cur = rng.standard_normal(cfg.dims)
    prev = rng.standard_normal(cfg.dims)
    f = B.Wavefield.allocate(cfg.dims, cfg.halo, dtype=torch.float64)
    outs = []
    for i in range(reps):
        f.it = 0
        for g in f.grids:
            g.zero_()
        f.set_interior(2, cur)
        f.set_interior(1, prev)
        B.run(f, cfg)
        torch.cuda.synchronize()
        outs.append(f.numpy(2).tobytes())
    print(f"float64 queue order {order}:", sum(o != outs[0] for o in outs), "of", reps - 1, "differ", flush=True)
    del f
