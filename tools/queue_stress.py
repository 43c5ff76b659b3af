"""Determinism of the production queue kernel at 512^3 (repeated runs from the
same levels; prints where later runs differ from the first)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config2

p = argparse.ArgumentParser()
p.add_argument("--order", type=int, default=2)
p.add_argument("--reps", type=int, default=6)
p.add_argument("--nt", type=int, default=9)
p.add_argument("--grid", type=int, default=512)
p.add_argument("--variant", default="queue")
p.add_argument("--nosponge", action="store_true")
p.add_argument("--norec", action="store_true")
p.add_argument("--nosrc", action="store_true")
p.add_argument("--scalarm", action="store_true")
p.add_argument("--tag", default="")
a = p.parse_args()
base = config2(order=a.order, n_t=a.nt, dims=(a.grid,) * 3)
cfg = B.KernelConfig(order=a.order, dims=base.dims, n_t=a.nt, dt=base.dt, h=base.h,
                     m=(float(np.median(base.m)) if a.scalarm else base.m),
                     source=None if a.nosrc else base.source,
                     receivers=None if a.norec else base.receivers,
                     sponge=None if a.nosponge else base.sponge)
rng = np.random.default_rng(42)
cur = rng.standard_normal(cfg.dims, dtype=np.float32)
prev = rng.standard_normal(cfg.dims, dtype=np.float32)
f = B.Wavefield.allocate(cfg.dims, cfg.halo)
res = None
bad = 0
for i in range(a.reps):
    f.it = 0
    for g in f.grids:
        g.zero_()
    f.set_interior(2, cur)
    f.set_interior(1, prev)
    torch.cuda.synchronize()
    B.run(f, cfg, variant=a.variant)
    torch.cuda.synchronize()
    out = f.numpy(2)
    if res is None:
        res = out
        continue
    d = np.argwhere(out.view(np.int32) != res.view(np.int32))
    if len(d):
        bad += 1
        xs = np.unique(d[:, 0])
        print(f"  rep {i}: {len(d)} diffs; x {xs[:10]} y {d[:,1].min()}..{d[:,1].max()} "
              f"z {d[:,2].min()}..{d[:,2].max()}", flush=True)
print(f"{a.tag} order {a.order} {a.variant} nosponge={a.nosponge} norec={a.norec} nosrc={a.nosrc} "
      f"scalarm={a.scalarm}: {bad} of {a.reps - 1} later runs differ", flush=True)
