"""Where does the two-step kernel differ from the single-step one?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config2

def run(order, n, nt, variant, seed=42):
    cfg = config2(order=order, n_t=nt, dims=(n, n, n))
    rng = np.random.default_rng(seed)
    cur = rng.standard_normal(cfg.dims, dtype=np.float32)
    prev = rng.standard_normal(cfg.dims, dtype=np.float32)
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    fld.set_interior(2, cur); fld.set_interior(1, prev)
    B.run(fld, cfg, variant=variant)
    return fld.numpy(2), fld.numpy(1)

for order, n, nt in [(2, 512, 2), (2, 512, 4), (2, 512, 9), (2, 256, 9), (2, 384, 9), (4, 512, 9), (2, 128, 9)]:
    a2, a1 = run(order, n, nt, "queue")
    b2, b1 = run(order, n, nt, "tb2")
    d2 = np.argwhere(a2.view(np.int32) != b2.view(np.int32))
    d1 = np.argwhere(a1.view(np.int32) != b1.view(np.int32))
    msg = f"order {order} n {n} nt {nt}: newest diff {len(d2)}, prev diff {len(d1)}"
    for name, d in (("newest", d2), ("prev", d1)):
        if len(d):
            msg += f" | {name} x {d[:,0].min()}..{d[:,0].max()} y {d[:,1].min()}..{d[:,1].max()} z {d[:,2].min()}..{d[:,2].max()}"
    print(msg, flush=True)
