"""Repeat the two-step kernel at 512^3 and compare with the single-step one."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config2

order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
nt = int(sys.argv[3]) if len(sys.argv) > 3 else 9
cfg = config2(order=order, n_t=nt, dims=(512, 512, 512))
rng = np.random.default_rng(40 + order)
cur = rng.standard_normal(cfg.dims, dtype=np.float32)
prev = rng.standard_normal(cfg.dims, dtype=np.float32)
fld = B.Wavefield.allocate(cfg.dims, cfg.halo)

def go(variant):
    fld.it = 0
    fld.set_interior(2, cur); fld.set_interior(1, prev)
    for g in fld.grids[:1]:
        g.zero_()
    B.run(fld, cfg, variant=variant)
    torch.cuda.synchronize()
    return fld.numpy(2), fld.numpy(1)

ref2, ref1 = go("queue")
bad = 0
for i in range(reps):
    b2, b1 = go("tb2")
    d2 = np.argwhere(ref2.view(np.int32) != b2.view(np.int32))
    d1 = np.argwhere(ref1.view(np.int32) != b1.view(np.int32))
    if len(d2) or len(d1):
        bad += 1
        for name, d in (("newest", d2), ("prev", d1)):
            if len(d):
                xs = np.unique(d[:, 0])
                print(f"rep {i}: {name} {len(d)} diffs; x planes {xs[:10]}..; y {d[:,1].min()}..{d[:,1].max()} z {d[:,2].min()}..{d[:,2].max()}", flush=True)
print(f"order {order}: {bad} of {reps} runs differ", flush=True)
