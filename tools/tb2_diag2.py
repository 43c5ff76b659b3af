import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1608_03984_b200 as B
from paper_1608_03984_b200.synthetic import config2

order = 2
cfg = config2(order=order, n_t=9, dims=(512, 512, 512))
rng = np.random.default_rng(42)
cur = rng.standard_normal(cfg.dims, dtype=np.float32)
prev = rng.standard_normal(cfg.dims, dtype=np.float32)

def fresh(variant):
    f = B.Wavefield.allocate(cfg.dims, cfg.halo)
    f.set_interior(2, cur); f.set_interior(1, prev)
    B.run(f, cfg, variant=variant)
    r = (f.numpy(2), f.numpy(1), f.traces.cpu().numpy().copy())
    del f
    return r

shared = B.Wavefield.allocate(cfg.dims, cfg.halo)
def reused(variant):
    f = shared
    f.it = 0
    f.grids[0].zero_()
    f.set_interior(2, cur); f.set_interior(1, prev)
    B.run(f, cfg, variant=variant)
    return (f.numpy(2), f.numpy(1), f.traces.cpu().numpy().copy())

def cmp(a, b):
    return [int((x.view(np.int32) != y.view(np.int32)).sum()) for x, y in zip(a, b)]

qf = fresh("queue")
tf = fresh("tb2")
print("tb2 fresh vs queue fresh", cmp(tf, qf), flush=True)
qr1 = reused("queue")
print("queue reused vs fresh", cmp(qr1, qf), flush=True)
tr1 = reused("tb2")
print("tb2 reused(after queue) vs queue fresh", cmp(tr1, qf), flush=True)
tr2 = reused("tb2")
print("tb2 reused(after tb2) vs queue fresh", cmp(tr2, qf), flush=True)
qr2 = reused("queue")
print("queue reused(after tb2) vs queue fresh", cmp(qr2, qf), flush=True)
tf2 = fresh("tb2")
print("tb2 fresh again vs queue fresh", cmp(tf2, qf), flush=True)
d = np.argwhere(tr1[0].view(np.int32) != qf[0].view(np.int32))
if len(d):
    x, y, z = d[0]
    print("first diff", d[0], "tb2", tr1[0][x, y, z], "queue", qf[0][x, y, z], flush=True)
    print("src", cfg.source.location, "sponge W planes", int((cfg.sponge.x < 1).sum()), flush=True)
