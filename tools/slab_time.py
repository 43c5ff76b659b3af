"""Cost of the library's x-slab exchange on one device: the config-2 run
(512^3, order 8) as 1, 2, 4, 8 slabs, all on this GPU (the slabs share it,
so the difference to one grid is the decomposition's overhead: the extra
boundary launches and the plane copies).  Device time of the library call
only (wavefields, plans and argument blocks built beforehand)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1608_03984_b200 as B
from paper_1608_03984_b200 import _lib
from paper_1608_03984_b200 import kernel as K
from paper_1608_03984_b200.slab import SlabPlan, slab_config
from paper_1608_03984_b200.synthetic import config2

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfg = config2(order=8, n_t=nt)
lib = _lib.load()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / nt


fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
base = timed(lambda: B.run(fld, cfg))
print(json.dumps({"slabs": "single grid", "ms_per_step": round(base, 4)}), flush=True)
del fld
mode = sys.argv[2] if len(sys.argv) > 2 else "one-stream"
for ns in (1, 2, 4, 8):
    plan = SlabPlan(cfg.dims[0], ns, cfg.halo)
    parts = [slab_config(cfg, plan, i) for i in range(ns)]
    flds = [K.Wavefield.allocate(c.dims, c.halo) for c, _ in parts]
    keep = [K.device_args(f, c, nt) for (c, _), f in zip(parts, flds)]
    arr = (_lib.AcousticArgs * ns)(*keep)
    dev = torch.cuda.current_device()
    devs = (ctypes.c_int * ns)(*([dev] * ns))
    cur = torch.cuda.current_stream()
    if mode == "one-stream":
        sts = [cur] * ns
    else:  # a stream per slab, as each slab would have its own GPU
        sts = [torch.cuda.Stream() for _ in range(ns)]
    streams = (ctypes.c_void_p * ns)(*[t.cuda_stream for t in sts])

    def call():
        for t in sts:
            t.wait_stream(cur)
        _lib.check(lib.fdr_acoustic_slabs_run(arr, ns, devs, streams))
        for t in sts:
            cur.wait_stream(t)

    ms = timed(call)
    print(json.dumps({"slabs": ns, "streams": mode, "ms_per_step": round(ms, 4),
                      "overhead_vs_single": round(ms / base - 1.0, 4),
                      "launches_per_step": lib.fdr_last_launch_count() / nt}), flush=True)
    del flds, keep, arr
    torch.cuda.empty_cache()
