"""Count slow-path division quads per segment (instrumented build: -DFDR_COUNT_SLOW).

    B200FD_LIB=build/variants/libb200fd_count.so python tools/slow_count.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import _lib
    from paper_1608_03984_b200.synthetic import config2

    lib = _lib.load()
    fn = lib.fdr_debug_slow_quads
    fn.restype = ctypes.c_ulonglong
    fn.argtypes = [ctypes.c_int]
    cfg = config2(order=8, n_t=500, dims=(512, 512, 512))
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    quads = float(np.prod(cfg.dims)) / 4
    fn(1)
    for seg in range(10):
        B.run(fld, cfg, 50)
        torch.cuda.synchronize()
        n = fn(1)
        print(json.dumps({"steps": f"{seg * 50}-{seg * 50 + 50}", "slow_quads_per_step": n / 50,
                          "frac": n / 50 / quads}), flush=True)


if __name__ == "__main__":
    main()
