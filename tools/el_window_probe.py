"""Elastic config 5 under the windowed schedule (B200FD_EL_WINDOW* knobs, read by
the library at first use): time per step, and a sha256 over the nine final
fields and the traces so that runs with different schedules can be compared
bit for bit.  usage: el_window_probe.py N_STEPS [--hash-steps M]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1608_03984_b200 import elastic

    nt = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    hash_steps = 12
    cfg = elastic.config5(n_t=max(nt, hash_steps))
    npts = float(np.prod(cfg.dims))
    fld = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo)
    elastic.elastic_run(fld, cfg, hash_steps, variant="queue")
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for k in elastic.FIELDS:
        h.update(np.ascontiguousarray(fld.numpy(k)).tobytes())
    if fld.traces is not None:
        h.update(np.ascontiguousarray(fld.traces.cpu().numpy()[:hash_steps]).tobytes())
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    elastic.elastic_run(fld, cfg, nt, variant="queue")
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / nt
    g = npts / ms / 1e6
    from paper_1608_03984_b200 import _lib
    pend = _lib.load().fdr_pending_error()
    print(json.dumps({"fuse": os.environ.get("B200FD_EL_FUSE", "0"),
                      "fuse_lag": os.environ.get("B200FD_EL_FUSE_LAG", "160"),
                      "pending_error": pend,
                      "window": os.environ.get("B200FD_EL_WINDOW", "0"),
                      "streams": os.environ.get("B200FD_EL_WINDOW_STREAMS", "1"),
                      "lead": os.environ.get("B200FD_EL_WINDOW_LEAD", "3"),
                      "sub": os.environ.get("B200FD_EL_WINDOW_SUB", "1"),
                      "ms_per_step": round(ms, 4), "gpts": round(g, 2),
                      "sha256_12_steps": h.hexdigest()[:16]}), flush=True)


if __name__ == "__main__":
    main()
