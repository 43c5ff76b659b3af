"""Phase timing of the host-buffer path on the config-2 workload: upload,
compute, download alone, the synchronous run(), and run_pipelined()."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import _lib
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=int(sys.argv[1]) if len(sys.argv) > 1 else 500)
    sim = B.HostSimulation(cfg)
    lib = sim.lib
    args = ctypes.byref(sim.args)
    st = torch.cuda.current_stream()
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    sx, sy, sz = (p(t) for t in sim.h_sponge)

    def ev_time(fn, reps=1):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        return a.elapsed_time(b) / reps

    ws = ctypes.c_void_p(sim.ws_ptr)
    s = ctypes.c_void_p(st.cuda_stream)
    up = lambda: _lib.check(lib.fdr_acoustic_host_upload(args, p(sim.h_m), sx, sy, sz, p(sim.h_series), p(sim.h_rec), ws, sim.ws_bytes, s))  # noqa: E731
    newest = [0]

    def comp():
        newest[0] = _lib.check(lib.fdr_acoustic_host_run_ws(args, 1, ws, sim.ws_bytes, s))

    down = lambda: _lib.check(lib.fdr_acoustic_host_download(args, newest[0], p(sim.h_final), p(sim.h_traces), ws, sim.ws_bytes, s))  # noqa: E731
    out = {"upload_ms": ev_time(up), "compute_ms": ev_time(comp), "download_ms": ev_time(down)}
    out["run_sync_ms"] = ev_time(sim.run)
    for n, d in ((3, 2), (6, 2), (6, 3)):
        t = ev_time(lambda: sim.run_pipelined(n, depth=d))
        out[f"pipelined_{n}x_depth{d}_ms_per_shot"] = t / n
    w0 = time.perf_counter()
    sim.run_pipelined(4, depth=2)
    torch.cuda.synchronize()
    out["pipelined_4_wall_ms_per_shot"] = (time.perf_counter() - w0) * 1e3 / 4
    print(json.dumps({k: round(v, 2) for k, v in out.items()}))


if __name__ == "__main__":
    main()
