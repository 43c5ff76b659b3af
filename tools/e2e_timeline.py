"""Event timeline of 4 pipelined shots: when each upload / compute / download
starts and ends on its stream (ms from the batch start)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import _lib
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=500)
    sim = B.HostSimulation(cfg)
    sim.run_pipelined(2, depth=2)
    torch.cuda.synchronize()
    lib, args = sim.lib, ctypes.byref(sim.args)
    up, comp, down = sim._streams
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    sx, sy, sz = (p(t) for t in sim.h_sponge)
    T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    t0 = T()
    t0.record(torch.cuda.current_stream())
    for s in (up, comp, down):
        s.wait_event(t0)
    marks, cdone, ddone = [], [None] * 4, [None] * 4
    for i in range(4):
        ws, hf, ht = sim._slot(i % 2)
        if i >= 2:
            up.wait_event(cdone[i - 2])
        a = T(); a.record(up)
        _lib.check(lib.fdr_acoustic_host_upload(args, p(sim.h_m), sx, sy, sz, p(sim.h_series), p(sim.h_rec), ctypes.c_void_p(ws), sim.ws_bytes, ctypes.c_void_p(up.cuda_stream)))
        b = T(); b.record(up)
        comp.wait_event(b)
        if i >= 2:
            comp.wait_event(ddone[i - 2])
        c = T(); c.record(comp)
        nw = _lib.check(lib.fdr_acoustic_host_run_ws(args, 1, ctypes.c_void_p(ws), sim.ws_bytes, ctypes.c_void_p(comp.cuda_stream)))
        d = T(); d.record(comp)
        cdone[i] = d
        down.wait_event(d)
        e = T(); e.record(down)
        _lib.check(lib.fdr_acoustic_host_download(args, nw, p(hf), p(ht), ctypes.c_void_p(ws), sim.ws_bytes, ctypes.c_void_p(down.cuda_stream)))
        f = T(); f.record(down)
        ddone[i] = f
        marks.append((a, b, c, d, e, f))
    torch.cuda.synchronize()
    for i, (a, b, c, d, e, f) in enumerate(marks):
        print(f"shot {i}: up {t0.elapsed_time(a):8.2f}-{t0.elapsed_time(b):8.2f}  "
              f"comp {t0.elapsed_time(c):8.2f}-{t0.elapsed_time(d):8.2f}  "
              f"down {t0.elapsed_time(e):8.2f}-{t0.elapsed_time(f):8.2f}")


if __name__ == "__main__":
    main()
