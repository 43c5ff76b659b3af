"""Benchmark of the acoustic hot path on B200 (driver contract).

One bench "step" = one complete BASELINE config-2 simulation at space order 8:
a 512^3 grid with the smooth random model, sponge, 15 Hz Ricker source and
512 receivers, advanced n_t = 500 time steps from zeroed levels (the zeroing
is inside the step).  `value` = whole-job grid-point updates per second
(GPts/s) with inputs resident in HBM; `e2e` = the same metric through the
public host-buffer API (HostSimulation.run_pipelined ->
fdr_acoustic_host_upload / _run_ws / _download), with every simulation's H2D upload of m /
sponge / series / receivers and D2H download of the final wavefield and
traces inside the timed region; two simulations are in flight, so one's
copies overlap the other's time steps (back-to-back shots).  Inputs (2.1 GB of
levels + m) exceed the 126 MB L2, so no flush is needed between steps.

--impl reference times the reference's own CPU implementation on the same
config: the unmodified fdroof.kernel.step (installed from /root/reference into
baseline/_ref, which travels to the GPU box; numpy ufuncs with x-slab threads
= host cores), driven like the reference's run loop (kernel.py:281-284) with
the sponge taper, injection and receivers applied around it (SURVEY.md
§8(a')).  One bench step = one time step of the 512^3 grid.  Without
baseline/_ref the numpy port in oracle/ stands in (kind "port").

Multi-GPU: replicas only: every rank runs its own independent
simulation; the timed region is bracketed by barriers, the time is the max
over ranks and `value` sums all ranks' updates ("scaling": "weak").
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "GPts/s (grid-point updates/sec) and % of roofline per space order, 1 B200"
UNIT = "GPts/s"
E2E_DEPTH = 2  # simulations in flight in the end-to-end leg (copies overlap steps)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--order", type=int, default=8)
    p.add_argument("--grid", type=int, default=512)
    p.add_argument("--nt", type=int, default=500)
    p.add_argument("--variant", default="auto")
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-steps", type=int, default=16)  # ~10 s of CPU work on the 16-core GPU box
    p.add_argument("--no-fp64", action="store_true", help="skip the float64 leg")
    p.add_argument("--no-configs", action="store_true",
                   help="skip the BASELINE configs 1, 3, 4, 5 lines")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        try:  # in-process NVML: microseconds per sample, no process spawn beside the timed work
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.02)
            pynvml.nvmlShutdown()
            return
        except Exception:  # noqa: BLE001  (no NVML binding: fall back to nvidia-smi)
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def max_over_ranks(x, pg, device):
    """The job's time is the slowest rank's device time (contract: max over ranks)."""
    if pg is None:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(world, per_rank_units, ms):
    """Units all ranks processed / the max-over-ranks time, in G units/s (weak
    scaling: every replica runs the full per-GPU workload)."""
    return world * float(per_rank_units) / (ms / 1e3) / 1e9


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_stepper(cfg, cores):
    """One time step of the reference on the CPU, as a closure, and its kind.

    "reference": the unmodified fdroof.kernel.step (baseline/_ref) on a
    source-free copy of the config, then the sponge taper on the new level,
    the injection of series[it] and the receiver sample -- the order of
    SURVEY.md §8(a') (tests/golden/make_golden.py::run_extended).
    "port": the numpy restatement oracle/acoustic.py::step (same result bit
    for bit, tests/test_oracle.py), when baseline/_ref is absent."""
    if os.path.isdir(os.path.join(REF_DIR, "fdroof")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from fdroof import kernel as K

        kcfg = K.KernelConfig(order=cfg.order, dims=tuple(cfg.dims), n_t=cfg.n_t, dt=cfg.dt,
                              h=cfg.h, m=np.asarray(cfg.m, np.float32))
        fld = K.Wavefield.allocate(kcfg.dims, kcfg.halo)
        from oracle import acoustic as O

        taper = O.sponge_taper(cfg)
        r = kcfg.halo
        series = np.asarray(cfg.source.series).astype(np.float32)
        loc = tuple(c + r for c in cfg.source.location)
        rec = cfg.receivers.locations
        traces = np.zeros((cfg.n_t, rec.shape[0]), np.float32)

        def one():
            it = fld.it
            K.step(fld, kcfg, slabs=cores)
            new = fld.interior(2)
            new *= taper
            if it < len(series):
                fld.grids[2][loc] += series[it]
            traces[it % cfg.n_t] = new[rec[:, 0], rec[:, 1], rec[:, 2]]

        one.latest = lambda: fld.interior(2)
        return one, "reference", "unmodified fdroof.kernel.step (baseline/_ref)"
    from oracle import acoustic as O

    st = O.OracleState(cfg.dims, cfg.halo)
    taper = O.sponge_taper(cfg)
    st.traces = np.zeros((cfg.n_t, cfg.receivers.count), np.float32)

    def one():
        O.step(st, cfg, slabs=cores, taper=taper)

    one.latest = st.latest
    return one, "port", "numpy port of fdroof.kernel.step (oracle/acoustic.py)"


def reference_arm(args):
    """The reference's CPU path (reference_stepper) on rank 0."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    from paper_1608_03984_b200.synthetic import config2

    cores = len(os.sched_getaffinity(0))
    dims = (args.grid,) * 3
    cfg = config2(order=args.order, n_t=args.nt, dims=dims)
    one, kind, what = reference_stepper(cfg, cores)
    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    wall = time.perf_counter() - t0
    pts = float(np.prod(dims))
    value = pts * args.steps / wall / 1e9
    sample = (f"{args.steps} timed time-steps (after {args.warmup} warm-up) of the "
              f"{dims[0]}^3 order-{args.order} update with sponge, source and receivers: "
              f"{what}, slabs={cores}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded smooth random model, BASELINE config 2)",
        "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args):
    return {"workload": f"acoustic order {args.order}, {args.grid}^3, {args.nt} time steps "
                        "(BASELINE config 2: smooth random model, sponge, Ricker, receivers)",
            "grid": [args.grid] * 3, "order": args.order, "n_t": args.nt, "h_m": 10.0,
            "l2": "inputs 4 x 0.54 GB > 126 MB L2 (no flush needed)",
            "parallelism": "replicas" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "single"}


def cpu_baseline(args, cfg):
    """The reference's CPU path on a bounded sample: args.cpu_steps time steps
    (after one warm-up) of the same 512^3 workload."""
    cores = len(os.sched_getaffinity(0))
    one, kind, what = reference_stepper(cfg, cores)
    one()  # warm
    t0 = time.perf_counter()
    for _ in range(args.cpu_steps):
        one()
    wall = time.perf_counter() - t0
    value = float(np.prod(cfg.dims)) * args.cpu_steps / wall / 1e9
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{args.cpu_steps} time steps (after 1 warm-up) of the {cfg.dims[0]}^3 "
                      f"order-{cfg.order} update with sponge, source and receivers: {what}, "
                      "x-slab threads = host cores"}


def time_device(fn, reps=1):
    """Device time (ms) of fn() on the current stream, after two warm calls
    (the second captures the CUDA graph small runs replay)."""
    import torch

    fn()
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def ncu_flops(key):
    """ncu-counted FLOPs / DRAM bytes per point of a production kernel
    (profiles/r02_ncu_flops.json, tools/ncu_flops.sh)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_flops.json"), encoding="utf-8") as fh:
            return json.load(fh).get(key, {})
    except (OSError, ValueError):
        return {}


def fp32_peak_tflops():
    """The FP32 roofline denominator measured here and now (fdr_fp32_fma_peak:
    FMA chains, no memory traffic), best of 3."""
    import ctypes

    from paper_1608_03984_b200 import _lib

    lib = _lib.load()
    best = 0.0
    for _ in range(3):
        tf = ctypes.c_double(0.0)
        _lib.check(lib.fdr_fp32_fma_peak(20000, 1, ctypes.byref(tf), None))
        best = max(best, tf.value)
    return best


def other_configs(dev, hbm):
    """BASELINE configs 1, 3, 4, 5, each run for its full n_t from zero fields
    (the acoustic ones with zeroed levels inside the timing)."""
    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import elastic, roofline as RL, tti
    from paper_1608_03984_b200.synthetic import config1, config3

    out = {}
    fp32_peak = fp32_peak_tflops() * 1e3  # GFLOP/s, measured
    for name, cfg in (("config1", config1()), ("config3", config3())):
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo, device=dev)

        def sim(c=cfg, f=fld):
            for g in f.grids:
                g.zero_()
            f.it = 0
            B.run(f, c)

        ms = time_device(sim)
        npts = float(np.prod(cfg.dims))
        g = npts * cfg.n_t / (ms / 1e3) / 1e9
        out[name] = {"workload": f"acoustic order {cfg.order}, {cfg.dims}, {cfg.n_t} steps",
                     "gpts_per_s": round(g, 2), "ms_per_sim": round(ms, 3),
                     "frac_hbm": round(g * 16 / hbm, 4), "bound": "hbm"}
        del fld
    cfg = tti.config4()
    fld = tti.TTIWavefield.allocate(cfg.dims, cfg.halo, device=dev)

    def sim4():
        for g in fld.p + fld.r:
            g.zero_()
        fld.it = 0
        tti.tti_run(fld, cfg)

    ms = time_device(sim4)
    g = float(np.prod(cfg.dims)) * cfg.n_t / (ms / 1e3) / 1e9
    fl = tti.tti_flops_per_point(cfg.order)
    counted = ncu_flops("tti_config4_384^3").get("void tti_pack<4, 1>", {})
    fl_ncu = counted.get("flops_per_point")
    out["config4"] = {
        "workload": f"TTI order 8, {cfg.dims}, {cfg.n_t} steps", "gpts_per_s": round(g, 2),
        "ms_per_sim": round(ms, 3),
        # the bound is set by the FLOPs the kernel executes (ncu), not the
        # catalogue's 964/pt: 242/pt over 60 B/pt is OI 4.0, below the ridge
        "bound": "hbm (60 B/pt; measured OI below the FP32 ridge)",
        "frac_hbm_60B": round(g * 60 / hbm, 4),
        "flops_per_point_ncu": fl_ncu, "dram_bytes_per_point_ncu": counted.get("dram_bytes_per_point"),
        "fp32_peak_gflops_measured": round(fp32_peak, 1),
        "frac_fp32_ncu_flops": round(g * fl_ncu / fp32_peak, 4) if fl_ncu else None,
        "gflops_catalog": round(g * fl, 1), "flops_per_point_catalog": fl}
    del fld
    cfg = elastic.config5()
    fld = elastic.ElasticWavefield.allocate(cfg.dims, cfg.halo, device=dev)

    def sim5():
        for g in fld.fields:
            g.zero_()
        fld.it = 0
        elastic.elastic_run(fld, cfg)

    ms = time_device(sim5)
    g = float(np.prod(cfg.dims)) * cfg.n_t / (ms / 1e3) / 1e9
    el = ncu_flops("elastic_config5_320^3")
    moved = sum(v.get("dram_bytes_per_point", 0.0) for v in el.values()) or None
    out["config5"] = {"workload": f"elastic velocity-stress order 8, {cfg.dims}, {cfg.n_t} steps",
                      "gpts_per_s": round(g, 2), "ms_per_sim": round(ms, 3),
                      "frac_hbm_84B": round(g * 84 / hbm, 4), "bound": "hbm (84 B/pt)",
                      "dram_bytes_per_point_ncu": moved,
                      "frac_hbm_moved": round(g * moved / hbm, 4) if moved else None}
    return out


def fp64_leg(dev, cfg, hbm, final32):
    """the config-2 simulation in float64 (fdr_acoustic64_run),
    timed on the device, and the float32 headline's final wavefield's relative
    L2 error against it."""
    import torch

    import paper_1608_03984_b200 as B

    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, device=dev, dtype=torch.float64)

    def sim():
        for g in fld.grids:
            g.zero_()
        fld.it = 0
        B.run(fld, cfg)

    ms = time_device(sim)
    g = float(np.prod(cfg.dims)) * cfg.n_t / (ms / 1e3) / 1e9
    ref = fld.interior(2).double()
    err = float(torch.linalg.vector_norm(final32.double() - ref) / torch.linalg.vector_norm(ref))
    return {"workload": f"acoustic order {cfg.order}, {tuple(cfg.dims)}, {cfg.n_t} steps, float64",
            "gpts_per_s": round(g, 2), "ms_per_sim": round(ms, 3), "bytes_per_point": 32,
            "frac_hbm": round(g * 32 / hbm, 4), "kernel": f"a64_queue<R={cfg.order // 2}> (AUTO)",
            "f32_rel_l2_vs_f64": err}


def step_loop_leg(cfg, dev, npts):
    """The reference's own calling pattern through the public API: one
    `step(fld, cfg)` call per time step (kernel.py:281-284).  Each timed shot
    uploads the config's inputs again (invalidate_plan, then the first step
    builds the device plan: m, sponge, series, receivers), zeroes the levels,
    makes n_t step() calls and downloads the final level and the traces;
    CUDA events bracket all of it on the compute stream."""
    import torch

    import paper_1608_03984_b200 as B

    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, device=dev)
    out = {}

    def shot():
        B.invalidate_plan(cfg)
        for g in fld.grids:
            g.zero_()
        fld.it = 0
        for _ in range(cfg.n_t):
            B.step(fld, cfg)
        out["final"] = fld.numpy(2)
        out["traces"] = fld.traces.cpu().numpy()

    shot()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    shot()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    h2d = int(np.asarray(cfg.m, np.float32).nbytes + 4 * sum(len(p) for p in
                                                             (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z))
              + 4 * len(cfg.source.series) + 12 * cfg.receivers.count)
    d2h = int(out["final"].nbytes + out["traces"].nbytes)
    del fld
    return {"value": round(npts * cfg.n_t / (ms / 1e3) / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_sim": round(ms, 3),
            "api": "invalidate_plan(cfg); n_t x step(fld, cfg); fld.numpy(); fld.traces.cpu() "
                   "(the reference's per-step loop, kernel.py:281-284)"}


def load_ncu_traffic(order):
    """DRAM bytes per launch of the step kernel from the committed ncu capture
    (profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path, encoding="utf-8") as fh:
            entry = json.load(fh).get(f"order{order}")
    except (OSError, ValueError):
        return None
    return None if entry is None else entry.get("traffic_bytes_per_launch")


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    import torch

    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200 import _lib
    from paper_1608_03984_b200.synthetic import config2

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    lib = _lib.load()

    dims = (args.grid,) * 3
    cfg = config2(order=args.order, n_t=args.nt, dims=dims)
    npts = float(np.prod(dims))
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one_sim(c=cfg, f=fld):
        for g in f.grids:
            g.zero_()
        f.it = 0
        B.run(f, c, variant=args.variant)

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        one_sim()
    launches_per_sim = int(lib.fdr_last_launch_count())
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for _ in range(args.steps):
            one_sim()
        t_end.record(stream)
        t_end.synchronize()
    barrier()
    ms = max_over_ranks(t_start.elapsed_time(t_end), pg, dev)
    per_rank_pts = npts * cfg.n_t * args.steps
    value = whole_job_rate(world, per_rank_pts, ms)

    from paper_1608_03984_b200 import roofline as RL

    peaks = RL.measured_peaks()
    hbm = float(peaks.get("hbm_gbs", RL.FALLBACK_HBM_GBS))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    launch_ms = ms / (args.steps * cfg.n_t)
    achieved = npts * RL.ACOUSTIC_BYTES_PER_POINT / (launch_ms / 1e3) / 1e9
    traffic = load_ncu_traffic(args.order)

    # e2e through the public host-buffer API
    e2e = None
    if not args.no_e2e:
        sim = B.HostSimulation(cfg, variant=args.variant, device=dev)
        sim.run_pipelined(E2E_DEPTH, depth=E2E_DEPTH)  # warm every slot
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.run_pipelined(args.steps, depth=E2E_DEPTH)
        e1.record(stream)
        e1.synchronize()
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1), pg, dev)
        e2e = {"value": whole_job_rate(world, per_rank_pts, ems), "unit": UNIT,
               "h2d_bytes_per_step": sim.h2d_bytes, "d2h_bytes_per_step": sim.d2h_bytes,
               "ms_per_step": ems / args.steps, "pipeline_depth": E2E_DEPTH,
               "api": "HostSimulation.run_pipelined -> fdr_acoustic_host_upload / _run_ws / "
                      "_download (each shot uploads its inputs and downloads its final level "
                      "and traces; steps on one stream, copies on two)"}
        del sim
        e2e["step_loop"] = step_loop_leg(cfg, dev, npts)

    # per-order sweep (config 2 is a sweep over orders 2..16)
    sweep = []
    if not args.no_sweep:
        for order in (2, 4, 8, 12, 16):
            c = B.KernelConfig(order=order, dims=cfg.dims, n_t=cfg.n_t, dt=cfg.dt, h=cfg.h, m=cfg.m,
                               source=cfg.source, receivers=cfg.receivers, sponge=cfg.sponge)
            f = B.Wavefield.allocate(c.dims, c.halo, device=dev)
            one_sim(c, f)
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            one_sim(c, f)
            b.record(stream)
            b.synchronize()
            sms = a.elapsed_time(b)
            g = npts * c.n_t / (sms / 1e3) / 1e9
            sweep.append({"order": order, "gpts_per_s": round(g, 3),
                          "achieved_gbs": round(g * 16, 1), "frac_hbm": round(g * 16 / hbm, 4),
                          "flops_per_pt": RL.acoustic_flops_per_point(order),
                          "gflops": round(g * RL.acoustic_flops_per_point(order), 1)})
            del f

    fp64 = None
    if rank == 0 and not args.no_fp64:
        one_sim()
        torch.cuda.synchronize(dev)
        fp64 = fp64_leg(dev, cfg, hbm, fld.interior(2))

    configs = None
    if rank == 0 and not args.no_configs:
        configs = other_configs(dev, hbm)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args, cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded smooth random model, BASELINE config 2)",
            "config": workload_config(args),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic,
                         "peak_source": peak_src,
                         "kernel": f"acoustic_queue<R={args.order // 2}> (one launch per time step)",
                         "bytes_per_launch": int(npts * 16), "launch_ms": round(launch_ms, 5)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_sim * args.steps,
            "clocks": clk.summary(),
            "per_order": sweep,
            "baseline_configs": configs,
            "fp64": fp64,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
