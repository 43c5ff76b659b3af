"""`python -m paper_1608_03984_b200` -- the bench front end of the reference's
CLI (/root/reference/pkg/src/fdroof/cli.py:306-342, parser at cli.py:413-422)
on the B200 kernel, plus `machines list|show` for the machine documents.

    python -m paper_1608_03984_b200 bench --order 8 --grid 512 --nt 100 \
        --machine b200 [--repeat 3] [--svg roof.svg] [--dump field.bin]

Same arguments, workload and report lines as `fdroof bench`: dt = 0.5 x the
CFL bound at h = 1, no source (seeded random start), GFLOPS from the
catalogue FLOPs per point, attainable from the machine's roof.  `--slabs` is
accepted for compatibility; the CTA grid replaces the reference's slab
threads.  Errors print `error: ...` and exit 2, as the reference does.
"""

import argparse
import statistics
import sys

from .errors import FdroofError


def fmt(x) -> str:
    """At most 4 decimals, integers bare, scientific outside [1e-4, 1e15)."""
    if isinstance(x, int):
        return str(x)
    x = float(x)
    if x != x:
        return "nan"
    if x in (float("inf"), float("-inf")):
        return "inf" if x > 0 else "-inf"
    if x == 0:
        return "0"
    if abs(x) < 1e15 and x == int(x):
        return str(int(x))
    if 1e-4 <= abs(x) < 1e15:
        s = f"{x:.4f}".rstrip("0").rstrip(".")
        return s if s not in ("", "-") else "0"
    mant, exp = f"{x:.4e}".split("e")
    return f"{mant.rstrip('0').rstrip('.')}e{exp}"


def _registry(args):
    from . import roofline as RL

    reg = RL.builtin_machines()
    reg["b200"] = RL.b200_machine()  # measured roof when MEASURED_PEAKS.json exists
    for path in args.machines_file:
        reg.update(RL.load_machines(path))
    return reg


def cmd_machines(args):
    reg = _registry(args)
    if args.action == "list":
        for name in sorted(reg):
            m = reg[name]
            print(f"{name:12s} {fmt(m.peak_gflops_achievable)} GFLOPS  "
                  f"{fmt(m.peak_bw_achievable)} GB/s  ridge {fmt(m.ridge_point)}")
        return 0
    if not args.name or args.name not in reg:
        raise FdroofError(f"unknown machine {args.name!r}; known: {sorted(reg)}")
    m = reg[args.name]
    print(f"name:              {m.name}")
    print(f"achievable:        {fmt(m.peak_gflops_achievable)} GFLOPS, {fmt(m.peak_bw_achievable)} GB/s")
    if m.peak_gflops_theoretical is not None or m.peak_bw_theoretical is not None:
        print(f"theoretical:       {fmt(m.peak_gflops_theoretical or 0)} GFLOPS, "
              f"{fmt(m.peak_bw_theoretical or 0)} GB/s")
    print(f"ridge point:       {fmt(m.ridge_point)} FLOPs/byte")
    print(f"precision:         {m.precision_bytes} bytes")
    if m.notes:
        print(f"notes:             {m.notes}")
    if m.source:
        print(f"source:            {m.source}")
    return 0


def cmd_bench(args):
    from . import charts, kernel
    from . import roofline as RL

    reg = _registry(args)
    if args.machine not in reg:
        raise FdroofError(f"unknown machine {args.machine!r}; known: {sorted(reg)}")
    machine = reg[args.machine]
    if args.repeat < 1:
        raise FdroofError("--repeat must be >= 1")
    dims = (args.grid,) * 3
    dt = 0.5 * kernel.max_stable_dt(args.order, 1.0)
    cfg = kernel.KernelConfig(order=args.order, dims=dims, n_t=args.nt, dt=dt)
    results = [kernel.run_benchmark(cfg, machine, slabs=args.slabs, variant=args.variant)
               for _ in range(args.repeat)]
    best = max(results, key=lambda r: r.measured_gflops)
    point = best.point
    print(f"order {args.order} (k={cfg.k}), grid {args.grid}^3, {args.nt} steps")
    print(f"oi:                {fmt(point.oi)} FLOPs/byte (grid-size independent)")
    print(f"attainable:        {fmt(point.attainable_gflops)} GFLOPS on {machine.name} "
          f"({point.bound}-bound)")
    if args.repeat > 1:
        vals = sorted(r.measured_gflops for r in results)
        print(f"measured:          min {fmt(vals[0])} / median {fmt(statistics.median(vals))} / "
              f"max {fmt(vals[-1])} GFLOPS over {args.repeat} runs")
    else:
        print(f"measured:          {fmt(best.measured_gflops)} GFLOPS in {best.wall_time_s:.3f} s")
    print(f"of attainable:     {best.measured_gflops / point.attainable_gflops * 100.0:.1f}%")
    gpts = float(args.grid) ** 3 * args.nt / best.wall_time_s / 1e9
    print(f"updates:           {fmt(gpts)} GPts/s")
    bad = best.wavefield.nonfinite_count()
    print(f"final field:       {'finite' if bad == 0 else f'{bad} NaN/inf values'}")
    if bad:  # the failure check: a diverged run is a computation error
        raise FdroofError(f"the final wavefield has {bad} non-finite values (unstable dt?)")
    if args.dump:
        kernel.dump_wavefield(results[-1].wavefield, args.dump)
        print(f"wrote {args.dump}")
    if args.svg:
        ds = RL.roofline_dataset(machine, (point,))
        charts.write_svg(charts.roofline_chart(ds), args.svg)
        print(f"wrote {args.svg}")
    return 0


def cmd_point(args):
    """Place a measured rate of any catalogue equation on a machine's roofline
    (the reference's `oi` / `predict` view for one equation, with a measured
    point): TTI and elastic-VS included (roofline.EQUATIONS, --equations-file)."""
    from . import charts
    from . import roofline as RL

    reg = _registry(args)
    if args.machine not in reg:
        raise FdroofError(f"unknown machine {args.machine!r}; known: {sorted(reg)}")
    machine = reg[args.machine]
    eqs = dict(RL.EQUATIONS)
    for path in args.equations_file:
        eqs.update(RL.load_equations(path))
    if args.equation not in eqs:
        raise FdroofError(f"unknown equation {args.equation!r}; known: {sorted(eqs)}")
    eq = eqs[args.equation]
    pt = RL.equation_point(machine, eq, args.k, measured_gpts=args.gpts)
    print(f"equation:          {eq.name} (k={args.k})")
    print(f"flops/point:       {RL.kernel_flops(eq, args.k)}")
    print(f"bytes/point:       {RL.equation_bytes_per_point(eq, machine.precision_bytes)}")
    print(f"oi:                {fmt(pt.oi)} FLOPs/byte")
    print(f"attainable:        {fmt(pt.attainable_gflops)} GFLOPS on {machine.name} ({pt.bound}-bound)")
    if args.gpts is not None:
        print(f"measured:          {fmt(pt.measured_gflops)} GFLOPS ({fmt(args.gpts)} GPts/s)")
        print(f"of attainable:     {pt.fraction * 100.0:.1f}%")
    if args.svg:
        charts.write_svg(charts.roofline_chart(RL.roofline_dataset(machine, (pt,))), args.svg)
        print(f"wrote {args.svg}")
    return 0


def build_parser():
    p = argparse.ArgumentParser(prog="paper_1608_03984_b200",
                                description="B200 time stepping for the fdroof acoustic kernel")
    p.add_argument("--machines-file", action="append", default=[], metavar="PATH",
                   help="extra machine YAML documents (reference schema)")
    sub = p.add_subparsers(dest="cmd", required=True)
    sp = sub.add_parser("machines", help="list or show machine documents")
    sp.add_argument("action", choices=("list", "show"))
    sp.add_argument("name", nargs="?")
    sp.set_defaults(func=cmd_machines)
    sp = sub.add_parser("bench", help="run the acoustic kernel on the GPU")
    sp.add_argument("--order", type=int, required=True)
    sp.add_argument("--grid", type=int, required=True, metavar="N_PER_DIM")
    sp.add_argument("--nt", type=int, required=True)
    sp.add_argument("--machine", required=True)
    sp.add_argument("--svg")
    sp.add_argument("--repeat", type=int, default=1)
    sp.add_argument("--slabs", type=int, default=1)
    sp.add_argument("--dump", metavar="PATH")
    sp.add_argument("--variant", default="auto", choices=("auto", "queue", "tma", "direct"))
    sp.set_defaults(func=cmd_bench)
    sp = sub.add_parser("point", help="one equation's roofline point (TTI, elastic-vs, ...)")
    sp.add_argument("--equation", required=True)
    sp.add_argument("--k", type=int, default=9, help="stencil points per line (order + 1)")
    sp.add_argument("--machine", required=True)
    sp.add_argument("--gpts", type=float, help="measured grid-point updates per second (1e9)")
    sp.add_argument("--equations-file", action="append", default=[], metavar="PATH")
    sp.add_argument("--svg")
    sp.set_defaults(func=cmd_point)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except FdroofError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
