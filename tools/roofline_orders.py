"""Roofline SVG of the acoustic step per space order: each order at its model
OI (FLOPs / 16 B) with its bound, the measurement from a bench.py JSON line
(per_order GPts/s x FLOPs per point), and a marker at the measured OI (FLOPs
/ ncu DRAM bytes per point, profiles/ncu_traffic.json).

    python tools/roofline_orders.py bench_line.json profiles/r01_roofline_orders.svg
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1608_03984_b200 import charts
    from paper_1608_03984_b200 import roofline as RL

    line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    m = RL.get_machine("b200")
    pts, moi = [], {}
    for row in line["per_order"]:
        o = row["order"]
        p = RL.roofline_point(m, o, measured_gflops=row["gpts_per_s"] * RL.acoustic_flops_per_point(o))
        pts.append(p)
        t = traffic.get(f"order{o}")
        if t:
            moi[p.label] = p.oi / t["traffic_over_algorithmic"]
    ds = RL.roofline_dataset(m, pts, margin=4.0)
    svg = charts.roofline_chart(ds, title="acoustic step per space order, 512^3 (B200)", measured_oi=moi)
    charts.write_svg(svg, sys.argv[2])
    sys.stdout.write(ds.to_csv())


if __name__ == "__main__":
    main()
