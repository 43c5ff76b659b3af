"""Summarise an `ncu --metrics ... --csv` run of tools/ncu_flops.sh: per kernel,
FLOPs per launch counted from the SASS thread-instruction counters (FADD, FMUL
= 1, FFMA, FADD2, FMUL2 = 2, FFMA2 = 4), DRAM bytes per launch and duration."""
import csv
import json
import sys
from collections import defaultdict

W = {"fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}


def summarise(path, points=None):
    rows = [ln for ln in open(path, encoding="utf-8") if ln.startswith('"')]
    rd = list(csv.DictReader(rows))
    per = defaultdict(dict)
    for r in rd:
        key = (r["ID"], r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        per[key][r["Metric Name"]] = v
    out = defaultdict(list)
    for (kid, name), m in per.items():
        fl = sum(W[k] * m.get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0) for k in W)
        dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        ns = m.get("gpu__time_duration.sum", 0.0)
        out[name.split("(")[0]].append({"flops": fl, "dram_bytes": dram, "ns": ns})
    res = {}
    for name, launches in out.items():
        n = len(launches)
        avg = {k: sum(x[k] for x in launches) / n for k in ("flops", "dram_bytes", "ns")}
        d = {"launches": n, "flops_per_launch": avg["flops"], "dram_bytes_per_launch": avg["dram_bytes"],
             "us_per_launch": avg["ns"] / 1e3}
        if points:
            d["flops_per_point"] = avg["flops"] / points
            d["dram_bytes_per_point"] = avg["dram_bytes"] / points
        res[name] = d
    return res


if __name__ == "__main__":
    pts = float(sys.argv[2]) if len(sys.argv) > 2 else None
    print(json.dumps(summarise(sys.argv[1], pts), indent=1))
