"""Summarise an ncu --import-source capture: stall samples by reason, by SASS
opcode and the hottest instructions (with their stall reasons).

usage: python tools/ncu_src_stalls.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         check=True, capture_output=True, text=True).stdout
    lines = out.splitlines()
    # first line is the kernel name
    return list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rs = rows(rep)
    reasons = [k for k in rs[0] if k.startswith("stall_") and "Not Issued" not in k]
    tot = Counter()
    by_op = defaultdict(Counter)
    execd = Counter()
    for r in rs:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        op = op.split(".")[0]
        execd[op] += int(r["Instructions Executed"] or 0)
        for k in reasons:
            v = int(r[k] or 0)
            tot[k] += v
            by_op[op][k] += v
    s = sum(tot.values())
    print(f"samples {s}; warp instructions executed {sum(execd.values())}")
    for k, v in tot.most_common():
        if v:
            print(f"  {k:24s} {v:7d} {100 * v / s:5.1f}%")
    print("by opcode (samples, top reasons; executed instructions)")
    for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
        n = sum(c.values())
        tops = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(3) if v)
        print(f"  {op:10s} {n:7d} {100 * n / s:5.1f}%  [{tops}]  exec {execd[op]}")
    print(f"hottest {top} instructions")
    hot = sorted(rs, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for r in hot:
        n = int(r["Warp Stall Sampling (All Samples)"] or 0)
        c = Counter({k: int(r[k] or 0) for k in reasons})
        tops = ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(3) if v)
        print(f"  {r['Address'][-5:]} {n:6d} {r['Source'].strip()[:60]:60s} [{tops}]")


if __name__ == "__main__":
    main()
