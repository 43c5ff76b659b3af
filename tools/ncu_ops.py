"""Executed-instruction histogram by SASS opcode from an ncu report's source page.

    python tools/ncu_ops.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = rows[2:]
    i_s, i_e = hdr.index("Source"), hdr.index("Instructions Executed")
    i_w = hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stall = Counter(), Counter()
    total = 0
    for r in data:
        if not r[i_e].isdigit():
            continue
        toks = r[i_s].strip().split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        n = int(r[i_e])
        cnt[op] += n
        stall[op] += int(r[i_w] or 0)
        total += n
    print(f"total warp instructions {total}")
    for op, n in cnt.most_common(top):
        print(f"{op:10s} {n:12d} {100 * n / total:5.1f}%  stall-samples {stall[op]}")


if __name__ == "__main__":
    main()
