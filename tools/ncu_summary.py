"""Summarise an ncu report (raw page) into the metrics DESIGN.md / profiles/ cite.

    python tools/ncu_summary.py report.ncu-rep [--json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = f"{vals[i]} {units[i]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               h.startswith("smsp__pcsamp_warps_issue_stalled_"):
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0:
                    stalls[h] = v
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:12]
        d["top_stalls"] = dict(top)
        res.append(d)
    return res


if __name__ == "__main__":
    r = raw(sys.argv[1])
    if "--json" in sys.argv:
        print(json.dumps(r, indent=1))
    else:
        for d in r:
            for k, v in d.items():
                print(f"{k:70s} {v}")
