"""Refresh profiles/ncu_traffic.json (the bench line's roofline.traffic) from an
ncu --metrics CSV of tools/ncu_flops.sh's acoustic leg (dram__bytes_read.sum +
dram__bytes_write.sum per acoustic_queue launch at 512^3).

    python tools/update_traffic.py gpurun_out/ncu_flops_o8.csv ORDER SOURCE_TAG
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_flops_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    csv_path, order, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    res = summarise(csv_path)
    name = next(k for k in res if "acoustic_queue" in k)
    d = res[name]
    alg = 16 * 512 ** 3
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    with open(path, encoding="utf-8") as fh:
        doc = json.load(fh)
    doc[f"order{order}"] = {
        "kernel": name,
        "traffic_bytes_per_launch": d["dram_bytes_per_launch"],
        "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": round(d["dram_bytes_per_launch"] / alg, 4),
        "ncu_duration_s": d["us_per_launch"] / 1e6,
        "launches": d["launches"],
        "source": tag,
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc[f"order{order}"], indent=1))


if __name__ == "__main__":
    main()
