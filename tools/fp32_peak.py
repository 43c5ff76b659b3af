"""Measured FP32 FMA-pipe peak on this B200 (fdr_fp32_fma_peak): scalar FFMA
and packed FFMA2 chains, best of 5, with the SM clock sampled during the run.
Writes profiles/fp32_peak.json when given --out."""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def measure(iters=20000, reps=5):
    from paper_1608_03984_b200 import _lib

    lib = _lib.load()
    out = {}
    for packed in (0, 1):
        best = 0.0
        for _ in range(reps):
            tf, ms = ctypes.c_double(0), ctypes.c_double(0)
            _lib.check(lib.fdr_fp32_fma_peak(iters, packed, ctypes.byref(tf), ctypes.byref(ms)))
            best = max(best, tf.value)
        out["ffma2_tflops" if packed else "ffma_tflops"] = round(best, 2)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out")
    a = p.parse_args()
    import bench

    with bench.ClockSampler(0) as clk:
        res = measure()
    res["clocks"] = clk.summary()
    res["how"] = ("fdr_fp32_fma_peak: 148 x 8 CTAs x 256 threads, 8 independent FMA chains per "
                  "thread, 16 x 8 FMAs per loop iteration, no memory traffic; best of 5")
    print(json.dumps(res))
    if a.out:
        with open(a.out, "w", encoding="utf-8") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
