"""Generate the full-length parity goldens for BASELINE configs 2-5 -- TEST INFRASTRUCTURE.

Runs the exact C oracles (multithreaded, strict IEEE float32) over the complete
BASELINE runs on the CPU and records:

* sha256 of every generated input the kernels consume (m / the 9 TTI parameter
  grids / the 3 elastic parameter grids, the float32 source series, receiver
  locations, sponge profiles), so that input drift on another host is caught
  before any comparison;
* sha256 of the final wavefield (acoustic: the newest level and the previous
  one; TTI: p and r, newest and previous; elastic: all 9 fields) and of the
  receiver traces;
* L2 norm / max |.| of each final field and a strided sample of the final
  fields and traces (`full_length_samples.npz`) so that a hash mismatch can
  still be quantified (relative L2 on the sample).

Configs and oracles:

    config2_o{2,4,8,12,16}  acoustic 512^3, 500 steps  oracle/acoustic_ref.c (cref.simulate)
    config3                 acoustic 1024x1024x768, order 8, 200 steps   (cref.simulate)
    config4                 TTI 384^3, order 8, 300 steps    oracle/tti_ref.c (tti.simulate_c)
    config5                 elastic 320^3, order 8, 300 steps  oracle/elastic_ref.c

The acoustic C oracle is pinned bit for bit to the unmodified reference
`fdroof.kernel.step` (/root/reference/pkg/src/fdroof/kernel.py:176-222, loop at
:281-284) by tests/test_oracle.py; TTI/elastic have no reference
implementation (SURVEY.md §8(a')) and are pinned to their own exact C oracles.

Usage: python tests/golden/make_full_goldens.py [name ...]   (default: all)
Wall time on an 8-core host: ~20 min (config 2, all orders), ~8 min (config 3),
~30 min (config 4), ~7 min (config 5).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

JSON_PATH = os.path.join(HERE, "full_length.json")
NPZ_PATH = os.path.join(HERE, "full_length_samples.npz")

# strided samples of the final fields / traces (diagnostics on a hash mismatch)
FIELD_STRIDE = {"config2": 16, "config3": 32, "config4": 16, "config5": 16}
TRACE_STRIDE = 8


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample(a, s):
    return np.ascontiguousarray(a[::s, ::s, ::s])


def acoustic_inputs(cfg) -> dict:
    """Hashes of exactly the float32/int32 arrays the acoustic kernels consume."""
    out = {"m": sha(np.asarray(cfg.m, dtype=np.float32)),
           "series": sha(np.asarray(cfg.source.series).astype(np.float32)),
           "receivers": sha(np.asarray(cfg.receivers.locations, dtype=np.int32)),
           "sponge": sha(np.concatenate([np.asarray(p, np.float32) for p in
                                         (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
           "dt": float(cfg.dt)}
    return out


def field_stats(a) -> dict:
    a64 = a.astype(np.float64)
    return {"sha256": sha(a), "l2": float(np.sqrt(np.sum(a64 * a64))),
            "maxabs": float(np.max(np.abs(a64))), "finite": bool(np.isfinite(a).all())}


def gen_acoustic(name, cfg, samples):
    from oracle import cref

    t = time.time()
    st = cref.simulate(cfg)
    secs = time.time() - t
    h = st.halo
    final = st.grids[2][h:-h, h:-h, h:-h]
    prev = st.grids[1][h:-h, h:-h, h:-h]
    base = name.split("_")[0]
    samples[f"{name}/final"] = sample(final, FIELD_STRIDE[base])
    samples[f"{name}/traces"] = np.ascontiguousarray(st.traces[:, ::TRACE_STRIDE])
    return {"kind": "acoustic", "order": cfg.order, "dims": list(cfg.dims), "n_t": cfg.n_t,
            "inputs": acoustic_inputs(cfg), "final": field_stats(final),
            "prev": field_stats(prev), "traces": field_stats(st.traces),
            "field_stride": FIELD_STRIDE[base], "trace_stride": TRACE_STRIDE,
            "oracle": "oracle/acoustic_ref.c (oracle/cref.py::simulate)", "oracle_s": secs}


def gen_tti(name, samples):
    from oracle import tti as T
    from paper_1608_03984_b200 import tti

    cfg = tti.config4()
    prm = cfg.params()
    w2, w1 = tti.tti_weights_f32(cfg.order)
    inputs = {f"param_{k}": sha(prm[k]) for k in tti.PARAM_NAMES}
    inputs.update(series=sha(np.asarray(cfg.source.series).astype(np.float32)),
                  receivers=sha(np.asarray(cfg.receivers.locations, np.int32)),
                  sponge=sha(np.concatenate([np.asarray(p, np.float32) for p in
                                             (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
                  dt=float(cfg.dt))
    t = time.time()
    st = T.simulate_c(cfg, prm, w2, w1)
    secs = time.time() - t
    rec = {"kind": "tti", "order": cfg.order, "dims": list(cfg.dims), "n_t": cfg.n_t,
           "inputs": inputs, "traces": field_stats(st.traces),
           "field_stride": FIELD_STRIDE["config4"], "trace_stride": TRACE_STRIDE,
           "oracle": "oracle/tti_ref.c (oracle/tti.py::simulate_c)", "oracle_s": secs}
    for f in ("p", "r"):
        rec[f"{f}_final"] = field_stats(st.interior(f, 2))
        rec[f"{f}_prev"] = field_stats(st.interior(f, 1))
        samples[f"{name}/{f}"] = sample(st.interior(f, 2), FIELD_STRIDE["config4"])
    samples[f"{name}/traces"] = np.ascontiguousarray(st.traces[:, ::TRACE_STRIDE])
    return rec


def gen_elastic(name, samples):
    from oracle import elastic as E
    from paper_1608_03984_b200 import elastic

    cfg = elastic.config5()
    prm = cfg.params()
    inputs = {f"param_{k}": sha(prm[k]) for k in ("bs", "lam", "mu")}
    inputs.update(series=sha(np.asarray(cfg.source.series).astype(np.float32)),
                  receivers=sha(np.asarray(cfg.receivers.locations, np.int32)),
                  sponge=sha(np.concatenate([np.asarray(p, np.float32) for p in
                                             (cfg.sponge.x, cfg.sponge.y, cfg.sponge.z)])),
                  dt=float(cfg.dt))
    t = time.time()
    st = E.simulate_c(cfg, prm, elastic.elastic_weights_f32(cfg.order))
    secs = time.time() - t
    rec = {"kind": "elastic", "order": cfg.order, "dims": list(cfg.dims), "n_t": cfg.n_t,
           "inputs": inputs, "traces": field_stats(st.traces),
           "field_stride": FIELD_STRIDE["config5"], "trace_stride": TRACE_STRIDE,
           "oracle": "oracle/elastic_ref.c (oracle/elastic.py::simulate_c)", "oracle_s": secs}
    for f in elastic.FIELDS:
        rec[f] = field_stats(st.interior(f))
        samples[f"{name}/{f}"] = sample(st.interior(f), FIELD_STRIDE["config5"])
    samples[f"{name}/traces"] = np.ascontiguousarray(st.traces[:, ::TRACE_STRIDE])
    return rec


ALL = [f"config2_o{o}" for o in (2, 4, 8, 12, 16)] + ["config3", "config4", "config5"]


def main(names):
    from paper_1608_03984_b200.synthetic import config2, config3

    meta = {}
    if os.path.exists(JSON_PATH):
        with open(JSON_PATH, encoding="utf-8") as fh:
            meta = json.load(fh)
    samples = {}
    if os.path.exists(NPZ_PATH):
        with np.load(NPZ_PATH) as z:
            samples = {k: z[k] for k in z.files}
    for name in names:
        t0 = time.time()
        if name.startswith("config2_o"):
            rec = gen_acoustic(name, config2(order=int(name[len("config2_o"):])), samples)
        elif name == "config3":
            rec = gen_acoustic(name, config3(), samples)
        elif name == "config4":
            rec = gen_tti(name, samples)
        elif name == "config5":
            rec = gen_elastic(name, samples)
        else:
            raise SystemExit(f"unknown golden {name!r}; choose from {ALL}")
        rec["threads"] = len(os.sched_getaffinity(0))
        meta[name] = rec
        with open(JSON_PATH, "w", encoding="utf-8") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        np.savez_compressed(NPZ_PATH, **samples)
        print(f"{name}: {time.time() - t0:.0f} s, final/p sha "
              f"{(rec.get('final') or rec.get('p_final') or rec.get('vz'))['sha256'][:16]}",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ALL)
