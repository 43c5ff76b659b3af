"""sha256-keyed cache of oracle outputs -- TEST INFRASTRUCTURE ONLY.

Long oracle runs (the full-length 512^3 config-2 simulation, ~minutes on the
host) are stored as .npz files named by the sha256 of everything that
determines them: the config's fields (arrays by dtype, shape and bytes), the
step count, the initial levels and a tag naming the oracle.  A changed input
gives a different key, so a stale entry can never be returned.  The directory
is FDR_ORACLE_CACHE or oracle/_cache/ (git-ignored).  Only tests/ use this.
"""

import dataclasses
import hashlib
import os

import numpy as np

CACHE_DIR = os.environ.get("FDR_ORACLE_CACHE") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_cache")


def _feed(h, obj):
    if obj is None:
        h.update(b"N")
    elif isinstance(obj, np.ndarray) or isinstance(obj, np.generic):
        a = np.ascontiguousarray(obj)
        h.update(f"A{a.dtype.str}{a.shape}".encode())
        h.update(a.tobytes())
    elif dataclasses.is_dataclass(obj):
        h.update(f"D{type(obj).__name__}".encode())
        for f in dataclasses.fields(obj):
            h.update(f.name.encode())
            _feed(h, getattr(obj, f.name))
    elif isinstance(obj, (list, tuple)):
        h.update(f"L{len(obj)}".encode())
        for v in obj:
            _feed(h, v)
    elif isinstance(obj, (int, float, str, bool)):
        h.update(f"S{type(obj).__name__}:{obj!r}".encode())
    else:
        raise TypeError(f"cannot key {type(obj).__name__}")


def key(*parts) -> str:
    h = hashlib.sha256()
    for p in parts:
        _feed(h, p)
    return h.hexdigest()


def cached(k: str, compute):
    """The dict of arrays stored under key k, computing (and storing) it with
    compute() -> dict[str, np.ndarray] on a miss."""
    path = os.path.join(CACHE_DIR, f"{k}.npz")
    if os.path.exists(path):
        with np.load(path) as z:
            return {name: z[name] for name in z.files}
    out = compute()
    os.makedirs(CACHE_DIR, exist_ok=True)
    tmp = f"{path}.{os.getpid()}.tmp.npz"
    np.savez(tmp, **out)
    os.replace(tmp, path)
    return out
