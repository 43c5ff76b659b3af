"""Host inputs behind a cached device plan: frozen while the plan lives.

The reference re-reads `cfg.m` and `source.series` on every step
(/root/reference/pkg/src/fdroof/kernel.py:188, :173).  This package uploads
them once per config (the device plan) and reuses the upload across `run` /
`step` calls.  To make that reuse safe, every numpy array a plan was built
from is made read-only (``flags.writeable = False``) for as long as a plan
uses it, so an in-place edit (an FWI-style model update) raises instead of
being silently ignored; assigning a new array to the config field changes the
plan key and rebuilds the plan.  `invalidate_plan(cfg)` drops a config's
plans and gives write access back once no other plan uses the array.
Non-ndarray array-likes (lists) cannot be write-protected: a snapshot is kept
and compared on every call.  Writes through some *other* view of the same
memory are not detected (documented in INTEGRATION.md).
"""

import threading
import weakref

import numpy as np

_lock = threading.Lock()
_frozen = {}  # id(array) -> [array, users, was_writeable]


def _freeze(arr: np.ndarray) -> None:
    with _lock:
        ent = _frozen.get(id(arr))
        if ent is not None and ent[0] is arr:
            ent[1] += 1
            return
        was = bool(arr.flags.writeable)
        if was:
            arr.flags.writeable = False
        _frozen[id(arr)] = [arr, 1, was]


def _thaw(arr: np.ndarray) -> None:
    with _lock:
        ent = _frozen.get(id(arr))
        if ent is None or ent[0] is not arr:
            return
        ent[1] -= 1
        if ent[1] == 0:
            del _frozen[id(arr)]
            if ent[2]:
                try:
                    arr.flags.writeable = True
                except ValueError:  # base became read-only meanwhile
                    pass


class InputGuard:
    """The host objects a device plan was built from (held, so their ids
    cannot be recycled while the plan is cached)."""

    def __init__(self, objs):
        self.refs = tuple(objs)
        arrays = []
        self.snapshots = []
        for o in self.refs:
            if isinstance(o, np.ndarray):
                if not any(o is a for a in arrays):
                    arrays.append(o)
            elif isinstance(o, (list, tuple)):  # array-likes that cannot be frozen
                self.snapshots.append((o, np.array(o, copy=True)))
        for a in arrays:
            _freeze(a)
        self._arrays = tuple(arrays)
        self._finalizer = weakref.finalize(self, _release_all, self._arrays)

    def key(self) -> tuple:
        return tuple(id(o) for o in self.refs)

    def unchanged(self) -> bool:
        return all(np.array_equal(np.asarray(o), s) for o, s in self.snapshots)

    def release(self) -> None:
        self._finalizer()


def _release_all(arrays):
    for a in arrays:
        _thaw(a)


def config_inputs(cfg, fields) -> list:
    """The config's array inputs: the named fields plus the source series,
    receiver coordinates and sponge profiles."""
    out = [getattr(cfg, f, None) for f in fields]
    src = getattr(cfg, "source", None)
    if src is not None:
        out.append(src)
        out.append(src.series)
    rec = getattr(cfg, "receivers", None)
    if rec is not None:
        out.append(rec)
        out.append(getattr(rec, "locations", getattr(rec, "positions", None)))
    sp = getattr(cfg, "sponge", None)
    if sp is not None:
        out.extend((sp, sp.x, sp.y, sp.z))
    return out


PLAN_ATTRS = ("_device_plan", "_device_plan64")


def cached_plan(cfg, attr, key, build):
    """cfg.<attr> if its key matches `key` and its guarded inputs are
    unchanged, else a new plan from build() (the old plan's inputs are
    released)."""
    plan = getattr(cfg, attr, None)
    if plan is not None and plan.key == key and plan.guard.unchanged():
        return plan
    if plan is not None:
        plan.guard.release()
    plan = build()
    setattr(cfg, attr, plan)
    return plan


def invalidate_plan(cfg) -> None:
    """Drop the device plans cached on `cfg` (acoustic, float64, TTI,
    elastic): the next run re-uploads every input, and arrays no other plan
    uses become writable again."""
    for attr in PLAN_ATTRS:
        plan = getattr(cfg, attr, None)
        if plan is not None:
            plan.guard.release()
            try:
                delattr(cfg, attr)
            except AttributeError:
                pass


def to_host(t):
    """Host numpy copy of a device tensor (or view) in one pass: the device to host
    copy lands in the result's own memory.  `.cpu().numpy().copy()` allocated and
    first-touched two host buffers; for a 512^3 float32 level that was 357 ms
    against 178 ms for the 500 time steps (tools/step_loop_breakdown.py)."""
    import torch

    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    torch.from_numpy(out).copy_(t)
    return out


def host_tensor(a):
    """torch.from_numpy for arrays that are only read (copied to the device or
    to pinned memory): write-protected inputs are fine, so torch's warning
    about non-writable arrays is silenced."""
    import warnings

    import torch

    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        return torch.from_numpy(a)


def grow_traces(fld, rows, n_rec, dtype, device):
    """A (rows, n_rec) trace view for `fld`, keeping the rows recorded so far.
    The backing store grows geometrically, so a step()-per-call loop that runs
    past cfg.n_t (one more row per call) copies O(rows) in total, not O(rows^2)."""
    import torch

    store = getattr(fld, "_trace_store", None)
    old = fld.traces
    if store is None or store.shape[1] != n_rec or store.dtype != dtype or store.shape[0] < rows:
        cap = rows if store is None or store.shape[1] != n_rec else max(rows, 2 * int(store.shape[0]))
        new = torch.zeros((cap, n_rec), dtype=dtype, device=device)
        if old is not None and old.shape[1] == n_rec:
            new[: old.shape[0]].copy_(old)
        store = new
        fld._trace_store = store
    elif old is None or old.data_ptr() != store.data_ptr():
        store.zero_()
        if old is not None and old.shape[1] == n_rec:
            store[: old.shape[0]].copy_(old)
    return store[:rows]
