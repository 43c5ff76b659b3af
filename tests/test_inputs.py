"""Device-plan input guard (paper_1608_03984_b200/_inputs.py), host only.

The reference re-reads cfg.m and source.series every step
(/root/reference/pkg/src/fdroof/kernel.py:188, :173); the cached device plan
must therefore never silently keep a stale upload: arrays it was built from
are write-protected while it lives, a new array rebuilds it, and
invalidate_plan() gives write access back.
"""

import numpy as np
import pytest

from paper_1608_03984_b200 import KernelConfig, Receivers, Source, Sponge, invalidate_plan
from paper_1608_03984_b200._inputs import InputGuard, cached_plan, config_inputs


class _Plan:
    builds = 0

    def __init__(self, cfg, key):
        _Plan.builds += 1
        self.key = key
        self.guard = InputGuard(config_inputs(cfg, ("m",)))


def _key(cfg):
    return tuple(id(o) for o in config_inputs(cfg, ("m",)))


def _get(cfg):
    return cached_plan(cfg, "_device_plan", _key(cfg), lambda: _Plan(cfg, _key(cfg)))


def _cfg():
    m = np.full((8, 8, 8), 1.5, np.float32)
    series = np.array([1.0, 2.0], np.float32)
    return KernelConfig(order=2, dims=(8, 8, 8), n_t=2, dt=0.1, m=m,
                        source=Source((3, 3, 3), series),
                        receivers=Receivers(np.array([[1, 2, 3]])),
                        sponge=Sponge(np.ones(8), np.ones(8), np.ones(8)))


def test_inputs_frozen_while_plan_cached():
    cfg = _cfg()
    p = _get(cfg)
    assert _get(cfg) is p
    with pytest.raises(ValueError):
        cfg.m[0, 0, 0] = 2.0
    with pytest.raises(ValueError):
        cfg.source.series[0] = 3.0
    with pytest.raises(ValueError):
        cfg.sponge.x[0] = 0.5
    invalidate_plan(cfg)
    cfg.m[0, 0, 0] = 2.0  # writable again
    cfg.source.series[0] = 3.0
    assert not hasattr(cfg, "_device_plan")


def test_new_array_rebuilds_plan():
    cfg = _cfg()
    p = _get(cfg)
    old = cfg.m
    cfg.m = np.full((8, 8, 8), 2.0, np.float32)
    q = _get(cfg)
    assert q is not p
    old[0, 0, 0] = 7.0  # the replaced array is released


def test_shared_array_stays_frozen_until_last_user():
    a, b = _cfg(), _cfg()
    b.m = a.m
    _get(a)
    _get(b)
    invalidate_plan(a)
    with pytest.raises(ValueError):
        a.m[0, 0, 0] = 2.0  # b's plan still uses it
    invalidate_plan(b)
    a.m[0, 0, 0] = 2.0


def test_list_inputs_compared_by_snapshot():
    cfg = _cfg()
    cfg.m = [[[1.5] * 8] * 8] * 8
    cfg.m = [[[1.5] * 8 for _ in range(8)] for _ in range(8)]
    p = _get(cfg)
    assert _get(cfg) is p
    cfg.m[0][0][0] = 2.5  # cannot be write-protected: detected by comparison
    assert _get(cfg) is not p
    invalidate_plan(cfg)


def test_readonly_input_left_readonly():
    cfg = _cfg()
    cfg.m.flags.writeable = False
    _get(cfg)
    invalidate_plan(cfg)
    assert not cfg.m.flags.writeable


def test_device_plan_reused_across_runs():
    """The plan key must be stable between calls: a rebuild per call would
    re-upload m every run (and every step() call)."""
    import torch

    from paper_1608_03984_b200 import kernel as K

    cfg = _cfg()
    p = K._plan(cfg, torch.device("cpu"), 8)
    assert K._plan(cfg, torch.device("cpu"), 8) is p
    assert K._plan(cfg, torch.device("cpu"), 12) is not p  # another pitch: another layout
    invalidate_plan(cfg)


def test_trace_store_grows_geometrically():
    import torch

    from paper_1608_03984_b200._inputs import grow_traces

    class F:
        traces = None

    f = F()
    f.traces = grow_traces(f, 4, 3, torch.float32, "cpu")
    f.traces[:] = 1.0
    allocs = set()
    for rows in range(5, 200):
        f.traces = grow_traces(f, rows, 3, torch.float32, "cpu")
        allocs.add(f._trace_store.data_ptr())
        assert f.traces.shape == (rows, 3) and f.traces.is_contiguous()
        assert (f.traces[:4] == 1.0).all() and (f.traces[4:] == 0.0).all()
    assert len(allocs) <= 7  # doublings, not one allocation per row
    f.traces = None  # a reset starts from zeros again
    f.traces = grow_traces(f, 10, 3, torch.float32, "cpu")
    assert (f.traces == 0).all()
