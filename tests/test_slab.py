"""x-slab decomposition with a per-step halo exchange (SURVEY.md §8(e),
§8(f)4): the plan, the exchange on gloo ranks and in one process, and the GPU
slabs, all bit-exact against the single-grid run."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import acoustic as O
from paper_1608_03984_b200.errors import ValidationError
from paper_1608_03984_b200.slab import SlabPlan, exchange_local, slab_config, slab_halo
from slab_cases import slab_case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_plan_tiles_and_messages():
    p = SlabPlan(64, 4, 2)
    assert [p.span(i) for i in range(4)] == [(0, 16), (16, 32), (32, 48), (48, 64)]
    assert p.local_range(0) == (0, 18) and p.local_range(3) == (46, 64)
    assert p.messages(0) == [(1, (14, 16), (16, 18))]
    assert p.messages(1) == [(0, (2, 4), (0, 2)), (2, (16, 18), (18, 20))]
    # every send lands on the peer's ghost planes covering the same global planes
    for i in range(4):
        g0 = p.local_range(i)[0]
        for peer, (sa, sb), _ in p.messages(i):
            back = [m for m in p.messages(peer) if m[0] == i][0]
            pg0 = p.local_range(peer)[0]
            assert (g0 + sa, g0 + sb) == (pg0 + back[2][0], pg0 + back[2][1])
    assert SlabPlan(10, 1, 4).messages(0) == []
    with pytest.raises(ValidationError):
        SlabPlan(10, 4, 4)  # 2-plane slabs cannot feed 4 ghost planes


def test_slab_config_owner_only_source_and_receivers():
    cfg, _ = slab_case()["o4"]
    plan = SlabPlan(cfg.dims[0], 2, cfg.halo)
    a, ia = slab_config(cfg, plan, 0)
    b, ib = slab_config(cfg, plan, 1)
    assert a.dims == (14, 14, 12) and b.dims == (14, 14, 12)
    assert a.source is not None and b.source is None  # x = 11 is owned by slab 0
    assert sorted(np.concatenate([ia, ib]).tolist()) == list(range(cfg.receivers.count))
    assert (b.receivers.locations[:, 0] >= 2).all()  # no receiver on a ghost plane
    assert np.array_equal(b.m, cfg.m[10:24])


def oracle_slabs(cfg, plan, n):
    """All slabs in one process (numpy oracle + exchange_local): the global
    final level and traces."""
    import torch

    parts = [slab_config(cfg, plan, i) for i in range(plan.n_slabs)]
    states = [O.OracleState(c.dims, c.halo) for c, _ in parts]
    for (c, _), st in zip(parts, states):
        if c.receivers is not None:
            st.traces = np.zeros((cfg.n_t, c.receivers.count), np.float32)
    tapers = [O.sponge_taper(c) for c, _ in parts]
    r = cfg.halo
    for _ in range(n):
        for (c, _), st, tp in zip(parts, states, tapers):
            O.step(st, c, taper=tp)
        exchange_local([torch.from_numpy(st.grids[2])[r: r + c.dims[0]]
                        for (c, _), st in zip(parts, states)], plan)
    got = np.concatenate([O.interior(st.grids[2], r)[plan.owned_local(i)]
                          for i, st in enumerate(states)])
    traces = np.zeros((cfg.n_t, cfg.receivers.count), np.float32)
    for (c, idx), st in zip(parts, states):
        if idx.size:
            traces[:, idx] = st.traces
    return got, traces


@pytest.mark.parametrize("n_slabs", [2, 3])
def test_local_exchange_oracle_bitexact(n_slabs):
    """All slabs in one process == full grid, field and traces (on- and off-grid)."""
    for cfg, n in slab_case().values():
        got, traces = oracle_slabs(cfg, SlabPlan(cfg.dims[0], n_slabs, slab_halo(cfg)), n)
        full = O.simulate(cfg, n)
        assert np.array_equal(got, full.latest())
        assert np.array_equal(traces, full.traces) and np.abs(full.traces).max() > 0


def test_offgrid_needs_the_wider_ghost_layer():
    cfg, n = slab_case()["off8"]
    assert slab_halo(cfg) == cfg.halo + 1 and slab_halo(slab_case()["o8"][0]) == 4
    with pytest.raises(ValidationError, match="slab_halo"):
        slab_config(cfg, SlabPlan(cfg.dims[0], 2, cfg.halo), 0)
    # the straddling source goes to both slabs, each receiver to exactly one
    plan = SlabPlan(cfg.dims[0], 2, slab_halo(cfg))
    (a, ia), (b, ib) = slab_config(cfg, plan, 0), slab_config(cfg, plan, 1)
    assert a.source.position[0] == 14.37 and b.source.position[0] == 14.37 - 10
    assert sorted(np.concatenate([ia, ib]).tolist()) == list(range(cfg.receivers.count))
    assert np.floor(b.receivers.positions[:, 0]).min() >= 5  # base plane owned by slab 1


def test_offgrid_receivers_wrong_with_only_r_ghost_planes(monkeypatch):
    """Why r + 1: with r ghost planes the receivers whose upper corner plane is
    the first ghost plane (x 14.6 for 2 slabs) sample a not-yet-exchanged,
    truncated-stencil value and diverge; everything else stays exact."""
    import paper_1608_03984_b200.slab as S

    cfg, n = slab_case()["off4"]
    monkeypatch.setattr(S, "slab_halo", lambda c: c.halo)
    got, traces = oracle_slabs(cfg, SlabPlan(cfg.dims[0], 2, cfg.halo), n)
    full = O.simulate(cfg, n)
    assert np.array_equal(got, full.latest())
    bad = np.nonzero((traces != full.traces).any(0))[0]
    assert cfg.receivers.positions[bad, 0].tolist() == [14.6]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_halo_exchange(tmp_path):
    out = tmp_path / "slab.json"
    env = dict(os.environ, FDR_MP_OUT=str(out), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp", "slab_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert set(res) == set(slab_case())
    for name, v in res.items():
        assert v == {"field_equal": True, "traces_equal": True, "nonzero": True}, name


@pytest.mark.gpu
@pytest.mark.parametrize("n_slabs", [2, 3])
def test_gpu_slabs_local_bitexact(cuda_device, n_slabs):
    """The GPU kernels on every slab with plane-block exchanges (one device)
    == the single-grid GPU run, field and traces."""
    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.slab import run_slabs_local

    for cfg, n in slab_case().values():
        plan = SlabPlan(cfg.dims[0], n_slabs, slab_halo(cfg))
        got, traces = run_slabs_local(cfg, plan, n)
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
        B.run(fld, cfg, n)
        assert np.array_equal(got, fld.numpy())
        assert np.array_equal(traces[:n], fld.traces.cpu().numpy()[:n])


@pytest.mark.gpu
@pytest.mark.parametrize("n_slabs", [1, 2, 3, 5])
def test_gpu_library_slabs_bitexact(cuda_device, n_slabs):
    """fdr_acoustic_slabs_run (the library's exchange: boundary planes first,
    peer copies into the neighbours' ghost planes overlapped with the interior)
    on one device == the single-grid run, field and traces."""
    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.slab import run_slabs

    for name, (cfg, n) in slab_case().items():
        if name.startswith("off"):
            continue
        plan = SlabPlan(cfg.dims[0], n_slabs, cfg.halo)
        got, traces = run_slabs(cfg, plan, n_steps=n)
        fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
        B.run(fld, cfg, n)
        assert np.array_equal(got, fld.numpy()), name
        assert np.array_equal(traces[:n], fld.traces.cpu().numpy()[:n]), name


@pytest.mark.gpu
def test_gpu_library_slabs_full_size(cuda_device):
    """Config-2 grid (512^3, order 8) split in 4 x-slabs on one device for 20
    steps from zero with the Ricker source: identical to the single-grid run."""
    import paper_1608_03984_b200 as B
    from paper_1608_03984_b200.slab import run_slabs
    from paper_1608_03984_b200.synthetic import config2

    cfg = config2(order=8, n_t=20)
    got, traces = run_slabs(cfg, SlabPlan(cfg.dims[0], 4, cfg.halo))
    fld = B.Wavefield.allocate(cfg.dims, cfg.halo)
    B.run(fld, cfg)
    assert np.array_equal(got, fld.numpy())
    assert np.array_equal(traces[:20], fld.traces.cpu().numpy()[:20])
