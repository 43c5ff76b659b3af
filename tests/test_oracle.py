"""Pin the CPU oracle (numpy + C restatements) to the real reference's outputs.

The goldens come from the unmodified fdroof.kernel.step / oracle_step
(tests/golden/make_golden.py).  Every comparison here is bit-for-bit (sha256
of the float32 bytes).  CPU only.
"""

import numpy as np
import pytest

from cases import (RAGGED, config1_case, medium_o8_case, mirror_case, random_case, ragged_case,
                   scalarm_case, sha, varm_case)
from oracle import acoustic as O
from oracle import cref
from paper_1608_03984_b200.stencils import first_derivative_weights, second_derivative_weights


def _state(cfg, levels):
    st = O.OracleState(cfg.dims, cfg.order // 2)
    if levels is not None:
        cur, prev = levels
        O.interior(st.grids[2], st.halo)[...] = cur
        O.interior(st.grids[1], st.halo)[...] = prev
    return st


def _run(kind, cfg, levels, n):
    st = _state(cfg, levels)
    if kind == "numpy":
        return O.simulate(cfg, n, state=st)
    return cref.simulate(cfg, n, threads=3, state=st)


KINDS = ["numpy", "c"]


@pytest.mark.parametrize("order", range(2, 34, 2))
def test_fornberg_restatement_matches_closed_forms(order):
    assert O.fornberg_weights(2, order) == second_derivative_weights(order)
    assert O.fornberg_weights(1, order) == first_derivative_weights(order)


@pytest.mark.parametrize("kind", KINDS)
def test_impulse_known_answer(kind, golden_arrays):
    from paper_1608_03984_b200 import KernelConfig

    cfg = KernelConfig(order=2, dims=(9, 9, 9), n_t=1, dt=0.3)
    cur = np.zeros((9, 9, 9), np.float32)
    cur[4, 4, 4] = 1.0
    st = _run(kind, cfg, (cur, np.zeros_like(cur)), 1)
    u = st.latest()
    assert (u == golden_arrays["impulse_o2"]).all()
    # the reference test's own known answer (test_kernel.py:42-52)
    assert u[4, 4, 4] == pytest.approx(2.0 - 6.0 * 0.09)
    assert np.count_nonzero(u) == 7


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("order", [2, 4, 6, 8, 12, 16])
def test_random_levels_bitexact(kind, order, golden_meta):
    cfg, levels = random_case(order)
    st = _run(kind, cfg, levels, 3)
    g = golden_meta[f"random_o{order}"]
    assert sha(st.latest()) == g["final_sha256"]
    assert sha(O.interior(st.grids[1], st.halo)) == g["prev_sha256"]


@pytest.mark.parametrize("order", [2, 8, 16])
def test_f64_convolution_oracle_matches_reference(order, golden_meta):
    cfg, levels = random_case(order)
    st = _state(cfg, levels)
    for _ in range(3):
        O.conv_step_f64(st, cfg)
    assert sha(st.latest()) == golden_meta[f"random_o{order}"]["f64oracle_sha256"]


@pytest.mark.parametrize("kind", KINDS)
def test_varying_and_scalar_slowness(kind, golden_meta):
    cfg, levels = varm_case()
    assert sha(_run(kind, cfg, levels, 2).latest()) == golden_meta["varm_o4"]["final_sha256"]
    cfg, levels = scalarm_case()
    assert sha(_run(kind, cfg, levels, 2).latest()) == golden_meta["scalarm_o6"]["final_sha256"]


@pytest.mark.parametrize("kind", KINDS)
def test_mirror_symmetry_case(kind, golden_arrays):
    cfg, _ = mirror_case()
    st = _state(cfg, None)
    for _ in range(4):
        st = (O.simulate if kind == "numpy" else cref.simulate)(cfg, 1, state=st)
        u = st.latest()
        for axis in range(3):
            assert (u == np.flip(u, axis=axis)).all()
    assert (st.latest() == golden_arrays["mirror_o8"]).all()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("order,dims,seed", RAGGED)
def test_ragged_dims_with_source(kind, order, dims, seed, golden_meta):
    cfg, levels = ragged_case(order, dims, seed)
    st = _run(kind, cfg, levels, 6)
    g = golden_meta[f"ragged_o{order}"]
    assert sha(st.latest()) == g["final_sha256"]
    assert sha(O.interior(st.grids[1], st.halo)) == g["prev_sha256"]


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("sponge", [False, True])
def test_config1_final_and_traces(kind, sponge, golden_meta, golden_arrays):
    cfg, _ = config1_case(sponge)
    st = _run(kind, cfg, None, cfg.n_t)
    key = "config1" if sponge else "config1_nosponge"
    assert sha(st.latest()) == golden_meta[key]["final_sha256"]
    assert sha(st.traces) == golden_meta[key]["traces_sha256"]
    assert (st.traces == golden_arrays[key + "_traces"]).all()
    # the halo of every level stays exactly zero (test_kernel.py:98-104)
    r = st.halo
    for g in st.grids:
        mask = np.ones(g.shape, bool)
        mask[r:-r, r:-r, r:-r] = False
        assert not g[mask].any()


def test_medium_o8_c_oracle(golden_meta):
    cfg, _ = medium_o8_case()
    st = _run("c", cfg, None, cfg.n_t)
    assert sha(st.latest()) == golden_meta["medium_o8"]["final_sha256"]
    assert sha(st.traces) == golden_meta["medium_o8"]["traces_sha256"]


def test_slab_threads_bitexact():
    cfg, levels = ragged_case(*RAGGED[1])
    ref = _state(cfg, levels)
    O.simulate(cfg, 2, slabs=1, state=ref)
    for slabs in (2, 3, 7):
        st = _state(cfg, levels)
        O.simulate(cfg, 2, slabs=slabs, state=st)
        assert (st.latest() == ref.latest()).all()
        st = _state(cfg, levels)
        cref.simulate(cfg, 2, threads=slabs, state=st)
        assert (st.latest() == ref.latest()).all()
