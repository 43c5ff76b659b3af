"""Equation catalogue (paper_1608_03984_b200/roofline.py) against the
reference's cost model (/root/reference/pkg/src/fdroof/equations.py:55-101,
its tests/test_equations.py:30-60) plus the TTI / elastic-VS entries of the
kernels built here."""

import pytest

from paper_1608_03984_b200 import roofline as RL
from paper_1608_03984_b200.errors import ValidationError


def test_reference_counts():
    assert RL.kernel_flops(RL.EQUATIONS["tti"], 7) == 604  # reference test_equations.py:36
    assert RL.kernel_flops(RL.EQUATIONS["tti"], 9) == 964
    for order in (2, 4, 8, 12, 16):
        assert RL.kernel_flops(RL.EQUATIONS["acoustic"], order + 1) == RL.acoustic_flops_per_point(order)
    assert RL.equation_bytes_per_point(RL.EQUATIONS["tti"]) == 60
    assert RL.equation_bytes_per_point(RL.EQUATIONS["elastic-vs"]) == 84


def test_points_on_the_b200_roof():
    m = RL.b200_machine()
    tti = RL.equation_point(m, RL.EQUATIONS["tti-b200"], 9, measured_gpts=74.3)
    assert tti.bound == "memory"  # 242 / 60 = 4.0 FLOP/B, below the ridge
    assert tti.fraction == pytest.approx(74.3 * 60 / m.peak_bw_achievable, rel=1e-9)
    cat = RL.equation_point(m, RL.EQUATIONS["tti"], 9)
    assert cat.bound == "compute"  # the catalogue's 964 FLOPs put it above the ridge
    el = RL.equation_point(m, RL.EQUATIONS["elastic-vs"], 9, measured_gpts=50.0)
    assert el.bound == "memory" and el.oi == pytest.approx(248 / 84)
    ds = RL.roofline_dataset(m, (tti, el))
    assert ds.inconsistencies() == []


def test_yaml_hook(tmp_path):
    p = tmp_path / "eq.yaml"
    p.write_text("name: my-eq\nfixed_kernel_flops: 100\nfields_moved: 10\n---\n"
                 "name: tti\nfields_moved: 16\nfactor: 2\noverride: true\n")
    eqs = RL.load_equations(str(p))
    assert RL.kernel_flops(eqs["my-eq"], 9) == 100 and eqs["tti"].fields_moved == 16
    p.write_text("name: tti\nfields_moved: 16\n")
    with pytest.raises(ValidationError):
        RL.load_equations(str(p))
    p.write_text("name: x\nbogus: 1\n")
    with pytest.raises(ValidationError):
        RL.load_equations(str(p))


def test_cli_point(capsys, tmp_path):
    from paper_1608_03984_b200 import cli

    svg = tmp_path / "p.svg"
    assert cli.main(["point", "--equation", "elastic-vs", "--machine", "b200", "--gpts", "50",
                     "--svg", str(svg)]) == 0
    out = capsys.readouterr().out
    assert "flops/point:       248" in out and "memory-bound" in out and svg.exists()
    assert cli.main(["point", "--equation", "nope", "--machine", "b200"]) == 2
