"""Report front end: machine documents in the reference's
schema, the roofline dataset, the SVG chart and the `bench` CLI."""

import xml.etree.ElementTree as ET

import numpy as np
import pytest

from paper_1608_03984_b200 import charts, cli
from paper_1608_03984_b200 import roofline as RL
from paper_1608_03984_b200.errors import ValidationError


def test_b200_document_theoretical_peaks_exact():
    m = RL.builtin_machines()["b200"]
    assert m.peak_gflops_theoretical == 74449.92  # 128 x 2 x 148 x 1.965
    assert m.peak_bw_theoretical == 8183.808  # 8 x 128 B x 7992 MT/s
    assert m.precision_bytes == 4
    live = RL.get_machine("b200")
    assert live.peak_bw_achievable == RL.measured_peaks().get("hbm_gbs", RL.FALLBACK_HBM_GBS)
    assert RL.b200_machine(precision_bytes=8).peak_gflops_achievable == live.peak_gflops_achievable / 2


def _write(tmp_path, text):
    p = tmp_path / "m.yaml"
    p.write_text(text)
    return str(p)


def test_machine_document_validation(tmp_path):
    good = _write(tmp_path, "name: x\npeak_bw_theoretical: 100\npeak_gflops_theoretical: 1000\n"
                  "---\nname: y\npeak_bw_achievable: 50\npeak_gflops_achievable: 400\n"
                  "precision_bytes: 8\n")
    reg = RL.load_machines(good)
    assert reg["x"].peak_bw_achievable == 80.0 and "defaulted to 80%" in reg["x"].notes
    assert reg["y"].precision_bytes == 8 and reg["y"].ridge_point == 8.0
    bad = {
        "name: x\nbogus: 1\npeak_bw_achievable: 1\npeak_gflops_achievable: 1\n": "unknown machine keys",
        "peak_bw_achievable: 1\npeak_gflops_achievable: 1\n": "missing 'name'",
        "name: x\narch: {cores: 2}\npeak_bw_achievable: 1\n": "arch keys",
        "name: x\npeak_bw_achievable: 1\n": "achievable or theoretical",
        "name: x\npeak_bw_achievable: 1\npeak_gflops_achievable: 1\n---\n"
        "name: x\npeak_bw_achievable: 1\npeak_gflops_achievable: 1\n": "duplicate",
        "name: x\npeak_bw_achievable: -1\npeak_gflops_achievable: 1\n": "must be > 0",
        "name: [x\n": "invalid YAML",
    }
    for text, msg in bad.items():
        with pytest.raises(ValidationError, match=msg.replace("(", r"\(")):
            RL.load_machines(_write(tmp_path, text))


def test_dataset_roof_and_csv():
    m = RL.MachineSpec("t", 1000.0, 100.0)
    pts = [RL.roofline_point(m, 8, measured_gflops=300.0),
           RL.roofline_point(m, 32, measured_gflops=2000.0)]
    ds = RL.roofline_dataset(m, pts)
    (a, b), (c, d) = ds.roof_segments
    assert b == c == (10.0, 1000.0) and d == (ds.oi_hi, 1000.0)
    assert a == (ds.oi_lo, ds.oi_lo * 100.0)
    assert ds.inconsistencies() == [pts[1]]  # 2000 GFLOPS above a 1000 roof
    lines = ds.to_csv().splitlines()
    assert lines[0] == "label,k,oi,attainable_gflops,bound,measured_gflops"
    assert lines[1].startswith("acoustic:k9,9,3.625,362.5,memory,300.0")
    # fp64 halves the operational intensity (4 fields x 8 bytes)
    m8 = RL.MachineSpec("t8", 500.0, 100.0, precision_bytes=8)
    assert RL.roofline_point(m8, 8).oi == 58 / 32
    with pytest.raises(ValidationError):
        RL.RooflineDataset(m, (), 1.0, 0.5)


def test_svg_chart_well_formed(tmp_path):
    m = RL.get_machine("b200")
    p = RL.roofline_point(m, 8, measured_gflops=335.6 * 58)
    ds = RL.roofline_dataset(m, (p,))
    svg = charts.roofline_chart(ds, measured_oi={p.label: 58 / 16 / 0.998})
    root = ET.fromstring(svg)
    ns = "{http://www.w3.org/2000/svg}"
    assert root.tag == ns + "svg"
    assert len(root.findall(ns + "polyline")) == 1
    assert len(root.findall(ns + "circle")) == 2 and len(root.findall(ns + "rect")) == 3
    text = " ".join(t.text or "" for t in root.iter(ns + "text"))
    bw = m.peak_bw_achievable  # the measured HBM rate (MEASURED_PEAKS.json) when present
    pct = round(100 * p.measured_gflops / p.attainable_gflops)
    assert f"{bw:,.1f} GB/s" in text and f"acoustic:k9 {pct}%" in text
    out = tmp_path / "r.svg"
    charts.write_svg(svg, out)
    assert out.read_text() == svg


def test_cli_machines_and_errors(tmp_path, capsys):
    extra = _write(tmp_path, "name: cpu\npeak_bw_achievable: 200\npeak_gflops_achievable: 2000\n")
    assert cli.main(["--machines-file", extra, "machines", "list"]) == 0
    out = capsys.readouterr().out
    assert "b200" in out and "cpu" in out
    assert cli.main(["machines", "show", "b200"]) == 0
    assert "8183.808 GB/s" in capsys.readouterr().out
    assert cli.main(["machines", "show", "nope"]) == 2
    assert "error: unknown machine" in capsys.readouterr().err
    assert cli.fmt(3.0) == "3" and cli.fmt(3.14159265) == "3.1416" and cli.fmt(1.5e-6) == "1.5e-06"


@pytest.mark.gpu
def test_cli_bench_runs_kernel_and_matches_oracle(cuda_device, tmp_path, capsys):
    """`bench` end to end on the GPU: the report lines, the SVG, and the dumped
    wavefield equal to the C oracle from the same seeded start."""
    from oracle import acoustic as O
    from oracle import cref
    from paper_1608_03984_b200 import kernel

    svg, dump = tmp_path / "r.svg", tmp_path / "f.bin"
    rc = cli.main(["bench", "--order", "4", "--grid", "48", "--nt", "12", "--machine", "b200",
                   "--repeat", "2", "--svg", str(svg), "--dump", str(dump)])
    assert rc == 0
    out = capsys.readouterr().out
    for key in ("oi:", "attainable:", "measured:", "of attainable:", "updates:"):
        assert key in out
    ET.fromstring(svg.read_text())
    cfg = kernel.KernelConfig(order=4, dims=(48, 48, 48), n_t=12,
                              dt=0.5 * kernel.max_stable_dt(4, 1.0))
    st = O.OracleState(cfg.dims, cfg.halo)
    O.interior(st.grids[2], st.halo)[...] = (
        np.random.default_rng(0).standard_normal(cfg.dims).astype(np.float32) * 1e-3)
    cref.simulate(cfg, cfg.n_t, state=st)
    got = np.fromfile(dump, dtype="<f4").reshape(cfg.dims, order="F")
    assert np.array_equal(got, st.latest())


def test_artifacts_byte_identical_across_runs(tmp_path):
    """Acceptance criterion 10 (test_acceptance.py:226-249) for this front end:
    the SVG and CSV of the same dataset are byte-identical across runs."""
    m = RL.get_machine("b200")
    pts = [RL.roofline_point(m, o, measured_gflops=100.0 * o) for o in (2, 8, 16)]
    outs = []
    for tag in ("a", "b"):
        svg, csv = tmp_path / f"r-{tag}.svg", tmp_path / f"r-{tag}.csv"
        ds = RL.roofline_dataset(m, pts)
        charts.write_svg(charts.roofline_chart(ds), svg)
        csv.write_text(ds.to_csv())
        outs.append((svg.read_bytes(), csv.read_bytes()))
    assert outs[0] == outs[1] and len(outs[0][0]) > 0 and len(outs[0][1]) > 0
