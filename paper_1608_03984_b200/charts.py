"""Roofline chart as a standalone SVG document (the report front end of
SURVEY.md §8(f)1; the reference's entry points are charts.py:75-105
`roofline_chart(dataset)` and `write_svg(chart, path)`).

Log-log axes: operational intensity (FLOPs/byte) against GFLOPS.  The roof
is drawn from `RooflineDataset.roof_segments`.  Each point is shown twice:
hollow at its model bound (attainable) and filled at its measurement.  When a
point also carries a measured OI (FLOPs / DRAM bytes from ncu), a third marker
sits at that OI.
"""

import math
from xml.sax.saxutils import escape

from .errors import ValidationError

W, H = 760, 500
ML, MR, MT, MB = 80, 30, 50, 60  # plot margins
PALETTE = ("#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b")


def _decades(lo, hi):
    return range(math.floor(math.log10(lo)), math.ceil(math.log10(hi)) + 1)


def roofline_chart(dataset, title=None, measured_oi=None) -> str:
    """SVG text of `dataset` (a roofline.RooflineDataset).  `measured_oi`
    optionally maps a point label to its measured operational intensity."""
    m = dataset.machine
    pts = list(dataset.points)
    ys = [m.peak_gflops_achievable, dataset.oi_lo * m.peak_bw_achievable]
    ys += [p.attainable_gflops for p in pts] + [p.measured_gflops for p in pts if p.measured_gflops]
    if min(ys) <= 0:
        raise ValidationError("roofline values must be positive")
    x0, x1 = math.log10(dataset.oi_lo), math.log10(dataset.oi_hi)
    y0, y1 = math.log10(min(ys) / 2.0), math.log10(max(ys) * 2.0)

    def px(oi):
        return ML + (math.log10(oi) - x0) / (x1 - x0) * (W - ML - MR)

    def py(g):
        return H - MB - (math.log10(g) - y0) / (y1 - y0) * (H - MT - MB)

    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" '
           f'viewBox="0 0 {W} {H}" font-family="sans-serif" font-size="12">',
           f'<rect x="0" y="0" width="{W}" height="{H}" fill="white"/>']
    head = title or f"Roofline: {m.name} ({m.precision_bytes * 8}-bit)"
    out.append(f'<text x="{W / 2:.1f}" y="24" text-anchor="middle" font-size="15">{escape(head)}</text>')
    # grid and decade ticks
    for e in _decades(dataset.oi_lo, dataset.oi_hi):
        v = 10.0 ** e
        if dataset.oi_lo <= v <= dataset.oi_hi:
            x = px(v)
            out.append(f'<line x1="{x:.1f}" y1="{MT}" x2="{x:.1f}" y2="{H - MB}" stroke="#ddd"/>')
            out.append(f'<text x="{x:.1f}" y="{H - MB + 16}" text-anchor="middle">{v:g}</text>')
    for e in _decades(10 ** y0, 10 ** y1):
        v = 10.0 ** e
        if 10 ** y0 <= v <= 10 ** y1:
            y = py(v)
            out.append(f'<line x1="{ML}" y1="{y:.1f}" x2="{W - MR}" y2="{y:.1f}" stroke="#ddd"/>')
            out.append(f'<text x="{ML - 6}" y="{y + 4:.1f}" text-anchor="end">{v:g}</text>')
    out.append(f'<rect x="{ML}" y="{MT}" width="{W - ML - MR}" height="{H - MT - MB}" '
               f'fill="none" stroke="#333"/>')
    out.append(f'<text x="{(ML + W - MR) / 2:.1f}" y="{H - 18}" text-anchor="middle">'
               f'operational intensity (FLOPs/byte)</text>')
    out.append(f'<text x="18" y="{(MT + H - MB) / 2:.1f}" text-anchor="middle" '
               f'transform="rotate(-90 18 {(MT + H - MB) / 2:.1f})">GFLOPS</text>')
    # roof
    slope, flat = dataset.roof_segments
    poly = " ".join(f"{px(a):.1f},{py(b):.1f}" for a, b in (slope[0], slope[1], flat[1]))
    out.append(f'<polyline points="{poly}" fill="none" stroke="#000" stroke-width="2"/>')
    rx = px(dataset.ridge)
    out.append(f'<line x1="{rx:.1f}" y1="{py(m.peak_gflops_achievable):.1f}" x2="{rx:.1f}" '
               f'y2="{H - MB}" stroke="#888" stroke-dasharray="4,3"/>')
    out.append(f'<text x="{rx + 4:.1f}" y="{H - MB - 6}" fill="#555">ridge {dataset.ridge:.2f}</text>')
    out.append(f'<text x="{px(dataset.oi_hi) - 4:.1f}" y="{py(m.peak_gflops_achievable) - 6:.1f}" '
               f'text-anchor="end">{m.peak_gflops_achievable:,.0f} GFLOPS</text>')
    out.append(f'<text x="{px(slope[0][0]) + 6:.1f}" y="{py(slope[0][1]) - 8:.1f}" '
               f'fill="#333">{m.peak_bw_achievable:,.1f} GB/s</text>')
    # points
    measured_oi = measured_oi or {}
    for i, p in enumerate(pts):
        c = PALETTE[i % len(PALETTE)]
        x = px(p.oi)
        out.append(f'<circle cx="{x:.1f}" cy="{py(p.attainable_gflops):.1f}" r="5" fill="white" '
                   f'stroke="{c}" stroke-width="2"><title>{escape(p.label)} bound '
                   f'{p.attainable_gflops:.1f}</title></circle>')
        if p.measured_gflops:
            y = py(p.measured_gflops)
            frac = p.measured_gflops / p.attainable_gflops
            out.append(f'<circle cx="{x:.1f}" cy="{y:.1f}" r="5" fill="{c}"><title>'
                       f'{escape(p.label)} measured {p.measured_gflops:.1f}</title></circle>')
            out.append(f'<text x="{x + 8:.1f}" y="{y + 4:.1f}" fill="{c}">{escape(p.label)} '
                       f'{frac * 100:.0f}%</text>')
            moi = measured_oi.get(p.label)
            if moi and dataset.oi_lo < moi < dataset.oi_hi:
                out.append(f'<rect x="{px(moi) - 4:.1f}" y="{y - 4:.1f}" width="8" height="8" '
                           f'fill="{c}"><title>{escape(p.label)} at measured OI {moi:.3f}'
                           f'</title></rect>')
    out.append("</svg>")
    return "\n".join(out) + "\n"


def write_svg(chart: str, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(chart)
