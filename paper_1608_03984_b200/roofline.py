"""Roofline bookkeeping for the measured kernels.

Algorithmic FLOPs and bytes per grid point follow the reference's cost model
(/root/reference/pkg/src/fdroof/equations.py:55-101): for the acoustic kernel
flops(k) = 3*2k + 3 + 5 - 4 = 6k + 4 with k = order + 1 (equations.py:122-132)
and 4 fields x 4 bytes = 16 bytes moved per point.  `roofline_point` mirrors
analysis.py:170-181 + machines.py:151-173: attainable = min(OI*B, F).

The B200 machine entry uses the driver-measured copy bandwidth from
MEASURED_PEAKS.json when present (else the profiling guide's fallback) and a
derived FP32 peak of 148 SMs x 128 lanes x 2 FLOP x SM clock.
"""

import json
import os
from dataclasses import dataclass, replace
from fractions import Fraction
from typing import Optional

from .errors import ValidationError

REPO_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
B200_SMS = 148
B200_FP32_LANES = 128
B200_MAX_SM_MHZ = 1965.0


def acoustic_flops_per_point(order: int) -> int:
    """6k + 4 with k = order + 1 (equations.py:55-71 with the acoustic entry)."""
    if order < 2 or order % 2:
        raise ValidationError(f"order must be even and >= 2, got {order}")
    return 6 * (order + 1) + 4


ACOUSTIC_BYTES_PER_POINT = 16  # m, u(t-2), u(t-1) read + u(t) written (equations.py:129)


@dataclass(frozen=True)
class ArchParams:
    """Core-side parameters of a machine document (machines.py:38-53)."""

    simd_lanes_sp: int
    fma_ops_per_cycle: int
    cores: int
    sockets: int
    clock_ghz: float


@dataclass(frozen=True)
class MemParams:
    """Memory-side parameters of a machine document (machines.py:56-67)."""

    transfer_rate_mts: float
    channels: int
    bytes_per_channel: int
    sockets: int


def _exact(x) -> Fraction:
    return Fraction(str(x))


def theoretical_peak_flops(arch: ArchParams) -> float:
    """lanes x fma x cores x sockets x clock in GFLOPS, in exact decimal
    arithmetic (the reference's rule, machines.py:70-83)."""
    return float(_exact(arch.simd_lanes_sp) * arch.fma_ops_per_cycle * arch.cores * arch.sockets
                 * _exact(arch.clock_ghz))


def theoretical_peak_bandwidth(mem: MemParams) -> float:
    """transfer rate x channels x bytes x sockets in GB/s (machines.py:86-95)."""
    return float(_exact(mem.transfer_rate_mts) * mem.channels * mem.bytes_per_channel
                 * mem.sockets / 1000)


@dataclass(frozen=True)
class MachineSpec:
    """fdroof.machines.MachineSpec (machines.py:98-148): achievable peaks are
    the roof; theoretical peaks, precision and provenance are carried along."""

    name: str
    peak_gflops_achievable: float
    peak_bw_achievable: float
    source: str = ""
    peak_gflops_theoretical: Optional[float] = None
    peak_bw_theoretical: Optional[float] = None
    precision_bytes: int = 4
    notes: str = ""
    arch: Optional[ArchParams] = None
    mem: Optional[MemParams] = None

    def __post_init__(self):
        if not (self.peak_gflops_achievable and self.peak_gflops_achievable > 0):
            raise ValidationError(f"machine {self.name!r}: peak_gflops_achievable must be > 0")
        if not (self.peak_bw_achievable and self.peak_bw_achievable > 0):
            raise ValidationError(f"machine {self.name!r}: peak_bw_achievable must be > 0")
        if self.precision_bytes not in (4, 8):
            raise ValidationError(f"machine {self.name!r}: precision_bytes must be 4 or 8")

    @property
    def ridge_point(self) -> float:
        return self.peak_gflops_achievable / self.peak_bw_achievable

    def attainable(self, oi: float) -> float:
        return min(oi * self.peak_bw_achievable, self.peak_gflops_achievable)


ACHIEVABLE_FRACTION_HINT = 0.8  # the reference's default when only theoretical peaks are given
_MACHINE_KEYS = {"name", "peak_gflops_theoretical", "peak_bw_theoretical", "peak_gflops_achievable",
                 "peak_bw_achievable", "precision_bytes", "notes", "arch", "mem"}
_ARCH_KEYS = {"simd_lanes_sp", "fma_ops_per_cycle", "cores", "sockets", "clock_ghz"}
_MEM_KEYS = {"transfer_rate_mts", "channels", "bytes_per_channel", "sockets"}
MACHINES_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "machines")


def _sub(doc, key, allowed, cls, where):
    sub = doc.get(key)
    if sub is None:
        return None
    if not isinstance(sub, dict):
        raise ValidationError(f"{where}: '{key}' must be a mapping")
    if set(sub) != allowed:
        extra, missing = sorted(set(sub) - allowed), sorted(allowed - set(sub))
        raise ValidationError(f"{where}: {key} keys: unknown {extra}, missing {missing}")
    return cls(**sub)


def machine_from_doc(doc, where="<doc>") -> MachineSpec:
    """Validate one machine document with the reference's schema and rules
    (machines.py:245-281): arch / mem give the theoretical peaks; missing
    achievable peaks default to 80% of theoretical, noted in `notes`."""
    if not isinstance(doc, dict):
        raise ValidationError(f"{where}: machine document must be a mapping")
    unknown = set(doc) - _MACHINE_KEYS
    if unknown:
        raise ValidationError(f"{where}: unknown machine keys: {sorted(unknown)}")
    if "name" not in doc:
        raise ValidationError(f"{where}: machine document missing 'name'")
    arch = _sub(doc, "arch", _ARCH_KEYS, ArchParams, where)
    mem = _sub(doc, "mem", _MEM_KEYS, MemParams, where)
    theo_f = theoretical_peak_flops(arch) if arch else doc.get("peak_gflops_theoretical")
    theo_b = theoretical_peak_bandwidth(mem) if mem else doc.get("peak_bw_theoretical")
    ach_f, ach_b = doc.get("peak_gflops_achievable"), doc.get("peak_bw_achievable")
    notes, defaulted = str(doc.get("notes", "")), []
    if ach_f is None and theo_f is not None:
        ach_f, _ = ACHIEVABLE_FRACTION_HINT * theo_f, defaulted.append("GFLOPS")
    if ach_b is None and theo_b is not None:
        ach_b, _ = ACHIEVABLE_FRACTION_HINT * theo_b, defaulted.append("bandwidth")
    if defaulted:
        hint = f"achievable {'/'.join(defaulted)} defaulted to 80% of theoretical"
        notes = f"{notes}; {hint}" if notes else hint
    if ach_f is None or ach_b is None:
        raise ValidationError(f"{where}: machine needs achievable or theoretical peaks")
    return MachineSpec(str(doc["name"]), float(ach_f), float(ach_b), where,
                       None if theo_f is None else float(theo_f),
                       None if theo_b is None else float(theo_b),
                       int(doc.get("precision_bytes", 4)), notes, arch, mem)


def load_machines(path) -> dict:
    """All machine documents of a YAML file (multi-document), by name."""
    import yaml

    try:
        with open(path, encoding="utf-8") as fh:
            docs = [d for d in yaml.safe_load_all(fh) if d is not None]
    except yaml.YAMLError as exc:
        raise ValidationError(f"{path}: invalid YAML ({exc})") from None
    out = {}
    for i, d in enumerate(docs):
        m = machine_from_doc(d, f"{path}[{i}]")
        if m.name in out:
            raise ValidationError(f"{path}: duplicate machine name {m.name!r}")
        out[m.name] = m
    return out


def builtin_machines() -> dict:
    out = {}
    for fn in sorted(os.listdir(MACHINES_DIR)):
        if fn.endswith((".yaml", ".yml")):
            out.update(load_machines(os.path.join(MACHINES_DIR, fn)))
    return out


def get_machine(name: str = "b200", registry: Optional[dict] = None) -> MachineSpec:
    """A machine by name from `registry` (default: the built-in documents).
    For the built-in B200 the achievable bandwidth is the driver-measured copy
    rate in MEASURED_PEAKS.json when that file is present."""
    reg = registry if registry is not None else builtin_machines()
    if name not in reg:
        raise ValidationError(f"unknown machine {name!r}; known: {sorted(reg)}")
    m = reg[name]
    if registry is None and name == "b200":
        return b200_machine()
    return m


@dataclass(frozen=True)
class RooflinePoint:
    """Mirror of fdroof.analysis.RooflinePoint."""

    label: str
    oi: float
    attainable_gflops: float
    bound: str
    k: int
    measured_gflops: Optional[float] = None

    @property
    def fraction(self) -> Optional[float]:
        if self.measured_gflops is None:
            return None
        return self.measured_gflops / self.attainable_gflops


def measured_peaks(path: Optional[str] = None) -> dict:
    path = path or os.path.join(REPO_ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path, encoding="utf-8") as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def b200_machine(sm_mhz: Optional[float] = None, precision_bytes: int = 4) -> MachineSpec:
    """B200 roofline from machines/b200.yaml: the measured HBM copy GB/s
    (MEASURED_PEAKS.json) when present, the derived FP32 (or FP64: half rate)
    GFLOPS at the given SM clock."""
    doc = load_machines(os.path.join(MACHINES_DIR, "b200.yaml"))["b200"]
    peaks = measured_peaks()
    bw = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    mhz = float(sm_mhz or peaks.get("sm_max_mhz", B200_MAX_SM_MHZ))
    flops = B200_SMS * B200_FP32_LANES * 2 * mhz * 1e-3  # GFLOPS
    if precision_bytes == 8:
        flops /= 2.0  # B200 FP64 FMA rate: half the FP32 rate
    return replace(doc, peak_gflops_achievable=flops, peak_bw_achievable=bw, source=src,
                   precision_bytes=precision_bytes)


def roofline_point(machine: MachineSpec, order: int,
                   measured_gflops: Optional[float] = None,
                   label: Optional[str] = None) -> RooflinePoint:
    """analysis.py:170-181 for the acoustic kernel: OI = flops / (4 fields x
    precision_bytes), attainable = min(OI B, F)."""
    k = order + 1
    oi = acoustic_flops_per_point(order) / (4 * machine.precision_bytes)
    bound = "memory" if oi < machine.ridge_point else "compute"
    return RooflinePoint(label or f"acoustic:k{k}", oi, machine.attainable(oi), bound, k,
                         measured_gflops)


# ------------------------------------------------------------ equations
# The reference's cost catalogue schema (equations.py:20-101, the equations
# YAML hook at :218-246) for the kernels this package time-steps, so the report
# front end can place TTI (config 4) and the elastic velocity-stress system
# (config 5) on the roofline next to the acoustic kernel.


@dataclass(frozen=True)
class EquationSpec:
    """fdroof.equations.EquationSpec: per-point FLOPs from derivative counts
    (or a fixed count) and the field values moved per point per step."""

    name: str
    factor: int = 1
    n_first: int = 0
    n_second: int = 0
    n_cross: int = 0
    extra_mult: int = 0
    extra_add: int = 0
    duplicates: int = 0
    fields_moved: int = 1
    fixed_kernel_flops: Optional[int] = None
    description: str = ""

    def __post_init__(self):
        if not self.name:
            raise ValidationError("equation name must be non-empty")
        if self.factor < 1:
            raise ValidationError(f"{self.name}: factor must be >= 1")
        for attr in ("n_first", "n_second", "n_cross", "extra_mult", "extra_add", "duplicates"):
            if getattr(self, attr) < 0:
                raise ValidationError(f"{self.name}: {attr} must be >= 0")
        if self.fields_moved < 1:
            raise ValidationError(f"{self.name}: fields_moved must be >= 1")
        if self.fixed_kernel_flops is not None and self.fixed_kernel_flops < 1:
            raise ValidationError(f"{self.name}: fixed_kernel_flops must be >= 1")


def kernel_flops(eq: EquationSpec, k: int) -> int:
    """equations.py:55-71: axis derivatives 2k FLOPs, cross derivatives
    2k^2 - 4k - 1 (stencils.py:116-128), plus the extras, minus duplicates,
    times the coupled-system factor; or the fixed count."""
    if eq.fixed_kernel_flops is not None:
        return eq.fixed_kernel_flops
    if k < 2:
        raise ValidationError(f"stencil size k must be >= 2, got {k}")
    per = ((eq.n_first + eq.n_second) * 2 * k + eq.n_cross * (2 * k * k - 4 * k - 1)
           + eq.extra_mult + eq.extra_add - eq.duplicates)
    return eq.factor * per


def equation_bytes_per_point(eq: EquationSpec, precision_bytes: int = 4) -> int:
    return eq.fields_moved * precision_bytes


EQUATIONS = {e.name: e for e in (
    EquationSpec("acoustic", factor=1, n_second=3, extra_mult=3, extra_add=5, duplicates=4,
                 fields_moved=4, description="the reference's acoustic entry (equations.py:122-132)"),
    EquationSpec("tti", factor=2, n_second=3, n_cross=3, extra_mult=44, extra_add=17,
                 duplicates=8, fields_moved=15,
                 description="the reference's TTI catalogue entry (equations.py:144-155): "
                             "964 FLOPs at k = 9, 60 B/pt"),
    # the kernels built here, with the FLOPs they execute per point (ncu:
    # FADD/FMUL 1, FFMA/FADD2/FMUL2 2, FFMA2 4; profiles/r02_ncu_flops.json)
    EquationSpec("tti-b200", fixed_kernel_flops=242, fields_moved=15,
                 description="tti_pack (csrc/tti.cu): p and r in f32x2 lanes, shared derivative "
                             "chains; ncu-counted FLOPs at order 8; 9 parameters + 2x2 levels "
                             "read, p and r written"),
    EquationSpec("elastic-vs", fixed_kernel_flops=248, fields_moved=21,
                 description="isotropic velocity-stress (csrc/elastic.cu, SURVEY.md §8(a')): 9 "
                             "fields read and written, buoyancy / lambda / mu read (infinite-cache "
                             "traffic, equations.py:7-8); ncu-counted FLOPs at order 8 (velocity "
                             "115.5 + stress 132.5)"),
)}

_EQ_KEYS = {"name", "factor", "n_first", "n_second", "n_cross", "extra_mult", "extra_add",
            "duplicates", "fields_moved", "fixed_kernel_flops", "description", "override"}


def load_equations(path) -> dict:
    """Equation documents of a YAML file (one per document), the reference's
    hook (equations.py:218-246): shadowing a built-in needs `override: true`."""
    import yaml

    with open(path, encoding="utf-8") as fh:
        docs = [d for d in yaml.safe_load_all(fh) if d is not None]
    out = {}
    for d in docs:
        if not isinstance(d, dict) or "name" not in d:
            raise ValidationError(f"{path}: equation document must be a mapping with a name")
        unknown = set(d) - _EQ_KEYS
        if unknown:
            raise ValidationError(f"{path}: unknown equation keys: {sorted(unknown)}")
        eq = EquationSpec(**{k: v for k, v in d.items() if k != "override"})
        if eq.name in EQUATIONS and not d.get("override", False):
            raise ValidationError(f"{path}: '{eq.name}' is a built-in equation; "
                                  "set 'override: true' to replace it")
        out[eq.name] = eq
    return out


def equation_point(machine: MachineSpec, eq: EquationSpec, k: int,
                   measured_gpts: Optional[float] = None,
                   label: Optional[str] = None) -> RooflinePoint:
    """The roofline point of any catalogue equation: OI = kernel_flops /
    bytes, attainable = min(OI B, F); a measured rate in grid points per
    second is converted with the same FLOP count (analysis.py:170-181)."""
    fl = kernel_flops(eq, k)
    oi = fl / equation_bytes_per_point(eq, machine.precision_bytes)
    bound = "memory" if oi < machine.ridge_point else "compute"
    meas = None if measured_gpts is None else measured_gpts * fl
    return RooflinePoint(label or f"{eq.name}:k{k}", oi, machine.attainable(oi), bound, k, meas)


@dataclass(frozen=True)
class RooflineDataset:
    """A machine's roof plus the points pinned against it (analysis.py:123-167)."""

    machine: MachineSpec
    points: tuple
    oi_lo: float
    oi_hi: float

    def __post_init__(self):
        if not (0 < self.oi_lo < self.oi_hi):
            raise ValidationError(f"need 0 < oi_lo < oi_hi, got {self.oi_lo}, {self.oi_hi}")

    @property
    def ridge(self) -> float:
        return self.machine.ridge_point

    @property
    def roof_segments(self):
        """The bandwidth slope and the flat compute roof, meeting at the ridge."""
        b, f = self.machine.peak_bw_achievable, self.machine.peak_gflops_achievable
        return ((self.oi_lo, self.oi_lo * b), (self.ridge, f)), ((self.ridge, f), (self.oi_hi, f))

    def inconsistencies(self, tolerance: float = 0.05):
        """Points measured above their bound by more than `tolerance`."""
        return [p for p in self.points if p.measured_gflops is not None
                and p.measured_gflops > p.attainable_gflops * (1.0 + tolerance)]

    def to_csv(self) -> str:
        lines = ["label,k,oi,attainable_gflops,bound,measured_gflops"]
        for p in self.points:
            m = "" if p.measured_gflops is None else repr(float(p.measured_gflops))
            lines.append(f"{p.label},{p.k},{p.oi!r},{p.attainable_gflops!r},{p.bound},{m}")
        return "\n".join(lines) + "\n"


def roofline_dataset(machine: MachineSpec, points, margin: float = 10.0) -> RooflineDataset:
    """Dataset spanning the points and the ridge with a factor `margin` each side."""
    ois = [p.oi for p in points] + [machine.ridge_point]
    return RooflineDataset(machine, tuple(points), min(ois) / margin, max(ois) * margin)
