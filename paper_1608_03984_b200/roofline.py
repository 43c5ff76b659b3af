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
from dataclasses import dataclass
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
class MachineSpec:
    """Subset of fdroof.machines.MachineSpec (machines.py:98-148) used for reporting."""

    name: str
    peak_gflops_achievable: float
    peak_bw_achievable: float
    source: str = ""

    @property
    def ridge_point(self) -> float:
        return self.peak_gflops_achievable / self.peak_bw_achievable

    def attainable(self, oi: float) -> float:
        return min(oi * self.peak_bw_achievable, self.peak_gflops_achievable)


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


def b200_machine(sm_mhz: Optional[float] = None) -> MachineSpec:
    """B200 roofline: measured HBM copy GB/s and the derived FP32 GFLOPS."""
    peaks = measured_peaks()
    bw = float(peaks.get("hbm_gbs", FALLBACK_HBM_GBS))
    src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    mhz = float(sm_mhz or peaks.get("sm_max_mhz", B200_MAX_SM_MHZ))
    fp32 = B200_SMS * B200_FP32_LANES * 2 * mhz * 1e-3  # GFLOPS
    return MachineSpec("b200", fp32, bw, src)


def roofline_point(machine: MachineSpec, order: int,
                   measured_gflops: Optional[float] = None) -> RooflinePoint:
    k = order + 1
    oi = acoustic_flops_per_point(order) / ACOUSTIC_BYTES_PER_POINT
    bound = "memory" if oi < machine.ridge_point else "compute"
    return RooflinePoint(f"acoustic:k{k}", oi, machine.attainable(oi), bound, k, measured_gflops)
