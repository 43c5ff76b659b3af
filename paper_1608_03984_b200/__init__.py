"""paper_1608_03984_b200: B200-native time stepping for the fdroof stencil hot path.

Re-exports the reference's kernel API (/root/reference/pkg/src/fdroof/
__init__.py:63-74: BenchResult, KernelConfig, Source, StabilityWarning,
Wavefield, dump_wavefield, max_stable_dt, oracle_step, run_benchmark, step) backed by the
sm_100a library libb200fd.so, plus the extensions the BASELINE configs need.
"""

from ._inputs import invalidate_plan
from .errors import DeviceError, ExtensionMissingError, FdroofError, ValidationError
from .kernel import (
    BenchResult,
    HostSimulation,
    KernelConfig,
    OffGridReceivers,
    OffGridSource,
    Receivers,
    Source,
    Sponge,
    StabilityWarning,
    Wavefield,
    dump_traces,
    dump_wavefield,
    load_traces,
    load_wavefield,
    max_stable_dt,
    oracle_step,
    run,
    run_benchmark,
    step,
    trilinear_weights,
)
from .roofline import (MachineSpec, RooflineDataset, RooflinePoint, b200_machine, get_machine,
                       load_machines, roofline_dataset, roofline_point)
from .stencils import a2_sum, acoustic_weights_f32, second_derivative_weights

__version__ = "0.1.0"
