"""`pwadvect` resolved to the B200 drop-in, for running the reference's own
test files unchanged (tests/test_gpu_reference_suite.py).

The hot-path modules `pwadvect.grid`, `pwadvect.kernel` and
`pwadvect.schedules` ARE this repository's package
(paper_2010_01545_b200.layout / .stencil / .engines, registered by the
package under the module paths .grid / .kernel / .schedules): every stencil
evaluation, generator fill and schedule run goes to libpwadv.so on the GPU.
The out-of-scope FPGA modelling modules (dataflow, transfer, params, refdata,
cli — SURVEY.md §2) are loaded unmodified from the stock reference installed
in baseline/_ref; they import `.grid` / `.kernel`, i.e. ours.
Test infrastructure only; nothing in the product imports it.
"""

import sys
from pathlib import Path

_STOCK = Path(__file__).resolve().parents[3] / "baseline" / "_ref" / "pwadvect"
if not (_STOCK / "__init__.py").exists():
    raise ImportError(f"stock reference not installed at {_STOCK}")

from paper_2010_01545_b200 import grid, kernel, schedules  # noqa: E402

for _name, _mod in (("grid", grid), ("kernel", kernel), ("schedules", schedules)):
    sys.modules[f"{__name__}.{_name}"] = _mod
# every other submodule is the stock file
__path__ = [str(_STOCK)]

# the stock facade's names (reference pkg/src/pwadvect/__init__.py:11-70)
from .grid import (Field3D, FieldSet, GeneratorSpec, GridDims, SourceSet,  # noqa: E402,F401
                   checksum, fill_fields, linear_index, make_grid, read_field, write_field)
from .kernel import (AdvectionCoefficients, FlopProfile, advect_point_u,  # noqa: E402,F401
                     advect_point_v, advect_point_w, default_coefficients, flops,
                     operation_census, run_reference)
from .schedules import (ScheduleSpec, Slab, TrafficReport, compare_outputs,  # noqa: E402,F401
                        partition_domain, run_schedule)
from .dataflow import (CycleReport, MemoryModel, PipelineSpec, calibrate,  # noqa: E402,F401
                       gflops, kernel_compute_cycles, kernel_memory_seconds, kernel_time,
                       pipeline_cycles, pipeline_latency)
from .transfer import (DmaConfig, ModelReport, dma_time, end_to_end,  # noqa: E402,F401
                       factor_cells, scaling_table, transfer_volume)
from .params import ModelParams, load_params  # noqa: E402,F401

__version__ = "0.1.0"
