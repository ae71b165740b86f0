"""B200-native PW-advection hot path of arXiv 2010.01545 (drop-in for pwadvect's stencil).

Import surface mirrors the reference package facade for the hot path
(pkg/src/pwadvect/__init__.py:11-34: grid, kernel and schedules names; the
reference's module paths `.grid`, `.kernel` and `.schedules` resolve to
`layout`, `stencil` and `engines` — registered below, no wrapper files) and
adds the device-resident API (`device`), the x-y decomposition with halo
exchange (`decomp`) and the fused time-stepping driver (`stepper`).
All compute runs in libpwadv.so (hand-written sm_100a CUDA); there is no CPU
fallback.
"""

from .layout import (Field3D, FieldSet, GeneratorSpec, GridDims, GridError, SourceSet,
                     checksum, fill_fields, lcg_doubles, linear_index, make_grid, read_field,
                     wrap_halos, write_field, zeros_sources)
from .stencil import (COMPUTE_ROLES, AdvectionCoefficients, FlopProfile, advect_point_u,
                      advect_point_v, advect_point_w, baseline_coefficients,
                      default_coefficients, flops, operation_census, reads_per_point,
                      run_reference)
from .engines import (VARIANTS, OutputComparison, ScheduleSpec, Slab, TrafficReport,
                      compare_outputs, partition_domain, run_schedule)

import sys as _sys

from . import engines as _engines, layout as _layout, stencil as _stencil

for _name, _mod in (("grid", _layout), ("kernel", _stencil), ("schedules", _engines)):
    _sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod

__version__ = "0.1.0"
