"""PW advection entry points (mirror of reference kernel.py), executed on the B200.

Drop-in for the reference's hot path: `run_reference(fields, coeffs) ->
SourceSet` (pkg/src/pwadvect/kernel.py:175-185) keeps its signature, argument
meaning and errors; the evaluation runs in libpwadv.so (K1, sm_100a) through
the host-buffer context (H2D, kernel, D2H pipelined over X slabs). Inputs can
be this package's FieldSet or the reference's own (duck-typed:
`fields.u.data`, `fields.dims.nx/ny/nz`, `coeffs.tcx/tcy/tzc1/tzc2`).

There is no CPU fallback: without a CUDA device or libpwadv.so these
functions raise.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from .layout import Field3D, GridDims, SourceSet

# ---------------------------------------------------------------------------
# coefficients (reference kernel.py:21-45)


@dataclass
class AdvectionCoefficients:
    """tcx/tcy scalars and per-level tzc1/tzc2 arrays of length nz."""

    tcx: float
    tcy: float
    tzc1: np.ndarray
    tzc2: np.ndarray

    def __post_init__(self):
        self.tzc1 = np.asarray(self.tzc1, dtype=np.float64)
        self.tzc2 = np.asarray(self.tzc2, dtype=np.float64)
        if self.tzc1.ndim != 1 or self.tzc1.shape != self.tzc2.shape:
            raise ValueError("tzc1/tzc2 must be 1-D arrays of equal length")
        if not (np.all(np.isfinite(self.tzc1)) and np.all(np.isfinite(self.tzc2))):
            raise ValueError("vertical coefficients must be finite")

    @property
    def nz(self) -> int:
        return int(self.tzc1.shape[0])


def default_coefficients(nz: int, value: float = 0.25) -> AdvectionCoefficients:
    """tcx = tcy = tzc1(k) = tzc2(k) = value (reference default 0.25)."""
    return AdvectionCoefficients(value, value, np.full(nz, value), np.full(nz, value))


def baseline_coefficients(seed: int, nz: int, dx: float = 50.0) -> AdvectionCoefficients:
    """BASELINE.json coefficients: tcx = tcy = 0.25/dx, tzc1/tzc2
    = 1e-3 + 4e-3*lcg(seed+1) in [1e-3, 5e-3). (tzd1/tzd2 of BASELINE are not
    used by the reference formulas.)"""
    from .layout import lcg_doubles
    t = lcg_doubles(seed + 1, 4 * nz)
    return AdvectionCoefficients(0.25 / dx, 0.25 / dx, 1e-3 + 4e-3 * t[:nz],
                                 1e-3 + 4e-3 * t[nz:2 * nz])


@dataclass(frozen=True)
class FlopProfile:
    """Paper's per-cell credit: 21 add + 32 mul = 53 (reference kernel.py:48-57)."""

    adds_per_cell: int = 21
    muls_per_cell: int = 32

    @property
    def total_per_cell(self) -> int:
        return self.adds_per_cell + self.muls_per_cell


def flops(dims: GridDims, profile: FlopProfile = FlopProfile()) -> int:
    return dims.cells * profile.total_per_cell


# The 17 input columns (field, dx, dy) one output column reads, from the
# operand wiring of kernel.py:117-128 (COMPUTE_ROLES, kernel.py:134-136).
COMPUTE_ROLES: tuple[tuple[str, int, int], ...] = (
    ("u", -1, 0), ("u", -1, 1), ("u", 0, -1), ("u", 0, 0), ("u", 0, 1), ("u", 1, 0),
    ("v", -1, 0), ("v", 0, -1), ("v", 0, 0), ("v", 0, 1), ("v", 1, -1), ("v", 1, 0),
    ("w", -1, 0), ("w", 0, -1), ("w", 0, 0), ("w", 0, 1), ("w", 1, 0),
)

# Per formula and point: multiplications, add/subs, operand reads, as the
# reference's symbolic census reports them (kernel.py:254-267): 10/11/18 below
# the top level, 8/9/15 at k = nz. The device kernel performs exactly these
# DMUL/DADD operations (63 per point below the top).
_CENSUS = {False: {"muls": 10, "adds": 11, "loads": 18}, True: {"muls": 8, "adds": 9, "loads": 15}}


def operation_census(top: bool = False) -> dict:
    return {name: dict(_CENSUS[bool(top)]) for name in ("su", "sv", "sw")}


def reads_per_point(top: bool = False) -> int:
    return 3 * _CENSUS[bool(top)]["loads"]


# ---------------------------------------------------------------------------
# drop-in execution

_CTX_LOCK = threading.Lock()
_CTX_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_CTX_MAX = 4


def _context(dims: GridDims):
    import torch
    from .device import HostContext
    if not torch.cuda.is_available():
        raise RuntimeError("run_reference needs a CUDA device: the B200 path has no CPU fallback")
    dev = torch.cuda.current_device()
    key = (dev, dims.nx, dims.ny, dims.nz)
    with _CTX_LOCK:
        ctx = _CTX_CACHE.get(key)
        if ctx is None:
            ctx = HostContext(GridDims(dims.nx, dims.ny, dims.nz), dev)
            _CTX_CACHE[key] = ctx
            while len(_CTX_CACHE) > _CTX_MAX:
                _, old = _CTX_CACHE.popitem(last=False)
                old.close()
        else:
            _CTX_CACHE.move_to_end(key)
        return ctx


def _host_array(f, dims):
    a = np.ascontiguousarray(f.data, dtype=np.float64)
    if a.shape != (dims.nx + 2, dims.ny + 2, dims.nz):
        raise ValueError(f"field shape {a.shape} != padded {(dims.nx + 2, dims.ny + 2, dims.nz)}")
    return a


def _output_array(shape) -> np.ndarray:
    """A new float64 output array in page-locked memory (torch's caching host
    allocator: blocks of released results are reused, and the D2H copies
    land in it directly instead of through staging and first-touch page
    faults); plain numpy memory if pinning is unavailable."""
    import torch
    try:
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    except RuntimeError:
        return np.empty(shape)


def run_reference(fields, coeffs) -> SourceSet:
    """Whole-grid PW advection; pure function of its inputs (reference kernel.py:175-185).
    Like the reference (zeros_sources, grid.py:129-130) the callee allocates the
    outputs; here they are page-locked numpy arrays."""
    dims = fields.dims
    nz_c = len(coeffs.tzc1)
    if nz_c != dims.nz:
        raise ValueError(f"coefficient length {nz_c} != nz {dims.nz}")
    gd = GridDims(dims.nx, dims.ny, dims.nz)
    u, v, w = (_host_array(f, dims) for f in (fields.u, fields.v, fields.w))
    outs = [_output_array(gd.padded_shape) for _ in range(3)]
    _context(gd).advect_host(u, v, w, *outs, coeffs.tcx, coeffs.tcy, coeffs.tzc1, coeffs.tzc2)
    return SourceSet(*(Field3D(gd, o) for o in outs))


def _advect_point(which: int, fields, coeffs, i: int, j: int, k: int) -> float:
    import torch
    from . import device
    dims = fields.dims
    assert 1 <= i <= dims.nx and 1 <= j <= dims.ny and 2 <= k <= dims.nz
    dev = torch.device("cuda")
    u, v, w = (torch.from_numpy(_host_array(f, dims)).to(dev) for f in (fields.u, fields.v, fields.w))
    out = device.alloc_fields(GridDims(dims.nx, dims.ny, dims.nz), dev)
    device.advect(u, v, w, coeffs, out, box=(i, i + 1, j, j + 1), opts=device.make_opts("simple"))
    return float(out[which][i, j, k - 1].item())


def advect_point_u(fields, coeffs, i: int, j: int, k: int) -> float:
    """su at one interior point (1-based i, j; 2 <= k <= nz), reference kernel.py:200-203."""
    return _advect_point(0, fields, coeffs, i, j, k)


def advect_point_v(fields, coeffs, i: int, j: int, k: int) -> float:
    return _advect_point(1, fields, coeffs, i, j, k)


def advect_point_w(fields, coeffs, i: int, j: int, k: int) -> float:
    return _advect_point(2, fields, coeffs, i, j, k)
