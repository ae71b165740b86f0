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
# the top level, 8/9/15 at k = nz (63 operations per point). K1 produces the
# same bits with 57: the x-direction sums it carries from plane to plane and
# the z-sums shared by a thread's two levels are computed once.
_CENSUS = {False: {"muls": 10, "adds": 11, "loads": 18}, True: {"muls": 8, "adds": 9, "loads": 15}}


def operation_census(top: bool = False) -> dict:
    return {name: dict(_CENSUS[bool(top)]) for name in ("su", "sv", "sw")}


def reads_per_point(top: bool = False) -> int:
    return 3 * _CENSUS[bool(top)]["loads"]


# ---------------------------------------------------------------------------
# array-level API (reference kernel.py:73-172), executed by K6 on the GPU

# Operand wiring (field, dx, dy, dk) per positional formula argument
# (kernel.py:117-128).
_SU_ARGS = (("u", 0, 0, 0), ("u", -1, 0, 0), ("u", 1, 0, 0), ("u", 0, -1, 0), ("u", 0, 1, 0),
            ("u", 0, 0, -1), ("u", 0, 0, 1), ("v", 0, -1, 0), ("v", 1, -1, 0), ("v", 0, 0, 0),
            ("v", 1, 0, 0), ("w", 0, 0, -1), ("w", 1, 0, -1), ("w", 0, 0, 0), ("w", 1, 0, 0))
_SV_ARGS = (("v", 0, 0, 0), ("v", -1, 0, 0), ("v", 1, 0, 0), ("v", 0, -1, 0), ("v", 0, 1, 0),
            ("v", 0, 0, -1), ("v", 0, 0, 1), ("u", -1, 0, 0), ("u", -1, 1, 0), ("u", 0, 0, 0),
            ("u", 0, 1, 0), ("w", 0, 0, -1), ("w", 0, 1, -1), ("w", 0, 0, 0), ("w", 0, 1, 0))
_SW_ARGS = (("w", 0, 0, 0), ("w", -1, 0, 0), ("w", 1, 0, 0), ("w", 0, -1, 0), ("w", 0, 1, 0),
            ("w", 0, 0, -1), ("w", 0, 0, 1), ("u", -1, 0, -1), ("u", -1, 0, 0), ("u", 0, 0, -1),
            ("u", 0, 0, 0), ("v", 0, -1, -1), ("v", 0, -1, 0), ("v", 0, 0, -1), ("v", 0, 0, 0))


def _device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path has no CPU fallback: a CUDA device is required")
    return torch.device("cuda", torch.cuda.current_device())


def _formula(which: int, args, top: bool):
    import ctypes
    import torch
    from . import _lib
    from .device import _stream_handle
    if len(args) != 19:
        raise TypeError(f"formula takes 19 positional arguments ({len(args)} given)")
    arrs = [np.asarray(a, dtype=np.float64) for a in args]
    shape = np.broadcast_shapes(*(a.shape for a in arrs))
    n = int(np.prod(shape, dtype=np.int64))
    dev = _device()
    keep, ptrs, strides = [], (ctypes.c_void_p * 19)(), (ctypes.c_int64 * 19)()
    for m, a in enumerate(arrs):
        if a.size == 1:
            t = torch.tensor([float(a.reshape(-1)[0])], dtype=torch.float64, device=dev)
            strides[m] = 0
        else:
            full = np.array(np.broadcast_to(a, shape), dtype=np.float64, order="C")  # writable copy
            t = torch.from_numpy(full.reshape(-1)).to(dev)
            strides[m] = 1
        keep.append(t)
        ptrs[m] = t.data_ptr()
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().pwadv_formula_f64(which, ptrs, strides, n, 1 if top else 0,
                                            ctypes.c_void_p(out.data_ptr()), 0,
                                            _stream_handle(None, dev)))
    res = out[:n].cpu().numpy().reshape(shape)
    if all(np.ndim(a) == 0 and not isinstance(a, np.ndarray) for a in args):
        return float(res)
    return res


def su_formula(tcx, tcy, tzc1_k, tzc2_k, u_c, u_xm1, u_xp1, u_jm1, u_jp1, u_km1, u_kp1,
               v_jm1, v_jm1_xp1, v_c, v_xp1, w_km1, w_km1_xp1, w_c, w_xp1, top=False):
    """su at broadcast points (kernel.py:73-84); the top branch drops the tzc2 half."""
    return _formula(0, (tcx, tcy, tzc1_k, tzc2_k, u_c, u_xm1, u_xp1, u_jm1, u_jp1, u_km1, u_kp1,
                        v_jm1, v_jm1_xp1, v_c, v_xp1, w_km1, w_km1_xp1, w_c, w_xp1), top)


def sv_formula(tcx, tcy, tzc1_k, tzc2_k, v_c, v_xm1, v_xp1, v_jm1, v_jp1, v_km1, v_kp1,
               u_xm1, u_xm1_jp1, u_c, u_jp1, w_km1, w_km1_jp1, w_c, w_jp1, top=False):
    """sv at broadcast points (kernel.py:87-98)."""
    return _formula(1, (tcx, tcy, tzc1_k, tzc2_k, v_c, v_xm1, v_xp1, v_jm1, v_jp1, v_km1, v_kp1,
                        u_xm1, u_xm1_jp1, u_c, u_jp1, w_km1, w_km1_jp1, w_c, w_jp1), top)


def sw_formula(tcx, tcy, tzc1_k, tzc2_k, w_c, w_xm1, w_xp1, w_jm1, w_jp1, w_km1, w_kp1,
               u_xm1_km1, u_xm1, u_km1, u_c, v_jm1_km1, v_jm1, v_km1, v_c, top=False):
    """sw at broadcast points (kernel.py:101-112)."""
    return _formula(2, (tcx, tcy, tzc1_k, tzc2_k, w_c, w_xm1, w_xp1, w_jm1, w_jp1, w_km1, w_kp1,
                        u_xm1_km1, u_xm1, u_km1, u_c, v_jm1_km1, v_jm1, v_km1, v_c), top)


_FORMULAS = ((su_formula, _SU_ARGS), (sv_formula, _SV_ARGS), (sw_formula, _SW_ARGS))


def compute_block(coeffs, roles: dict):
    """su/sv/sw of columns given their 17 role arrays (kernel.py:139-162).

    `roles` maps each COMPUTE_ROLES key to an array shaped (..., nz) with a
    common leading shape; returns three arrays of that shape with level 0
    zeroed, the mid formula at levels 1..nz-2 and the top formula at nz-1.
    Runs as one K6 launch on the GPU."""
    import ctypes
    import torch
    from . import _lib
    from .device import _stream_handle
    base = np.asarray(roles[("u", 0, 0)])
    shape = base.shape
    if len(shape) < 1:
        raise ValueError("role arrays must be shaped (..., nz)")
    nz = shape[-1]
    if nz < 2:
        raise ValueError(f"nz {nz} < 2")
    tz1 = np.ascontiguousarray(coeffs.tzc1, dtype=np.float64)
    tz2 = np.ascontiguousarray(coeffs.tzc2, dtype=np.float64)
    if tz1.shape != (nz,) or tz2.shape != (nz,):
        raise ValueError(f"coefficient length {tz1.shape[0]} != nz {nz}")
    ncols = int(np.prod(shape[:-1], dtype=np.int64))
    dev = _device()
    keep, ptrs = [], (ctypes.c_void_p * 17)()
    for m, key in enumerate(COMPUTE_ROLES):
        a = np.asarray(roles[key], dtype=np.float64)
        if a.shape != shape:
            raise ValueError(f"role {key} shape {a.shape} != {shape}")
        if a.size:
            host = a if a.flags.c_contiguous and a.flags.writeable else np.array(a, order="C")
            t = torch.from_numpy(host.reshape(-1)).to(dev)
        else:
            t = torch.empty(1, dtype=torch.float64, device=dev)
        keep.append(t)
        ptrs[m] = t.data_ptr()
    tz = torch.from_numpy(np.concatenate([tz1, tz2])).to(dev)
    outs = [torch.empty(max(ncols * nz, 1), dtype=torch.float64, device=dev) for _ in range(3)]
    _lib.check(_lib.lib().pwadv_compute_block_f64(
        ptrs, *(ctypes.c_void_p(o.data_ptr()) for o in outs), ncols, nz, float(coeffs.tcx),
        float(coeffs.tcy), ctypes.c_void_p(tz.data_ptr()), ctypes.c_void_p(tz.data_ptr() + 8 * nz),
        0, _stream_handle(None, dev)))
    return tuple(o[:ncols * nz].cpu().numpy().reshape(shape) for o in outs)


def grid_roles(fields, x0: int, x1: int) -> dict:
    """Role views over interior columns i in [x0, x1) (1-based), full Y range
    (kernel.py:165-172): zero-copy strided views of the padded fields."""
    arrs = {"u": fields.u.data, "v": fields.v.data, "w": fields.w.data}
    ny = fields.dims.ny
    return {(f, dx, dy): arrs[f][x0 + dx:x1 + dx, 1 + dy:1 + dy + ny, :]
            for f, dx, dy in COMPUTE_ROLES}


# ---------------------------------------------------------------------------
# drop-in execution

_CTX_LOCK = threading.Lock()
_CTX_CACHE: "OrderedDict[tuple, object]" = OrderedDict()
_CTX_MAX = 4


def _context(dims: GridDims):
    """The cached HostContext for this shape on the current device (created on
    first use). At most _CTX_MAX shapes are kept, and their device buffers (6
    padded fields each) within a quarter of the device memory; evicted
    contexts are closed outside the cache lock — close() waits for a call in
    progress on another thread, and that caller's next call re-fetches
    (ContextClosed)."""
    import torch
    from .device import HostContext
    if not torch.cuda.is_available():
        raise RuntimeError("run_reference needs a CUDA device: the B200 path has no CPU fallback")
    dev = torch.cuda.current_device()
    key = (dev, dims.nx, dims.ny, dims.nz)
    evicted = []
    with _CTX_LOCK:
        ctx = _CTX_CACHE.get(key)
        if ctx is None:
            ctx = HostContext(GridDims(dims.nx, dims.ny, dims.nz), dev)
            _CTX_CACHE[key] = ctx
            budget = torch.cuda.get_device_properties(dev).total_memory // 4

            def held():
                return sum(6 * 8 * (k[1] + 2) * (k[2] + 2) * k[3] for k in _CTX_CACHE)
            while len(_CTX_CACHE) > 1 and (len(_CTX_CACHE) > _CTX_MAX or held() > budget):
                evicted.append(_CTX_CACHE.popitem(last=False)[1])
        else:
            _CTX_CACHE.move_to_end(key)
    for old in evicted:
        old.close()
    return ctx


def _host_array(f, dims):
    a = np.ascontiguousarray(f.data, dtype=np.float64)
    if a.shape != (dims.nx + 2, dims.ny + 2, dims.nz):
        raise ValueError(f"field shape {a.shape} != padded {(dims.nx + 2, dims.ny + 2, dims.nz)}")
    return a


# Outputs up to this size come from torch's caching page-locked allocator
# (released results are reused; the D2H lands in them directly). Larger ones
# are plain numpy memory, filled through the context's staging buffers: the
# caching allocator rounds every block up to a power of two and never returns
# it to the OS (three C3 outputs would pin ~3 x 4 GiB for the process's life).
_PINNED_OUTPUT_MAX = 512 << 20


def _output_array(shape) -> np.ndarray:
    """A new float64 output array (page-locked below _PINNED_OUTPUT_MAX)."""
    import torch
    nbytes = 8 * int(np.prod(shape, dtype=np.int64))
    if nbytes <= _PINNED_OUTPUT_MAX:
        try:
            return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
        except RuntimeError:
            pass
    return np.empty(shape)


def run_reference(fields, coeffs) -> SourceSet:
    """Whole-grid PW advection; pure function of its inputs (reference kernel.py:175-185).
    Like the reference (zeros_sources, grid.py:129-130) the callee allocates the
    outputs: numpy arrays, page-locked up to _PINNED_OUTPUT_MAX bytes each. Safe
    to call from several threads (each shape's context serialises its calls)."""
    dims = fields.dims
    nz_c = len(coeffs.tzc1)
    if nz_c != dims.nz:
        raise ValueError(f"coefficient length {nz_c} != nz {dims.nz}")
    gd = GridDims(dims.nx, dims.ny, dims.nz)
    u, v, w = (_host_array(f, dims) for f in (fields.u, fields.v, fields.w))
    outs = [_output_array(gd.padded_shape) for _ in range(3)]
    planes = _slab_planes(gd)
    from ._lib import PwadvError
    while True:
        try:
            if planes >= gd.nx:
                _advect_host(gd, (u, v, w), outs, coeffs)
            else:
                _advect_host_slabs(gd, (u, v, w), outs, coeffs, planes)
            break
        except PwadvError as exc:
            # the device buffers did not fit beside what else lives on the
            # GPU: halve the slab and try again (loud once one plane fails)
            if "out of memory" not in str(exc) or planes <= 1:
                raise
            planes = max(1, min(planes, gd.nx) // 2)
    return SourceSet(*(Field3D(gd, o) for o in outs))


def _advect_host(gd, ins, outs, coeffs) -> None:
    from .device import ContextClosed
    for attempt in range(3):
        try:
            _context(gd).advect_host(*ins, *outs, coeffs.tcx, coeffs.tcy, coeffs.tzc1, coeffs.tzc2)
            return
        except ContextClosed:  # evicted by another thread between fetch and call
            if attempt == 2:
                raise


# Share of the device memory the drop-in's six padded device arrays may take
# before a grid is evaluated X slab by X slab (PWADV_DROPIN_DEVICE_BYTES
# overrides the byte limit: tests force slabs on small grids with it).
_DEVICE_SHARE = 0.65


def _slab_planes(gd) -> int:
    """Interior X planes per device-resident slab: nx when the whole grid fits."""
    import os

    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("run_reference needs a CUDA device: the B200 path has no CPU fallback")
    limit = int(os.environ.get("PWADV_DROPIN_DEVICE_BYTES", "0")) or int(
        _DEVICE_SHARE * torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)
    per_plane = 6 * 8 * (gd.ny + 2) * gd.nz
    if per_plane * (gd.nx + 2) <= limit:
        return gd.nx
    n = limit // per_plane - 2
    if n < 1:
        raise ValueError(f"one X plane of {gd.ny + 2} x {gd.nz} with its two halo planes "
                         f"({3 * per_plane} bytes on the device) exceeds the limit of {limit} bytes")
    return int(n)


def _advect_host_slabs(gd, ins, outs, coeffs, planes: int) -> None:
    """Out-of-core evaluation of a grid larger than the device: X slabs of
    `planes` interior planes, each with its two neighbouring planes as halo —
    a contiguous run of the padded host arrays, X being the slowest axis — go
    through the slab shape's context, in and out of the same runs of the
    caller's arrays (no staging copy of a slab). A slab's output run starts
    one plane early, on the previous slab's last interior plane, which the
    slab's own (zero) halo plane would overwrite: that one plane is saved and
    put back; the plane after the run is the next slab's first, written later,
    or the grid's halo plane. Bit-identical to the whole-grid evaluation (the
    reference's X-slab engines, schedules.py:65-75, rest on the same
    independence); halo planes, halo columns and level 0 are +0.0 as
    zeros_sources leaves them (grid.py:129-130)."""
    nx = gd.nx
    i0 = 1
    while i0 <= nx:
        n = min(planes, nx + 1 - i0)
        sd = GridDims(n, gd.ny, gd.nz)
        keep = [o[i0 - 1].copy() for o in outs] if i0 > 1 else None
        _advect_host(sd, [a[i0 - 1:i0 + n + 1] for a in ins], [o[i0 - 1:i0 + n + 1] for o in outs],
                     coeffs)
        if keep is not None:
            for o, k in zip(outs, keep):
                o[i0 - 1] = k
        i0 += n
    for o in outs:
        o[0] = 0.0
        o[nx + 1] = 0.0


def _advect_point(which: int, fields, coeffs, i: int, j: int, k: int) -> float:
    """One point through the GPU formula kernel (K6) on its 15 operands, as
    the reference's _advect_point (kernel.py:186-195): 1-based i, j and
    k (2 <= k <= nz); at the top (k == nz) the k+1 operands are passed as 0.0.
    Only the operands cross to the device, not the fields."""
    dims = fields.dims
    assert 1 <= i <= dims.nx and 1 <= j <= dims.ny and 2 <= k <= dims.nz
    top = k == dims.nz
    arrs = {"u": fields.u.data, "v": fields.v.data, "w": fields.w.data}
    fn, spec = _FORMULAS[which]
    ops = [0.0 if (top and dk == 1) else float(arrs[f][i + dx, j + dy, k - 1 + dk])
           for f, dx, dy, dk in spec]
    return float(fn(float(coeffs.tcx), float(coeffs.tcy), float(coeffs.tzc1[k - 1]),
                    float(coeffs.tzc2[k - 1]), *ops, top=top))


def advect_point_u(fields, coeffs, i: int, j: int, k: int) -> float:
    """su at one interior point (1-based i, j; 2 <= k <= nz), reference kernel.py:200-203."""
    return _advect_point(0, fields, coeffs, i, j, k)


def advect_point_v(fields, coeffs, i: int, j: int, k: int) -> float:
    return _advect_point(1, fields, coeffs, i, j, k)


def advect_point_w(fields, coeffs, i: int, j: int, k: int) -> float:
    return _advect_point(2, fields, coeffs, i, j, k)
