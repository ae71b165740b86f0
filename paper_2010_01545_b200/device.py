"""Device-resident API: the hot path on torch CUDA tensors, no host copies.

Fields are torch.float64 CUDA tensors of shape (nx+2, ny+2, nz), C-contiguous,
k fastest — byte-for-byte the reference's `Field3D.data` layout
(pkg/src/pwadvect/grid.py:61-88), so there are no transposes at the boundary.
torch only allocates memory and supplies streams; every kernel is ours
(libpwadv.so through `_lib`). This is the API the benchmark times.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .layout import GeneratorSpec, GridDims, GridError, make_grid

__all__ = ["DeviceCoefficients", "make_opts", "advect", "step", "wrap_halos", "fill",
           "describe_plan", "HostContext", "BoundLaunch", "dims_of", "alloc_fields",
           "save_field", "load_field"]


def _stream_handle(stream, device) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _p(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def dims_of(t: torch.Tensor) -> GridDims:
    if t.dim() != 3:
        raise GridError(f"fields are 3-D (nx+2, ny+2, nz), got shape {tuple(t.shape)}")
    return make_grid(t.shape[0] - 2, t.shape[1] - 2, t.shape[2])


def _check_field(t: torch.Tensor, dims: GridDims, name: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if tuple(t.shape) != dims.padded_shape:
        raise GridError(f"{name} shape {tuple(t.shape)} != padded {dims.padded_shape}")
    if t.dtype != torch.float64:
        raise GridError(f"fields are float64, got {t.dtype} for {name}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the PW path has no CPU fallback)")
    if not t.is_contiguous():
        raise GridError(f"{name} must be C-contiguous (k fastest)")


def alloc_fields(dims: GridDims, device=None, zero: bool = True):
    """Three padded float64 fields on `device` (zeroed: +0.0 halos, as zeros_sources)."""
    mk = torch.zeros if zero else torch.empty
    return tuple(mk(dims.padded_shape, dtype=torch.float64, device=device) for _ in range(3))


@dataclass
class DeviceCoefficients:
    """tcx/tcy scalars + tzc1/tzc2 resident on the device (tz[0] = tzc1, tz[1] = tzc2)."""

    tcx: float
    tcy: float
    tz: torch.Tensor  # (2, nz) float64 CUDA

    @property
    def nz(self) -> int:
        return int(self.tz.shape[1])

    @classmethod
    def from_host(cls, coeffs, device=None) -> "DeviceCoefficients":
        """From a (reference or mirror) AdvectionCoefficients-like object."""
        tz = np.stack([np.asarray(coeffs.tzc1, dtype=np.float64),
                       np.asarray(coeffs.tzc2, dtype=np.float64)])
        t = torch.from_numpy(np.ascontiguousarray(tz)).to(device or "cuda")
        return cls(float(coeffs.tcx), float(coeffs.tcy), t)


def _as_device_coeffs(coeffs, device) -> DeviceCoefficients:
    if isinstance(coeffs, DeviceCoefficients):
        if coeffs.tz.device != device:
            return DeviceCoefficients(coeffs.tcx, coeffs.tcy, coeffs.tz.to(device))
        return coeffs
    return DeviceCoefficients.from_host(coeffs, device)


def make_opts(variant: str = "xmarch", *, tile_j: int = 0, stages: int = 0, grid: int = 0,
              max_threads: int = 0, chunks: int = 0, flags: int = 0) -> _lib.Opts:
    """Kernel selection: "xmarch" (bulk-copy plane ring, default), "simple"
    (one thread per point), "xmarch_generic" (the X-march with a run-time
    tile layout even where a compile-time one exists), "xmarch_elem" (the
    X-march with unaligned tile runs and scalar shared loads — what odd nz
    and 8-byte-aligned fields run on), "xmarch_ct" (the column-tile X-march:
    k-slab work units, every pair on the 16-byte grid; tile_j 6/12/24 selects
    the slab height 128/64/32), "xmarch_noct" (the X-march without the column-
    tile form), "march" (the general march K1m, no plane ring); suffix "_fma"
    for the DFMA (not bit-exact) build."""
    base = variant
    if variant.endswith("_fma"):
        flags |= _lib.FLAG_FMA
        base = variant[:-4]
    if base == "simple":
        flags |= _lib.FLAG_SIMPLE
    elif base == "xmarch_generic":
        flags |= _lib.FLAG_GENERIC
    elif base == "xmarch_elem":
        flags |= _lib.FLAG_UNALIGNED
    elif base == "xmarch_ct":
        flags |= _lib.FLAG_CTILE
    elif base == "xmarch_noct":
        flags |= _lib.FLAG_NO_CTILE
    elif base == "march":
        flags |= _lib.FLAG_MARCH
    elif base != "xmarch":
        raise ValueError(f"unknown kernel variant {variant!r}")
    return _lib.Opts(flags, tile_j, stages, grid, max_threads, chunks, None)


def _box(dims: GridDims, box):
    if box is None:
        return 1, dims.nx + 1, 1, dims.ny + 1
    x0, x1, y0, y1 = (int(b) for b in box)
    if not (1 <= x0 <= x1 <= dims.nx + 1 and 1 <= y0 <= y1 <= dims.ny + 1):
        raise ValueError(f"box {box} outside interior {dims.nx}x{dims.ny}")
    return x0, x1, y0, y1


def advect(u, v, w, coeffs, out=None, *, box=None, opts: _lib.Opts | None = None,
           stream=None):
    """K1: su, sv, sw = PW advection of (u, v, w); returns the output tensors.

    `out` (su, sv, sw) must be zero-initialised once by the caller (halo
    columns are never written); allocated with +0.0 halos when None.
    `box` = (x_begin, x_end, y_begin, y_end) restricts to interior columns
    (1-based, half-open), like the reference's X slabs (schedules.py:53-75).
    """
    dims = dims_of(u)
    for t, n in ((u, "u"), (v, "v"), (w, "w")):
        _check_field(t, dims, n)
    dc = _as_device_coeffs(coeffs, u.device)
    if dc.nz != dims.nz:
        raise ValueError(f"coefficient length {dc.nz} != nz {dims.nz}")
    if out is None:
        out = alloc_fields(dims, u.device)
    for t, n in zip(out, ("su", "sv", "sw")):
        _check_field(t, dims, n)
    x0, x1, y0, y1 = _box(dims, box)
    L = _lib.lib()
    _lib.check(L.pwadv_advect_box_f64(_p(u), _p(v), _p(w), _p(out[0]), _p(out[1]), _p(out[2]),
                                      dims.nx, dims.ny, dims.nz, dc.tcx, dc.tcy, _p(dc.tz[0]),
                                      _p(dc.tz[1]), x0, x1, y0, y1, _lib.opts_ptr(opts),
                                      _stream_handle(stream, u.device)))
    return out


def step(u, v, w, coeffs, dt: float, out, *, box=None, opts: _lib.Opts | None = None,
         stream=None):
    """K4: out = (u, v, w) + dt*(su, sv, sw) on interior columns (halos untouched)."""
    dims = dims_of(u)
    for t, n in ((u, "u"), (v, "v"), (w, "w")):
        _check_field(t, dims, n)
    for t, n in zip(out, ("u_new", "v_new", "w_new")):
        _check_field(t, dims, n)
    dc = _as_device_coeffs(coeffs, u.device)
    if dc.nz != dims.nz:
        raise ValueError(f"coefficient length {dc.nz} != nz {dims.nz}")
    x0, x1, y0, y1 = _box(dims, box)
    _lib.check(_lib.lib().pwadv_step_box_f64(
        _p(u), _p(v), _p(w), _p(out[0]), _p(out[1]), _p(out[2]), dims.nx, dims.ny, dims.nz,
        dc.tcx, dc.tcy, _p(dc.tz[0]), _p(dc.tz[1]), float(dt), x0, x1, y0, y1,
        _lib.opts_ptr(opts), _stream_handle(stream, u.device)))
    return out


class BoundLaunch:
    """A K1 (advect) or K4 (dt given: step) launch on one box with every
    argument validated and converted once; calling it costs one ctypes call.
    For loops that launch the same box on the same buffers many times (the
    multi-GPU interior / rim launches), where per-call Python overhead would
    otherwise exceed the kernel time of a small per-GPU block."""

    def __init__(self, fields, coeffs, out, *, box=None, opts: _lib.Opts | None = None,
                 dt: float | None = None, pull: "_lib.Peers | None" = None,
                 gather: bool = False):
        """pull: the neighbours' buffers — fused into the kernel's bulk copies
        (the aligned X-march), or with gather=True as the K2p halo gather
        (pwadv_pull_halos_f64 into this block's halos) followed by the plain
        launch with the planner's kernel (any shape: K1c, odd nz, ...)."""
        u, v, w = fields
        dims = dims_of(u)
        if pull is not None and box is not None:
            raise ValueError("a halo-pull launch covers the whole interior (no box)")
        if gather and pull is None:
            raise ValueError("gather needs the peer table")
        for t, n in zip(tuple(fields) + tuple(out), ("u", "v", "w", "o0", "o1", "o2")):
            _check_field(t, dims, n)
        dc = _as_device_coeffs(coeffs, u.device)
        if dc.nz != dims.nz:
            raise ValueError(f"coefficient length {dc.nz} != nz {dims.nz}")
        x0, x1, y0, y1 = _box(dims, box)
        self._keep = (tuple(fields), tuple(out), dc, opts)
        self.device = u.device
        L = _lib.lib()
        head = [_p(u), _p(v), _p(w), _p(out[0]), _p(out[1]), _p(out[2]), dims.nx, dims.ny,
                dims.nz, dc.tcx, dc.tcy, _p(dc.tz[0]), _p(dc.tz[1])]
        self._pre = None
        if pull is not None and gather:
            self._keep += (pull,)
            self._pre = (L.pwadv_pull_halos_f64,
                         [_p(u), _p(v), _p(w), dims.nx, dims.ny, dims.nz, ctypes.byref(pull)])
            pull = None
        if pull is not None:
            self._keep += (pull,)
            pp = ctypes.byref(pull)
            if dt is None:
                self._fn = L.pwadv_advect_pull_f64
                self._args = head + [pp, _lib.opts_ptr(opts)]
            else:
                self._fn = L.pwadv_step_pull_f64
                self._args = head + [float(dt), pp, _lib.opts_ptr(opts)]
        elif dt is None:
            self._fn = L.pwadv_advect_box_f64
            self._args = head + [x0, x1, y0, y1, _lib.opts_ptr(opts)]
        else:
            self._fn = L.pwadv_step_box_f64
            self._args = head + [float(dt), x0, x1, y0, y1, _lib.opts_ptr(opts)]

    def __call__(self, stream=None) -> None:
        h = _stream_handle(stream, self.device)
        if self._pre is not None:
            _lib.check(self._pre[0](*self._pre[1], h))
        _lib.check(self._fn(*self._args, h))


def event_pair(events, stream=None):
    """Start a timing event pair on `stream` if `events` is a list (else None)."""
    if events is None:
        return None
    s = stream or torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    events.append((a, b))
    return b


def close_event_pair(end, stream=None) -> None:
    if end is not None:
        end.record(stream or torch.cuda.current_stream())


def self_peers(fields) -> _lib.Peers:
    """Peer table naming this block as all eight of its neighbours: a halo-pull
    launch with it evaluates the periodic domain without a halo wrap."""
    dims = dims_of(fields[0])
    p = _lib.Peers()
    for d in range(8):
        p.u[d], p.v[d], p.w[d] = (_p(t) for t in fields)
        p.nx[d], p.ny[d] = dims.nx, dims.ny
    return p


def pull_halos(u, v, w, peers: _lib.Peers, stream=None) -> None:
    """K2p: this block's halo cells gathered from the neighbours' current
    interiors (pwadv_pull_halos_f64) — the cells a two-phase periodic exchange
    delivers (reference wrap_halos, grid.py:203-208), for any shape."""
    dims = dims_of(u)
    for t, n in ((u, "u"), (v, "v"), (w, "w")):
        _check_field(t, dims, n)
    _lib.check(_lib.lib().pwadv_pull_halos_f64(_p(u), _p(v), _p(w), dims.nx, dims.ny, dims.nz,
                                               ctypes.byref(peers), _stream_handle(stream, u.device)))


def advect_pull(u, v, w, coeffs, peers: _lib.Peers, out=None, *, opts: _lib.Opts | None = None,
                stream=None):
    """K1 with the halo exchange fused in: su, sv, sw of the whole interior
    with halo cells loaded from the neighbours' current (u, v, w) in `peers`
    (pwadv_advect_pull_f64); this block's halos are not read."""
    if out is None:
        out = alloc_fields(dims_of(u), u.device)
    BoundLaunch((u, v, w), coeffs, out, opts=opts, pull=peers)(stream)
    return out


def step_pull(u, v, w, coeffs, dt: float, out, peers: _lib.Peers, *, opts: _lib.Opts | None = None,
              stream=None):
    """K4 with the halo pull (pwadv_step_pull_f64): out = (u, v, w) + dt*PW on
    the whole interior; out's halos are not written."""
    BoundLaunch((u, v, w), coeffs, out, opts=opts, dt=float(dt), pull=peers)(stream)
    return out


def wrap_halos(*fields, stream=None) -> None:
    """K2: periodic halo wrap in place (reference grid.py:203-208)."""
    if not fields:
        return
    dims = dims_of(fields[0])
    for t in fields:
        _check_field(t, dims, "field")
    L = _lib.lib()
    h = _stream_handle(stream, fields[0].device)
    if len(fields) == 3:
        _lib.check(L.pwadv_wrap_halos3_f64(_p(fields[0]), _p(fields[1]), _p(fields[2]),
                                           dims.nx, dims.ny, dims.nz, h))
    else:
        for t in fields:
            _lib.check(L.pwadv_wrap_halos_f64(_p(t), dims.nx, dims.ny, dims.nz, h))


def fill(dims: GridDims, spec: GeneratorSpec, device=None, stream=None, out=None):
    """K5: (u, v, w) on the device, bit-identical to the reference fill_fields."""
    if spec.mode == "trig":
        raise ValueError("the trig test pattern is host-generated (layout.fill_fields)")
    code = {"random": 0, "baseline": 1, "uniform": 2}[spec.mode]
    if out is None:
        out = alloc_fields(dims, device or "cuda", zero=False)
    for t, n in zip(out, "uvw"):
        _check_field(t, dims, n)
    _lib.check(_lib.lib().pwadv_fill_f64(_p(out[0]), _p(out[1]), _p(out[2]), dims.nx, dims.ny,
                                         dims.nz, code, int(spec.seed) & (2**64 - 1),
                                         float(spec.a), float(spec.b), float(spec.c),
                                         _stream_handle(stream, out[0].device)))
    return out


def describe_plan(dims: GridDims, box=None, opts: _lib.Opts | None = None, device: int = 0) -> dict:
    x0, x1, y0, y1 = _box(dims, box)
    info = _lib.PlanInfo()
    _lib.check(_lib.lib().pwadv_describe_plan(dims.nx, dims.ny, dims.nz, x0, x1, y0, y1,
                                              _lib.opts_ptr(opts), int(device), ctypes.byref(info)))
    return {"kernel": {1: "xmarch", 2: "simple", 3: "march", 4: "xmarch_elem", 5: "xmarch_ct"}[info.kernel], "tile_j": info.tile_j,
            "threads_per_column": info.threads_per_column, "stages": info.stages,
            "threads": info.threads, "grid": info.grid, "smem_bytes": info.smem_bytes,
            "strips": info.strips, "chunks": info.chunks, "long_strips": info.long_strips,
            "spare_ctas": info.spare_ctas, "main_chunk_planes": info.main_chunk_planes}


# ---------------------------------------------------------------------------
# field files (the reference's format, grid.py:252-270) straight to / from
# device tensors through a page-locked buffer

def save_field(t: torch.Tensor, path) -> None:
    """Write a padded device field as the reference's field file: 24-byte
    little-endian (nx, ny, nz) header + the padded float64 data."""
    from .layout import _HEADER
    dims = dims_of(t)
    _check_field(t, dims, "field")
    host = torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True)
    host.copy_(t)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(dims.nx, dims.ny, dims.nz))
        fh.write(memoryview(host.numpy()).cast("B"))


def load_field(path, device=None) -> torch.Tensor:
    """Read a reference field file into a new device tensor (GridError on a
    truncated file, as read_field)."""
    from .layout import _HEADER
    with open(path, "rb") as fh:
        nx, ny, nz = _HEADER.unpack(fh.read(_HEADER.size))
        dims = make_grid(nx, ny, nz)
        host = torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True)
        got = fh.readinto(memoryview(host.numpy()).cast("B"))
    if got != dims.padded_len * 8:
        raise GridError(f"truncated field file {path}")
    return host.to(device or "cuda")


class ContextClosed(RuntimeError):
    """A HostContext was closed (e.g. evicted) before or while it was fetched."""


class HostContext:
    """pwadv_ctx: device buffers + 3 streams for host-buffer (end-to-end) calls."""

    def __init__(self, dims: GridDims, device: int = 0):
        import threading
        self.dims = dims
        self.device = int(device)
        # a pwadv_ctx takes one call at a time (its buffers and streams are
        # shared); concurrent callers of one context are serialised here
        self.lock = threading.RLock()
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().pwadv_ctx_create(ctypes.byref(h), self.device, dims.nx, dims.ny,
                                               dims.nz))
        self._h = h

    def close(self) -> None:
        """Free the context. Waits for a call in progress on another thread
        (it holds self.lock); later calls raise ContextClosed."""
        lock = getattr(self, "lock", None)
        if lock is None:
            return
        with lock:
            if getattr(self, "_h", None) is not None and self._h.value:
                _lib.lib().pwadv_ctx_destroy(self._h)
            self._h = None

    def _handle(self) -> ctypes.c_void_p:
        if self._h is None:  # caller holds self.lock
            raise ContextClosed("pwadv_ctx was closed (evicted from the drop-in's cache)")
        return self._h

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _hp(a) -> ctypes.c_void_p:
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
                raise ValueError("host buffers must be contiguous float64 CPU tensors")
            return ctypes.c_void_p(a.data_ptr())
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise GridError("host buffers must be C-contiguous float64 arrays")
        return ctypes.c_void_p(a.ctypes.data)

    def advect_host(self, u, v, w, su, sv, sw, tcx, tcy, tzc1, tzc2, chunks: int = 0,
                    opts: _lib.Opts | None = None) -> tuple[int, int]:
        """Host in, host out: pipelined H2D / K1 / D2H. Returns (h2d, d2h) bytes.
        chunks <= 0: automatic (1 below 32 MiB per field, else 16)."""
        d = self.dims
        for a in (u, v, w, su, sv, sw):
            if tuple(a.shape) != d.padded_shape:
                raise GridError(f"field shape {tuple(a.shape)} != padded {d.padded_shape}")
        tz1 = np.ascontiguousarray(tzc1, dtype=np.float64)
        tz2 = np.ascontiguousarray(tzc2, dtype=np.float64)
        if tz1.shape != (d.nz,) or tz2.shape != (d.nz,):
            raise ValueError(f"coefficient length {tz1.shape} != nz {d.nz}")
        with self.lock:
            _lib.check(_lib.lib().pwadv_ctx_advect_host(
                self._handle(), self._hp(u), self._hp(v), self._hp(w), self._hp(su), self._hp(sv),
                self._hp(sw), float(tcx), float(tcy), ctypes.c_void_p(tz1.ctypes.data),
                ctypes.c_void_p(tz2.ctypes.data), int(chunks), _lib.opts_ptr(opts)))
            a, b = ctypes.c_uint64(), ctypes.c_uint64()
            _lib.check(_lib.lib().pwadv_ctx_last_bytes(self._handle(), ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def submit_host(self, u, v, w, su, sv, sw, tcx, tcy, tzc1, tzc2, chunks: int = 0,
                    opts: _lib.Opts | None = None) -> tuple[int, int]:
        """Asynchronous advect_host for page-locked buffers (consecutive submissions
        pipeline H2D / K1 / D2H across grids); call sync() before reading outputs.
        chunks <= 0: automatic (about 64 MiB per field and chunk)."""
        d = self.dims
        tz1 = np.ascontiguousarray(tzc1, dtype=np.float64)
        tz2 = np.ascontiguousarray(tzc2, dtype=np.float64)
        if tz1.shape != (d.nz,) or tz2.shape != (d.nz,):
            raise ValueError(f"coefficient length {tz1.shape} != nz {d.nz}")
        with self.lock:
            self._keep = (tz1, tz2)  # the coefficient upload is asynchronous
            _lib.check(_lib.lib().pwadv_ctx_submit_host(
                self._handle(), self._hp(u), self._hp(v), self._hp(w), self._hp(su), self._hp(sv),
                self._hp(sw), float(tcx), float(tcy), ctypes.c_void_p(tz1.ctypes.data),
                ctypes.c_void_p(tz2.ctypes.data), int(chunks), _lib.opts_ptr(opts)))
            a, b = ctypes.c_uint64(), ctypes.c_uint64()
            _lib.check(_lib.lib().pwadv_ctx_last_bytes(self._handle(), ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def sync(self) -> None:
        with self.lock:
            _lib.check(_lib.lib().pwadv_ctx_sync(self._handle()))
