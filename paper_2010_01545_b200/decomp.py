"""x-y domain decomposition with a 1-cell periodic halo exchange.

The reference parallelises only over X slabs of threads sharing one array
(schedules.py:65-75, 207-232); MONC halo-swaps every prognostic field between
MPI ranks before advection. Here the global interior is split
into a px x py grid of blocks, one per GPU (rank = cx*py + cy, x = i is the
slowest axis; "AxB" means px x py). Each rank holds a padded local block of
shape (nx_l+2, ny_l+2, nz) in the reference layout; k is never split.

The exchange reproduces `wrap_halos` (grid.py:203-208) exactly, with no
diagonal messages, in two phases:

  X: my plane 1 -> the x- neighbour's halo plane nx+1, my plane nx -> the x+
     neighbour's halo plane 0 (all j, including the stale y halos);
  Y: my column 1 -> the y- neighbour's halo column ny+1, my column ny -> the
     y+ neighbour's halo column 0, for every i including the X halos just
     received — which carries the corner values (u(x-lo, y-hi), v(x-hi, y-lo)
     are the corners the stencil reads, SURVEY.md probe P4).

An undivided axis (p = 1) is a local periodic copy (K2 per axis). Faces are
packed/unpacked by libpwadv kernels (CUDA) or by tensor slicing (CPU, for the
gloo tests); messages go through a Transport: NCCL point-to-point via
torch.distributed (one process per GPU), gloo on CPU, or an in-process
loopback hub that emulates several ranks on one device for the tests.

`advect_overlapped` runs the exchange on a side stream while K1 computes the
interior box whose stencil stays inside the block, then computes the
one-cell rim. Outputs are bitwise identical to a single-domain evaluation.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from .layout import GridDims, make_grid

__all__ = ["split_extent", "Decomposition", "TorchFaceOps", "CudaFaceOps", "DistTransport",
           "LoopbackHub", "HaloExchanger", "exchange_all_loopback"]


def split_extent(n: int, parts: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of n cells into (offset, length), wider first
    (the rule of partition_domain, schedules.py:65-75)."""
    if not 1 <= parts <= n:
        raise ValueError(f"cannot split {n} cells into {parts} parts")
    q, r = divmod(n, parts)
    out, off = [], 0
    for p in range(parts):
        ln = q + (1 if p < r else 0)
        out.append((off, ln))
        off += ln
    return out


@dataclass(frozen=True)
class Decomposition:
    global_dims: GridDims
    px: int
    py: int
    rank: int

    def __post_init__(self):
        if self.px < 1 or self.py < 1:
            raise ValueError("px, py must be >= 1")
        if not 0 <= self.rank < self.px * self.py:
            raise ValueError(f"rank {self.rank} outside a {self.px}x{self.py} decomposition")
        split_extent(self.global_dims.nx, self.px)
        split_extent(self.global_dims.ny, self.py)

    @property
    def size(self) -> int:
        return self.px * self.py

    @property
    def coords(self) -> tuple[int, int]:
        return divmod(self.rank, self.py)

    def rank_of(self, cx: int, cy: int) -> int:
        return (cx % self.px) * self.py + (cy % self.py)

    def block(self, rank: int | None = None) -> tuple[int, int, int, int]:
        """(x_off, nx_l, y_off, ny_l) of a rank's interior (0-based offsets)."""
        r = self.rank if rank is None else rank
        cx, cy = divmod(r, self.py)
        xo, nxl = split_extent(self.global_dims.nx, self.px)[cx]
        yo, nyl = split_extent(self.global_dims.ny, self.py)[cy]
        return xo, nxl, yo, nyl

    @property
    def local_dims(self) -> GridDims:
        _, nxl, _, nyl = self.block()
        return make_grid(nxl, nyl, self.global_dims.nz)

    @property
    def neighbours(self) -> dict:
        cx, cy = self.coords
        return {"xm": self.rank_of(cx - 1, cy), "xp": self.rank_of(cx + 1, cy),
                "ym": self.rank_of(cx, cy - 1), "yp": self.rank_of(cx, cy + 1)}

    def for_rank(self, rank: int) -> "Decomposition":
        return Decomposition(self.global_dims, self.px, self.py, rank)

    # -- data placement -----------------------------------------------------
    def local_view(self, padded_global):
        """The rank's padded block cut from a wrapped global padded array: its
        halos are the neighbours' edge cells / the periodic images."""
        xo, nxl, yo, nyl = self.block()
        return padded_global[xo:xo + nxl + 2, yo:yo + nyl + 2, :]

    def fill_local(self, spec, device=None, stream=None):
        """Device fields of this block, generated from the global stream (K5);
        halos are filled by the first exchange."""
        from . import _lib, device as dv
        dims = self.local_dims
        out = dv.alloc_fields(dims, device or "cuda", zero=True)
        if spec.mode == "uniform":
            return dv.fill(dims, spec, device=device, stream=stream, out=out)
        code = {"random": 0, "baseline": 1}[spec.mode]
        xo, _, yo, _ = self.block()
        g = self.global_dims
        _lib.check(_lib.lib().pwadv_fill_box_f64(
            dv._p(out[0]), dv._p(out[1]), dv._p(out[2]), dims.nx, dims.ny, dims.nz, g.nx, g.ny, xo,
            yo, code, int(spec.seed) & (2**64 - 1), float(spec.a), float(spec.b), float(spec.c),
            dv._stream_handle(stream, out[0].device)))
        return out


# ---------------------------------------------------------------------------
# face pack/unpack backends

class TorchFaceOps:
    """Tensor-slicing pack/unpack (CPU tensors; used by the gloo tests)."""

    @staticmethod
    def pack(fields, buf, axis: int, index: int, stream=None) -> None:
        for m, f in enumerate(fields):
            src = f[index] if axis == 0 else f[:, index]
            buf[m].copy_(src.reshape(-1))

    @staticmethod
    def unpack(fields, buf, axis: int, index: int, stream=None) -> None:
        for m, f in enumerate(fields):
            dst = f[index] if axis == 0 else f[:, index]
            dst.copy_(buf[m].view_as(dst))

    @classmethod
    def pack2(cls, fields, buf_lo, buf_hi, axis: int, n: int, stream=None) -> None:
        cls.pack(fields, buf_lo, axis, 1, stream)
        cls.pack(fields, buf_hi, axis, n, stream)

    @classmethod
    def unpack2(cls, fields, buf_lo, buf_hi, axis: int, n: int, stream=None) -> None:
        cls.unpack(fields, buf_hi, axis, n + 1, stream)
        cls.unpack(fields, buf_lo, axis, 0, stream)

    @staticmethod
    def wrap_axis(fields, axis: int, stream=None) -> None:
        for f in fields:
            if axis == 0:
                f[0].copy_(f[-2])
                f[-1].copy_(f[1])
            else:
                f[:, 0].copy_(f[:, -2])
                f[:, -1].copy_(f[:, 1])


class CudaFaceOps:
    """libpwadv pack/unpack kernels (one launch packs u, v and w)."""

    @staticmethod
    def _call(name, fields, buf, axis, index, stream):
        from . import _lib, device as dv
        d = dv.dims_of(fields[0])
        fn = getattr(_lib.lib(), name)
        _lib.check(fn(dv._p(fields[0]), dv._p(fields[1]), dv._p(fields[2]), dv._p(buf), d.nx, d.ny,
                      d.nz, int(index), dv._stream_handle(stream, fields[0].device)))

    @classmethod
    def pack(cls, fields, buf, axis, index, stream=None):
        cls._call("pwadv_pack_xface3_f64" if axis == 0 else "pwadv_pack_yface3_f64",
                  fields, buf, axis, index, stream)

    @classmethod
    def unpack(cls, fields, buf, axis, index, stream=None):
        cls._call("pwadv_unpack_xface3_f64" if axis == 0 else "pwadv_unpack_yface3_f64",
                  fields, buf, axis, index, stream)

    @staticmethod
    def _call2(name, fields, buf_lo, buf_hi, axis, stream):
        from . import _lib, device as dv
        d = dv.dims_of(fields[0])
        _lib.check(getattr(_lib.lib(), name)(
            dv._p(fields[0]), dv._p(fields[1]), dv._p(fields[2]), dv._p(buf_lo), dv._p(buf_hi),
            d.nx, d.ny, d.nz, int(axis), dv._stream_handle(stream, fields[0].device)))

    @classmethod
    def pack2(cls, fields, buf_lo, buf_hi, axis, n, stream=None):
        """faces 1 and n of `axis` in one launch (pwadv_pack_faces3_f64)."""
        cls._call2("pwadv_pack_faces3_f64", fields, buf_lo, buf_hi, axis, stream)

    @classmethod
    def unpack2(cls, fields, buf_lo, buf_hi, axis, n, stream=None):
        """halos 0 and n+1 of `axis` in one launch (pwadv_unpack_faces3_f64)."""
        cls._call2("pwadv_unpack_faces3_f64", fields, buf_lo, buf_hi, axis, stream)

    @staticmethod
    def wrap_axis(fields, axis, stream=None):
        from . import _lib, device as dv
        d = dv.dims_of(fields[0])
        _lib.check(_lib.lib().pwadv_wrap_axis3_f64(
            dv._p(fields[0]), dv._p(fields[1]), dv._p(fields[2]), d.nx, d.ny, d.nz, int(axis),
            dv._stream_handle(stream, fields[0].device)))


# ---------------------------------------------------------------------------
# transports. An op is (kind, tensor, peer, tag): kind "send" or "recv"; tag 0
# marks a message travelling toward the minus neighbour, 1 toward the plus one.

class DistTransport:
    """torch.distributed point-to-point (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.backend = dist.get_backend(group)

    def run(self, ops) -> None:
        dist = self.dist
        if not ops:
            return
        if self.backend == "nccl":
            # one NCCL group; sends/recvs between a pair match in posting order
            p2p = [dist.P2POp(dist.isend if k == "send" else dist.irecv, t, peer, self.group)
                   for k, t, peer, _ in ops]
            for req in dist.batch_isend_irecv(p2p):
                req.wait()
        elif any(t.is_cuda for _, t, _, _ in ops):
            # gloo has no point-to-point for CUDA tensors: stage through the
            # host (dry runs of the multi-rank paths with the ranks sharing
            # one GPU, tests/test_gpu_multi.py; never a measured path)
            torch.cuda.current_stream().synchronize()  # the packed faces are final
            staged = [(k, t, t.cpu() if k == "send" else torch.empty(t.shape, dtype=t.dtype), peer, tag)
                      for k, t, peer, tag in ops]
            reqs = [(dist.isend if k == "send" else dist.irecv)(h, peer, group=self.group, tag=tag)
                    for k, _, h, peer, tag in staged]
            for r in reqs:
                r.wait()
            for k, t, h, _, _ in staged:
                if k == "recv":
                    t.copy_(h)
        else:
            reqs = [(dist.isend if k == "send" else dist.irecv)(t, peer, group=self.group, tag=tag)
                    for k, t, peer, tag in ops]
            for r in reqs:
                r.wait()


class LoopbackHub:
    """Emulates the ranks of a decomposition inside one process: every posted
    send is matched to the recv with the same (src, dst, tag), in order."""

    def run_all(self, ops_by_rank: dict) -> None:
        queues: dict = {}
        for r, ops in ops_by_rank.items():
            for k, t, peer, tag in ops:
                if k == "send":
                    queues.setdefault((r, peer, tag), []).append(t)
        for r, ops in ops_by_rank.items():
            for k, t, peer, tag in ops:
                if k == "recv":
                    t.copy_(queues[(peer, r, tag)].pop(0))
        left = sum(len(q) for q in queues.values())
        if left:
            raise RuntimeError(f"{left} unmatched loopback sends")


class ThreadHubTransport:
    """Emulates NCCL point-to-point for ranks run as host threads of one
    process (several ranks on one GPU, for tests). Each rank calls `run` from
    its own thread inside its stream context: sends are published with a CUDA
    event, the ranks meet at a host barrier, each receiver's stream waits on
    the sender's event and copies, and a second barrier plus events keep send
    buffers alive until every receiver has copied. No kernel ever waits on
    another rank's kernel (only streams wait on recorded events)."""

    def __init__(self, nranks: int):
        import threading
        self.n = nranks
        self.barrier = threading.Barrier(nranks)
        self.lock = threading.Lock()
        self.queues: dict = {}
        self.done: dict = {}

    def bind(self, rank: int) -> "_BoundHub":
        return _BoundHub(self, rank)


class _BoundHub:
    def __init__(self, hub: ThreadHubTransport, rank: int):
        self.hub, self.rank = hub, rank

    def run(self, ops) -> None:
        hub, me = self.hub, self.rank
        cur = torch.cuda.current_stream()
        ready = torch.cuda.Event()
        ready.record(cur)
        with hub.lock:
            for k, t, peer, tag in ops:
                if k == "send":
                    hub.queues.setdefault((me, peer, tag), []).append((t, ready))
        hub.barrier.wait()
        for k, t, peer, tag in ops:
            if k == "recv":
                with hub.lock:
                    src, ev = hub.queues[(peer, me, tag)].pop(0)
                cur.wait_event(ev)
                t.copy_(src)
        copied = torch.cuda.Event()
        copied.record(cur)
        with hub.lock:
            hub.done[me] = copied
        hub.barrier.wait()
        for ev in list(hub.done.values()):
            cur.wait_event(ev)
        hub.barrier.wait()


# ---------------------------------------------------------------------------

class HaloExchanger:
    """Two-phase periodic halo exchange of (u, v, w) for one rank."""

    def __init__(self, dec: Decomposition, device=None, transport=None, faceops=None):
        self.dec = dec
        d = dec.local_dims
        self.dims = d
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.device = dev
        self.faceops = faceops or (CudaFaceOps if dev.type == "cuda" else TorchFaceOps)
        self.transport = transport  # default (torch.distributed) created on first use
        xf, yf = (d.ny + 2) * d.nz, (d.nx + 2) * d.nz

        def buf(n):
            return torch.empty((3, n), dtype=torch.float64, device=dev)
        self.xbuf = {k: buf(xf) for k in ("send_m", "send_p", "recv_m", "recv_p")}
        self.ybuf = {k: buf(yf) for k in ("send_m", "send_p", "recv_m", "recv_p")}
        self._side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
        self._launch_cache: dict = {}

    # phase pieces (shared by the real transports and the loopback emulation)
    def _axis(self, axis):
        p = self.dec.px if axis == 0 else self.dec.py
        n = self.dims.nx if axis == 0 else self.dims.ny
        nb = self.dec.neighbours
        m, pl = (nb["xm"], nb["xp"]) if axis == 0 else (nb["ym"], nb["yp"])
        return p, n, m, pl, (self.xbuf if axis == 0 else self.ybuf)

    def pre(self, fields, axis, stream=None) -> list:
        p, n, m, pl, b = self._axis(axis)
        if p == 1:
            self.faceops.wrap_axis(fields, axis, stream)
            return []
        self.faceops.pack2(fields, b["send_m"], b["send_p"], axis, n, stream)
        # order matters when both neighbours are one rank (p == 2): the peer
        # receives my first message into its plus-side halo
        return [("send", b["send_m"], m, 0), ("send", b["send_p"], pl, 1),
                ("recv", b["recv_p"], pl, 0), ("recv", b["recv_m"], m, 1)]

    def post(self, fields, axis, stream=None) -> None:
        p, n, _, _, b = self._axis(axis)
        if p == 1:
            return
        self.faceops.unpack2(fields, b["recv_m"], b["recv_p"], axis, n, stream)

    def exchange(self, fields, stream=None) -> None:
        """Refresh the halos of `fields` (X phase, then Y phase)."""
        for axis in (0, 1):
            ops = self.pre(fields, axis, stream)
            if ops:
                if self.transport is None:
                    self.transport = DistTransport()
                if self.device.type == "cuda":
                    s = stream or torch.cuda.current_stream(self.device)
                    with torch.cuda.stream(s):
                        self.transport.run(ops)
                else:
                    self.transport.run(ops)
            self.post(fields, axis, stream)

    # -- compute with overlap ----------------------------------------------
    def boxes(self):
        """(interior box, rim boxes) in local 1-based interior coordinates."""
        nx, ny = self.dims.nx, self.dims.ny
        if nx < 3 or ny < 3:
            return None, [(1, nx + 1, 1, ny + 1)]
        inner = (2, nx, 2, ny)
        rims = [(1, 2, 1, ny + 1), (nx, nx + 1, 1, ny + 1), (2, nx, 1, 2), (2, nx, ny, ny + 1)]
        return inner, rims

    def _launches(self, fields, coeffs, out, opts, dt):
        """(interior, rim) BoundLaunch pair for these buffers, built once and
        reused: per-step Python cost is then two ctypes calls."""
        from . import _lib, device as dv
        key = (tuple(t.data_ptr() for t in tuple(fields) + tuple(out)), id(coeffs),
               None if opts is None else (opts.flags, opts.tile_j, opts.stages, opts.grid,
                                          opts.max_threads, opts.chunks), dt)
        cache = self._launch_cache
        hit = cache.get(key)
        if hit is not None and hit[2] is coeffs:
            return hit[0], hit[1]
        inner, rims = self.boxes()
        rim = dv.make_opts("simple")  # same arithmetic build (FMA or exact) as the interior
        rim.flags |= (opts.flags & _lib.FLAG_FMA) if opts is not None else 0
        if inner is None:
            li, lr = None, dv.BoundLaunch(fields, coeffs, out, box=rims[0], opts=rim, dt=dt)
        else:  # the four one-cell strips in one launch
            rim.flags |= _lib.FLAG_RIM
            li = dv.BoundLaunch(fields, coeffs, out, box=inner, opts=opts, dt=dt)
            lr = dv.BoundLaunch(fields, coeffs, out, box=(1, self.dims.nx + 1, 1, self.dims.ny + 1),
                                opts=rim, dt=dt)
        if len(cache) > 8:
            cache.clear()
        cache[key] = (li, lr, coeffs)
        return li, lr

    def run_overlapped(self, fields, coeffs, out, opts=None, stream=None, dt=None) -> None:
        """Exchange halos and then compute the one-cell rim on a side stream
        while the interior is computed on the main stream (the rim needs the
        halos, not the interior: it runs on the SMs the interior grid leaves
        free, or as the interior's CTAs retire); the main stream then joins."""
        li, lr = self._launches(fields, coeffs, out, opts, dt)
        main = stream or torch.cuda.current_stream(self.device)
        side = self._side
        side.wait_stream(main)
        self.exchange(fields, stream=side)
        lr(side)
        if li is not None:
            li(main)
        main.wait_stream(side)

    def advect_overlapped(self, fields, coeffs, out, opts=None, stream=None) -> None:
        self.run_overlapped(fields, coeffs, out, opts, stream)

    def step_overlapped(self, fields, coeffs, dt, out, opts=None, stream=None) -> None:
        self.run_overlapped(fields, coeffs, out, opts, stream, dt=float(dt))


def exchange_all_loopback(exchangers: list, fields_by_rank: list, stream=None) -> None:
    """Run one halo exchange for all emulated ranks of a decomposition in one
    process (the same pack / message / unpack code as the real transports)."""
    hub = LoopbackHub()
    for axis in (0, 1):
        ops = {ex.dec.rank: ex.pre(f, axis, stream) for ex, f in zip(exchangers, fields_by_rank)}
        hub.run_all(ops)
        for ex, f in zip(exchangers, fields_by_rank):
            ex.post(f, axis, stream)


# ---------------------------------------------------------------------------
# Fused stepping: K4 pushes boundary values straight into the neighbours'
# halos (pwadv_step_push_f64) — the exchange is part of the compute kernel,
# stores over NVLink to peer memory; one barrier per step.

_DIRS = ((-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (-1, 1), (1, -1), (1, 1))  # PWADV_NB_* order


def neighbour_ranks(dec: Decomposition) -> list[int]:
    cx, cy = dec.coords
    return [dec.rank_of(cx + dx, cy + dy) for dx, dy in _DIRS]


class LocalPeerRegistry:
    """Peer buffers of ranks living in this process (emulation on one GPU):
    rank -> ((u, v, w) of set 0, (u, v, w) of set 1) as device pointers."""

    def __init__(self):
        self.sets: dict = {}

    def publish(self, rank: int, sets) -> None:
        self.sets[rank] = tuple(tuple(t.data_ptr() for t in s) for s in sets)

    def pointers(self, rank: int, set_index: int):
        return self.sets[rank][set_index]


class IpcPeerRegistry:
    """Peer buffers across processes (one per GPU): each rank exports CUDA IPC
    handles of its two buffer sets, all ranks exchange them with
    torch.distributed, and each rank maps its neighbours' buffers (NVLink P2P)."""

    def __init__(self, dec: Decomposition, group=None):
        self.dec, self.group = dec, group
        self.sets: dict = {}
        self._opened: list = []
        self._bases: dict = {}

    def publish(self, rank: int, sets) -> None:
        import torch.distributed as dist
        from . import _lib
        try:  # a rank that cannot export still joins the gather (no rank left waiting)
            mine = [self.export(s) for s in sets]
        except _lib.PwadvError as exc:
            mine = f"rank {rank}: {exc}"
        everyone = [None] * self.dec.size
        dist.all_gather_object(everyone, mine, group=self.group)
        failed = [e for e in everyone if isinstance(e, str)]
        if failed:
            raise _lib.PwadvError(-1, "CUDA IPC export failed: " + "; ".join(failed))
        self.sets[rank] = tuple(tuple(t.data_ptr() for t in s) for s in sets)
        for r in set(neighbour_ranks(self.dec)) - {rank}:
            self.sets[r] = self.map_remote(everyone[r])

    def map_remote(self, exported):
        """Device pointers for another process's exported buffers: each
        distinct allocation handle is opened once (several tensors may live in
        one allocation), plus the tensor's offset inside it."""
        from . import _lib
        L = _lib.lib()
        ptrs = []
        for entry in exported:
            row = []
            for hb, off in entry:
                base = self._bases.get(hb)
                if base is None:
                    p = ctypes.c_void_p()
                    _lib.check(L.pwadv_ipc_open((ctypes.c_ubyte * 64)(*hb), 0, ctypes.byref(p)))
                    base = self._bases[hb] = p.value
                    self._opened.append(base)
                row.append(base + off)
            ptrs.append(tuple(row))
        return tuple(ptrs)

    @staticmethod
    def export(tensors):
        """(handle bytes, offset) of each tensor, for another process's map_remote."""
        from . import _lib
        L = _lib.lib()
        out = []
        for t in tensors:
            h = (ctypes.c_ubyte * 64)()
            off = ctypes.c_uint64()
            _lib.check(L.pwadv_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)))
            out.append((bytes(h), int(off.value)))
        return out

    def pointers(self, rank: int, set_index: int):
        return self.sets[rank][set_index]

    def close(self) -> None:
        from . import _lib
        for base in self._opened:
            _lib.lib().pwadv_ipc_close(ctypes.c_void_p(base), 0)
        self._opened = []
        self._bases = {}


def pull_mode(dims, opts, device_index: int) -> str:
    """How a block's halo cells are pulled: "fused" into K1 / K4's own bulk
    copies where the planner runs the block on the aligned X-march, else
    "gather" — the K2p gather kernel (pwadv_pull_halos_f64) followed by the
    planner's kernel (deep columns on K1c, odd nz, ...). The choice is a
    rank's own: both forms read only the neighbours' interiors and write only
    this block."""
    from . import device as dv
    try:
        plan = dv.describe_plan(dims, None, opts, device_index)
    except Exception:  # noqa: BLE001  (no plan report: let the fused launch decide)
        return "fused"
    return "fused" if plan["kernel"] == "xmarch" else "gather"


def peer_tables(dec: "Decomposition", registry, nsets: int) -> list:
    """One pwadv_peers table per published buffer set: the eight neighbours'
    (u, v, w) of that set and their interior extents."""
    from . import _lib
    tables = []
    nbr = neighbour_ranks(dec)
    for set_index in range(nsets):
        p = _lib.Peers()
        for d, r in enumerate(nbr):
            p.u[d], p.v[d], p.w[d] = registry.pointers(r, set_index)
            _, nxl, _, nyl = dec.block(r)
            p.nx[d], p.ny[d] = nxl, nyl
        tables.append(p)
    return tables


class PullEvaluator:
    """PW advection of one block with the halo exchange fused into K1 (pull):
    the kernel's bulk copies load the halo cells straight from the
    neighbours' current u, v, w — over NVLink for another GPU's block (CUDA IPC
    through `registry`), from this block's own buffers along an undivided axis
    — so an evaluation is one launch, with no pack/unpack, no separate
    exchange and nothing to overlap by hand. `barrier(stream)` (all ranks)
    orders each evaluation after every rank's previous writes to its fields;
    the first evaluation always passes one (all blocks published and filled)."""

    def __init__(self, dec: Decomposition, fields, coeffs, registry, barrier=None, *, opts=None):
        from . import device as dv
        self.dec = dec
        self.fields = tuple(fields)
        self.coeffs = dv._as_device_coeffs(coeffs, self.fields[0].device)
        self.registry = registry
        self.barrier = barrier
        self.opts = opts
        registry.publish(dec.rank, (self.fields,))
        self.peers = None
        self._launches: dict = {}
        # "fused": the halo cells loaded by K1's own bulk copies (the aligned
        # X-march); "gather": the K2p gather kernel fills this block's halos
        # from the neighbours, then the planner's kernel runs — for blocks the
        # planner gives to another kernel (deep columns on K1c, odd nz) or
        # that the fused pull does not take. The choice is this rank's own:
        # both forms read only the neighbours' interiors and write only here.
        self.mode = pull_mode(dec.local_dims, opts, self.fields[0].device.index or 0)

    def _build_peers(self):
        return peer_tables(self.dec, self.registry, 1)[0]

    def evaluate(self, out, stream=None, *, sync: bool = True, dt: float | None = None,
                 events=None) -> None:
        """su, sv, sw (or, with dt, the forward-Euler update) of this block into
        `out`; with `events` (a list) an event pair around the launch is appended."""
        from . import _lib, device as dv
        first = self.peers is None
        if (first or sync) and self.barrier is not None:
            self.barrier(stream)
        if first:
            self.peers = self._build_peers()
        key = (tuple(t.data_ptr() for t in out), dt)
        launch = self._launches.get(key)
        if launch is None:
            if len(self._launches) > 8:
                self._launches.clear()
            launch = self._launches[key] = dv.BoundLaunch(self.fields, self.coeffs, out,
                                                          opts=self.opts, dt=dt, pull=self.peers,
                                                          gather=self.mode == "gather")
        ev = dv.event_pair(events, stream)
        try:
            launch(stream)
        except _lib.PwadvError as exc:
            if self.mode != "fused" or exc.code != _lib.PWADV_E_ARG:
                raise
            # a block the fused pull does not take (the launch was refused
            # before anything ran): gather + the planner's kernel from now on
            self.mode = "gather"
            self._launches.clear()
            launch = self._launches[key] = dv.BoundLaunch(self.fields, self.coeffs, out,
                                                          opts=self.opts, dt=dt, pull=self.peers,
                                                          gather=True)
            launch(stream)
        dv.close_event_pair(ev, stream)


class NcclBarrier:
    """Stream-ordered barrier across ranks: a one-element all-reduce on the
    compute stream completes only after every rank's preceding kernels."""

    def __init__(self, device, group=None):
        self.flag = torch.zeros(1, device=device)
        self.group = group

    def __call__(self, stream=None) -> None:
        import torch.distributed as dist
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            dist.all_reduce(self.flag, group=self.group)


class FlagHandshake:
    """Neighbour-only, stream-ordered barrier for the fused steps
    (pwadv_signal_peers / pwadv_wait_peers, csrc/pwadv_sync.cu).

    Call k (after step k's launches on `stream`): write k into my slot of
    every neighbour's flag array (remote stores over NVLink into their
    IPC-mapped memory, fenced after the step's writes), then make the stream
    wait until every neighbour's slot in MY array holds >= k — i.e. until the
    neighbours have finished step k too. Ranks that are not neighbours never
    synchronise; no kernel and no NCCL call is involved, the GPU front end
    carries both the writes and the wait. `registry` maps the flag arrays
    (IpcPeerRegistry across processes, LocalPeerRegistry for ranks emulated
    as threads — every rank must construct its handshake before any calls
    one). Replaces NcclBarrier (one global all-reduce per step) on the fused
    paths."""

    def __init__(self, dec: Decomposition, registry, device=None, *, mode: str = "memop",
                 timeout_s: float = 10.0):
        """mode "memop": one batch of stream memory operations per call (the
        default; validated with 8 ranks emulated on one GPU and across
        processes). mode "kernel": a 32-thread kernel chained by programmatic
        dependent launch doing release stores / acquire polls, with a
        timeout that sets `err` instead of hanging (lower latency with 2-6
        emulated ranks; see tools/handshake_latency.cu)."""
        from . import _lib
        if mode not in ("memop", "kernel"):
            raise ValueError(f"unknown handshake mode {mode!r}")
        self.mode = mode
        self.timeout_ns = int(timeout_s * 1e9)
        self.dec = dec
        self.flags = torch.zeros(dec.size, dtype=torch.int64, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.flags.device)
        self.registry = registry
        registry.publish(dec.rank, ((self.flags,),))
        self.nbrs = sorted(set(neighbour_ranks(dec)) - {dec.rank})
        self.k = 0
        self._sig = self._wait = None
        dev = self.flags.device.index or 0
        m64, fl = ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.lib().pwadv_handshake_caps(dev, ctypes.byref(m64), ctypes.byref(fl)))
        self.caps = {"mem64": bool(m64.value), "flush_remote_writes": bool(fl.value)}
        if not m64.value:
            raise _lib.PwadvError(_lib.PWADV_E_CUDA, "64-bit stream memory operations unsupported")

    @staticmethod
    def slot_table(dec: Decomposition, my_flags: int, flags_of) -> tuple[list, list]:
        """(signal, wait) device addresses for rank dec.rank: my slot in each
        distinct neighbour's flag array (flags_of(rank) = its base address),
        and each neighbour's slot in mine; slot r = byte offset 8*r."""
        nbrs = sorted(set(neighbour_ranks(dec)) - {dec.rank})
        return ([flags_of(r) + 8 * dec.rank for r in nbrs], [my_flags + 8 * r for r in nbrs])

    def _build(self):
        sig, wait = self.slot_table(self.dec, self.flags.data_ptr(),
                                    lambda r: self.registry.pointers(r, 0)[0])
        n = len(sig)
        self._sig = (ctypes.c_void_p * max(n, 1))(*sig)
        self._wait = (ctypes.c_void_p * max(n, 1))(*wait)

    def __call__(self, stream=None) -> None:
        from . import _lib, device as dv
        if not self.nbrs:
            return
        if self._sig is None:
            self._build()
        self.k += 1
        h = dv._stream_handle(stream, self.flags.device)
        n = len(self.nbrs)
        if self.mode == "memop":
            _lib.check(_lib.lib().pwadv_handshake(self._sig, n, self._wait, n, self.k, h))
        else:
            _lib.check(_lib.lib().pwadv_handshake_kernel(self._sig, n, self._wait, n, self.k,
                                                         ctypes.c_void_p(self.err.data_ptr()),
                                                         self.timeout_ns, h))

    def timed_out(self) -> bool:
        """Kernel mode: some wait gave up after timeout_s (results are void)."""
        return bool(int(self.err.item()))

    def release(self) -> None:
        """Unblock this rank's own pending waits (after a failed probe): write
        the last awaited value into every slot of my flag array."""
        self.flags.fill_(self.k)


class ThreadStreamBarrier:
    """Barrier for ranks emulated as host threads on one GPU: every rank's
    stream waits on every other rank's event (kernels never wait on kernels)."""

    def __init__(self, nranks: int):
        import threading
        self.b = threading.Barrier(nranks)
        self.lock = threading.Lock()
        self.events: dict = {}

    def bind(self, rank: int):
        def barrier(stream=None):
            s = stream or torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(s)
            with self.lock:
                self.events[rank] = ev
            self.b.wait()
            for e in list(self.events.values()):
                s.wait_event(e)
            self.b.wait()
        return barrier


class PullStepper:
    """Forward-Euler steps of one block with the halo cells pulled from the
    neighbours' current buffers every step — for ANY block shape.

    Two buffer sets (ping-pong), both published; step n reads set n%2 — its
    own interior and, for the halo cells, the neighbours' interiors of the
    same set: inside K4's bulk copies where the block runs on the aligned
    X-march (mode "fused", pwadv_step_pull_f64), else through the K2p gather
    kernel followed by K4 with the planner's kernel (mode "gather": deep
    columns on K1c, odd nz) — and writes the interior of set (n+1)%2; then
    `barrier` (the neighbour flag handshake): before step n+1 every neighbour
    has finished step n, so its new interior is final (RAW) and it is done
    reading the set this rank overwrites next (WAR). No halo is ever pushed,
    packed or sent. PushStepper (peer stores from K4's epilogue) is the
    cheaper form where it applies; this one covers the other shapes."""

    def __init__(self, dec: Decomposition, fields, coeffs, dt: float, registry, barrier, *,
                 opts=None):
        from . import device as dv
        self.dec = dec
        self.dims = dec.local_dims
        u = fields[0]
        self.coeffs = dv._as_device_coeffs(coeffs, u.device)
        self.dt = float(dt)
        self.opts = opts
        self.sets = (tuple(fields), dv.alloc_fields(self.dims, u.device))
        self.cur = 0
        self.registry = registry
        self.barrier = barrier
        registry.publish(dec.rank, self.sets)
        self._peers = None
        self._launches: dict = {}
        self.steps_done = 0
        self.mode = pull_mode(self.dims, opts, u.device.index or 0)

    @property
    def fields(self):
        """The current fields (halos as the last gather / wrap left them; use
        refreshed_fields() for valid halos)."""
        return self.sets[self.cur]

    def _build_peers(self):
        return peer_tables(self.dec, self.registry, 2)

    def _launch(self, cur: int):
        from . import device as dv
        launch = self._launches.get(cur)
        if launch is None:
            launch = self._launches[cur] = dv.BoundLaunch(
                self.sets[cur], self.coeffs, self.sets[1 - cur], opts=self.opts, dt=self.dt,
                pull=self._peers[cur], gather=self.mode == "gather")
        return launch

    def step(self, n: int = 1, stream=None, events=None) -> None:
        from . import _lib, device as dv
        if self._peers is None:  # every rank published and filled its fields
            self.barrier(stream)
            self._peers = self._build_peers()
        for _ in range(n):
            ev = dv.event_pair(events, stream)
            try:
                self._launch(self.cur)(stream)
            except _lib.PwadvError as exc:
                if self.mode != "fused" or exc.code != _lib.PWADV_E_ARG:
                    raise
                self.mode = "gather"  # refused before anything ran: gather + the planner's kernel
                self._launches.clear()
                self._launch(self.cur)(stream)
            dv.close_event_pair(ev, stream)
            self.barrier(stream)
            self.cur = 1 - self.cur
            self.steps_done += 1

    def refreshed_fields(self, stream=None):
        """The current fields with their halos gathered from the neighbours (as
        an exchange / wrap_halos would leave them)."""
        from . import device as dv
        if self._peers is None:
            self.barrier(stream)
            self._peers = self._build_peers()
        dv.pull_halos(*self.sets[self.cur], self._peers[self.cur], stream=stream)
        return self.sets[self.cur]


class PushStepper:
    """Forward-Euler steps of one block with the halo exchange fused into K4.

    Two buffer sets (ping-pong); step n reads set n%2 (halos valid) and writes
    set (n+1)%2 — its interior and, through peer stores, the halos of every
    block that mirrors its boundary — then all ranks meet at `barrier`.
    `initial_exchange(fields)` fills the halos of the starting fields once.
    """

    def __init__(self, dec: Decomposition, fields, coeffs, dt: float, registry, barrier, *,
                 opts=None, initial_exchange=None):
        from . import device as dv
        self.dec = dec
        self.dims = dec.local_dims
        u = fields[0]
        self.coeffs = dv._as_device_coeffs(coeffs, u.device)
        self.dt = float(dt)
        self.opts = opts
        self.sets = (tuple(fields), dv.alloc_fields(self.dims, u.device))
        self.cur = 0
        self.registry = registry
        self.barrier = barrier
        registry.publish(dec.rank, self.sets)
        self._initial = initial_exchange
        self._peers = None
        self.steps_done = 0

    def _build_peers(self):
        return peer_tables(self.dec, self.registry, 2)

    def step(self, n: int = 1, stream=None, events=None) -> None:
        from . import _lib, device as dv
        if self._peers is None:  # all ranks have published by the first step
            if self._initial is not None:
                self._initial(self.sets[0])
            self.barrier(stream)
            self._peers = self._build_peers()
        L = _lib.lib()
        dc = self.coeffs
        d = self.dims
        for _ in range(n):
            src, dst = self.sets[self.cur], self.sets[1 - self.cur]
            h = dv._stream_handle(stream, src[0].device)
            ev = dv.event_pair(events, stream)
            _lib.check(L.pwadv_step_push_f64(
                dv._p(src[0]), dv._p(src[1]), dv._p(src[2]), dv._p(dst[0]), dv._p(dst[1]),
                dv._p(dst[2]), d.nx, d.ny, d.nz, dc.tcx, dc.tcy, dv._p(dc.tz[0]), dv._p(dc.tz[1]),
                self.dt, ctypes.byref(self._peers[1 - self.cur]), _lib.opts_ptr(self.opts), h))
            dv.close_event_pair(ev, stream)
            self.barrier(stream)
            self.cur = 1 - self.cur
            self.steps_done += 1

    @property
    def fields(self):
        return self.sets[self.cur]
