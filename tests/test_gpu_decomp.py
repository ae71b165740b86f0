"""GPU tests of the multi-GPU path, emulated on one B200.

Every emulated rank is a host thread with its own CUDA streams running the
production code (fill_local, HaloExchanger.exchange / advect_overlapped /
step_overlapped, libpwadv pack/unpack kernels); only the message transport is
the in-process ThreadHubTransport instead of NCCL (kernels never wait on one
another). Results must be bitwise identical to the single-domain evaluation.
"""

import ctypes
import threading

import numpy as np
import pytest
import torch

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import device
from paper_2010_01545_b200.decomp import Decomposition, HaloExchanger, ThreadHubTransport
from paper_2010_01545_b200.stepper import Stepper

pytestmark = pytest.mark.gpu


def run_ranks(n, fn):
    errs, out = [], [None] * n

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r)
            s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if errs:
        raise errs[0][1]
    return out


@pytest.mark.parametrize("shape", [(40, 36, 64), (24, 21, 8), (64, 48, 128)])
@pytest.mark.parametrize("px,py", [(1, 2), (2, 1), (2, 2), (2, 4), (3, 2)])
def test_emulated_decomposition_bitwise(shape, px, py):
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(7)
    co = pw.baseline_coefficients(7, gd.nz)
    gfields = device.fill(gd, spec)
    want = device.advect(*gfields, co)
    torch.cuda.synchronize()
    hub = ThreadHubTransport(px * py)

    def rank(r):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
        out = device.alloc_fields(dec.local_dims, "cuda")
        ex.advect_overlapped(fs, co, out)
        torch.cuda.current_stream().synchronize()
        halos_ok = all(torch.equal(f, dec.local_view(g)) for f, g in zip(fs, gfields))
        return dec, halos_ok, out

    res = run_ranks(px * py, rank)
    for dec, halos_ok, out in res:
        assert halos_ok, dec.rank
        xo, bx, yo, by = dec.block()
        for o, w in zip(out, want):
            a = o[1:-1, 1:-1].contiguous().view(torch.int64)
            b = w[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].contiguous().view(torch.int64)
            assert torch.equal(a, b), dec.rank


@pytest.mark.parametrize("px,py", [(2, 4), (1, 2)])
def test_emulated_decomposed_time_stepping(px, py):
    gd = pw.make_grid(48, 40, 16)
    spec = pw.GeneratorSpec.baseline(3)
    co = pw.baseline_coefficients(3, gd.nz)
    single = Stepper(device.fill(gd, spec), co, 0.1)
    single.step(5)
    want = single.fields
    torch.cuda.synchronize()
    hub = ThreadHubTransport(px * py)

    def rank(r):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
        st = Stepper(fs, co, 0.1, exchanger=ex)
        st.step(5)
        final = st.fields  # refreshes halos through the exchange
        torch.cuda.current_stream().synchronize()
        return dec, final

    for dec, final in run_ranks(px * py, rank):
        for f, w in zip(final, want):
            assert torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64)), dec.rank


@pytest.mark.parametrize("px,py,shape", [(2, 4, (48, 40, 16)), (1, 2, (30, 26, 64)), (2, 2, (25, 23, 6)),
                                         (1, 1, (20, 18, 64)), (3, 2, (36, 30, 128)),
                                         (2, 2, (25, 23, 7)), (2, 4, (48, 40, 33))])
def test_emulated_fused_push_stepping(px, py, shape):
    """K4 with the exchange fused in (peer stores + one barrier per step) ==
    single-domain stepping, bitwise, halos included."""
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PushStepper, ThreadStreamBarrier
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(11)
    co = pw.baseline_coefficients(11, gd.nz)
    single = Stepper(device.fill(gd, spec), co, 0.1)
    single.step(4)
    want = single.fields
    torch.cuda.synchronize()
    n = px * py
    hub = ThreadHubTransport(n)
    reg = LocalPeerRegistry()
    bar = ThreadStreamBarrier(n)

    def rank(r):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
        st = PushStepper(dec, fs, co, 0.1, reg, bar.bind(r), initial_exchange=ex.exchange)
        st.step(4)
        torch.cuda.current_stream().synchronize()
        return dec, st.fields

    for dec, final in run_ranks(n, rank):
        for f, w in zip(final, want):
            assert torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64)), dec.rank


@pytest.mark.parametrize("px,py,shape", [(2, 2, (25, 23, 64)), (1, 2, (30, 26, 128)), (2, 4, (48, 40, 33)),
                                         (2, 2, (16, 24, 300)), (3, 2, (36, 30, 7)), (1, 1, (9, 8, 63)),
                                         (2, 1, (10, 40, 1031))])
def test_emulated_pull_stepping(px, py, shape):
    """PullStepper (halo cells pulled every step: inside K4 on the aligned
    X-march, through the K2p gather kernel + the planner's K4 for odd nz and
    deep columns) == single-domain stepping, bitwise, halos included after
    refreshed_fields()."""
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PullStepper, ThreadStreamBarrier
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(13)
    co = pw.baseline_coefficients(13, gd.nz)
    single = Stepper(device.fill(gd, spec), co, 0.1)
    single.step(5)
    want = single.fields
    torch.cuda.synchronize()
    n = px * py
    reg = LocalPeerRegistry()
    bar = ThreadStreamBarrier(n)

    def rank(r):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        _poison_halos(fs)
        st = PullStepper(dec, fs, co, 0.1, reg, bar.bind(r))
        assert st.mode == ("fused" if gd.nz in (64, 128) else "gather")
        st.step(5)
        final = st.refreshed_fields()
        torch.cuda.current_stream().synchronize()
        return dec, final

    for dec, final in run_ranks(n, rank):
        for f, w in zip(final, want):
            assert torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64)), dec.rank


def _misaligned_fields(dims):
    """Zeroed padded fields that are 8- but not 16-byte aligned."""
    n = dims.padded_len
    out = []
    for _ in range(3):
        base = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
        out.append(base[1:].view(dims.padded_shape))
    assert all(t.data_ptr() % 16 == 8 for t in out)
    return tuple(out)


@pytest.mark.parametrize("px,py", [(1, 2), (2, 1), (2, 2)])
def test_emulated_fused_push_8byte_aligned_peers(px, py):
    """Blocks whose NEW buffers are only 8-byte aligned, next to blocks with
    16-byte-aligned buffers: the aligned blocks' boundary stores into those
    peers must take the 8-byte form (no misaligned 16-byte store), bitwise
    equal to single-domain stepping."""
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PushStepper, ThreadStreamBarrier
    gd = pw.make_grid(30, 26, 16)
    spec = pw.GeneratorSpec.baseline(5)
    co = pw.baseline_coefficients(5, gd.nz)
    single = Stepper(device.fill(gd, spec), co, 0.1)
    single.step(3)
    want = single.fields
    torch.cuda.synchronize()
    n = px * py
    hub = ThreadHubTransport(n)
    reg = LocalPeerRegistry()
    bar = ThreadStreamBarrier(n)

    def rank(r):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
        st = PushStepper(dec, fs, co, 0.1, reg, bar.bind(r), initial_exchange=ex.exchange)
        if r % 2 == 1:  # odd ranks: 8-byte-aligned new buffers
            st.sets = (st.sets[0], _misaligned_fields(dec.local_dims))
            reg.publish(r, st.sets)
        st.step(3)
        torch.cuda.current_stream().synchronize()
        return dec, st.fields

    for dec, final in run_ranks(n, rank):
        for f, w in zip(final, want):
            assert torch.equal(f.contiguous().view(torch.int64),
                               dec.local_view(w).contiguous().view(torch.int64)), dec.rank


@pytest.mark.parametrize("axis", [0, 1])
def test_cuda_face_ops_match_tensor_slicing(axis):
    """pwadv_pack/unpack_faces3_f64 (both faces of an axis in one launch) ==
    the tensor-slicing reference implementation, bitwise."""
    from paper_2010_01545_b200.decomp import CudaFaceOps, TorchFaceOps
    d = pw.make_grid(7, 5, 6)
    g = torch.Generator(device="cuda").manual_seed(3)
    a = [torch.randn(d.padded_shape, dtype=torch.float64, device="cuda", generator=g) for _ in range(3)]
    b = [t.clone() for t in a]
    n = d.nx if axis == 0 else d.ny
    face = (d.ny + 2) * d.nz if axis == 0 else (d.nx + 2) * d.nz
    bufs = [torch.empty((3, face), dtype=torch.float64, device="cuda") for _ in range(4)]
    CudaFaceOps.pack2(a, bufs[0], bufs[1], axis, n)
    TorchFaceOps.pack2(b, bufs[2], bufs[3], axis, n)
    torch.cuda.synchronize()
    assert torch.equal(bufs[0], bufs[2]) and torch.equal(bufs[1], bufs[3])
    src_lo, src_hi = bufs[0] * 2.0, bufs[1] - 1.0
    CudaFaceOps.unpack2(a, src_lo, src_hi, axis, n)
    TorchFaceOps.unpack2(b, src_lo, src_hi, axis, n)
    torch.cuda.synchronize()
    assert all(torch.equal(x, y) for x, y in zip(a, b))


def _ipc_reader(q_in, q_out):
    """Second process: map the first process's buffers and fill them with K5."""
    try:
        import paper_2010_01545_b200 as pw2
        from paper_2010_01545_b200 import _lib, decomp as dc
        torch.cuda.set_device(0)
        exported, dims = q_in.get(timeout=120)
        reg = dc.IpcPeerRegistry.__new__(dc.IpcPeerRegistry)
        reg._opened, reg._bases = [], {}
        (ptrs,) = reg.map_remote([exported])
        g = pw2.make_grid(*dims)
        _lib.check(_lib.lib().pwadv_fill_f64(*(ctypes.c_void_p(p) for p in ptrs), g.nx, g.ny, g.nz,
                                             1, 77, 0.0, 0.0, 0.0, None))
        torch.cuda.synchronize()
        n_bases = len(reg._bases)
        reg.close()
        q_out.put(("ok", n_bases))
    except Exception as e:  # pragma: no cover - reported to the parent
        q_out.put(("error", repr(e)))


def test_ipc_export_map_and_write_across_processes():
    """CUDA IPC as the fused step uses it, between two processes on one GPU
    (no kernel waits on another: the writer finishes before the owner reads):
    three fields carved out of ONE allocation (shared handle, nonzero
    offsets) are mapped by the other process, which writes them with K5; the
    owner then sees exactly the K5 fields."""
    import torch.multiprocessing as mp
    from paper_2010_01545_b200.decomp import IpcPeerRegistry
    d = pw.make_grid(20, 18, 16)
    n = d.padded_len
    block = torch.zeros(3 * n + 64, dtype=torch.float64, device="cuda")
    fields = [block[8 + m * n: 8 + (m + 1) * n].view(d.padded_shape) for m in range(3)]
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_reader, args=(q_in, q_out))
    p.start()
    q_in.put((IpcPeerRegistry.export(fields), (d.nx, d.ny, d.nz)))
    status, info = q_out.get(timeout=180)
    p.join(timeout=60)
    assert status == "ok", info
    assert info == 1  # one allocation, opened once
    want = device.fill(d, pw.GeneratorSpec.baseline(77))
    torch.cuda.synchronize()
    for f, w in zip(fields, want):
        assert torch.equal(f.view(torch.int64), w.view(torch.int64))


def _ipc_puller(q_in, q_out):
    """Second process: K1 with the halo pull whose eight neighbours are the
    first process's buffers, mapped by CUDA IPC (the bulk copies read them
    through the IPC mapping, as they read another GPU's buffers over NVLink)."""
    try:
        import paper_2010_01545_b200 as pw2
        from paper_2010_01545_b200 import _lib, decomp as dc, device as dv
        torch.cuda.set_device(0)
        exported, dims = q_in.get(timeout=120)
        reg = dc.IpcPeerRegistry.__new__(dc.IpcPeerRegistry)
        reg._opened, reg._bases = [], {}
        (ptrs,) = reg.map_remote([exported])
        g = pw2.make_grid(*dims)
        mine = dv.fill(g, pw2.GeneratorSpec.baseline(13))  # the same values as the owner's
        for f in mine:
            f[0].fill_(float("nan")); f[-1].fill_(float("nan"))  # noqa: E702
            f[:, 0].fill_(float("nan")); f[:, -1].fill_(float("nan"))  # noqa: E702
        peers = _lib.Peers()
        for d_ in range(8):
            peers.u[d_], peers.v[d_], peers.w[d_] = ptrs
            peers.nx[d_], peers.ny[d_] = g.nx, g.ny
        out = dv.advect_pull(*mine, pw2.baseline_coefficients(13, g.nz), peers)
        torch.cuda.synchronize()
        q_out.put(("ok", [o.cpu().numpy() for o in out]))
        reg.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        q_out.put(("error", repr(e)))


def test_ipc_pull_reads_mapped_peer_buffers():
    """The halo pull's bulk copies reading CUDA-IPC-mapped buffers of another
    process (on this one GPU; the owner is idle while they are read): the
    result equals K1 on valid halos, bit for bit."""
    import torch.multiprocessing as mp
    from paper_2010_01545_b200.decomp import IpcPeerRegistry
    d = pw.make_grid(40, 36, 64)
    n = d.padded_len
    block = torch.zeros(3 * n + 64, dtype=torch.float64, device="cuda")
    fields = [block[8 + m * n: 8 + (m + 1) * n].view(d.padded_shape) for m in range(3)]
    for f, w in zip(fields, device.fill(d, pw.GeneratorSpec.baseline(13))):
        f.copy_(w)
    want = device.advect(*fields, pw.baseline_coefficients(13, d.nz))
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_puller, args=(q_in, q_out))
    p.start()
    q_in.put((IpcPeerRegistry.export(fields), (d.nx, d.ny, d.nz)))
    status, got = q_out.get(timeout=180)
    p.join(timeout=60)
    assert status == "ok", got
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.int64), w.cpu().numpy().view(np.int64))


# --- K1 / K4 with the halo exchange fused in (pull) ---------------------------

def _poison_halos(fields):
    for f in fields:
        f[0].fill_(float("nan"))
        f[-1].fill_(float("nan"))
        f[:, 0].fill_(float("nan"))
        f[:, -1].fill_(float("nan"))


@pytest.mark.parametrize("shape", [(40, 36, 64), (7, 300, 64), (33, 5, 128), (1, 1, 2), (150, 13, 6),
                                   (40, 24, 64), (40, 30, 64), (3, 2000, 64)])
def test_pull_single_block_self_peers(shape):
    """An undivided domain pulling from itself: halos never read (NaN-poisoned),
    results bit-identical to wrap + K1 (and wrap + K4)."""
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(5)
    co = pw.baseline_coefficients(5, gd.nz)
    f = device.fill(gd, spec)
    want = device.advect(*f, co)
    want_step = device.step(*f, co, 0.1, device.alloc_fields(gd, "cuda"))
    g = [t.clone() for t in f]
    _poison_halos(g)
    peers = device.self_peers(g)
    got = device.advect_pull(*g, co, peers)
    nxt = device.alloc_fields(gd, "cuda")
    device.step_pull(*g, co, 0.1, nxt, peers)
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert torch.equal(a.view(torch.int64), b.view(torch.int64))
    for a, b in zip(nxt, want_step):
        assert torch.equal(a[1:-1, 1:-1].contiguous().view(torch.int64),
                           b[1:-1, 1:-1].contiguous().view(torch.int64))
    assert all(torch.equal(t[0], torch.zeros_like(t[0])) for t in nxt)  # new halos untouched


@pytest.mark.parametrize("shape", [(40, 36, 64), (64, 48, 128), (25, 23, 6),
                                   (24, 26, 63), (12, 16, 300), (9, 40, 1031)])
@pytest.mark.parametrize("px,py", [(1, 2), (2, 1), (2, 2), (2, 4), (3, 2)])
def test_emulated_pull_decomposition_bitwise(shape, px, py):
    """PullEvaluator on every block of a px x py decomposition (peer buffers on
    this GPU, halos NaN-poisoned): bit-identical to the undivided evaluation;
    and a pulled forward step too. Blocks on the aligned X-march pull inside
    the kernel; odd nz and deep columns (K1c) take the K2p gather kernel."""
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PullEvaluator
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(9)
    co = pw.baseline_coefficients(9, gd.nz)
    gfields = device.fill(gd, spec)
    want = device.advect(*gfields, co)
    want_step = device.step(*gfields, co, 0.1, device.alloc_fields(gd, "cuda"))
    # the undivided reference is itself the oracle's result (checker only)
    from oracle import oracle
    host = [f.cpu().numpy() for f in gfields]
    ow = oracle.advect(*host, co.tcx, co.tcy, co.tzc1, co.tzc2, engines=oracle.host_threads())
    assert oracle.compare([t.cpu().numpy() for t in want], ow)["bitwise_equal"]
    reg = LocalPeerRegistry()
    evs = []
    for r in range(px * py):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(spec)
        _poison_halos(fs)
        evs.append((dec, PullEvaluator(dec, fs, co, reg)))
    torch.cuda.synchronize()
    if gd.nz % 2:
        assert all(ev.mode == "gather" for _, ev in evs)
    elif gd.nz in (64, 128):
        assert all(ev.mode == "fused" for _, ev in evs)
    for dec, ev in evs:  # every block published before any evaluation
        out = device.alloc_fields(dec.local_dims, "cuda")
        ev.evaluate(out)
        nxt = device.alloc_fields(dec.local_dims, "cuda")
        ev.evaluate(nxt, dt=0.1)
        torch.cuda.synchronize()
        xo, bx, yo, by = dec.block()
        for o, w in zip(out, want):
            assert torch.equal(o[1:-1, 1:-1].contiguous().view(torch.int64),
                               w[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].contiguous().view(torch.int64)), dec.rank
        for o, w in zip(nxt, want_step):
            assert torch.equal(o[1:-1, 1:-1].contiguous().view(torch.int64),
                               w[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].contiguous().view(torch.int64)), dec.rank


@pytest.mark.parametrize("shape", [(8, 8, 7), (13, 6, 64), (5, 9, 130), (1, 1, 2), (1, 7, 5)])
def test_pull_halos_gather_kernel(shape):
    """K2p (pwadv_pull_halos_f64): with the block as its own eight neighbours
    it is the periodic wrap (reference wrap_halos, grid.py:203-208), every halo
    cell incl. the corners; over a 2x3 decomposition every block's halos equal
    the wrapped global field's."""
    gd = pw.make_grid(*shape)
    f = device.fill(gd, pw.GeneratorSpec.random(5))
    want = [t.clone() for t in f]
    device.wrap_halos(*want)
    _poison_halos(f)
    device.pull_halos(*f, device.self_peers(f))
    torch.cuda.synchronize()
    for a, b in zip(f, want):
        assert torch.equal(a.view(torch.int64), b.view(torch.int64))
    px, py = 2, 3
    if gd.nx < px or gd.ny < py:
        return
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PullEvaluator
    reg = LocalPeerRegistry()
    co = pw.baseline_coefficients(5, gd.nz)
    evs = []
    for r in range(px * py):
        dec = Decomposition(gd, px, py, r)
        fs = dec.fill_local(pw.GeneratorSpec.random(5))
        _poison_halos(fs)
        evs.append((dec, fs, PullEvaluator(dec, fs, co, reg)))
    for dec, fs, ev in evs:
        device.pull_halos(*fs, ev._build_peers())
    torch.cuda.synchronize()
    for dec, fs, _ in evs:
        for a, w in zip(fs, want):
            assert torch.equal(a.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64)), dec.rank


def test_pull_rejects_shapes_off_the_aligned_xmarch():
    from paper_2010_01545_b200 import _lib
    gd = pw.make_grid(8, 8, 7)  # odd nz
    f = device.fill(gd, pw.GeneratorSpec.baseline(1))
    co = pw.baseline_coefficients(1, 7)
    with pytest.raises(_lib.PwadvError):
        device.advect_pull(*f, co, device.self_peers(f))
    gd = pw.make_grid(8, 8, 8)
    f = device.fill(gd, pw.GeneratorSpec.baseline(1))
    p = device.self_peers(f)
    p.ny[0] = 9  # an x neighbour with another y extent
    with pytest.raises(_lib.PwadvError):
        device.advect_pull(*f, pw.baseline_coefficients(1, 8), p)


@pytest.mark.parametrize("kw", [dict(grid=3, chunks=4), dict(grid=5, chunks=2, tile_j=5), dict(grid=7),
                                dict(grid=4), dict(grid=4, tile_j=7)])
def test_pull_multi_unit_plans(kw):
    """Halo pull with several work units per CTA (forced small grids / chunks):
    y-face and interior units interleaved in one CTA's plane sequence; with
    whole-X rounds plus a chunked tail (grid=4) the strips are rotated so the
    y-face strips fall in the tail."""
    gd = pw.make_grid(50, 70, 64)
    spec = pw.GeneratorSpec.baseline(3)
    co = pw.baseline_coefficients(3, gd.nz)
    f = device.fill(gd, spec)
    want = device.advect(*f, co)
    g = [t.clone() for t in f]
    _poison_halos(g)
    got = device.advect_pull(*g, co, device.self_peers(g), opts=device.make_opts("xmarch", **kw))
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert torch.equal(a.view(torch.int64), b.view(torch.int64)), kw


# --- neighbour flag handshake (pwadv_signal_peers / pwadv_wait_peers) --------

@pytest.mark.parametrize("px,py,shape,mode", [(1, 2, (30, 26, 64), "memop"), (2, 2, (25, 23, 6), "memop"),
                                              (2, 4, (48, 40, 16), "memop"), (3, 2, (36, 30, 128), "memop"),
                                              (1, 2, (30, 26, 64), "kernel"), (2, 2, (25, 23, 6), "kernel")])
def test_emulated_fused_push_with_flag_handshake(px, py, shape, mode):
    """PushStepper ordered by the neighbour-only flag handshake (stream-ordered
    flag writes/waits, no host barrier, no kernel waiting on a kernel) ==
    single-domain stepping, bitwise, halos included."""
    from paper_2010_01545_b200.decomp import FlagHandshake, LocalPeerRegistry, PushStepper
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(11)
    co = pw.baseline_coefficients(11, gd.nz)
    single = Stepper(device.fill(gd, spec), co, 0.1)
    single.step(6)
    want = single.fields
    torch.cuda.synchronize()
    n = px * py
    hub = ThreadHubTransport(n)
    reg, flag_reg = LocalPeerRegistry(), LocalPeerRegistry()
    decs = [Decomposition(gd, px, py, r) for r in range(n)]
    hs = [FlagHandshake(d, flag_reg, device="cuda", mode=mode, timeout_s=20.0)
          for d in decs]  # all published up front

    def rank(r):
        dec = decs[r]
        fs = dec.fill_local(spec)
        ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
        st = PushStepper(dec, fs, co, 0.1, reg, hs[r], initial_exchange=ex.exchange)
        st.step(6)
        torch.cuda.current_stream().synchronize()
        return dec, st.fields

    for dec, final in run_ranks(n, rank):
        for f, w in zip(final, want):
            assert torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64)), dec.rank
    assert all(h.k == 7 for h in hs)  # the initial handshake + one per step
    assert not any(h.timed_out() for h in hs)


@pytest.mark.parametrize("px,py,shape", [(1, 2, (40, 36, 64)), (2, 4, (64, 48, 64))])
def test_emulated_pull_with_flag_handshake(px, py, shape):
    """PullEvaluator (K1 pulling its halos from the neighbours' fields)
    ordered by the flag handshake, evaluations interleaved with in-place
    updates of the fields (so a missing order would read stale or torn
    halos) == the single-domain result, bitwise, every round."""
    import threading
    from paper_2010_01545_b200.decomp import FlagHandshake, LocalPeerRegistry, PullEvaluator
    gd = pw.make_grid(*shape)
    spec = pw.GeneratorSpec.baseline(4)
    co = pw.baseline_coefficients(4, gd.nz)
    rounds = 4
    g = device.fill(gd, spec)
    wants = []
    for k in range(rounds):
        for f in g:  # in-place update of the fields between evaluations
            f.mul_(1.0 + 0.25 * (k > 0))
        device.wrap_halos(*g)
        wants.append([o.clone() for o in device.advect(*g, co)])
    torch.cuda.synchronize()
    n = px * py
    reg, flag_reg = LocalPeerRegistry(), LocalPeerRegistry()
    decs = [Decomposition(gd, px, py, r) for r in range(n)]
    hs = [FlagHandshake(d, flag_reg, device="cuda") for d in decs]
    ready = threading.Barrier(n)

    def rank(r):
        dec = decs[r]
        fs = dec.fill_local(spec)
        ev = PullEvaluator(dec, fs, co, reg, hs[r])
        ready.wait()  # every rank published its fields
        got = []
        for k in range(rounds):
            if k:
                hs[r]()  # neighbours done reading round k-1 before the update
                for f in fs:
                    f.mul_(1.25)
            out = device.alloc_fields(dec.local_dims, "cuda")
            ev.evaluate(out)  # handshake: neighbours' updates done, then K1 pulls
            got.append(out)
        torch.cuda.current_stream().synchronize()
        return dec, got

    for dec, got in run_ranks(n, rank):
        for k in range(rounds):
            for o, w in zip(got[k], wants[k]):
                wl = dec.local_view(w).contiguous()
                assert torch.equal(o[1:-1, 1:-1].contiguous().view(torch.int64),
                                   wl[1:-1, 1:-1].contiguous().view(torch.int64)), (dec.rank, k)


def _handshake_proc(rank, port, q):
    """Rank of a 2-process (1x2) run on one GPU: ping-pong mailboxes in the
    OTHER process's memory (CUDA IPC), ordered only by the flag handshake."""
    try:
        import torch.distributed as dist
        import paper_2010_01545_b200 as pw2
        from paper_2010_01545_b200 import _lib, decomp as dc, device as dv
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
        g = pw2.make_grid(8, 6, 4)
        dec = dc.Decomposition(pw2.make_grid(8, 12, 4), 1, 2, rank)
        hs = dc.FlagHandshake(dec, dc.IpcPeerRegistry(dec), device="cuda")
        boxes = (dv.alloc_fields(g, "cuda"), dv.alloc_fields(g, "cuda"))  # my mailboxes (ping-pong)
        mreg = dc.IpcPeerRegistry(dec)
        mreg.publish(rank, boxes)
        other = 1 - rank
        seen = []
        rounds = 40
        for k in range(1, rounds + 1):
            # my "step": read my mailbox written by the other rank in step k-1,
            # write the other rank's mailbox k % 2 (K5 fill with seed k)
            if k > 1:
                seen.append([t.clone() for t in boxes[(k - 1) % 2]])
            ptrs = mreg.pointers(other, k % 2)
            _lib.check(_lib.lib().pwadv_fill_f64(*(ctypes.c_void_p(p) for p in ptrs), g.nx, g.ny, g.nz,
                                                 0, 1000 * (rank + 1) + k, 0.0, 0.0, 0.0,
                                                 dv._stream_handle(None, torch.device("cuda", 0))))
            hs()
        torch.cuda.synchronize()
        bad = 0
        for k, got in zip(range(1, rounds), seen):
            want = dv.fill(g, pw2.GeneratorSpec.random(1000 * (other + 1) + k))
            bad += sum(0 if torch.equal(a.view(torch.int64), b.view(torch.int64)) else 1
                       for a, b in zip(got, want))
        torch.cuda.synchronize()
        dist.barrier()
        mreg.close()
        hs.registry.close()
        q.put((rank, "ok", bad, hs.k, int(hs.flags[other].item())))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e), 0, 0))


def test_flag_handshake_across_processes_ipc():
    """The handshake as bench.py runs it (IpcPeerRegistry over torch.distributed,
    remote flag writes into CUDA-IPC-mapped memory), two processes on one GPU:
    40 ping-pong rounds of cross-process mailbox writes, each read only after
    the handshake — every mailbox holds exactly the other rank's round-k fill."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_handshake_proc, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, status, bad, k, peer_flag in res:
        assert status == "ok", (rank, bad)
        assert bad == 0 and k == 40 and peer_flag == 40, (rank, bad, k, peer_flag)
