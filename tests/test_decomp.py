"""Host-side tests of the x-y decomposition and halo exchange.

CPU only: the exchange runs on CPU tensors (TorchFaceOps) through the same
pre/post + transport code as on GPUs — an in-process loopback hub for many
decompositions, and real multi-process torch.distributed (gloo, world sizes
2 and 4, rendezvous on 127.0.0.1). After the exchange every block must equal
its view of the globally wrapped field (reference wrap_halos semantics,
grid.py:203-208), and the oracle evaluated block by block must reassemble
the single-domain result bit for bit (the reference's engine-count
independence, test_schedules.py:72-77, extended to x-y blocks).
"""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200.decomp import (Decomposition, DistTransport, HaloExchanger,
                                          TorchFaceOps, exchange_all_loopback, split_extent)
from oracle import oracle


def test_split_extent_and_blocks_cover():
    assert split_extent(10, 3) == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(ValueError):
        split_extent(3, 4)
    g = pw.make_grid(13, 11, 4)
    for px, py in ((1, 1), (1, 2), (2, 2), (2, 4), (3, 3), (13, 1)):
        seen = np.zeros((13, 11), dtype=int)
        for r in range(px * py):
            xo, nx, yo, ny = Decomposition(g, px, py, r).block()
            seen[xo:xo + nx, yo:yo + ny] += 1
        assert np.all(seen == 1)


def test_neighbours_are_periodic():
    d = Decomposition(pw.make_grid(8, 8, 2), 2, 4, 0)
    assert d.coords == (0, 0)
    assert d.neighbours == {"xm": 4, "xp": 4, "ym": 3, "yp": 1}
    d5 = d.for_rank(5)
    assert d5.coords == (1, 1) and d5.neighbours == {"xm": 1, "xp": 1, "ym": 4, "yp": 6}
    with pytest.raises(ValueError):
        Decomposition(pw.make_grid(8, 8, 2), 2, 4, 8)


def _global_case(nx, ny, nz, seed=5):
    u, v, w = oracle.fill_random(nx, ny, nz, seed, baseline=True)
    co = oracle.baseline_coefficients(seed, nz)
    return (u, v, w), co


def _stale_blocks(dec, glob):
    """Each rank's block with its halos poisoned (the exchange must fill them)."""
    blocks = []
    for r in range(dec.size):
        d = dec.for_rank(r)
        fs = [torch.from_numpy(np.ascontiguousarray(d.local_view(g))).clone() for g in glob]
        for f in fs:
            f[0] = f[-1] = f[:, 0] = f[:, -1] = np.nan
        blocks.append(fs)
    return blocks


@pytest.mark.parametrize("px,py", [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (3, 3), (4, 2)])
def test_loopback_exchange_and_blockwise_oracle(px, py):
    nx, ny, nz = 17, 13, 6
    glob, co = _global_case(nx, ny, nz)
    dec = Decomposition(pw.make_grid(nx, ny, nz), px, py, 0)
    blocks = _stale_blocks(dec, glob)
    ex = [HaloExchanger(dec.for_rank(r), device="cpu", faceops=TorchFaceOps) for r in range(dec.size)]
    exchange_all_loopback(ex, blocks)
    want = oracle.advect(*glob, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
    for r, fs in enumerate(blocks):
        d = dec.for_rank(r)
        for f, g in zip(fs, glob):
            assert np.array_equal(f.numpy(), d.local_view(g)), (r, "halo")
        got = oracle.advect(*(f.numpy() for f in fs), co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
        xo, bx, yo, by = d.block()
        for gb, wn in zip(got, want):
            assert gb[1:-1, 1:-1].tobytes() == wn[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].tobytes()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, px, py, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nx, ny, nz = 12, 10, 5
        glob, co = _global_case(nx, ny, nz, seed=9)
        dec = Decomposition(pw.make_grid(nx, ny, nz), px, py, rank)
        fs = _stale_blocks(dec, glob)[rank]
        ex = HaloExchanger(dec, device="cpu", transport=DistTransport(), faceops=TorchFaceOps)
        ex.exchange(fs)
        ok = all(np.array_equal(f.numpy(), dec.local_view(g)) for f, g in zip(fs, glob))
        got = oracle.advect(*(f.numpy() for f in fs), co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
        want = oracle.advect(*glob, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
        xo, bx, yo, by = dec.block()
        ok &= all(gb[1:-1, 1:-1].tobytes() == wn[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].tobytes()
                  for gb, wn in zip(got, want))
        # a second exchange on updated data (buffers are reused)
        for f in fs:
            f.mul_(2.0)
        ex.exchange(fs)
        ok &= all(np.array_equal(f.numpy(), 2.0 * dec.local_view(g)) for f, g in zip(fs, glob))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("px,py", [(1, 2), (2, 1), (2, 2)])
def test_gloo_multiprocess_exchange(px, py):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = px * py
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, px, py, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in results) == list(range(world))
    for r, ok, err in results:
        assert ok, (r, err)


@pytest.mark.parametrize("px,py,shape", [(2, 4, (21, 30, 4)), (1, 2, (9, 11, 4)), (3, 1, (10, 5, 4))])
def test_pull_evaluator_peer_table(px, py, shape):
    """PullEvaluator's peer table (host side, no launch): entry d names the
    neighbour in direction d (PWADV_NB_* order) — the buffers that rank
    published and its block extents; an undivided axis names the block itself."""
    from paper_2010_01545_b200 import _lib
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, PullEvaluator
    gd = pw.make_grid(*shape)
    co = pw.AdvectionCoefficients(0.005, 0.005, np.full(gd.nz, 2e-3), np.full(gd.nz, 3e-3))
    reg = LocalPeerRegistry()
    evs = []
    for r in range(px * py):
        dec = Decomposition(gd, px, py, r)
        d = dec.local_dims
        fs = tuple(torch.zeros(d.padded_shape, dtype=torch.float64) for _ in range(3))
        evs.append((dec, fs, PullEvaluator(dec, fs, co, reg)))
    ptrs = {dec.rank: tuple(t.data_ptr() for t in fs) for dec, fs, _ in evs}
    dirs = {_lib.NB_XM: (-1, 0), _lib.NB_XP: (1, 0), _lib.NB_YM: (0, -1), _lib.NB_YP: (0, 1),
            _lib.NB_XMYM: (-1, -1), _lib.NB_XMYP: (-1, 1), _lib.NB_XPYM: (1, -1), _lib.NB_XPYP: (1, 1)}
    for dec, _, ev in evs:
        p = ev._build_peers()
        cx, cy = dec.coords
        for d, (dx, dy) in dirs.items():
            r = dec.rank_of(cx + dx, cy + dy)
            assert (p.u[d], p.v[d], p.w[d]) == ptrs[r], (dec.rank, d)
            _, nxl, _, nyl = dec.block(r)
            assert (p.nx[d], p.ny[d]) == (nxl, nyl)
        # x neighbours share this block's y extent, y neighbours its x extent
        assert p.ny[_lib.NB_XM] == p.ny[_lib.NB_XP] == dec.local_dims.ny
        assert p.nx[_lib.NB_YM] == p.nx[_lib.NB_YP] == dec.local_dims.nx
        # the corner neighbours sit on the x neighbours' rows and the y neighbours'
        # columns (what pwadv_pull_halos_f64 requires of a peer table)
        for c, xn, yn in ((_lib.NB_XMYM, _lib.NB_XM, _lib.NB_YM), (_lib.NB_XMYP, _lib.NB_XM, _lib.NB_YP),
                          (_lib.NB_XPYM, _lib.NB_XP, _lib.NB_YM), (_lib.NB_XPYP, _lib.NB_XP, _lib.NB_YP)):
            assert p.nx[c] == p.nx[xn] and p.ny[c] == p.ny[yn], (dec.rank, c)
        if px == 1:
            assert (p.u[_lib.NB_XM], p.u[_lib.NB_XP]) == (ptrs[dec.rank][0],) * 2


def test_peer_tables_one_per_buffer_set():
    """peer_tables (PushStepper / PullStepper): table s names the neighbours'
    set-s buffers; extents are the same in both."""
    from paper_2010_01545_b200 import _lib
    from paper_2010_01545_b200.decomp import LocalPeerRegistry, peer_tables
    gd = pw.make_grid(7, 9, 4)
    px, py = 2, 3
    reg = LocalPeerRegistry()
    sets = {}
    for r in range(px * py):
        d = Decomposition(gd, px, py, r).local_dims
        sets[r] = tuple(tuple(torch.zeros(d.padded_shape, dtype=torch.float64) for _ in range(3))
                        for _ in range(2))
        reg.publish(r, sets[r])
    for r in range(px * py):
        dec = Decomposition(gd, px, py, r)
        t0, t1 = peer_tables(dec, reg, 2)
        cx, cy = dec.coords
        nb = dec.rank_of(cx + 1, cy)  # NB_XP
        assert t0.u[_lib.NB_XP] == sets[nb][0][0].data_ptr()
        assert t1.w[_lib.NB_XP] == sets[nb][1][2].data_ptr()
        assert list(t0.nx) == list(t1.nx) and list(t0.ny) == list(t1.ny)


@pytest.mark.parametrize("px,py", [(1, 2), (2, 2), (2, 4), (3, 2), (1, 1)])
def test_flag_handshake_slot_table_pairs_up(px, py):
    """Neighbour handshake wiring (host side): every signal rank r sends lands
    in exactly the slot its neighbour waits on for r, neighbours are the
    distinct 8-neighbourhood ranks (an undivided axis: none / itself), and
    nobody signals or waits on a non-neighbour."""
    from paper_2010_01545_b200.decomp import FlagHandshake, neighbour_ranks
    g = pw.make_grid(6 * px, 6 * py, 4)
    base = {r: 0x10000 * (r + 1) for r in range(px * py)}  # fake device addresses
    sig, wait = {}, {}
    for r in range(px * py):
        dec = Decomposition(g, px, py, r)
        sig[r], wait[r] = FlagHandshake.slot_table(dec, base[r], base.__getitem__)
        nb = set(neighbour_ranks(dec)) - {r}
        assert len(sig[r]) == len(wait[r]) == len(nb)
        assert sorted((a - base[r]) // 8 for a in wait[r]) == sorted(nb)
    for r in range(px * py):
        for a in sig[r]:
            owner = next(q for q in base if base[q] <= a < base[q] + 8 * px * py)
            assert (a - base[owner]) // 8 == r and a in wait[owner]


def _agree_worker(rank, port, oks, q):
    try:
        import torch.distributed as dist
        import bench
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=len(oks))
        q.put((rank, bench.agree_all(oks[rank], torch.device("cpu"))))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("oks", [(True, True), (True, False), (False, False)])
def test_bench_ranks_agree_on_the_fused_path(oks):
    """bench.agree_all: every rank takes the fused path only if every rank can
    (a rank-local fallback would mix collectives and hang)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_agree_worker, args=(r, port, oks, q)) for r in range(len(oks))]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {r: all(oks) for r in range(len(oks))}, res
