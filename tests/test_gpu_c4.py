"""BASELINE config 4 at full size: 4096x4096x128, 100 forward-Euler steps.

Parity at 2.1e9 points uses the light-cone check of SURVEY.md §8f1: after n
steps a tile depends only on its n-cell neighbourhood, so the C oracle steps
that neighbourhood alone (oracle.lightcone_tile: box fill by LCG skip-ahead,
open-box stepping whose valid region shrinks one cell per side per step) and
the GPU's tile must match it bit for bit. Tiles are placed across the
periodic domain edge, across the 2x4 block boundaries and in the interior.
Step 1 is checked on full-length bands. Both the single-GPU stepper (K2 wrap
+ K4, CUDA graph) and the 2x4 decomposition with the exchange fused into K4
(8 emulated ranks on one GPU, peer stores + a barrier per step) run the
whole 103 GB problem.
"""

import threading

import numpy as np
import pytest
import torch

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import device
from paper_2010_01545_b200.stepper import Stepper
from oracle import oracle

pytestmark = pytest.mark.gpu

NX = NY = 4096
NZ = 128
SEED = 42
DT = 0.1
STEPS = 100
TILE = 16
# (i0, j0): 1-based first interior row/column of each 16x16 tile (periodic)
TILES = [(2041, 1017),   # corner of four 2x4 blocks
         (4089, 4089),   # global corner: neighbourhood wraps in x and y
         (1000, 3000),   # block interior
         (1, 2041)]      # x edge, across a y block boundary
BANDS = [(4093, 1, 8, NY),   # step 1: 8 full rows across the x wrap
         (1, 2045, NX, 8)]   # step 1: 8 full columns across the y block boundary


def _need_memory():
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    need = 2 * 3 * (NX + 2) * (NY + 2) * NZ * 8 + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB of free device memory, {free / 1e9:.0f} free")


def _coeffs():
    return pw.baseline_coefficients(SEED, NZ)


@pytest.fixture(scope="module")
def cone_tiles():
    co = oracle.baseline_coefficients(SEED, NZ)
    eng = oracle.host_threads()
    return {t: oracle.lightcone_tile(NX, NY, NZ, SEED, co, DT, STEPS, t[0], t[1], TILE, TILE, eng)
            for t in TILES}


def _idx(first, count, n):
    return ((np.arange(first, first + count) - 1) % n) + 1


def _tile_single(fields, i0, j0, ti, tj):
    ii = torch.as_tensor(_idx(i0, ti, NX), device=fields[0].device)
    jj = torch.as_tensor(_idx(j0, tj, NY), device=fields[0].device)
    return [f.index_select(0, ii).index_select(1, jj).cpu().numpy() for f in fields]


def _assert_tile(got, want, what):
    for name, g, w in zip("uvw", got, want):
        bad = np.argwhere(g.view(np.int64) != w.view(np.int64))
        assert bad.size == 0, f"{what} {name}: {len(bad)} cells differ, first at {bad[0]}"


def _whole_grid_sane(fields):
    for f in fields:
        for x in range(1, f.shape[0] - 1, 512):   # bounded temporaries
            assert bool(torch.isfinite(f[x:min(x + 512, f.shape[0] - 1), 1:-1]).all())
    assert not bool(fields[2][1:-1, 1:-1, 0].ne(0).any())


def test_c4_single_gpu_lightcone(cone_tiles):
    _need_memory()
    dims = pw.make_grid(NX, NY, NZ)
    st = Stepper(device.fill(dims, pw.GeneratorSpec.baseline(SEED)), _coeffs(), DT)
    st.step(1)
    torch.cuda.synchronize()
    co = oracle.baseline_coefficients(SEED, NZ)
    for i0, j0, ti, tj in BANDS:
        want = oracle.lightcone_tile(NX, NY, NZ, SEED, co, DT, 1, i0, j0, ti, tj,
                                     oracle.host_threads())
        _assert_tile(_tile_single(st.a, i0, j0, ti, tj), want, f"step-1 band {(i0, j0)}")
    st.capture(2)          # steps 2-3 (warm-up outside the graph), then replay
    st.step(STEPS - 4)
    st.step(1)             # one eager step: mixed graph / eager sequence
    assert st.steps_done == STEPS
    torch.cuda.synchronize()
    for (i0, j0), want in cone_tiles.items():
        _assert_tile(_tile_single(st.a, i0, j0, TILE, TILE), want, f"tile {(i0, j0)}")
    _whole_grid_sane(st.a)


def test_c4_2x4_fused_exchange_lightcone(cone_tiles):
    from paper_2010_01545_b200.decomp import (Decomposition, HaloExchanger, LocalPeerRegistry,
                                              PushStepper, ThreadHubTransport,
                                              ThreadStreamBarrier)
    _need_memory()
    gd = pw.make_grid(NX, NY, NZ)
    px, py = 2, 4
    n = px * py
    hub, reg, bar = ThreadHubTransport(n), LocalPeerRegistry(), ThreadStreamBarrier(n)
    co = _coeffs()
    spec = pw.GeneratorSpec.baseline(SEED)
    out, errs = [None] * n, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                dec = Decomposition(gd, px, py, r)
                fs = dec.fill_local(spec)
                ex = HaloExchanger(dec, device="cuda", transport=hub.bind(r))
                st = PushStepper(dec, fs, co, DT, reg, bar.bind(r), initial_exchange=ex.exchange)
                st.step(STEPS)
            s.synchronize()
            out[r] = (dec, st.fields)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0][1]
    torch.cuda.synchronize()

    for (i0, j0), want in cone_tiles.items():
        got = [np.empty((TILE, TILE, NZ)) for _ in range(3)]
        ii, jj = _idx(i0, TILE, NX), _idx(j0, TILE, NY)
        for dec, fs in out:
            xo, nxl, yo, nyl = dec.block()
            a = np.nonzero((ii > xo) & (ii <= xo + nxl))[0]
            b = np.nonzero((jj > yo) & (jj <= yo + nyl))[0]
            if a.size == 0 or b.size == 0:
                continue
            li = torch.as_tensor(ii[a] - xo, device=fs[0].device)
            lj = torch.as_tensor(jj[b] - yo, device=fs[0].device)
            for g, f in zip(got, fs):
                g[np.ix_(a, b)] = f.index_select(0, li).index_select(1, lj).cpu().numpy()
        _assert_tile(got, want, f"2x4 tile {(i0, j0)}")
    for _, fs in out:
        _whole_grid_sane(fs)
