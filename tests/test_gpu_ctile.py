"""GPU parity of the column-tile X-march (K1c, k_advect_ctile) against the C
oracle, bitwise: every slab height (KT 32 / 64 / 128) over even nz (3-D
tensor maps) and odd nz (column-pair rows, both y parities),
slabs that cut columns unevenly, partial y-strips, thin X, sub-boxes, the
fused step K4 and the DFMA build (normwise 1e-12), the deep-column default
plan (nz > 768, formerly K1m) and the shapes that must stay off it."""

import numpy as np
import pytest
import torch

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import device
from oracle import oracle

pytestmark = pytest.mark.gpu


def _inputs(nx, ny, nz, seed):
    u, v, w = oracle.fill_random(nx, ny, nz, seed, baseline=True)
    co = oracle.baseline_coefficients(seed, nz)
    return (u, v, w), (co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])


def _dev(arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


def _bits_equal(got, want, what):
    for g, w_ in zip(got, want):
        g = g.cpu().numpy() if isinstance(g, torch.Tensor) else g
        assert np.array_equal(g.view(np.int64), w_.view(np.int64)), what


SHAPES = [(9, 7, 64), (13, 30, 63), (20, 25, 96), (7, 26, 97), (5, 12, 130), (6, 9, 2),
          (4, 6, 3), (3, 40, 255), (17, 4, 256), (2, 3, 777), (2, 2, 1030), (3, 14, 1025),
          (1, 24, 64), (11, 1, 65), (4, 12, 31)]


@pytest.mark.parametrize("tile_j", [6, 8, 12, 16, 24])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_ctile_bitwise_against_oracle(shape, tile_j):
    nx, ny, nz = shape
    ins, args = _inputs(nx, ny, nz, 5 + nz)
    dims = pw.make_grid(nx, ny, nz)
    want = oracle.advect(*ins, *args)
    opts = device.make_opts("xmarch_ct", tile_j=tile_j)
    plan = device.describe_plan(dims, opts=opts)
    if nz % 2 and tile_j in (8, 16, 24):  # odd nz needs one column parity per warp: KT 64 / 128
        assert plan["kernel"] != "xmarch_ct", plan
    else:
        assert plan["kernel"] == "xmarch_ct", plan
        assert plan["threads_per_column"] * 2 == 768 // tile_j
    fin = _dev(ins)
    co = pw.AdvectionCoefficients(*args)
    out = device.advect(*fin, co, opts=opts)
    _bits_equal(out, want, (shape, tile_j))


@pytest.mark.parametrize("shape", [(12, 30, 62), (12, 29, 63), (10, 13, 128), (6, 25, 300), (3, 5, 1030), (4, 7, 1031)],
                         ids=lambda s: "x".join(map(str, s)))
def test_ctile_box_step_and_fma(shape):
    nx, ny, nz = shape
    ins, args = _inputs(nx, ny, nz, 77)
    dims = pw.make_grid(nx, ny, nz)
    want = oracle.advect(*ins, *args)
    fin = _dev(ins)
    co = pw.AdvectionCoefficients(*args)
    opts = device.make_opts("xmarch_ct")
    assert device.describe_plan(dims, opts=opts)["kernel"] == "xmarch_ct"
    # a sub-box: only its interior is written
    box = (1 + nx // 3, nx + 1, 2, max(3, ny))
    out = device.alloc_fields(dims, "cuda")
    device.advect(*fin, co, out, box=box, opts=opts)
    x0, x1, y0, y1 = box
    for o, w_ in zip(out, want):
        o = o.cpu().numpy()
        assert np.array_equal(o[x0:x1, y0:y1].view(np.int64), w_[x0:x1, y0:y1].view(np.int64))
        rest = o.copy()
        rest[x0:x1, y0:y1] = 0.0
        assert not rest.any()
    # the fused step K4: f + dt*s (mul then add)
    nxt = device.alloc_fields(dims, "cuda")
    device.step(*fin, co, 0.1, nxt, opts=opts)
    for g, f, s in zip(nxt, ins, want):
        assert np.array_equal(g.cpu().numpy()[1:-1, 1:-1].view(np.int64),
                              (f + 0.1 * s)[1:-1, 1:-1].view(np.int64))
    # DFMA build within the normwise tolerance of BASELINE's north_star
    out_f = device.advect(*fin, co, opts=device.make_opts("xmarch_ct_fma"))
    r = oracle.compare([o.cpu().numpy() for o in out_f], want)
    assert r["normwise_rel"] <= 1e-12, r


def test_ctile_is_the_default_for_deep_columns_and_matches_k1m():
    nx, ny, nz = 6, 20, 1500
    ins, args = _inputs(nx, ny, nz, 3)
    dims = pw.make_grid(nx, ny, nz)
    assert device.describe_plan(dims)["kernel"] == "xmarch_ct"
    want = oracle.advect(*ins, *args)
    fin = _dev(ins)
    co = pw.AdvectionCoefficients(*args)
    _bits_equal(device.advect(*fin, co), want, "default")
    _bits_equal(device.advect(*fin, co, opts=device.make_opts("march")), want, "K1m")


@pytest.mark.parametrize("nz", [40, 41])
def test_ctile_declines_8_byte_aligned_fields(nz):
    # 8-byte-aligned fields: the forced form is declined, results stay exact
    nx, ny = 6, 8
    ins, args = _inputs(nx, ny, nz, 9)
    want = oracle.advect(*ins, *args)
    n = (nx + 2) * (ny + 2) * nz
    bufs = [torch.empty(n + 1, dtype=torch.float64, device="cuda") for _ in range(6)]
    shp = pw.make_grid(nx, ny, nz).padded_shape
    fin = [b[1:].view(shp) for b in bufs[:3]]
    fout = [b[1:].view(shp) for b in bufs[3:]]
    for t, a in zip(fin, ins):
        t.copy_(torch.from_numpy(a))
    for t in fout:
        t.zero_()
    device.advect(*fin, pw.AdvectionCoefficients(*args), fout, opts=device.make_opts("xmarch_ct"))
    _bits_equal(fout, want, "8-byte aligned")


@pytest.mark.parametrize("shape", [(512, 64, 1030), (96, 96, 514), (300, 77, 63), (64, 96, 777)], ids=lambda s: "x".join(map(str, s)))
def test_ctile_medium_grids_every_plane(shape):
    """Multi-round plans (full rounds of whole (strip, slab) units plus X
    chunks) at sizes where every CTA runs several units, every plane
    against the streamed oracle."""
    nx, ny, nz = shape
    dims = pw.make_grid(nx, ny, nz)
    fields = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = pw.baseline_coefficients(42, nz)
    out = device.advect(*fields, co, opts=device.make_opts("xmarch_ct"))
    torch.cuda.synchronize()
    r = oracle.compare_streamed(fields, out, co.tcx, co.tcy, co.tzc1, co.tzc2)
    assert r["bitwise_equal"] and r["planes_checked"] == nx, r


@pytest.mark.parametrize("nz", [16, 24, 40, 56, 72, 88, 100, 104, 110])
def test_compile_time_depths_every_plane(nz):
    """Depths with their own compile-time tile layout (the whole-column
    X-march's NZC depths, K1c's 128-level slab at 110): the default plan's K1
    and K4 on a multi-round grid, every plane against the oracle."""
    nx, ny = 300, 200
    dims = pw.make_grid(nx, ny, nz)
    fields = device.fill(dims, pw.GeneratorSpec.baseline(8))
    co = pw.baseline_coefficients(8, nz)
    plan = device.describe_plan(dims)
    assert plan["kernel"] == ("xmarch_ct" if nz == 110 else "xmarch"), plan
    out = device.advect(*fields, co)
    torch.cuda.synchronize()
    r = oracle.compare_streamed(fields, out, co.tcx, co.tcy, co.tzc1, co.tzc2)
    assert r["bitwise_equal"] and r["planes_checked"] == nx, r
    nxt = device.alloc_fields(dims, "cuda")
    device.step(*fields, co, 0.1, nxt)
    torch.cuda.synchronize()
    r = oracle.compare_streamed(fields, nxt, co.tcx, co.tcy, co.tzc1, co.tzc2, dt=0.1)
    assert r["bitwise_equal"], r


@pytest.mark.parametrize("shape", [(1024, 512, 256), (512, 514, 255), (256, 256, 2048)],
                         ids=lambda s: "x".join(map(str, s)))
def test_ctile_large_grids_every_plane(shape):
    """K1c at full size (134-136M points; even slabs, odd nz pair rows,
    2048-level columns in 16 slabs): the default plan, every plane of su, sv,
    sw against the streamed C oracle, bitwise."""
    nx, ny, nz = shape
    dims = pw.make_grid(nx, ny, nz)
    assert device.describe_plan(dims)["kernel"] == "xmarch_ct"
    fields = device.fill(dims, pw.GeneratorSpec.baseline(21))
    co = pw.baseline_coefficients(21, nz)
    out = device.advect(*fields, co)
    torch.cuda.synchronize()
    r = oracle.compare_streamed(fields, out, co.tcx, co.tcy, co.tzc1, co.tzc2, slab=32)
    assert r["bitwise_equal"] and r["planes_checked"] == nx, r
