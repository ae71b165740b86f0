"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Checks the C restatement and the numpy restatement against the reference's
own goldens.json digests (reference pkg/tests/goldens.json, test_kernel.py:114-121,
test_grid.py:111-116) and against the fixtures made by importing the reference
(tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from oracle import oracle
from tests.golden_data import (case_inputs, load_cases, reference_goldens, small_arrays,
                               step_cases)

CASES = load_cases()


def test_reference_goldens_json_8x8x8():
    g = reference_goldens()
    u, v, w = oracle.fill_random(8, 8, 8, 42)
    assert [oracle.checksum(a) for a in (u, v, w)] == [g["fields"][k] for k in "uvw"]
    c = np.full(8, 0.25)
    su, sv, sw = oracle.advect(u, v, w, 0.25, 0.25, c, c)
    assert [oracle.checksum(a) for a in (su, sv, sw)] == [g["sources"][k] for k in ("su", "sv", "sw")]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_fixtures(case):
    u, v, w = case_inputs(case)
    assert [oracle.checksum(a) for a in (u, v, w)] == [case["inputs"][k] for k in "uvw"]
    outs = oracle.advect(u, v, w, case["tcx"], case["tcy"], case["tzc1"], case["tzc2"])
    assert [oracle.checksum(a) for a in outs] == [case["sources"][k] for k in ("su", "sv", "sw")]
    if case["arrays"]:
        arrs = small_arrays()
        for key, got in zip(("u", "v", "w", "su", "sv", "sw"), (u, v, w) + outs):
            ref = arrs[f"{case['name']}/{key}"]
            assert ref.tobytes() == got.tobytes(), key  # full padded arrays incl. halos, signed zeros
    # the independent numpy restatement agrees bit-for-bit too
    nouts = oracle.advect_numpy(u, v, w, case["tcx"], case["tcy"], case["tzc1"], case["tzc2"])
    assert oracle.compare(outs, nouts)["bitwise_equal"]


@pytest.mark.parametrize("engines", [2, 3, 8])
def test_oracle_engine_count_independence(engines):
    u, v, w = oracle.fill_random(13, 7, 9, 5, baseline=True)
    co = oracle.baseline_coefficients(5, 9)
    a = oracle.advect(u, v, w, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"], engines=1)
    b = oracle.advect(u, v, w, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"], engines=engines)
    assert oracle.compare(a, b)["bitwise_equal"]
    # the numpy restatement of run_schedule (bench.py's reference arm) too
    c = oracle.run_schedule_numpy(u, v, w, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"], engines)
    assert oracle.compare(a, c)["bitwise_equal"]


def test_lcg_skip_ahead_and_naive_recurrence():
    seq = oracle.lcg_doubles(2**63 + 5, 4097)
    state, naive = (2**63 + 5), []
    for _ in range(4097):
        state = (6364136223846793005 * state + 1442695040888963407) & (2**64 - 1)
        naive.append((state >> 11) * 2.0**-53)
    assert np.array_equal(seq, np.array(naive))
    assert np.array_equal(oracle.lcg_doubles(2**63 + 5, 100, start=3000), seq[3000:3100])


def test_baseline_coefficients_match_fixture():
    case = next(c for c in CASES if c["name"] == "baseline_64x64x64_s42")
    co = oracle.baseline_coefficients(42, 64)
    assert np.array_equal(co["tzc1"], case["tzc1"]) and np.array_equal(co["tzc2"], case["tzc2"])
    assert co["tcx"] == case["tcx"] == 0.005
    assert 1e-3 <= co["tzc1"].min() and co["tzc1"].max() < 5e-3


@pytest.mark.parametrize("sc", step_cases(), ids=lambda s: f"{s['nx']}x{s['ny']}x{s['nz']}x{s['steps']}")
def test_composed_time_stepping_oracle(sc):
    u, v, w = oracle.fill_random(sc["nx"], sc["ny"], sc["nz"], sc["seed"], baseline=True)
    co = oracle.baseline_coefficients(sc["seed"], sc["nz"])
    oracle.step(u, v, w, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"], sc["dt"], sc["steps"])
    assert [oracle.checksum(a) for a in (u, v, w)] == [sc["fields"][k] for k in "uvw"]


def test_compare_semantics_signed_zero_and_ulp():
    a = [np.zeros((3, 3, 2))]
    b = [np.zeros((3, 3, 2))]
    b[0][1, 1, 1] = -0.0
    r = oracle.compare(a, b)
    assert not r["bitwise_equal"] and r["max_ulp_diff"] == 1
    b[0][1, 1, 1] = np.nextafter(0.0, 1.0)
    assert oracle.compare(a, b)["max_ulp_diff"] == 1


def test_fill_box_is_the_periodic_padded_fill():
    """oracle.fill_box (LCG skip-ahead per column) == cells of the full fill,
    halo ring included, and periodic at any distance (boxes past the edge)."""
    g = (9, 7, 6)
    full = oracle.fill_random(*g, 42, baseline=True)
    box = oracle.fill_box(*g, 42, 0, 0, g[0] + 2, g[1] + 2, baseline=True)
    assert all(np.array_equal(a, b) for a, b in zip(full, box))
    box = oracle.fill_box(*g, 42, -12, 5, 30, 25, baseline=True)
    ii = (np.arange(-12, 18) - 1) % g[0] + 1
    jj = (np.arange(5, 30) - 1) % g[1] + 1
    assert all(np.array_equal(b, a[np.ix_(ii, jj)]) for a, b in zip(full, box))


@pytest.mark.parametrize("steps,i0,j0,ti,tj", [(1, 1, 1, 9, 7), (3, 2, 6, 4, 3), (5, 8, 7, 3, 2)])
def test_lightcone_tile_equals_periodic_stepping(steps, i0, j0, ti, tj):
    """The light-cone check's CPU side: stepping only the n-cell neighbourhood
    of a tile (open box, no wrap) reproduces the periodic full-grid steps."""
    g = (9, 7, 6)
    co = oracle.baseline_coefficients(42, g[2])
    u, v, w = oracle.fill_random(*g, 42, baseline=True)
    oracle.step(u, v, w, co["tcx"], co["tcy"], co["tzc1"], co["tzc2"], 0.1, steps)
    tile = oracle.lightcone_tile(*g, 42, co, 0.1, steps, i0, j0, ti, tj)
    ii = (np.arange(i0, i0 + ti) - 1) % g[0] + 1
    jj = (np.arange(j0, j0 + tj) - 1) % g[1] + 1
    for got, full in zip(tile, (u, v, w)):
        assert np.array_equal(got.view(np.int64), full[np.ix_(ii, jj)].view(np.int64))


def test_array_api_oracle_matches_reference_fixtures():
    """compute_block / su,sv,sw_formula restated in numpy (oracle) == the
    reference's own outputs (tests/golden/arrays.npz), bit for bit."""
    from tests.golden_data import compute_block_cases, formula_cases
    for c in compute_block_cases():
        got = oracle.compute_block_numpy(c["tcx"], c["tcy"], c["tzc1"], c["tzc2"], c["roles"])
        for g, w in zip(got, c["want"]):
            assert g.shape == w.shape and np.array_equal(g.view(np.int64), w.view(np.int64))
    for c in formula_cases():
        got = np.asarray(oracle.formula_numpy(c["which"], c["args"], c["top"]))
        assert np.array_equal(got.view(np.int64), c["want"].view(np.int64))


def test_grid_roles_views_reproduce_reference_compute_block():
    """grid_roles (kernel.py:165-172) are views of the padded fields; fed to
    compute_block they give the reference's fixture for columns 2..5."""
    import paper_2010_01545_b200 as pw
    from paper_2010_01545_b200.stencil import COMPUTE_ROLES, grid_roles
    from tests.golden_data import array_api_fixtures
    z = array_api_fixtures()
    d = pw.make_grid(7, 6, 5)
    u, v, w = oracle.fill_random(7, 6, 5, 99)
    f = pw.FieldSet(*(pw.Field3D(d, a) for a in (u, v, w)))
    roles = grid_roles(f, 2, 6)
    assert all(np.shares_memory(roles[r], {"u": u, "v": v, "w": w}[r[0]]) for r in COMPUTE_ROLES)
    assert roles[("v", 1, -1)].shape == (4, 6, 5)
    c = z["gr/coeffs"]
    got = oracle.compute_block_numpy(c[0], c[1], c[2:7], c[7:], [roles[r] for r in COMPUTE_ROLES])
    for g, name in zip(got, ("su", "sv", "sw")):
        assert np.array_equal(g.view(np.int64), z[f"gr/{name}"].view(np.int64))
