"""CPU-only tests: the C-ABI library loads and exports the declared symbols,
argument validation happens before any compute, and the host-side mirror of the
reference interface (layout, coefficients, engines, comparator) behaves like
the reference's own unit tests (pkg/tests/test_grid.py, test_kernel.py,
test_schedules.py). No CUDA device is needed.
"""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import _lib
from paper_2010_01545_b200.engines import plan_traffic
from tests.golden_data import GOLDEN

ROOT = Path(__file__).resolve().parent.parent


def header_functions(name="pwadv.h"):
    text = (ROOT / "include" / name).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pwadv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes binding"
    assert set(_lib.SIGNATURES) == set(names)
    assert L.pwadv_abi_version() == _lib.ABI_VERSION


def test_traffic_library_exports_every_header_symbol():
    """include/pwadv_traffic.h against libpwadv_traffic.so (the optional CUPTI
    counters library). Its exports are read with nm (it links libcuda, absent
    without a driver); where it loads, the value count and the no-session
    error are checked too, without touching a GPU."""
    import subprocess
    from paper_2010_01545_b200 import traffic
    if not traffic._LIB.exists():
        pytest.skip("libpwadv_traffic.so not built")
    names = header_functions("pwadv_traffic.h")
    assert names == ["pwadv_traffic_begin", "pwadv_traffic_end", "pwadv_traffic_last_error",
                     "pwadv_traffic_max_ranges", "pwadv_traffic_num_values"]
    nm = subprocess.run(["nm", "-D", "--defined-only", str(traffic._LIB)], capture_output=True,
                        text=True, check=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    assert set(names) <= exported, set(names) - exported
    nvals = int(re.search(r"PWADV_TRAFFIC_NVALUES\s+(\d+)",
                          (ROOT / "include" / "pwadv_traffic.h").read_text()).group(1))
    assert nvals == 5
    try:
        L = traffic.lib()
    except OSError:
        return
    assert L.pwadv_traffic_num_values() == nvals
    assert L.pwadv_traffic_max_ranges() >= 1
    vals, n = (ctypes.c_double * nvals)(), ctypes.c_int(0)
    assert L.pwadv_traffic_end(vals, ctypes.byref(n)) == -1
    assert b"no active traffic session" in L.pwadv_traffic_last_error()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_validation_before_compute():
    L = _lib.lib()
    p = ctypes.c_void_p(256)
    rc = L.pwadv_advect_f64(p, p, p, p, p, p, 0, 4, 4, 0.1, 0.1, p, p, None, None)
    assert rc == _lib.PWADV_E_DIMS
    assert b"horizontal extents" in L.pwadv_last_error()
    rc = L.pwadv_advect_f64(p, p, p, p, p, p, 4, 4, 1, 0.1, 0.1, p, p, None, None)
    assert rc == _lib.PWADV_E_DIMS and b"nz must be >= 2" in L.pwadv_last_error()
    rc = L.pwadv_advect_f64(p, None, p, p, p, p, 4, 4, 4, 0.1, 0.1, p, p, None, None)
    assert rc == _lib.PWADV_E_NULL
    rc = L.pwadv_advect_f64(p, ctypes.c_void_p(257), p, p, p, p, 4, 4, 4, 0.1, 0.1, p, p, None, None)
    assert rc == _lib.PWADV_E_ALIGN
    rc = L.pwadv_advect_box_f64(p, p, p, p, p, p, 4, 4, 4, 0.1, 0.1, p, p, 0, 3, 1, 5, None, None)
    assert rc == _lib.PWADV_E_RANGE
    rc = L.pwadv_step_box_f64(p, p, p, p, p, p, 4, 4, 4, 0.1, 0.1, p, p, 0.1, 1, 5, 1, 5, None, None)
    assert rc == _lib.PWADV_E_ARG  # in-place step refused (needs ping-pong buffers)
    rc = L.pwadv_fill_f64(p, p, p, 4, 4, 4, 7, 0, 0.0, 0.0, 0.0, None)
    assert rc == _lib.PWADV_E_ARG
    with pytest.raises(_lib.PwadvError):
        _lib.check(_lib.PWADV_E_DIMS)


def test_fused_exchange_entry_points_validate_their_peer_tables():
    """pwadv_advect_pull_f64 / pwadv_step_pull_f64 / pwadv_step_push_f64
    reject bad peer tables before touching the device (no GPU needed)."""
    L = _lib.lib()
    p, q = ctypes.c_void_p(256), ctypes.c_void_p(4096)

    def table(ptr=256, nx=4, ny=4):
        t = _lib.Peers()
        for d in range(8):
            t.u[d] = t.v[d] = t.w[d] = ptr
            t.nx[d], t.ny[d] = nx, ny
        return t

    head = (p, p, p, q, q, q, 4, 4, 4, 0.1, 0.1, p, p)
    assert L.pwadv_advect_pull_f64(*head, None, None, None) == _lib.PWADV_E_NULL
    assert L.pwadv_advect_pull_f64(*head, ctypes.byref(table(264)), None, None) == _lib.PWADV_E_ALIGN
    assert b"16-byte" in L.pwadv_last_error()  # the pull's bulk copies want 16 bytes
    bad = table()
    bad.ny[_lib.NB_XM] = 5  # an x neighbour with another y extent
    assert L.pwadv_advect_pull_f64(*head, ctypes.byref(bad), None, None) == _lib.PWADV_E_RANGE
    bad = table()
    bad.u[_lib.NB_YP] = None
    assert L.pwadv_advect_pull_f64(*head, ctypes.byref(bad), None, None) == _lib.PWADV_E_NULL
    assert L.pwadv_advect_pull_f64(*head, ctypes.byref(table(nx=0)), None, None) == _lib.PWADV_E_DIMS
    same = (p, p, p, p, p, p, 4, 4, 4, 0.1, 0.1, p, p, 0.1)
    assert L.pwadv_step_pull_f64(*same, ctypes.byref(table()), None, None) == _lib.PWADV_E_ARG
    assert L.pwadv_step_push_f64(*same, ctypes.byref(table(264)), None, None) == _lib.PWADV_E_ARG
    assert L.pwadv_step_push_f64(*same, None, None, None) == _lib.PWADV_E_NULL


# --- layout (reference test_grid.py) ------------------------------------------

def test_make_grid_and_rejects():
    assert pw.make_grid(512, 512, 64).cells == 16_777_216
    assert pw.make_grid(1, 1, 2).cells == 2
    for bad in [(0, 4, 4), (4, 0, 4), (4, 4, 1), (4, 4, 0), (-1, 4, 4)]:
        with pytest.raises(pw.GridError):
            pw.make_grid(*bad)
    assert issubclass(pw.GridError, ValueError)


def test_linear_index_bijection():
    dims = pw.make_grid(3, 2, 4)
    offs = {pw.linear_index(i, j, k, dims) for i in range(dims.nx + 2)
            for j in range(dims.ny + 2) for k in range(1, dims.nz + 1)}
    assert offs == set(range(dims.padded_len))
    arr = np.arange(dims.padded_len, dtype=np.float64).reshape(dims.padded_shape)
    assert arr[2, 1, 3] == pw.linear_index(2, 1, 4, dims)


def test_field_validation_and_io(tmp_path):
    dims = pw.make_grid(2, 2, 2)
    with pytest.raises(pw.GridError):
        pw.Field3D(dims, np.zeros((2, 2, 2)))
    with pytest.raises(pw.GridError):
        pw.Field3D(dims, np.zeros(dims.padded_shape, dtype=np.float32))
    d5 = pw.make_grid(5, 4, 3)
    f = pw.Field3D(d5, np.random.default_rng(1).random(d5.padded_shape))
    pw.write_field(f, tmp_path / "u.field")
    back = pw.read_field(tmp_path / "u.field")
    assert back.dims == d5 and np.array_equal(back.data, f.data)
    assert (tmp_path / "u.field").stat().st_size == 24 + d5.padded_len * 8
    (tmp_path / "t.field").write_bytes((tmp_path / "u.field").read_bytes()[:-8])
    with pytest.raises(pw.GridError):
        pw.read_field(tmp_path / "t.field")


def test_host_wrap_and_checksum_semantics():
    from oracle import oracle
    u, _, _ = oracle.fill_random(5, 3, 4, 3)
    a = u.copy()
    a[0] = a[-1] = 0.0
    a[:, 0] = a[:, -1] = 0.0
    pw.wrap_halos(a)
    assert np.array_equal(a, u)
    dims = pw.make_grid(5, 3, 4)
    f = pw.Field3D(dims, u.copy())
    g = f.copy()
    g.data[0, 0, 0] = 99.0  # halo-only change keeps the digest
    assert pw.checksum(f) == pw.checksum(g) == oracle.checksum(u)
    g.data[2, 2, 1] = np.nextafter(g.data[2, 2, 1], 1.0)
    assert pw.checksum(g) != pw.checksum(f)


def test_generator_spec():
    with pytest.raises(pw.GridError):
        pw.GeneratorSpec("bogus")
    assert pw.GeneratorSpec.random(3).seed == 3
    assert pw.GeneratorSpec.baseline(5).mode == "baseline"


# --- coefficients / census (reference test_kernel.py) -------------------------

def test_coefficients_validation():
    with pytest.raises(ValueError):
        pw.AdvectionCoefficients(0.1, 0.1, np.ones(3), np.ones(4))
    with pytest.raises(ValueError):
        pw.AdvectionCoefficients(0.1, 0.1, np.ones((2, 2)), np.ones((2, 2)))
    with pytest.raises(ValueError):
        pw.AdvectionCoefficients(0.1, 0.1, np.array([1.0, np.nan]), np.ones(2))
    c = pw.default_coefficients(7)
    assert c.nz == 7 and c.tcx == 0.25 and np.all(c.tzc2 == 0.25)


def test_census_and_roles_match_reference():
    ref = json.loads((GOLDEN / "cases.json").read_text())
    assert [list(r) for r in pw.COMPUTE_ROLES] == ref["compute_roles"]
    assert pw.operation_census(False) == ref["operation_census"]["mid"]
    assert pw.operation_census(True) == ref["operation_census"]["top"]
    assert pw.reads_per_point(False) == ref["operation_census"]["reads_mid"] == 54
    assert pw.reads_per_point(True) == ref["operation_census"]["reads_top"] == 45
    assert pw.FlopProfile().total_per_cell == 53
    assert pw.flops(pw.make_grid(1, 1, 2)) == 106


# --- engines / comparator (reference test_schedules.py) -----------------------

def test_partition_domain():
    assert pw.partition_domain(pw.make_grid(512, 4, 2), 1) == [pw.Slab(1, 513)]
    assert [s.width for s in pw.partition_domain(pw.make_grid(512, 4, 2), 4)] == [128] * 4
    assert [s.width for s in pw.partition_domain(pw.make_grid(10, 4, 2), 3)] == [4, 3, 3]
    for nx in (1, 2, 7, 13):
        for e in range(1, nx + 1):
            slabs = pw.partition_domain(pw.make_grid(nx, 2, 2), e)
            assert [i for s in slabs for i in range(s.x_begin, s.x_end)] == list(range(1, nx + 1))
    for e in (0, 5, -1):
        with pytest.raises(ValueError):
            pw.partition_domain(pw.make_grid(4, 4, 4), e)


def test_schedule_spec_validation():
    with pytest.raises(ValueError):
        pw.ScheduleSpec("nonsense")
    with pytest.raises(ValueError):
        pw.ScheduleSpec("xmarch", y_batch=0)
    d = pw.make_grid(4, 4, 4)
    with pytest.raises(ValueError):
        pw.ScheduleSpec("y_batched", y_batch=5).validate(d)
    with pytest.raises(ValueError):
        pw.ScheduleSpec("reference", engines=5).validate(d)
    pw.ScheduleSpec("x_reordered", y_batch=4, engines=4).validate(d)
    assert pw.ScheduleSpec("x_reordered").kernel_variant == "xmarch"
    assert pw.ScheduleSpec("simple_fma").kernel_variant == "simple_fma"


def _srcset(arrs):
    d = pw.make_grid(arrs[0].shape[0] - 2, arrs[0].shape[1] - 2, arrs[0].shape[2])
    return pw.SourceSet(*(pw.Field3D(d, a) for a in arrs))


def test_compare_outputs_semantics():
    rng = np.random.default_rng(0)
    base = [rng.random((4, 4, 3)) for _ in range(3)]
    a, b = _srcset([x.copy() for x in base]), _srcset([x.copy() for x in base])
    assert pw.compare_outputs(a, b) == pw.OutputComparison(True, 0.0, 0)
    b.sv.data[2, 2, 1] = np.nextafter(b.sv.data[2, 2, 1], np.inf)
    r = pw.compare_outputs(a, b)
    assert not r.bitwise_equal and r.max_ulp_diff == 1
    c = _srcset([np.zeros((4, 4, 3)) for _ in range(3)])
    d = _srcset([np.zeros((4, 4, 3)) for _ in range(3)])
    d.su.data[1, 1, 1] = -0.0
    r = pw.compare_outputs(c, d)
    assert not r.bitwise_equal and r.max_ulp_diff == 1
    with pytest.raises(ValueError):
        pw.compare_outputs(c, _srcset([np.zeros((5, 4, 3)) for _ in range(3)]))


def test_plan_traffic_accounting():
    dims = pw.make_grid(512, 512, 64)
    plan = {"kernel": "xmarch", "tile_j": 12, "grid": 148, "strips": 43, "smem_bytes": 200000,
            "chunks": 10}
    tr = plan_traffic(dims, (1, 513, 1, 513), plan)
    interior_in = 3 * 512 * 512 * 64
    # staged input traffic is within (1 + halo columns + boundary planes) of the interior
    assert interior_in < tr.external_reads < 1.25 * interior_in
    assert tr.external_writes == interior_in
    simple = plan_traffic(dims, (1, 513, 1, 513), {"kernel": "simple"})
    assert simple.external_reads == 27 * 512 * 512 * 63
    # two-phase schedule (whole strips for the full rounds, the rest chunked):
    # 2048^2 -> 148 whole strips + 23 strips in 6 chunks; closed form
    d3 = pw.make_grid(2048, 2048, 64)
    p3 = {"kernel": "xmarch", "tile_j": 12, "strips": 171, "long_strips": 148, "chunks": 6,
          "smem_bytes": 0}
    t3 = plan_traffic(d3, (1, 2049, 1, 2049), p3)
    widths = [12] * 170 + [2048 - 170 * 12]
    want = 2050 * sum(w + 2 for w in widths[:148])
    want += sum((2048 * (c + 1) // 6 - 2048 * c // 6 + 2) * (w + 2) for w in widths[148:] for c in range(6))
    assert t3.external_reads == 3 * 64 * want


# --- the reference's traffic counters (schedules.py:117-191) in closed form ---

def _stock_schedules():
    ref = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
    if not (ref / "pwadvect" / "schedules.py").exists():
        pytest.skip("stock reference not installed in baseline/_ref")
    import importlib.util
    import sys as _sys
    # import the stock package under its own name in a private module table
    saved = {k: v for k, v in _sys.modules.items() if k == "pwadvect" or k.startswith("pwadvect.")}
    for k in saved:
        del _sys.modules[k]
    _sys.path.insert(0, str(ref))
    try:
        import pwadvect.grid as g
        import pwadvect.kernel as k
        import pwadvect.schedules as s
        assert Path(s.__file__).resolve().parent == (ref / "pwadvect").resolve()
        return g, k, s
    finally:
        _sys.path.remove(str(ref))
        for key in [k for k in _sys.modules if k == "pwadvect" or k.startswith("pwadvect.")]:
            del _sys.modules[key]
        _sys.modules.update(saved)
        del importlib


def test_reference_traffic_matches_stock_counters():
    """reference_traffic() equals what the stock reference counts while it
    moves the data, for every variant, random dims, y_batch and engines."""
    from paper_2010_01545_b200.engines import ScheduleSpec, partition_domain, reference_traffic
    g, k, s = _stock_schedules()
    rng = np.random.default_rng(5)
    for _ in range(40):
        nx, ny, nz = int(rng.integers(1, 9)), int(rng.integers(1, 8)), int(rng.integers(2, 7))
        dims = g.make_grid(nx, ny, nz)
        fields = g.fill_fields(dims, g.GeneratorSpec.random(int(rng.integers(0, 99))))
        co = k.default_coefficients(nz)
        yb = int(rng.integers(1, ny + 1))
        eng = int(rng.integers(1, nx + 1))
        for variant in s.VARIANTS:
            _, want, _ = s.run_schedule(fields, co, s.ScheduleSpec(variant, yb, eng))
            spec = ScheduleSpec(variant, yb, eng)
            got = reference_traffic(pw.make_grid(nx, ny, nz), spec,
                                    partition_domain(pw.make_grid(nx, ny, nz), eng))
            assert (got.external_reads, got.external_writes, got.local_reads, got.local_writes,
                    got.scratch_bytes_peak) == (want.external_reads, want.external_writes,
                                                want.local_reads, want.local_writes,
                                                want.scratch_bytes_peak), (variant, nx, ny, nz, yb, eng)


def test_schedule_spec_and_variants_mirror_reference():
    from paper_2010_01545_b200.engines import (ALL_VARIANTS, REFERENCE_VARIANTS, VARIANTS,
                                               XSHIFT_ROLES, ScheduleSpec)
    assert ScheduleSpec().variant == "reference"
    assert VARIANTS == REFERENCE_VARIANTS == ("reference", "column_buffered", "y_batched",
                                              "x_reordered")
    assert set(ALL_VARIANTS) >= set(VARIANTS) | {"xmarch", "xmarch_fma"}
    with pytest.raises(ValueError):
        ScheduleSpec("nonsense")
    assert len(XSHIFT_ROLES) == 22
    assert sum(1 for r in XSHIFT_ROLES if r[1] <= 0) == 13  # shifted blocks per X step
