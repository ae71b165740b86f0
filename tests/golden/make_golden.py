"""Generate the golden parity fixtures by importing the REFERENCE itself.

Run in the dev container (the reference is only present there):

    python tests/golden/make_golden.py

It imports pwadvect from /root/reference/pkg/src (read-only), evaluates the
reference's own `run_reference` (pkg/src/pwadvect/kernel.py:175-185) on seeded
inputs built with the reference's own generator (`fill_fields` /
`lcg_doubles`, pkg/src/pwadvect/grid.py:164-239), and writes:

* tests/golden/cases.json — per case: dims, generator, coefficients (exact,
  as float.hex), blake2b-64 digests (reference `checksum`, grid.py:242-249)
  of the inputs u/v/w and of the reference outputs su/sv/sw;
* tests/golden/small.npz — full padded input/output arrays of the small cases;
* tests/golden/steps.json — digests of a composed time-stepping oracle built
  from the reference's `run_reference` + numpy `f + dt*s` + `wrap_halos`
  (the reference has no time integration);
* tests/golden/arrays.npz — the array-level API: the reference's
  `compute_block` (kernel.py:139-162) on independent random role arrays and
  on `grid_roles` views, and `su/sv/sw_formula` (kernel.py:73-112) on
  broadcast scalar/array arguments, mid and top branches.

The BASELINE.json value distributions are applied on top of
the reference LCG: x*20.0-10.0 (numpy mul then sub), w=0 at k=0 and k=nz-1,
then the reference `wrap_halos`; tzc1/tzc2 = 1e-3 + 4e-3*lcg_doubles(seed+1).
Nothing under tests/ reads /root/reference at run time; only this script does.
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from pwadvect.grid import (FieldSet, Field3D, GeneratorSpec, checksum,  # noqa: E402
                           fill_fields, lcg_doubles, make_grid, wrap_halos)
from pwadvect.kernel import (COMPUTE_ROLES, AdvectionCoefficients,  # noqa: E402
                             compute_block, grid_roles, operation_census, reads_per_point,
                             run_reference, su_formula, sv_formula, sw_formula)

OUT = Path(__file__).resolve().parent


def baseline_fields(dims, seed):
    vals = lcg_doubles(seed, 3 * dims.cells)
    shape = (dims.nx, dims.ny, dims.nz)
    arrs = []
    for n in range(3):
        a = np.empty(dims.padded_shape)
        a[1:-1, 1:-1, :] = (vals[n * dims.cells:(n + 1) * dims.cells] * 20.0 - 10.0).reshape(shape)
        if n == 2:
            a[1:-1, 1:-1, 0] = 0.0
            a[1:-1, 1:-1, dims.nz - 1] = 0.0
        wrap_halos(a)
        arrs.append(Field3D(dims, a))
    return FieldSet(*arrs)


def baseline_coeffs(seed, nz):
    t = lcg_doubles(seed + 1, 4 * nz)
    tz = [1e-3 + 4e-3 * t[m * nz:(m + 1) * nz] for m in range(4)]
    return AdvectionCoefficients(0.25 / 50.0, 0.25 / 50.0, tz[0], tz[1]), tz[2], tz[3]


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    goldens = json.loads((REF / "tests" / "goldens.json").read_text())
    cases, small = [], {}

    def add(name, dims, gen, fields, coeffs, keep_arrays, extra=None):
        src = run_reference(fields, coeffs)
        case = {
            "name": name, "nx": dims.nx, "ny": dims.ny, "nz": dims.nz, "generator": gen,
            "tcx": float(coeffs.tcx).hex(), "tcy": float(coeffs.tcy).hex(),
            "tzc1": hexs(coeffs.tzc1), "tzc2": hexs(coeffs.tzc2),
            "inputs": {"u": checksum(fields.u), "v": checksum(fields.v), "w": checksum(fields.w)},
            "sources": {"su": checksum(src.su), "sv": checksum(src.sv), "sw": checksum(src.sw)},
            "arrays": keep_arrays,
        }
        if extra:
            case.update(extra)
        cases.append(case)
        if keep_arrays:
            for key, f in (("u", fields.u), ("v", fields.v), ("w", fields.w),
                           ("su", src.su), ("sv", src.sv), ("sw", src.sw)):
                small[f"{name}/{key}"] = f.data.copy()
        return src

    # 1. the reference's own golden case (goldens.json): 8x8x8, random(42), 0.25
    dims = make_grid(8, 8, 8)
    fields = fill_fields(dims, GeneratorSpec.random(42))
    coeffs = AdvectionCoefficients(0.25, 0.25, np.full(8, 0.25), np.full(8, 0.25))
    src = add("ref_goldens_8x8x8", dims, {"mode": "random", "seed": 42}, fields, coeffs, True)
    assert checksum(src.su) == goldens["sources"]["su"]
    assert checksum(src.sv) == goldens["sources"]["sv"]
    assert checksum(src.sw) == goldens["sources"]["sw"]
    assert checksum(fields.u) == goldens["fields"]["u"]

    # 2. random shapes / random coefficients (as test_kernel.py:101-111)
    rng = np.random.default_rng(2010_01545)
    shapes = [(1, 1, 2), (1, 1, 3), (2, 1, 2), (1, 7, 5), (9, 1, 4), (3, 3, 2),
              (5, 4, 6), (6, 5, 7), (13, 11, 9), (16, 16, 16), (33, 17, 10), (7, 40, 12)]
    for nx, ny, nz in shapes:
        dims = make_grid(nx, ny, nz)
        seed = int(rng.integers(0, 2**31))
        fields = fill_fields(dims, GeneratorSpec.random(seed))
        coeffs = AdvectionCoefficients(float(rng.random()), float(rng.random()),
                                       rng.random(nz), rng.random(nz))
        add(f"random_{nx}x{ny}x{nz}", dims, {"mode": "random", "seed": seed}, fields, coeffs, True)

    # 3. uniform fields (symmetry / closed forms, test_kernel.py:42-85)
    for (a, b, c), tz in (((1.7, -0.3, 2.4), 0.25), ((1.25, -0.75, 2.5), 0.25), ((1.0, 1.0, 1.0), 0.25)):
        dims = make_grid(5, 5, 6)
        fields = fill_fields(dims, GeneratorSpec.uniform(a, b, c))
        coeffs = AdvectionCoefficients(tz, tz, np.full(6, tz), np.full(6, tz))
        add(f"uniform_{a}_{b}_{c}", dims, {"mode": "uniform", "a": a, "b": b, "c": c},
            fields, coeffs, True)

    # 4. trig generator (host-generated sin/cos test aid, grid.py:211-220)
    dims = make_grid(12, 10, 8)
    fields = fill_fields(dims, GeneratorSpec.trig())
    coeffs = AdvectionCoefficients(0.3, 0.2, np.linspace(0.1, 0.8, 8), np.linspace(0.9, 0.2, 8))
    add("trig_12x10x8", dims, {"mode": "trig"}, fields, coeffs, True)

    # 5. BASELINE distributions: C0 (configs[0]) and ragged / nz=128 / odd-nz shapes
    for nx, ny, nz, seed, keep in ((64, 64, 64, 42, False), (37, 29, 64, 3, False),
                                   (16, 24, 128, 7, False), (33, 17, 63, 11, False),
                                   (20, 18, 64, 5, True), (150, 3, 64, 9, False),
                                   (3, 150, 64, 10, False)):
        dims = make_grid(nx, ny, nz)
        fields = baseline_fields(dims, seed)
        coeffs, tzd1, tzd2 = baseline_coeffs(seed, nz)
        add(f"baseline_{nx}x{ny}x{nz}_s{seed}", dims, {"mode": "baseline", "seed": seed},
            fields, coeffs, keep, {"tzd1": hexs(tzd1), "tzd2": hexs(tzd2)})

    # 5b. non-finite inputs: a NaN with a payload and +-Inf propagate through
    # the formulas exactly as numpy evaluates them (payloads included)
    dims = make_grid(8, 7, 6)
    fields = baseline_fields(dims, 3)
    fields.u.data[3, 3, 2] = np.nan
    fields.u.data[5, 5, 1] = np.frombuffer(np.uint64(0x7FF8000000000123).tobytes(), np.float64)[0]
    fields.v.data[4, 2, 3] = np.inf
    fields.w.data[2, 5, 4] = -np.inf
    for f in (fields.u, fields.v, fields.w):
        wrap_halos(f.data)
    coeffs, _, _ = baseline_coeffs(3, 6)
    add("nonfinite_8x7x6", dims, {"mode": "nonfinite"}, fields, coeffs, True)

    (OUT / "cases.json").write_text(json.dumps({
        "generated_by": "tests/golden/make_golden.py (imports reference pwadvect 0.1.0)",
        "reference_goldens_json": goldens,
        "cases": cases,
        "compute_roles": [list(r) for r in COMPUTE_ROLES],
        "operation_census": {"mid": operation_census(False), "top": operation_census(True),
                             "reads_mid": reads_per_point(False),
                             "reads_top": reads_per_point(True)}}, indent=1))
    np.savez_compressed(OUT / "small.npz", **small)

    # 6. composed time stepping: f <- f + dt*s, then wrap
    steps_out = []
    for nx, ny, nz, seed, nsteps in ((12, 10, 16, 5, 5), (24, 20, 128, 6, 3), (9, 7, 8, 4, 10)):
        dims = make_grid(nx, ny, nz)
        fields = baseline_fields(dims, seed)
        coeffs, _, _ = baseline_coeffs(seed, nz)
        dt = 0.1
        for _ in range(nsteps):
            src = run_reference(fields, coeffs)
            for f, s in ((fields.u, src.su), (fields.v, src.sv), (fields.w, src.sw)):
                f.data[1:-1, 1:-1, :] = f.data[1:-1, 1:-1, :] + dt * s.data[1:-1, 1:-1, :]
                wrap_halos(f.data)
        steps_out.append({"nx": nx, "ny": ny, "nz": nz, "seed": seed, "steps": nsteps, "dt": dt,
                          "fields": {"u": checksum(fields.u), "v": checksum(fields.v),
                                     "w": checksum(fields.w)}})
    (OUT / "steps.json").write_text(json.dumps({"cases": steps_out}, indent=1))

    # 7. array-level API: compute_block on independent role arrays (leading
    # shapes (2, 3), (5,), (0, 4)), on grid_roles views, and the formulas
    arrays = {}
    rng = np.random.default_rng(2010)
    for n, (lead, nz) in enumerate((((2, 3), 9), ((5,), 2), ((3, 2), 3), ((0, 4), 4))):
        roles = {r: rng.uniform(-10.0, 10.0, lead + (nz,)) for r in COMPUTE_ROLES}
        co = AdvectionCoefficients(float(rng.uniform(0, 1)), float(rng.uniform(0, 1)),
                                   rng.uniform(0, 1, nz), rng.uniform(0, 1, nz))
        outs = compute_block(co, roles)
        arrays[f"cb{n}/coeffs"] = np.concatenate([[co.tcx, co.tcy], co.tzc1, co.tzc2])
        for m, r in enumerate(COMPUTE_ROLES):
            arrays[f"cb{n}/role{m}"] = roles[r]
        for name, o in zip(("su", "sv", "sw"), outs):
            arrays[f"cb{n}/{name}"] = o
    dims = make_grid(7, 6, 5)
    fields = fill_fields(dims, GeneratorSpec.random(99))
    co = AdvectionCoefficients(0.3, 0.7, rng.uniform(0, 1, 5), rng.uniform(0, 1, 5))
    for name, o in zip(("su", "sv", "sw"), compute_block(co, grid_roles(fields, 2, 6))):
        arrays[f"gr/{name}"] = o
    arrays["gr/coeffs"] = np.concatenate([[co.tcx, co.tcy], co.tzc1, co.tzc2])
    for which, fn in enumerate((su_formula, sv_formula, sw_formula)):
        for top in (False, True):
            args = [float(rng.uniform(0, 1)), float(rng.uniform(0, 1)), rng.uniform(0, 1, 5),
                    float(rng.uniform(0, 1))]
            args += [rng.uniform(-10, 10, (4, 5)) if m % 3 else rng.uniform(-10, 10, 5)
                     for m in range(15)]
            out = fn(*args, top=top)
            key = f"f{which}{int(top)}"
            for m, a in enumerate(args):
                arrays[f"{key}/arg{m}"] = np.asarray(a, dtype=np.float64)
            arrays[f"{key}/out"] = out
    np.savez_compressed(OUT / "arrays.npz", **arrays)
    print(f"{len(cases)} cases, {len(small)} arrays, {len(steps_out)} stepping cases, "
          f"{len(arrays)} array-API arrays")


if __name__ == "__main__":
    main()
