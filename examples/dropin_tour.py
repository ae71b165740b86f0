"""A user's view of the drop-in: the reference's hot-path calls, unchanged,
running on the B200 (run with `python examples/dropin_tour.py` on a GPU box).

Every call below exists under the same name in the reference package
(`pwadvect`, pkg/src/pwadvect/__init__.py); the identities printed are the
ones the reference's own test suite checks (bit-exact results).
"""

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2010_01545_b200 as pwadvect  # noqa: E402  (instead of `import pwadvect`)
from paper_2010_01545_b200 import kernel  # noqa: E402  (pwadvect.kernel)


def main():
    dims = pwadvect.make_grid(96, 80, 64)
    fields = pwadvect.fill_fields(dims, pwadvect.GeneratorSpec.random(seed=42))  # K5 on the GPU
    again = pwadvect.fill_fields(dims, pwadvect.GeneratorSpec.random(seed=42))
    print(f"grid {dims.nx}x{dims.ny}x{dims.nz}: u checksum {pwadvect.checksum(fields.u)} "
          f"(regenerated: {pwadvect.checksum(again.u)})")
    assert np.array_equal(fields.u.data[0], fields.u.data[-2])  # periodic halos

    coeffs = pwadvect.default_coefficients(dims.nz)
    src = pwadvect.run_reference(fields, coeffs)                # K1 on the GPU
    print("su checksum", pwadvect.checksum(src.su), "| level 0 is zero:",
          bool(np.all(src.su.data[:, :, 0] == 0.0)))

    # scalar point evaluation equals the grid value bit for bit
    p = pwadvect.advect_point_u(fields, coeffs, 3, 5, 7)
    assert p == src.su.data[3, 5, 6]
    # the array-level API: compute_block over grid_roles views
    su, sv, sw = kernel.compute_block(coeffs, kernel.grid_roles(fields, 1, dims.nx + 1))
    assert np.array_equal(su[..., 1:], src.su.data[1:-1, 1:-1, 1:])

    # uniform winds with tzc1 == tzc2 cancel exactly below the top level
    uni = pwadvect.fill_fields(dims, pwadvect.GeneratorSpec.uniform(1.5, -2.0, 3.0))
    sym = pwadvect.run_reference(uni, coeffs)
    print("uniform winds: zero below the top:", bool(np.all(sym.su.data[1:-1, 1:-1, :-1] == 0.0)),
          "| top", sym.su.data[1, 1, -1], "== closed form", 2 * 0.25 * 1.5 * 3.0)

    # every schedule name and engine count gives the same bits
    for name in ("reference", "column_buffered", "y_batched", "x_reordered"):
        for engines in (1, 4):
            out, traffic, wall = pwadvect.run_schedule(
                fields, coeffs, pwadvect.ScheduleSpec(name, y_batch=16, engines=engines))
            assert pwadvect.compare_outputs(src, out).bitwise_equal
    print("all schedules x engines bitwise equal")

    # throughput of the drop-in on a BASELINE-sized grid (numpy in, numpy out)
    big = pwadvect.make_grid(512, 512, 64)
    bf = pwadvect.fill_fields(big, pwadvect.GeneratorSpec.baseline(42))
    bc = pwadvect.baseline_coefficients(42, 64)
    pwadvect.run_reference(bf, bc)
    t = time.perf_counter()
    for _ in range(5):
        pwadvect.run_reference(bf, bc)
    dt = (time.perf_counter() - t) / 5
    print(f"run_reference 512x512x64 from numpy arrays: {dt * 1e3:.1f} ms "
          f"({big.cells / dt / 1e9:.2f} Gpoints/s incl. host<->device copies)")


if __name__ == "__main__":
    main()
