"""The numpy drop-in on a grid evaluated X slab by X slab (out of core) beside
the whole-grid call: rate and bitwise equality. The slab form is what
run_reference does by itself when the six padded device arrays exceed its
share of the device memory; PWADV_DROPIN_DEVICE_BYTES forces it here.

    python tools/out_of_core.py [--shape 2048x2048x64] [--limit-gb 4]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device, stencil  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="2048x2048x64")
    ap.add_argument("--limit-gb", type=float, default=4.0)
    a = ap.parse_args()
    nx, ny, nz = (int(x) for x in a.shape.split("x"))
    dims = pw.make_grid(nx, ny, nz)
    dev = device.fill(dims, pw.GeneratorSpec.baseline(42))
    fields = pw.FieldSet(*(pw.Field3D(dims, t.cpu().numpy()) for t in dev))
    del dev
    co = pw.baseline_coefficients(42, nz)
    os.environ.pop("PWADV_DROPIN_DEVICE_BYTES", None)
    r = {"shape": a.shape, "points": dims.cells}

    def timed(n=3):
        pw.run_reference(fields, co)
        t = time.perf_counter()
        for _ in range(n):
            out = pw.run_reference(fields, co)
        return (time.perf_counter() - t) / n, out
    dt, whole = timed()
    r["whole_grid"] = {"s": round(dt, 4), "gpts": round(dims.cells / dt / 1e9, 3)}
    os.environ["PWADV_DROPIN_DEVICE_BYTES"] = str(int(a.limit_gb * 1e9))
    planes = stencil._slab_planes(stencil.GridDims(nx, ny, nz))
    dt, sl = timed()
    r["slabs"] = {"planes_per_slab": planes, "slabs": -(-nx // planes), "s": round(dt, 4),
                  "gpts": round(dims.cells / dt / 1e9, 3), "device_limit_GB": a.limit_gb}
    r["bitwise_equal"] = all(np.array_equal(x.data.view(np.int64), y.data.view(np.int64))
                             for x, y in zip((whole.su, whole.sv, whole.sw), (sl.su, sl.sv, sl.sw)))
    print(json.dumps(r))


if __name__ == "__main__":
    main()
