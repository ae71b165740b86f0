"""Where the numpy drop-in's time goes: pageable vs pinned inputs/outputs, fresh vs reused outputs."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def timeit(fn, n=5):
    fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n


def main():
    nx, ny, nz = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512x512x64").split("x"))  # noqa
    dims = pw.make_grid(nx, ny, nz)
    f = pw.fill_fields(dims, pw.GeneratorSpec.baseline(42))
    co = pw.baseline_coefficients(42, nz)
    ctx = device.HostContext(dims, 0)
    args = (co.tcx, co.tcy, co.tzc1, co.tzc2)
    page_in = [f.u.data, f.v.data, f.w.data]
    pin_in = [torch.from_numpy(a).pin_memory() for a in page_in]
    pin_out = [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    reuse_out = [np.zeros(dims.padded_shape) for _ in range(3)]
    r = {}
    r["run_reference"] = timeit(lambda: pw.run_reference(f, co))
    r["fresh_np_empty_x3_touch"] = timeit(lambda: [np.empty(dims.padded_shape).fill(1.0) for _ in range(3)])
    r["pageable_in_fresh_out"] = timeit(lambda: ctx.advect_host(*page_in, *[np.empty(dims.padded_shape) for _ in range(3)], *args))
    r["pageable_in_reused_out"] = timeit(lambda: ctx.advect_host(*page_in, *reuse_out, *args))
    r["pageable_in_pinned_out"] = timeit(lambda: ctx.advect_host(*page_in, *pin_out, *args))
    r["pinned_in_pinned_out"] = timeit(lambda: ctx.advect_host(*pin_in, *pin_out, *args))
    r["torch_pinned_alloc_x3"] = timeit(lambda: [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)])
    r["host_memcpy_406MB_numpy"] = timeit(lambda: [np.copyto(o, i) for o, i in zip(reuse_out, page_in)])
    for k, v in r.items():
        print(json.dumps({"case": k, "ms": round(v * 1e3, 2), "gpts": round(dims.cells / v / 1e9, 3)}))
    ctx.close()


if __name__ == "__main__" and "--register" not in sys.argv:
    main()


def register_cost(shape=(514, 514, 64)):
    """cudaHostRegister / Unregister of three fresh-but-touched pageable fields."""
    cudart = torch.cuda.cudart()
    arrs = [np.ones(shape) for _ in range(3)]
    for _ in range(2):
        t = time.perf_counter()
        for a in arrs:
            rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
            assert int(rc) == 0, rc
        t1 = time.perf_counter()
        for a in arrs:
            cudart.cudaHostUnregister(a.ctypes.data)
        t2 = time.perf_counter()
        print(json.dumps({"case": "host_register_x3", "register_ms": round((t1 - t) * 1e3, 2),
                          "unregister_ms": round((t2 - t1) * 1e3, 2)}))


if __name__ == "__main__" and "--register" in sys.argv:
    register_cost()
