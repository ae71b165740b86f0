"""Device cost of the overlapped multi-GPU evaluation on one GPU: a 1x1
decomposition (the exchange degenerates to the local periodic copy) runs
HaloExchanger.advect_overlapped — interior X-march box on the main stream,
exchange on the side stream, then the rim — against one whole-grid K1."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import decomp, device  # noqa: E402


def rate(fn, dims, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return dims.cells * reps / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    nx, ny, nz = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512x512x64").split("x"))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    gd = pw.make_grid(nx, ny, nz)
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), "cuda")
    f = device.fill(gd, pw.GeneratorSpec.baseline(42))
    out = device.alloc_fields(gd, "cuda")
    dec = decomp.Decomposition(gd, 1, 1, 0)
    ex = decomp.HaloExchanger(dec, device="cuda", transport=decomp.ThreadHubTransport(1).bind(0))
    inner = (2, nx, 2, ny)
    res = {}
    for _ in range(3):
        res.setdefault("k1_whole", []).append(rate(lambda: device.advect(*f, co, out), gd, reps))
        res.setdefault("overlapped", []).append(
            rate(lambda: ex.advect_overlapped(f, co, out), gd, reps))
        res.setdefault("k1_interior_box_only", []).append(
            rate(lambda: device.advect(*f, co, out, box=inner), gd, reps))
        res.setdefault("exchange_only", []).append(rate(lambda: ex.exchange(f), gd, reps))
    print(json.dumps({"grid": f"{nx}x{ny}x{nz}", **{k: round(sorted(v)[1], 2) for k, v in res.items()},
                      "plan_interior": device.describe_plan(gd, inner)}))


if __name__ == "__main__" and "--host" not in sys.argv:
    main()


def host_overhead(shape=(512, 256, 64), reps=200):
    """Host time per advect_overlapped call vs device time per call."""
    import time
    nx, ny, nz = shape
    gd = pw.make_grid(nx, ny, nz)
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), "cuda")
    f = device.fill(gd, pw.GeneratorSpec.baseline(42))
    out = device.alloc_fields(gd, "cuda")
    dec = decomp.Decomposition(gd, 1, 1, 0)
    ex = decomp.HaloExchanger(dec, device="cuda", transport=decomp.ThreadHubTransport(1).bind(0))
    for _ in range(10):
        ex.advect_overlapped(f, co, out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        ex.advect_overlapped(f, co, out)
    host = (time.perf_counter() - t) / reps
    torch.cuda.synchronize()
    dev_t = (time.perf_counter() - t) / reps
    rim = device.make_opts("simple")
    from paper_2010_01545_b200 import _lib
    rim.flags |= _lib.FLAG_RIM
    r = rate(lambda: device.advect(*f, co, out, box=(1, nx + 1, 1, ny + 1), opts=rim), gd, reps)
    print(json.dumps({"grid": f"{nx}x{ny}x{nz}", "host_us_per_call": round(host * 1e6, 1),
                      "wall_us_per_call": round(dev_t * 1e6, 1),
                      "rim_kernel_us": round(gd.cells / (r * 1e9) * 1e6, 1)}))


if __name__ == "__main__" and "--host" in sys.argv:
    host_overhead()
