"""Streamed e2e rate (pwadv_ctx_submit_host + sync) vs chunk count and stream length."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def main():
    nx, ny, nz = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "512x512x64").split("x"))
    dims = pw.make_grid(nx, ny, nz)
    f = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), "cuda")
    hin = [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    hout = [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    for a, b in zip(hin, f):
        a.copy_(b)
    tz = [co.tz[0].cpu().numpy(), co.tz[1].cpu().numpy()]
    ctx = device.HostContext(dims, 0)
    for steps in (20, 50):
        for ch in (1, 2, 4, 8, 16, 32):
            ctx.submit_host(*hin, *hout, co.tcx, co.tcy, *tz, chunks=ch)
            ctx.sync()
            t = time.perf_counter()
            for _ in range(steps):
                ctx.submit_host(*hin, *hout, co.tcx, co.tcy, *tz, chunks=ch)
            ctx.sync()
            dt = (time.perf_counter() - t) / steps
            print(json.dumps({"grid": f"{nx}x{ny}x{nz}", "steps": steps, "chunks": ch,
                              "ms": round(dt * 1e3, 3), "gpts": round(dims.cells / dt / 1e9, 3)}),
                  flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
