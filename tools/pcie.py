"""Pinned host<->device bandwidth (alone / concurrent) and e2e rate vs chunking."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def bw():
    n = 3 * 514 * 514 * 64  # three C1 fields
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = n * 8
    for label, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                      ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        print(json.dumps({"copy": label, "GBs": round(5 * nb / (time.perf_counter() - t) / 1e9, 1)}))
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps({"copy": "both", "GBs_each": round(5 * nb / dt / 1e9, 1)}))


def e2e():
    dims = pw.make_grid(512, 512, 64)
    f = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, 64), "cuda")
    hin = [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    hout = [torch.empty(dims.padded_shape, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    for a, b in zip(hin, f):
        a.copy_(b)
    tz = [co.tz[0].cpu().numpy(), co.tz[1].cpu().numpy()]
    ctx = device.HostContext(dims, 0)
    for ch in (1, 8, 12, 16, 24, 32, 48, 64):
        for _ in range(2):
            ctx.advect_host(*hin, *hout, co.tcx, co.tcy, *tz, chunks=ch)
        t = time.perf_counter()
        for _ in range(10):
            ctx.advect_host(*hin, *hout, co.tcx, co.tcy, *tz, chunks=ch)
        dt = (time.perf_counter() - t) / 10
        print(json.dumps({"e2e_chunks": ch, "ms": round(dt * 1e3, 3), "gpts": round(dims.cells / dt / 1e9, 3)}))


if __name__ == "__main__":
    bw()
    e2e()
