"""Arrival-time gaps of CTA 0 around work-unit boundaries (profiling aid)."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def run(nx, ny, nz, chunks):
    dims = pw.make_grid(nx, ny, nz)
    fields = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), fields[0].device)
    out = device.alloc_fields(dims, fields[0].device)
    opts = device.make_opts("xmarch", chunks=chunks)
    for _ in range(3):
        device.advect(*fields, co, out, opts=opts)
    tr = torch.zeros(2 * 4096, dtype=torch.int64, device="cuda")
    opts.trace = ctypes.c_void_p(tr.data_ptr())
    device.advect(*fields, co, out, opts=opts)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(-1, 2).astype(np.float64)
    n = int((t[:, 1] > 0).sum())
    arr = (t[:n, 1] - t[0, 0]) / 1e3
    iss = (t[:n, 0] - t[0, 0]) / 1e3
    plan = device.describe_plan(dims, None, opts)
    ns, nch = plan["strips"], plan["chunks"]
    g = plan["grid"]
    firsts, q = [], 0
    for u in range(0, ns * nch, g):
        chunk = u // ns
        ib, ie = nx * chunk // nch, nx * (chunk + 1) // nch
        firsts.append(q)
        q += ie - ib + 2
    gaps = np.diff(arr)
    around = {int(f): [round(float(x), 2) for x in gaps[max(0, f - 3):f + 4]] for f in firsts[1:4]}
    print(json.dumps({"shape": [nx, ny, nz], "chunks": nch, "planes": n, "total_us": round(arr[-1], 1),
                      "median_gap": round(float(np.median(gaps)), 3), "unit_first": firsts[:6],
                      "gaps_around_unit_starts": around,
                      "lat_median": round(float(np.median(arr - iss)), 2),
                      "top_gaps": sorted([(round(float(x), 2), int(i)) for i, x in enumerate(gaps)], reverse=True)[:8]}))


if __name__ == "__main__":
    for ch in (19, 4):
        run(2048, 2048, 64, ch)
    run(512, 512, 64, 10)
