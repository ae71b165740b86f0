"""Per-plane copy latency of CTA 0 (issue -> arrival) from %globaltimer stamps."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402

SHAPES = {"c1": (512, 512, 64), "c3": (2048, 2048, 64)}


def run(cfg, **kw):
    nx, ny, nz = SHAPES[cfg]
    dims = pw.make_grid(nx, ny, nz)
    fields = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), fields[0].device)
    out = device.alloc_fields(dims, fields[0].device)
    dbg = kw.pop("debug", 0)
    opts = device.make_opts("xmarch_generic", **kw)  # stamps exist in the generic kernel only
    opts.flags |= dbg << 8
    for _ in range(3):
        device.advect(*fields, co, out, opts=opts)
    tr = torch.zeros(2 * 4096, dtype=torch.int64, device="cuda")
    opts.trace = ctypes.c_void_p(tr.data_ptr())
    device.advect(*fields, co, out, opts=opts)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(-1, 2).astype(np.float64)
    n = int((t[:, 1] > 0).sum())
    t = t[:n]
    t0 = t[0, 0]
    lat = (t[:, 1] - t[:, 0]) / 1e3  # us
    arr = np.diff(t[:, 1]) / 1e3
    plan = device.describe_plan(dims, None, opts)
    print(json.dumps({"cfg": cfg, "kw": kw, "debug": dbg, "planes": n,
                      "lat_us_p10_50_90": [round(float(np.percentile(lat, p)), 2) for p in (10, 50, 90)],
                      "interarrival_us_p10_50_90": [round(float(np.percentile(arr, p)), 3) for p in (10, 50, 90)],
                      "total_us": round((t[-1, 1] - t0) / 1e3, 1), "stages": plan["stages"],
                      "first20_issue_us": [round((x - t0) / 1e3, 2) for x in t[:20, 0]],
                      "first20_arrive_us": [round((x - t0) / 1e3, 2) for x in t[:20, 1]]}))


if __name__ == "__main__":
    for cfg in ("c1",):
        for kw in ({}, {"debug": 5}, {"debug": 1}, {"stages": 4}, {"stages": 6}):
            run(cfg, **dict(kw))
