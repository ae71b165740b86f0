"""Default-plan throughput over a range of grid shapes (one GPU).

For each (nx, ny, nz) the fields are filled on the device, the default plan
(`describe_plan`) is reported, and K1 is timed in a burst after a clock
pre-warm (the bench's shape). One JSON line per shape: Gpts/s, GB/s at the
algorithmic 48 B/point, fraction of the measured HBM peak.

    python tools/shape_sweep.py [--shapes 512x512x64,128x128x1030] [--reps 30]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402

DEFAULT = ("512x512x64,512x512x63,512x512x32,512x512x33,1024x1024x16,512x512x96,512x512x128,"
           "512x512x127,256x256x256,256x256x255,256x256x384,256x256x512,256x256x511,128x128x768,"
           "128x128x769,128x128x1024,128x128x1030,64x64x2048,64x64x4096,2048x2048x63")


def peak_gbs():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6550.4


def time_burst(fn, reps, prewarm_ms=40.0):
    torch.cuda.synchronize()
    time.sleep(0.2)
    t_end = time.perf_counter() + prewarm_ms / 1e3
    while time.perf_counter() < t_end:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--variants", default='[{"variant": "xmarch"}]',
                    help="JSON list of make_opts kwargs (variant + options)")
    args = ap.parse_args()
    peak = peak_gbs()
    variants = json.loads(args.variants)
    for s in args.shapes.split(","):
        nx, ny, nz = (int(t) for t in s.split("x"))
        dims = pw.make_grid(nx, ny, nz)
        fields = device.fill(dims, pw.GeneratorSpec.baseline(42))
        co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), fields[0].device)
        out = device.alloc_fields(dims, fields[0].device)
        ref = None
        for v in variants:
            kw = dict(v)
            name = kw.pop("variant")
            opts = device.make_opts(name, **kw)
            rec = {"shape": s, "variant": v}
            try:
                rec["plan"] = device.describe_plan(dims, None, opts)
                ms = time_burst(lambda: device.advect(*fields, co, out, opts=opts), args.reps)
            except Exception as e:  # noqa: BLE001
                rec["error"] = str(e)
                print(json.dumps(rec), flush=True)
                continue
            snap = [int(o.view(torch.int64).sum().item()) for o in out]
            if ref is None:
                ref = snap
            gbs = 48 * dims.cells / (ms / 1e3) / 1e9
            rec.update(ms=round(ms, 4), gpts=round(dims.cells / ms / 1e6, 2), GBs=round(gbs, 1),
                       frac=round(gbs / peak, 4), same_as_first=snap == ref)
            print(json.dumps(rec), flush=True)
        del fields, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
