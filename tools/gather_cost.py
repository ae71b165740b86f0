"""K2p (pwadv_pull_halos_f64, the halo gather from the neighbours' buffers)
beside K2 (the local periodic wrap) and the evaluation that follows it, block
as its own eight neighbours on one GPU: the cost the gather form of the halo
pull adds to an evaluation of a block off the aligned X-march.

    python tools/gather_cost.py [--shapes 256x256x512,512x512x63]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def timed(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="256x256x512,512x512x63,512x256x300,2048x2048x63,128x128x1030")
    a = ap.parse_args()
    for shp in a.shapes.split(","):
        nx, ny, nz = (int(x) for x in shp.split("x"))
        dims = pw.make_grid(nx, ny, nz)
        f = device.fill(dims, pw.GeneratorSpec.baseline(42))
        co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), f[0].device)
        out = device.alloc_fields(dims, "cuda")
        peers = device.self_peers(f)
        k1 = device.BoundLaunch(f, co, out)
        k1g = device.BoundLaunch(f, co, out, pull=peers, gather=True)
        want = [t.clone() for t in device.advect(*f, co)]
        k1g()
        torch.cuda.synchronize()
        same = all(torch.equal(x.view(torch.int64), y.view(torch.int64)) for x, y in zip(out, want))
        halo_bytes = 2 * 3 * 8 * (2 * (ny + 2) + 2 * nx) * nz  # read + written
        r = {"shape": shp, "plan": device.describe_plan(dims)["kernel"],
             "wrap_us": round(timed(lambda: device.wrap_halos(*f)), 2),
             "gather_us": round(timed(lambda: device.pull_halos(*f, peers)), 2),
             "halo_MB": round(halo_bytes / 1e6, 2), "bitwise_equal": bool(same)}
        # alternated bursts, best of each (a sustained loop drifts to the power cap)
        import time
        a_, b_ = [], []
        for _ in range(4):
            time.sleep(0.3)
            a_.append(timed(k1, 20))
            time.sleep(0.3)
            b_.append(timed(k1g, 20))
        r["k1_us"], r["gather_plus_k1_us"] = round(min(a_), 2), round(min(b_), 2)
        r["added_pct"] = round(100 * (r["gather_plus_k1_us"] / r["k1_us"] - 1), 2)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
