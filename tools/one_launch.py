"""Fill a grid on the device and launch K1 (or K4 with --step) a few times with
the given options — a small target for ncu metric runs.

    python tools/one_launch.py 4096x4096x128 --chunks 8 [--step] [--n 3]
        [--variant xmarch_elem] [--pull]   (--pull: the block as its own neighbours)
        [--stages S] [--flags 0x1000]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("grid")
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--step", action="store_true")
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--variant", default="xmarch")
    ap.add_argument("--pull", action="store_true")
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0)
    a = ap.parse_args()
    nx, ny, nz = (int(x) for x in a.grid.split("x"))
    dims = pw.make_grid(nx, ny, nz)
    f = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), f[0].device)
    out = device.alloc_fields(dims, f[0].device)
    opts = device.make_opts(a.variant, chunks=a.chunks, stages=a.stages, flags=a.flags)
    print(device.describe_plan(dims, None, opts))
    peers = device.self_peers(f) if a.pull else None
    for _ in range(a.n):
        if peers is not None:
            device.BoundLaunch(f, co, out, opts=opts, dt=0.1 if a.step else None, pull=peers)()
        elif a.step:
            device.step(*f, co, 0.1, out, opts=opts)
        else:
            device.advect(*f, co, out, opts=opts)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
