"""Probe the column-tile kernel case by case, each in its own process (a
device fault is sticky): prints one line per (shape, tile_j) with the plan and
the outcome against the oracle.

    python tools/ct_probe.py 13x30x63:6 13x30x64:12 ...
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import device
from oracle import oracle
nx, ny, nz = map(int, sys.argv[2].split("x")); tj = int(sys.argv[3]); variant = sys.argv[4]
u, v, w = oracle.fill_random(nx, ny, nz, 5, baseline=True)
co = oracle.baseline_coefficients(5, nz)
args = (co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
want = oracle.advect(u, v, w, *args)
dims = pw.make_grid(nx, ny, nz)
opts = device.make_opts(variant, tile_j=tj)
plan = device.describe_plan(dims, opts=opts)
f = [torch.from_numpy(a).cuda() for a in (u, v, w)]
out = device.advect(*f, pw.AdvectionCoefficients(*args), opts=opts)
torch.cuda.synchronize()
r = oracle.compare([o.cpu().numpy() for o in out], want)
bad = None
if not r["bitwise_equal"]:
    g = out[0].cpu().numpy(); d = np.argwhere(g.view(np.int64) != want[0].view(np.int64))
    bad = {"n": int(len(d)), "first": d[:6].tolist(), "levels": sorted(set(d[:, 2].tolist()))[:20],
           "cols": sorted(set(d[:, 1].tolist()))[:20]}
print(json.dumps({"plan": plan, "equal": r["bitwise_equal"], "bad_su": bad}))
'''


def main():
    variant = "xmarch_ct"
    for arg in sys.argv[1:]:
        if arg.startswith("--variant="):
            variant = arg.split("=", 1)[1]
            continue
        shape, tj = arg.split(":")
        res = subprocess.run([sys.executable, "-c", CHILD, str(ROOT), shape, tj, variant],
                             capture_output=True, text=True, timeout=300)
        line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else ""
        print(json.dumps({"case": arg, "rc": res.returncode, "out": line,
                          "err": res.stderr.strip().splitlines()[-1][:200] if res.returncode else ""}),
              flush=True)


if __name__ == "__main__":
    main()
