"""Pin the oracle to the reference on random cases (dev container only: it
imports the reference package from /root/reference, read-only). Random
shapes and seeds, the reference's own generator and run_reference against
oracle.advect (C) and oracle.run_schedule_numpy; prints one JSON line.

    python tools/oracle_vs_reference.py [--cases 200]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402

import pwadvect as ref  # noqa: E402  (the reference, read-only)
from oracle import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    a = ap.parse_args()
    rng = np.random.default_rng(5)
    bad = 0
    for _ in range(a.cases):
        nx, ny, nz = int(rng.integers(1, 24)), int(rng.integers(1, 24)), int(rng.integers(2, 40))
        seed = int(rng.integers(0, 2**63))
        dims = ref.make_grid(nx, ny, nz)
        f = ref.fill_fields(dims, ref.GeneratorSpec.random(seed))
        t = rng.random(2 * nz) * 4e-3 + 1e-3
        tc = float(rng.random() * 0.01)
        co = ref.AdvectionCoefficients(tc, tc * 1.5, t[:nz], t[nz:])
        want = ref.run_reference(f, co)
        u, v, w = f.u.data, f.v.data, f.w.data
        a1 = oracle.advect(u, v, w, co.tcx, co.tcy, co.tzc1, co.tzc2, engines=3)
        a2 = oracle.run_schedule_numpy(u, v, w, co.tcx, co.tcy, co.tzc1, co.tzc2, 2)
        wd = (want.su.data, want.sv.data, want.sw.data)
        bad += not (oracle.compare(a1, wd)["bitwise_equal"] and oracle.compare(a2, wd)["bitwise_equal"])
    print(json.dumps({"cases": a.cases, "mismatches": bad,
                      "what": "oracle.advect (C) and oracle.run_schedule_numpy vs the reference's run_reference, bitwise"}))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
