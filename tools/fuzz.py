"""Randomised parity fuzz of K1 / K4 plans against the C oracle: random grid
shapes (odd and even nz, thin and wide), random plan options (tile width,
ring depth, chunks, grid), every kernel form (aligned X-march, UA forced,
K1m, one-thread), the halo pull with the block as its own neighbours (NaN
halos), the fused step, and the halo pull and the fused push step over
random x-y decompositions. Prints one JSON line; exit 1 on any mismatch.

    python tools/fuzz.py [--cases 200] [--seed 1]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402
from oracle import oracle  # noqa: E402  (checker)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    bad, done = [], 0
    for n in range(a.cases):
        nz = int(rng.choice([2, 3, 5, 8, 16, 24, 31, 32, 33, 40, 48, 56, 63, 64, 65, 72, 88, 96, 99, 100,
                              104, 110, 112, 120, 127, 128, 136, 152, 160, 176, 192, 200, 257,
                              300, 514, 1030]))
        nx = int(rng.integers(1, 90))
        ny = int(rng.integers(1, 400 if nz <= 64 else (120 if nz <= 300 else 40)))
        seed = int(rng.integers(0, 2**31))
        u, v, w = oracle.fill_random(nx, ny, nz, seed, baseline=True)
        co = oracle.baseline_coefficients(seed, nz)
        args = (co["tcx"], co["tcy"], co["tzc1"], co["tzc2"])
        want = oracle.advect(u, v, w, *args, engines=oracle.host_threads())
        dims = pw.make_grid(nx, ny, nz)
        f = [torch.from_numpy(x).cuda() for x in (u, v, w)]
        dco = pw.AdvectionCoefficients(*args)
        kw = {}
        if rng.random() < 0.5:
            kw["tile_j"] = int(rng.integers(1, 13))
        if rng.random() < 0.3:
            kw["stages"] = int(rng.integers(3, 8))
        if rng.random() < 0.3:
            kw["chunks"] = int(rng.integers(1, 9))
        if rng.random() < 0.3:
            kw["grid"] = int(rng.integers(1, 160))
        variant = str(rng.choice(["xmarch", "xmarch_elem", "xmarch_ct", "march", "simple"]))
        if variant == "xmarch_ct":  # tile_j selects the slab height (0: the planner's)
            kw["tile_j"] = int(rng.choice([0, 6, 12, 24]))
        case = {"shape": [nx, ny, nz], "variant": variant, **kw}
        try:
            out = device.advect(*f, dco, opts=device.make_opts(variant, **kw))
            torch.cuda.synchronize()
            if not oracle.compare([o.cpu().numpy() for o in out], want)["bitwise_equal"]:
                bad.append({**case, "what": "advect"})
            if nz % 2 == 0 and nz <= 768 and variant == "xmarch":
                g = [t.clone() for t in f]
                for t in g:
                    t[0].fill_(float("nan")); t[-1].fill_(float("nan"))  # noqa: E702
                    t[:, 0].fill_(float("nan")); t[:, -1].fill_(float("nan"))  # noqa: E702
                outp = device.advect_pull(*g, dco, device.self_peers(g), opts=device.make_opts(variant, **kw))
                torch.cuda.synchronize()
                if not oracle.compare([o.cpu().numpy() for o in outp], want)["bitwise_equal"]:
                    bad.append({**case, "what": "pull"})
            nxt = device.alloc_fields(dims, "cuda")
            device.step(*f, dco, 0.1, nxt, opts=device.make_opts(variant, **kw))
            torch.cuda.synchronize()
            for gtn, fh, s in zip(nxt, (u, v, w), want):
                if not np.array_equal(gtn.cpu().numpy()[1:-1, 1:-1].view(np.int64),
                                      (fh + 0.1 * s)[1:-1, 1:-1].view(np.int64)):
                    bad.append({**case, "what": "step"})
                    break
        except Exception as e:  # noqa: BLE001
            bad.append({**case, "what": f"error {type(e).__name__}: {e}"[:200]})
        done += 1
    # the halo pull over random x-y decompositions (every block's neighbours
    # are the other blocks' buffers on this GPU; blocks evaluated in turn)
    from paper_2010_01545_b200.decomp import Decomposition, LocalPeerRegistry, PullEvaluator
    for n in range(max(1, a.cases // 10)):
        # even nz on the aligned X-march pull inside K1; odd nz and deep columns
        # (UA form, K1c) take the K2p gather kernel and the planner's kernel
        nz = int(rng.choice([2, 6, 16, 64, 96, 128, 5, 33, 63, 127, 160, 300, 514]))
        px, py = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        nx, ny = int(rng.integers(px, 70)), int(rng.integers(py, 150 if nz <= 128 else 40))
        seed = int(rng.integers(0, 2**31))
        gd = pw.make_grid(nx, ny, nz)
        spec = pw.GeneratorSpec.baseline(seed)
        co = pw.baseline_coefficients(seed, nz)
        host = oracle.fill_random(nx, ny, nz, seed, baseline=True)
        want = oracle.advect(*host, co.tcx, co.tcy, co.tzc1, co.tzc2, engines=oracle.host_threads())
        case = {"pull_decomposition": [nx, ny, nz, px, py]}
        try:
            reg, evs = LocalPeerRegistry(), []
            for r in range(px * py):
                dec = Decomposition(gd, px, py, r)
                fs = dec.fill_local(spec)
                for t in fs:
                    t[0].fill_(float("nan")); t[-1].fill_(float("nan"))  # noqa: E702
                    t[:, 0].fill_(float("nan")); t[:, -1].fill_(float("nan"))  # noqa: E702
                evs.append((dec, PullEvaluator(dec, fs, co, reg)))
            for dec, ev in evs:
                o = device.alloc_fields(dec.local_dims, "cuda")
                ev.evaluate(o)
                torch.cuda.synchronize()
                xo, bx, yo, by = dec.block()
                for got, wnt in zip(o, want):
                    if not np.array_equal(got.cpu().numpy()[1:-1, 1:-1].view(np.int64),
                                          wnt[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].view(np.int64)):
                        bad.append({**case, "rank": dec.rank})
                        break
        except Exception as e:  # noqa: BLE001
            bad.append({**case, "what": f"error {type(e).__name__}: {e}"[:200]})
        done += 1
    # the fused push step over random decompositions, a few steps, ranks
    # stepped in turn on one stream (no kernel waits on another)
    from paper_2010_01545_b200.decomp import PushStepper
    from paper_2010_01545_b200.stepper import Stepper
    for n in range(max(1, a.cases // 20)):
        nz = int(rng.choice([2, 5, 16, 33, 64, 128]))
        px, py = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        nx, ny = int(rng.integers(px, 60)), int(rng.integers(py, 120))
        steps = int(rng.integers(1, 5))
        seed = int(rng.integers(0, 2**31))
        gd = pw.make_grid(nx, ny, nz)
        spec = pw.GeneratorSpec.baseline(seed)
        co = pw.baseline_coefficients(seed, nz)
        case = {"push_decomposition": [nx, ny, nz, px, py, steps]}
        try:
            g = device.fill(gd, spec)
            single = Stepper([t.clone() for t in g], co, 0.1)
            single.step(steps)
            want = single.fields
            reg, sts = LocalPeerRegistry(), []
            for r in range(px * py):
                dec = Decomposition(gd, px, py, r)
                fs = tuple(dec.local_view(t).contiguous() for t in g)
                sts.append((dec, PushStepper(dec, fs, co, 0.1, reg, lambda stream=None: None)))
            for _ in range(steps):
                for _, st in sts:
                    st.step(1)
            torch.cuda.synchronize()
            for dec, st in sts:
                for got, wnt in zip(st.fields, want):
                    if not torch.equal(got.view(torch.int64), dec.local_view(wnt).contiguous().view(torch.int64)):
                        bad.append({**case, "rank": dec.rank})
                        break
        except Exception as e:  # noqa: BLE001
            bad.append({**case, "what": f"error {type(e).__name__}: {e}"[:200]})
        done += 1
    print(json.dumps({"cases": done, "mismatches": len(bad), "first": bad[:5]}))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
