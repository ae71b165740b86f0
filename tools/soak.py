"""Soak test of the ring protocol: many back-to-back launches must keep giving
the same bits (a rare race in the mbarrier / refill protocol would show up as
a changed digest or a hang). Prints one JSON line.

    python tools/soak.py [--launches 100000] [--steps 3000] [--only k1,k4,pull,ua,ct]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import device  # noqa: E402
from paper_2010_01545_b200.stepper import Stepper  # noqa: E402


def digest(ts):
    return tuple(int(t.view(torch.int64).sum().item()) for t in ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=100000)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--only", default="k1,k4,pull,ua")
    a = ap.parse_args()
    which = set(a.only.split(","))
    res = {}
    if "pull" in which:  # K1 with the halo pull (block as its own neighbours), 2048^2x64
        dp = pw.make_grid(2048, 2048, 64)
        fp = device.fill(dp, pw.GeneratorSpec.baseline(7))
        cop = device.DeviceCoefficients.from_host(pw.baseline_coefficients(7, 64), "cuda")
        want = device.advect(*fp, cop)
        for t_ in fp:  # halos must not matter
            t_[0].fill_(float("nan"))
            t_[:, 0].fill_(float("nan"))
        outp = device.alloc_fields(dp, "cuda")
        launch = device.BoundLaunch(fp, cop, outp, pull=device.self_peers(fp))
        ref = digest(want)
        n_pull = max(1, a.launches // 20)
        bad = 0
        t = time.perf_counter()
        for n in range(n_pull):
            launch()
            if n % 100 == 99:
                bad += digest(outp) != ref
        torch.cuda.synchronize()
        res["k1_pull_2048sq"] = {"launches": n_pull, "mismatches": bad, "s": round(time.perf_counter() - t, 1)}
        del fp, outp, want, launch
        torch.cuda.empty_cache()
    if "ua" in which:  # the UA form, odd nz
        du = pw.make_grid(512, 512, 63)
        fu = device.fill(du, pw.GeneratorSpec.baseline(5))
        cou = device.DeviceCoefficients.from_host(pw.baseline_coefficients(5, 63), "cuda")
        outu = device.alloc_fields(du, "cuda")
        ua = device.make_opts("xmarch_elem")  # forced: the default plan here is K1c's pair rows
        device.advect(*fu, cou, outu, opts=ua)
        ref = digest(outu)
        n_ua = max(1, a.launches // 4)
        bad = 0
        t = time.perf_counter()
        for n in range(n_ua):
            device.advect(*fu, cou, outu, opts=ua)
            if n % 1000 == 999:
                bad += digest(outu) != ref
        torch.cuda.synchronize()
        res["k1_ua_512x512x63"] = {"launches": n_ua, "mismatches": bad, "s": round(time.perf_counter() - t, 1)}
    if "ct" in which:  # the column-tile form K1c: deep even columns and odd nz (pair rows)
        for shape, seed in (((256, 256, 512), 3), ((128, 130, 1031), 4), ((130, 129, 1031), 6)):
            dc = pw.make_grid(*shape)
            fc = device.fill(dc, pw.GeneratorSpec.baseline(seed))
            coc = device.DeviceCoefficients.from_host(pw.baseline_coefficients(seed, shape[2]), "cuda")
            outc = device.alloc_fields(dc, "cuda")
            assert device.describe_plan(dc)["kernel"] == "xmarch_ct"
            device.advect(*fc, coc, outc)
            ref = digest(outc)
            n_ct = max(1, a.launches // 4)
            bad = 0
            t = time.perf_counter()
            for n in range(n_ct):
                device.advect(*fc, coc, outc)
                if n % 1000 == 999:
                    bad += digest(outc) != ref
            torch.cuda.synchronize()
            res["k1c_" + "x".join(map(str, shape))] = {"launches": n_ct, "mismatches": bad,
                                                        "s": round(time.perf_counter() - t, 1)}
            del fc, outc
            torch.cuda.empty_cache()
    if not which & {"k1", "k4"}:
        print(json.dumps(res))
        return
    # K1, C1: same inputs, same outputs, every 1000 launches compared
    d = pw.make_grid(512, 512, 64)
    f = device.fill(d, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, 64), "cuda")
    out = device.alloc_fields(d, "cuda")
    device.advect(*f, co, out)
    ref = digest(out)
    bad = 0
    t = time.perf_counter()
    for n in range(a.launches):
        device.advect(*f, co, out)
        if n % 1000 == 999:
            bad += digest(out) != ref
    torch.cuda.synchronize()
    res["k1_c1"] = {"launches": a.launches, "mismatches": bad, "s": round(time.perf_counter() - t, 1)}
    # K4, C4 block: two identical runs of `steps` steps end in the same bits
    d4 = pw.make_grid(2048, 1024, 128)
    co4 = pw.baseline_coefficients(42, 128)
    digests = []
    t = time.perf_counter()
    for _ in range(2):
        st = Stepper(device.fill(d4, pw.GeneratorSpec.baseline(42)), co4, 0.01)
        st.step(a.steps)
        digests.append(digest(st.fields))
        del st
        torch.cuda.empty_cache()
    res["k4_c4"] = {"steps": a.steps, "runs_equal": digests[0] == digests[1],
                    "s": round(time.perf_counter() - t, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
