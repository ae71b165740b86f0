"""Cost of the fused halo pull in K1 on one GPU.

    python tools/pull_cost.py [NXxNYxNZ] [reps] [flags]

(a) K1 on a block whose halos are already valid; (b) K2 wrap + K1 (the
periodic evaluation without the pull); (c) K1-pull with the block as all
eight of its own neighbours (the periodic evaluation in one launch: halo
planes / columns come from the block's own interior); (d) the global grid cut
2x4 on this GPU, each block's K1-pull reading the other blocks' buffers
(the copies of the 2x4 decomposition minus NVLink), timed back to back.
Prints Gpts/s of each (median of 3 interleaved rounds) and whether (c) and
(d) equal (a) bitwise."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import decomp, device  # noqa: E402


def rate(fn, cells, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return cells * reps / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    nx, ny, nz = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048x2048x64").split("x"))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # e.g. 128: ordinary launches (no PDL)
    opts = device.make_opts("xmarch", flags=flags)
    gd = pw.make_grid(nx, ny, nz)
    spec = pw.GeneratorSpec.baseline(42)
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), "cuda")
    f = device.fill(gd, spec)
    ref = device.advect(*f, co)
    out = device.alloc_fields(gd, "cuda")
    peers = device.self_peers(f)
    pull = device.BoundLaunch(f, co, out, pull=peers, opts=opts)
    plain = device.BoundLaunch(f, co, out, opts=opts)
    # 2x4 blocks of the same grid on this GPU
    reg = decomp.LocalPeerRegistry()
    blocks = []
    for r in range(8):
        dec = decomp.Decomposition(gd, 2, 4, r)
        fs = dec.fill_local(spec)
        ev = decomp.PullEvaluator(dec, fs, co, reg)
        blocks.append((dec, ev, device.alloc_fields(dec.local_dims, "cuda")))

    def wrap_k1():
        device.wrap_halos(*f)
        plain()

    def blocks_2x4():
        for _, ev, o in blocks:
            ev.evaluate(o, sync=False)

    res = {}
    for _ in range(3):  # interleaved
        res.setdefault("k1_valid_halos", []).append(rate(plain, gd.cells, reps))
        res.setdefault("k2_wrap_plus_k1", []).append(rate(wrap_k1, gd.cells, reps))
        res.setdefault("k1_pull_self", []).append(rate(pull, gd.cells, reps))
        res.setdefault("k1_pull_2x4_blocks", []).append(rate(blocks_2x4, gd.cells, reps))
    pull()
    torch.cuda.synchronize()
    same_self = all(torch.equal(a.view(torch.int64), b.view(torch.int64)) for a, b in zip(out, ref))
    same_blocks = True
    for dec, _, o in blocks:
        xo, bx, yo, by = dec.block()
        for a, b in zip(o, ref):
            same_blocks &= torch.equal(a[1:-1, 1:-1].contiguous().view(torch.int64),
                                       b[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].contiguous().view(torch.int64))
    print(json.dumps({"grid": f"{nx}x{ny}x{nz}", **{k: round(sorted(v)[1], 2) for k, v in res.items()},
                      "pull_self_bitwise": same_self, "pull_2x4_bitwise": bool(same_blocks)}))


if __name__ == "__main__":
    main()
