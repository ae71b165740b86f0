"""Cost of the fused halo push in K4 on one GPU: a 1x1 decomposition whose
eight neighbours are the block itself (every boundary value is also stored
into the mirroring halo cells, as on 2x4 GPUs minus NVLink), against the
plain K4 step (wrap_halos + step). Prints Gpts/s of each."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import decomp, device  # noqa: E402
from paper_2010_01545_b200.stepper import Stepper  # noqa: E402


def rate(fn, dims, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return dims.cells * reps / (a.elapsed_time(b) / 1e3) / 1e9


def main():
    nx, ny, nz = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2048x1024x128").split("x"))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    gd = pw.make_grid(nx, ny, nz)
    spec = pw.GeneratorSpec.baseline(42)
    co = pw.baseline_coefficients(42, nz)
    plain = Stepper(device.fill(gd, spec), co, 0.1)
    dec = decomp.Decomposition(gd, 1, 1, 0)
    fs = dec.fill_local(spec)
    ex = decomp.HaloExchanger(dec, device="cuda", transport=decomp.ThreadHubTransport(1).bind(0))
    push = decomp.PushStepper(dec, fs, co, 0.1, decomp.LocalPeerRegistry(),
                              decomp.ThreadStreamBarrier(1).bind(0), initial_exchange=ex.exchange)
    res = {}
    for _ in range(3):  # interleaved
        res.setdefault("k2_wrap_plus_k4", []).append(rate(lambda: plain.step(1), gd, reps))
        res.setdefault("k4_fused_push", []).append(rate(lambda: push.step(1), gd, reps))
    torch.cuda.synchronize()
    same = all(torch.equal(a.view(torch.int64), b.view(torch.int64))
               for a, b in zip(plain.fields, push.fields)) if plain.steps_done == push.steps_done else None
    print(json.dumps({"grid": f"{nx}x{ny}x{nz}", **{k: round(sorted(v)[1], 2) for k, v in res.items()},
                      "bitwise_equal": same}))


if __name__ == "__main__":
    main()
