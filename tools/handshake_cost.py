"""Cost of the per-step ordering of the fused multi-GPU paths, on one GPU.

    python tools/handshake_cost.py [--rounds 2000] [--steps 200]

1. Latency: n ranks emulated as host threads, each with its own stream, run
   R rounds of a ~100 us one-thread spin kernel followed by the barrier —
   the neighbour flag handshake (decomp.FlagHandshake: stream-ordered flag
   writes + waits) or the thread-emulation barrier (events + a host barrier,
   a stand-in for the round-1 NCCL all-reduce, which cannot run with 8 ranks
   on one GPU) — and without any; the difference per round is the barrier's
   GPU-side critical-path cost (the host enqueues ahead of the GPU).
2. In context: the C2 strong-scaling cut (1024x1024x64 over 2x4 blocks of
   512x256x64), every block evaluated with the halo pull, 8 threads on one
   GPU, with the flag handshake / the thread barrier / no ordering at all.
3. Projection for 8 GPUs (one block per GPU): t_step = t_block + t_handshake,
   efficiency = t_C2_on_1_GPU / (8 * t_step).
Prints one JSON line per measurement.
"""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2010_01545_b200 as pw  # noqa: E402
from paper_2010_01545_b200 import decomp, device  # noqa: E402


def run_threads(n, fn):
    out, errs = [None] * n, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, s)
            s.synchronize()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
    ts = [threading.Thread(target=worker, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


def latency(px, py, rounds, kind, sleep_cycles=0):
    gd = pw.make_grid(8 * px, 8 * py, 4)
    n = px * py
    decs = [decomp.Decomposition(gd, px, py, r) for r in range(n)]
    if kind == "flags":
        reg = decomp.LocalPeerRegistry()
        bars = [decomp.FlagHandshake(d, reg, device="cuda") for d in decs]
    elif kind == "thread_barrier":
        tb = decomp.ThreadStreamBarrier(n)
        bars = [tb.bind(r) for r in range(n)]
    else:
        bars = [None] * n
    go = threading.Barrier(n)

    def rank(r, s):
        if bars[r] is not None:
            bars[r](s)
        s.synchronize()
        go.wait()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(s)
        for _ in range(rounds):
            if sleep_cycles:
                torch.cuda._sleep(sleep_cycles)  # one thread spinning: the "step"
            if bars[r] is not None:
                bars[r](s)
        b.record(s)
        s.synchronize()
        return a.elapsed_time(b) * 1e3 / rounds, (time.perf_counter() - t0) * 1e6 / rounds
    res = run_threads(n, rank)
    return max(x[0] for x in res), max(x[1] for x in res)


def pull_c2(kind, steps):
    gd = pw.make_grid(1024, 1024, 64)
    px, py = 2, 4
    n = px * py
    spec = pw.GeneratorSpec.baseline(42)
    co = pw.baseline_coefficients(42, 64)
    decs = [decomp.Decomposition(gd, px, py, r) for r in range(n)]
    reg = decomp.LocalPeerRegistry()
    if kind == "flags":
        freg = decomp.LocalPeerRegistry()
        bars = [decomp.FlagHandshake(d, freg, device="cuda") for d in decs]
    elif kind == "thread_barrier":
        tb = decomp.ThreadStreamBarrier(n)
        bars = [tb.bind(r) for r in range(n)]
    else:
        bars = [None] * n
    ready = threading.Barrier(n)

    def rank(r, s):
        dec = decs[r]
        fs = dec.fill_local(spec)
        ev = decomp.PullEvaluator(dec, fs, co, reg, bars[r])
        out = device.alloc_fields(dec.local_dims, "cuda")
        ready.wait()
        if bars[r] is None:
            ev.barrier = None
        for _ in range(5):
            ev.evaluate(out, stream=s)
        s.synchronize()
        ready.wait()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(steps):
            ev.evaluate(out, stream=s)
        b.record(s)
        s.synchronize()
        return a.elapsed_time(b) * 1e3 / steps
    return max(run_threads(n, rank))


def block_alone(steps):
    """One 512x256x64 block (C2 at 2x4) evaluated with the halo pull, its
    neighbours being itself: the per-GPU kernel time of the 8-GPU run."""
    gd = pw.make_grid(512, 256, 64)
    f = device.fill(gd, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, 64), f[0].device)
    out = device.alloc_fields(gd, f[0].device)
    launch = device.BoundLaunch(f, co, out, pull=device.self_peers(f))
    full = pw.make_grid(1024, 1024, 64)
    g = device.fill(full, pw.GeneratorSpec.baseline(42))
    o2 = device.alloc_fields(full, g[0].device)
    whole = device.BoundLaunch(g, co, o2)
    res = {}
    for name, fn in (("block_pull_us", launch), ("c2_whole_1gpu_us", whole)):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[name] = a.elapsed_time(b) * 1e3 / steps
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=2000)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    # each round: a one-thread spin kernel of ~100 us (the "step", long enough
    # that the host enqueues ahead and only the GPU-side cost remains), then
    # the barrier; handshake latency = round time - spin-only round time
    try:
        cyc = int(100e-6 * torch.cuda.clock_rate() * 1e6)
    except Exception:  # noqa: BLE001 - no NVML
        cyc = 196500
    lat = {}
    for px, py in ((1, 2), (2, 4)):
        base = None
        for kind in ("none", "flags", "thread_barrier"):
            dev_us, host_us = latency(px, py, a.rounds // 4, kind, sleep_cycles=cyc)
            if kind == "none":
                base = dev_us
            lat[(px, py, kind)] = dev_us - base
            print(json.dumps({"what": "latency", "decomposition": f"{px}x{py}", "barrier": kind,
                              "us_per_round_device": round(dev_us, 2),
                              "us_per_round_host": round(host_us, 2),
                              "barrier_us": round(dev_us - base, 2)}), flush=True)
    for kind in ("flags", "thread_barrier", "none"):
        us = pull_c2(kind, a.steps)
        print(json.dumps({"what": "C2 2x4 pulled evaluations, 8 emulated ranks on one GPU",
                          "barrier": kind, "us_per_step_all_8_blocks": round(us, 1)}), flush=True)
    blk = block_alone(a.steps)
    hs = lat[(2, 4, "flags")]
    t_step = blk["block_pull_us"] + hs
    print(json.dumps({"what": "projection, C2 strong scaling on 8 GPUs (2x4)", **{k: round(v, 2) for k, v in blk.items()},
                      "handshake_us": round(hs, 2), "t_step_us": round(t_step, 2),
                      "efficiency": round(blk["c2_whole_1gpu_us"] / (8 * t_step), 4),
                      "note": "handshake latency measured with 8 emulated ranks on one GPU "
                              "(local writes; over NVLink add the remote write latency, ~1-2 us)"}),
          flush=True)


if __name__ == "__main__":
    main()
