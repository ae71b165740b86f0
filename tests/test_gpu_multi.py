"""Multi-process multi-GPU tests (one process per rank, CUDA IPC).

With >= 2 GPUs: one process per GPU, NCCL + CUDA IPC over NVLink — the
production paths exactly as `bench.py --gpus N` runs them. With fewer GPUs
than ranks (this round's boxes have one) the same workers and the same
bench command run as a DRY RUN with every rank on cuda:0: the processes
time-slice the GPU, torch.distributed runs on gloo (NCCL refuses two ranks
on one device) with the halo messages staged through the host, and the
fused paths map each other's buffers through CUDA IPC as they would across
GPUs. No kernel waits on another kernel (the handshake is stream memory
operations; the barrier fallback is a host-side all-reduce), so sharing a
GPU cannot deadlock; rates from a dry run mean nothing and are not read.
They run:
HaloExchanger over DistTransport (NCCL batch_isend_irecv) with
advect_overlapped, the halo-pull PullEvaluator and the fused PushStepper with IpcPeerRegistry +
NcclBarrier, each compared bitwise with the single-domain result computed in
the same process.
"""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _shared_gpu_ok() -> bool:
    """Several processes may open cuda:0 (compute mode Default): the dry run
    needs it; an exclusive-process GPU skips those cases instead of failing."""
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=compute_mode", "--format=csv,noheader", "-i", "0"],
                             capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception:  # noqa: BLE001
        return True
    return out in ("", "Default")


def _skip_unless_shareable(share: bool) -> None:
    if share and not _shared_gpu_ok():
        pytest.skip("GPU 0 is in an exclusive compute mode: no shared-GPU dry run")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, px, py, q, share=False, nz=64):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        import paper_2010_01545_b200 as pw
        from paper_2010_01545_b200 import decomp, device
        from paper_2010_01545_b200.stepper import Stepper
        gpu = 0 if share else rank
        torch.cuda.set_device(gpu)
        dev = torch.device("cuda", gpu)
        if share:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        gd = pw.make_grid(64, 48, nz)
        spec = pw.GeneratorSpec.baseline(21)
        co = pw.baseline_coefficients(21, gd.nz)
        dec = decomp.Decomposition(gd, px, py, rank)
        # single-domain references on this GPU
        full = device.fill(gd, spec, device=dev)
        want_adv = device.advect(*full, co)
        single = Stepper(device.fill(gd, spec, device=dev), co, 0.1)
        single.step(5)
        want_step = single.fields
        torch.cuda.synchronize()
        ok = True
        # advect with the NCCL exchange overlapped with the interior
        fs = dec.fill_local(spec, device=dev)
        ex = decomp.HaloExchanger(dec, dev)
        out = device.alloc_fields(dec.local_dims, dev)
        ex.advect_overlapped(fs, co, out)
        torch.cuda.synchronize()
        xo, bx, yo, by = dec.block()
        for o, w in zip(out, want_adv):
            ok &= torch.equal(o[1:-1, 1:-1].view(torch.int64),
                              w[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].view(torch.int64))
        # the fused step: peer stores over CUDA IPC + one NCCL barrier per step
        fs2 = dec.fill_local(spec, device=dev)
        reg = decomp.IpcPeerRegistry(dec)
        st = decomp.PushStepper(dec, fs2, co, 0.1, reg, decomp.NcclBarrier(dev),
                                initial_exchange=lambda f: ex.exchange(f))
        st.step(5)
        torch.cuda.synchronize()
        for f, w in zip(st.fields, want_step):
            ok &= torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64))
        # K1 with the halo pull: neighbours' buffers over CUDA IPC, halos NaN
        fs3 = dec.fill_local(spec, device=dev)
        for f in fs3:
            f[0].fill_(float("nan")); f[-1].fill_(float("nan"))  # noqa: E702
            f[:, 0].fill_(float("nan")); f[:, -1].fill_(float("nan"))  # noqa: E702
        reg3 = decomp.IpcPeerRegistry(dec)
        ev = decomp.PullEvaluator(dec, fs3, co, reg3, decomp.NcclBarrier(dev))
        out3 = device.alloc_fields(dec.local_dims, dev)
        ev.evaluate(out3)
        torch.cuda.synchronize()
        ok &= ev.mode == ("fused" if nz == 64 else "gather")
        for o, w in zip(out3, want_adv):
            ok &= torch.equal(o[1:-1, 1:-1].contiguous().view(torch.int64),
                              w[1 + xo:1 + xo + bx, 1 + yo:1 + yo + by].contiguous().view(torch.int64))
        # steps with the halo cells pulled every step (fused on the aligned
        # X-march, K2p gather + the planner's K4 otherwise)
        fs4 = dec.fill_local(spec, device=dev)
        reg4 = decomp.IpcPeerRegistry(dec)
        ps = decomp.PullStepper(dec, fs4, co, 0.1, reg4, decomp.NcclBarrier(dev))
        ps.step(5)
        final = ps.refreshed_fields()
        torch.cuda.synchronize()
        for f, w in zip(final, want_step):
            ok &= torch.equal(f.view(torch.int64), dec.local_view(w).contiguous().view(torch.int64))
        dist.barrier()
        reg4.close()
        reg3.close()
        reg.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


def _run_torchrun(cmd, env, cwd, timeout):
    """subprocess.run for a torchrun command in its own process group: on a
    timeout the whole group (torchrun and its ranks) is killed, so no rank is
    left holding the GPU."""
    import signal
    import subprocess
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=cwd,
                         env=env, start_new_session=True)
    try:
        out, err = p.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, err = p.communicate()
        raise AssertionError(f"timed out after {timeout} s: {err[-2000:]}")
    return subprocess.CompletedProcess(cmd, p.returncode, out, err)


def _run_ranks(world, px, py, share, nz=64):
    """One process per rank running _worker; (rank, ok, error) of every rank.
    Ranks still alive at the end — a hang, a crash of their peers — are killed,
    so none is left holding the GPU for the tests that follow."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, py, q, share, nz)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        results = [q.get(timeout=600) for _ in range(world)]
        for p in procs:
            p.join(timeout=120)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    assert sorted(r for r, _, _ in results) == list(range(world))
    return results


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
@pytest.mark.parametrize("px,py", [(1, 2), (2, 1), (2, 2), (2, 4)])
def test_nccl_exchange_and_fused_ipc_step(px, py):
    world = px * py
    share = world > NGPU  # dry run: the ranks share cuda:0 (module docstring)
    if share and world > 4:
        pytest.skip(f"needs {world} GPUs (the shared-GPU dry run stops at 4 ranks)")
    _skip_unless_shareable(share)
    for r, ok, err in _run_ranks(world, px, py, share):
        assert ok, (r, err)


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
@pytest.mark.parametrize("px,py,nz", [(1, 2, 63), (2, 2, 300)])
def test_off_xmarch_blocks_across_processes(px, py, nz):
    """Odd nz / deep columns (blocks the planner gives to the UA form or K1c):
    the exchange, the fused push step and the pull evaluation — there the K2p
    gather kernel reading the other processes' buffers, then the planner's
    kernel — bitwise against the single-domain result."""
    world = px * py
    share = world > NGPU
    _skip_unless_shareable(share)
    for r, ok, err in _run_ranks(world, px, py, share, nz):
        assert ok, (r, err)


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
@pytest.mark.parametrize("config", ["c1", "c4"])
def test_bench_under_torchrun(config):
    """bench.py as the driver launches it for N=2 (torchrun, one rank per GPU;
    on a one-GPU box the shared-GPU dry run): one JSON line from rank 0, the
    fused multi-GPU path in use (halo pull for evaluations, peer-store push
    for steps), every rank's block bit-exact against the oracle."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"),
           "--gpus", "2", "--config", config, "--steps", "10", "--warmup", "3", "--no-cpu", "--no-e2e"]
    env = dict(os.environ)
    _skip_unless_shareable(NGPU < 2)
    if NGPU < 2:
        env["PWADV_BENCH_SHARE_GPU"] = "1"
    r = _run_torchrun(cmd, env, root, 900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    step = d["config"].get("multi_gpu_step", "")
    assert ("halo pull" in step) if config == "c1" else ("peer stores" in step), (step, r.stderr[-1500:])
    assert d["parity"]["bitwise_equal"] is True, d["parity"]
    assert ("dry_run" in d["config"]) == (NGPU < 2)


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
@pytest.mark.parametrize("where,config", [("handshake", "c1"), ("fused", "c1"), ("fused", "c4")])
def test_bench_ranks_fall_back_together(where, config):
    """A failure on ONE rank (injected on the last: PWADV_BENCH_FAIL) while the
    others succeed: all ranks must take the same fallback — the all-reduce
    barrier when the flag handshake cannot be set up, the exchange-and-overlap
    step when the fused path cannot — and still print the line (ADVICE r1:
    ranks that diverge here hang in mismatched collectives)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(root / "bench.py"),
           "--gpus", "2", "--config", config, "--steps", "5", "--warmup", "3", "--no-cpu", "--no-e2e",
           "--no-traffic"]
    env = dict(os.environ, PWADV_BENCH_FAIL=where)
    _skip_unless_shareable(NGPU < 2)
    if NGPU < 2:
        env["PWADV_BENCH_SHARE_GPU"] = "1"
    r = _run_torchrun(cmd, env, root, 240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    step = d["config"].get("multi_gpu_step", "")
    assert d["n_gpus"] == 2 and d["value"] > 0
    if where == "handshake":
        assert "all-reduce barrier" in step, step
        assert d["parity"]["bitwise_equal"] is True, d["parity"]
    else:
        assert step.startswith("NCCL exchange overlapped"), step
