"""Live DRAM traffic from the hardware counters (libpwadv_traffic.so, CUPTI
range profiler) against the plan: K1 at C1 must move close to
its algorithmic 48 B/point (reads about once, writes once) — traffic well
above it would mean wasted re-reads."""

import pytest
import torch

import paper_2010_01545_b200 as pw
from paper_2010_01545_b200 import device, traffic

pytestmark = pytest.mark.gpu


def _case(nx, ny, nz):
    dims = pw.make_grid(nx, ny, nz)
    f = device.fill(dims, pw.GeneratorSpec.baseline(42))
    co = device.DeviceCoefficients.from_host(pw.baseline_coefficients(42, nz), f[0].device)
    return dims, f, co


def test_k1_c1_dram_bytes_near_plan():
    dims, f, co = _case(512, 512, 64)
    out = device.alloc_fields(dims, f[0].device)
    r = traffic.measure(lambda: device.advect(*f, co, out), plan_bytes=48 * dims.cells)
    assert r["kernels"] == 1, r
    # reads: the padded inputs once (+ halo planes/columns mostly from L2);
    # writes: the outputs once — some may still be dirty in L2 at kernel end
    assert 0.97 * 24 * dims.cells <= r["dram_read_bytes"] <= 1.10 * 24 * dims.cells, r
    assert 0.70 * 24 * dims.cells <= r["dram_write_bytes"] <= 1.05 * 24 * dims.cells, r
    assert 0.8 <= r["ratio_to_plan"] <= 1.1, r
    assert r["kernel_us"] > 50, r
    # fp64 pipe (no tensor cores: not a contraction): busy but not the bound;
    # the census is 63 flop per point (operation_census), carried sums reuse
    # some of them across levels, every flop is one lane of a DADD/DMUL
    assert 20.0 <= r["fp64_pipe_pct"] <= 100.0, r
    assert 20 * dims.cells / 32 <= r["fp64_warp_inst"] <= 130 * dims.cells / 32, r


def test_sum_over_several_launches_and_step():
    dims, f, co = _case(256, 256, 64)
    out = device.alloc_fields(dims, f[0].device)
    nxt = device.alloc_fields(dims, f[0].device)

    def three():
        device.advect(*f, co, out)
        device.advect(*f, co, out)
        device.step(*f, co, 0.1, nxt)
    r = traffic.measure(three, plan_bytes=3 * 48 * dims.cells)
    assert r["kernels"] == 3, r
    assert r["dram_read_bytes"] > 0 and r["dram_write_bytes"] > 0
    assert 0.0 < r["fp64_pipe_pct"] <= 100.0 and r["fp64_warp_inst"] > 0, r


def test_run_schedule_reports_measured_traffic():
    dims = pw.make_grid(128, 96, 64)
    fields = pw.fill_fields(dims, pw.GeneratorSpec.random(3))
    co = pw.default_coefficients(64)
    src, tr, wall = pw.run_schedule(fields, co, pw.ScheduleSpec("xmarch", engines=2,
                                                                measure_traffic=True))
    m = tr.measured
    assert m is not None and "error" not in m, m
    assert m["kernels"] == 2
    assert m["plan_bytes"] == 8 * (tr.device.external_reads + tr.device.external_writes)
    assert 0.5 < m["ratio_to_plan"] < 1.5, m
    # the reference variants keep the reference's counters; equality ignores `measured`
    _, tr2, _ = pw.run_schedule(fields, co, pw.ScheduleSpec("reference", engines=2))
    assert tr2.measured is None and tr2.device is not None
    assert wall > 0
