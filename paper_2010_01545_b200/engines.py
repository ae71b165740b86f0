"""Execution variants, X-slab engines and the bitwise comparator (mirror of
reference schedules.py:27-272), executed on the B200.

`run_schedule(fields, coeffs, spec) -> (SourceSet, TrafficReport, wall)` keeps
the reference's signature and errors. Variants:

* "xmarch" (default) — K1, the bulk-copy plane-ring X-march kernel;
* "simple" — K1, one thread per point (independent second implementation);
* "xmarch_fma" / "simple_fma" — DFMA-contracted builds (not bit-exact;
  normwise error <= 1e-12, reported by compare_outputs);
* the reference's FPGA data-movement variants ("reference",
  "column_buffered", "y_batched", "x_reordered", schedules.py:27) are
  accepted for drop-in compatibility and all run as "xmarch": the reference
  guarantees they are bitwise identical (schedules.py:1-8), and the X-march
  is the GPU form of "x_reordered" (schedules.py:160-191).

`engines` splits the interior into balanced X slabs exactly like
partition_domain (schedules.py:65-75); each slab is one box launch, outputs
are bitwise independent of the engine count. `wall` is device time measured
with CUDA events around the launches (inputs already resident), the analogue
of the reference's perf_counter around its compute (schedules.py:220-228).
`TrafficReport` counts element traffic of the chosen GPU plan: HBM reads
(staged plane tiles, halo columns and segment-boundary planes included),
HBM writes, shared-memory reads/fills, and shared memory per CTA.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .layout import Field3D, GridDims, SourceSet

GPU_VARIANTS = ("xmarch", "simple", "xmarch_fma", "simple_fma")
REFERENCE_VARIANTS = ("reference", "column_buffered", "y_batched", "x_reordered")
VARIANTS = GPU_VARIANTS + REFERENCE_VARIANTS


@dataclass(frozen=True)
class Slab:
    """One engine's interior X range, 1-based, half-open (reference schedules.py:53-62)."""

    x_begin: int
    x_end: int

    @property
    def width(self) -> int:
        return self.x_end - self.x_begin


def partition_domain(dims, engines: int) -> list[Slab]:
    """Contiguous X slabs, widths differing by <= 1, wider first (schedules.py:65-75)."""
    if engines < 1 or engines > dims.nx:
        raise ValueError(f"engines must be in 1..nx={dims.nx}, got {engines}")
    q, r = divmod(dims.nx, engines)
    out, start = [], 1
    for e in range(engines):
        end = start + q + (1 if e < r else 0)
        out.append(Slab(start, end))
        start = end
    return out


@dataclass(frozen=True)
class ScheduleSpec:
    variant: str = "xmarch"
    y_batch: int = 64
    engines: int = 1

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}; one of {VARIANTS}")
        if self.y_batch < 1:
            raise ValueError("y_batch must be >= 1")
        if self.engines < 1:
            raise ValueError("engines must be >= 1")

    def validate(self, dims) -> None:
        if self.engines > dims.nx:
            raise ValueError(f"engines={self.engines} exceeds nx={dims.nx}")
        if self.variant in ("y_batched", "x_reordered") and self.y_batch > dims.ny:
            raise ValueError(f"y_batch={self.y_batch} exceeds ny={dims.ny}")

    @property
    def kernel_variant(self) -> str:
        return self.variant if self.variant in GPU_VARIANTS else "xmarch"


@dataclass
class TrafficReport:
    """Element traffic of one run (units: float64 elements; scratch in bytes)."""

    external_reads: int = 0
    external_writes: int = 0
    local_reads: int = 0
    local_writes: int = 0
    scratch_bytes_peak: int = 0

    def merge(self, other: "TrafficReport") -> None:
        self.external_reads += other.external_reads
        self.external_writes += other.external_writes
        self.local_reads += other.local_reads
        self.local_writes += other.local_writes
        self.scratch_bytes_peak = max(self.scratch_bytes_peak, other.scratch_bytes_peak)


def plan_traffic(dims: GridDims, box, plan: dict) -> TrafficReport:
    """Traffic of one box launch under `plan` (device.describe_plan)."""
    x0, x1, y0, y1 = box
    nbx, nby, nz = x1 - x0, y1 - y0, dims.nz
    tr = TrafficReport()
    if nbx <= 0 or nby <= 0:
        return tr
    tr.external_writes = 3 * nbx * nby * nz  # all levels of interior columns (level 0 = +0.0)
    if plan["kernel"] == "simple":
        # 27 distinct operands per point at k >= 1 (9 per field), via L1/L2
        tr.external_reads = 27 * nbx * nby * (nz - 1)
        return tr
    tj, nch = plan["tile_j"], plan.get("chunks", 1)
    nstrips, nlong = plan["strips"], plan.get("long_strips", 0)
    widths = [min(tj, nby - s * tj) for s in range(nstrips)]
    if plan.get("spare_ctas", 0) > 0:
        # spare-tail plan: nch main chunks of mlen planes + one tail chunk per strip
        mlen = plan["main_chunk_planes"]
        per_col = nch * (mlen + 2) + (nbx - nch * mlen + 2)
        tr.external_reads = 3 * nz * per_col * sum(w + 2 for w in widths)
        tr.local_writes = tr.external_reads
        tr.local_reads = 9 * nbx * nby * nz
        tr.scratch_bytes_peak = int(plan["smem_bytes"])
        return tr
    # work units (pwadv_advect.cu unit_at): strips 0..nlong-1 whole, the rest
    # in nch X chunks; each unit streams its planes + one on each side
    planes = sum((nbx + 2) * (widths[s] + 2) for s in range(nlong))
    for s in range(nlong, nstrips):
        for chunk in range(nch):
            ib, ie = nbx * chunk // nch, nbx * (chunk + 1) // nch
            planes += (ie - ib + 2) * (widths[s] + 2)
    tr.external_reads = 3 * nz * planes
    tr.local_writes = tr.external_reads
    # 9 paired shared loads per thread per plane step (2 points) = 9 per point
    tr.local_reads = 9 * nbx * nby * nz
    tr.scratch_bytes_peak = int(plan["smem_bytes"])
    return tr


def run_schedule(fields, coeffs, spec: ScheduleSpec):
    """Execute one schedule on the GPU; returns (sources, traffic, wall seconds)."""
    import torch
    from . import device

    dims = fields.dims
    if len(coeffs.tzc1) != dims.nz:
        raise ValueError(f"coefficient length {len(coeffs.tzc1)} != nz {dims.nz}")
    spec.validate(dims)
    slabs = partition_domain(dims, spec.engines)
    gd = GridDims(dims.nx, dims.ny, dims.nz)
    dev = torch.device("cuda")
    u, v, w = (torch.from_numpy(np.ascontiguousarray(f.data, dtype=np.float64)).to(dev)
               for f in (fields.u, fields.v, fields.w))
    dc = device.DeviceCoefficients.from_host(coeffs, dev)
    out = device.alloc_fields(gd, dev)
    opts = device.make_opts(spec.kernel_variant)
    traffic = TrafficReport()
    for s in slabs:
        box = (s.x_begin, s.x_end, 1, gd.ny + 1)
        traffic.merge(plan_traffic(gd, box, device.describe_plan(gd, box, opts, dev.index or 0)))
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in slabs:
        device.advect(u, v, w, dc, out, box=(s.x_begin, s.x_end, 1, gd.ny + 1), opts=opts)
    t1.record()
    t1.synchronize()
    wall = t0.elapsed_time(t1) / 1e3
    res = SourceSet(*(Field3D(gd, t.cpu().numpy()) for t in out))
    return res, traffic, wall


@dataclass(frozen=True)
class OutputComparison:
    bitwise_equal: bool
    max_abs_diff: float
    max_ulp_diff: int


def _ordered(arr: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(arr).reshape(-1).view(np.int64)
    return np.where(b >= 0, b, np.int64(-(2**63)) - b)


def _ulp_distance(a: np.ndarray, b: np.ndarray) -> int:
    oa, ob = _ordered(a), _ordered(b)
    same = (oa >= 0) == (ob >= 0)
    worst = int(np.abs(oa[same] - ob[same]).max()) if same.any() else 0
    if (~same).any():
        cross = np.abs(oa[~same]).astype(np.uint64) + np.abs(ob[~same]).astype(np.uint64)
        worst = max(worst, int(cross.max()))
    return worst


def compare_outputs(a: SourceSet, b: SourceSet) -> OutputComparison:
    """Exact comparison over the full padded arrays (reference schedules.py:261-272);
    a signed-zero difference counts as 1 ULP."""
    if a.dims != b.dims:
        raise ValueError(f"dims mismatch: {a.dims} vs {b.dims}")
    pairs = [(np.asarray(x.data), np.asarray(y.data))
             for x, y in ((a.su, b.su), (a.sv, b.sv), (a.sw, b.sw))]
    if all(np.array_equal(np.ascontiguousarray(x).view(np.int64),
                          np.ascontiguousarray(y).view(np.int64)) for x, y in pairs):
        return OutputComparison(True, 0.0, 0)
    max_abs = max(float(np.abs(x - y).max()) for x, y in pairs)
    return OutputComparison(False, max_abs, max(1, max(_ulp_distance(x, y) for x, y in pairs)))
