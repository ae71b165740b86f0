"""Execution variants, X-slab engines and the bitwise comparator (mirror of
reference schedules.py:27-272), executed on the B200.

`run_schedule(fields, coeffs, spec) -> (SourceSet, TrafficReport, wall)` keeps
the reference's signature, defaults and errors. Variants:

* the reference's four ("reference" — the default, as in
  schedules.py:80 —, "column_buffered", "y_batched", "x_reordered",
  schedules.py:27) all run as K1, the bulk-copy plane-ring X-march kernel:
  the reference guarantees they are bitwise identical (schedules.py:1-8),
  and the X-march is the GPU form of "x_reordered" (schedules.py:160-191).
  Their TrafficReport keeps the reference's contract: the element traffic
  of that variant's data movement, in closed form from dims and spec
  (schedules.py:117-191; docs/model-notes.md §3), identical to what the
  reference counts;
* the GPU's own: "xmarch" (K1), "simple" (one thread per point, an
  independent second implementation), "xmarch_fma" / "simple_fma" (DFMA-
  contracted builds: not bit-exact; normwise error <= 1e-12, reported by
  compare_outputs). Their TrafficReport counts the chosen GPU plan's element
  traffic: HBM reads (staged plane tiles, halo columns and segment-boundary
  planes included), HBM writes, shared-memory reads/fills, shared memory
  per CTA.

Every report also carries `device` — the GPU plan's counts — and, with
`ScheduleSpec(measure_traffic=True)`, `measured`: the DRAM bytes the launches
actually moved, read from the hardware counters (CUPTI range profiler,
libpwadv_traffic.so), beside the plan's bytes and their ratio. Neither takes
part in equality, so the reference's determinism checks hold.

`engines` splits the interior into balanced X slabs exactly like
partition_domain (schedules.py:65-75); each slab is one box launch, outputs
are bitwise independent of the engine count. `wall` is perf_counter time of
the whole call after the output allocation, as the reference measures it
(schedules.py:218-228): the upload of u, v, w, the launches and the download
of su, sv, sw.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .layout import Field3D, GridDims, SourceSet

GPU_VARIANTS = ("xmarch", "simple", "xmarch_fma", "simple_fma")
REFERENCE_VARIANTS = ("reference", "column_buffered", "y_batched", "x_reordered")
# the reference's variant tuple, exactly (schedules.py:27: code that loops over
# VARIANTS expects bitwise-identical results from each); the GPU's own
# variants are accepted by ScheduleSpec too, listed in ALL_VARIANTS
VARIANTS = REFERENCE_VARIANTS
ALL_VARIANTS = REFERENCE_VARIANTS + GPU_VARIANTS


def _xshift_roles(roles) -> tuple:
    """Scratch blocks of the X-reordered schedule: the compute roles, closed
    under "a role with dx <= 0 has its dx+1 parent" (the plane shift feeds
    dx from dx+1), as schedules.py:30-50 defines them: 22 for COMPUTE_ROLES."""
    have = set(roles)
    todo = list(have)
    while todo:
        f, dx, dy = todo.pop()
        if dx <= 0 and (f, dx + 1, dy) not in have:
            have.add((f, dx + 1, dy))
            todo.append((f, dx + 1, dy))
    return tuple(sorted(have))


def _compute_roles():
    from .stencil import COMPUTE_ROLES
    return COMPUTE_ROLES


XSHIFT_ROLES = _xshift_roles(_compute_roles())


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
    variant: str = "reference"
    y_batch: int = 64
    engines: int = 1
    measure_traffic: bool = False  # GPU extension: DRAM bytes from the hardware counters

    def __post_init__(self):
        if self.variant not in ALL_VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}; one of {ALL_VARIANTS}")
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
    """Element traffic of one run (units: float64 elements; scratch in bytes).
    `device` (GPU plan counts) and `measured` (DRAM bytes from the counters)
    are extensions that do not take part in equality."""

    external_reads: int = 0
    external_writes: int = 0
    local_reads: int = 0
    local_writes: int = 0
    scratch_bytes_peak: int = 0
    device: "TrafficReport | None" = field(default=None, compare=False, repr=False)
    measured: "dict | None" = field(default=None, compare=False)

    def merge(self, other: "TrafficReport") -> None:
        self.external_reads += other.external_reads
        self.external_writes += other.external_writes
        self.local_reads += other.local_reads
        self.local_writes += other.local_writes
        self.scratch_bytes_peak = max(self.scratch_bytes_peak, other.scratch_bytes_peak)


def reference_traffic(dims, spec: "ScheduleSpec", slabs) -> TrafficReport:
    """The element traffic the reference counts for its variant `spec.variant`
    over `slabs` (schedules.py:117-191), in closed form — it depends only on
    dims and spec (docs/model-notes.md §3): per output column 54 operand
    touches per mid level and 45 at the top; column_buffered / y_batched
    copy the 17 role columns of every output column into scratch;
    x_reordered prefetches all XSHIFT_ROLES blocks once per slab and Y batch,
    then per X step shifts the dx <= 0 blocks down and fetches the dx = +1
    ones."""
    from .stencil import COMPUTE_ROLES, reads_per_point
    nx, ny, nz = dims.nx, dims.ny, dims.nz
    col = reads_per_point(False) * (nz - 2) + reads_per_point(True)
    nrole = len(COMPUTE_ROLES)
    tr = TrafficReport(external_writes=3 * nx * ny * (nz - 1))
    v = spec.variant
    if v == "reference":
        tr.external_reads = nx * ny * col
    elif v in ("column_buffered", "y_batched"):
        batch = 1 if v == "column_buffered" else spec.y_batch
        tr.external_reads = nrole * nx * ny * nz
        tr.local_writes = tr.external_reads
        tr.local_reads = nx * ny * col
        tr.scratch_bytes_peak = nrole * min(batch, ny) * nz * 8
    else:  # x_reordered
        nshift = sum(1 for r in XSHIFT_ROLES if r[1] <= 0)
        nfetch = len(XSHIFT_ROLES) - nshift
        for s in slabs:
            steps = s.width - 1
            fetched = ny * nz * (len(XSHIFT_ROLES) + nfetch * steps)
            shifted = nshift * steps * ny * nz
            tr.external_reads += fetched
            tr.local_writes += fetched + shifted
            tr.local_reads += shifted + s.width * ny * col
        tr.scratch_bytes_peak = len(XSHIFT_ROLES) * min(spec.y_batch, ny) * nz * 8
    return tr


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
    """Execute one schedule on the GPU; returns (sources, traffic, wall seconds)
    (reference schedules.py:207-232)."""
    import torch
    from . import device

    dims = fields.dims
    if len(coeffs.tzc1) != dims.nz:
        raise ValueError(f"coefficient length {len(coeffs.tzc1)} != nz {dims.nz}")
    spec.validate(dims)
    slabs = partition_domain(dims, spec.engines)
    gd = GridDims(dims.nx, dims.ny, dims.nz)
    dev = torch.device("cuda", torch.cuda.current_device())
    opts = device.make_opts(spec.kernel_variant)
    boxes = [(s.x_begin, s.x_end, 1, gd.ny + 1) for s in slabs]
    plan = TrafficReport()
    for box in boxes:
        plan.merge(plan_traffic(gd, box, device.describe_plan(gd, box, opts, dev.index)))
    if spec.variant in REFERENCE_VARIANTS:
        traffic = reference_traffic(gd, spec, slabs)
    else:
        traffic = TrafficReport(plan.external_reads, plan.external_writes, plan.local_reads,
                                plan.local_writes, plan.scratch_bytes_peak)
    traffic.device = plan
    hosts = [np.ascontiguousarray(f.data, dtype=np.float64) for f in (fields.u, fields.v, fields.w)]
    res = SourceSet(*(Field3D(gd, np.zeros(gd.padded_shape)) for _ in range(3)))
    dc = device.DeviceCoefficients.from_host(coeffs, dev)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    u, v, w = (torch.from_numpy(h).to(dev) for h in hosts)
    out = device.alloc_fields(gd, dev)
    for box in boxes:
        device.advect(u, v, w, dc, out, box=box, opts=opts)
    for r, o in zip((res.su, res.sv, res.sw), out):
        r.data[...] = o.cpu().numpy()
    wall = time.perf_counter() - t0
    if spec.measure_traffic:  # one more pass of the same launches under the counters
        from . import traffic as tmod

        def launches():
            for box in boxes:
                device.advect(u, v, w, dc, out, box=box, opts=opts)
        try:
            traffic.measured = tmod.measure(launches, device=dev.index,
                                            plan_bytes=8 * (plan.external_reads + plan.external_writes))
        except tmod.TrafficUnavailable as exc:
            traffic.measured = {"error": str(exc)}
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
