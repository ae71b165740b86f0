"""Command line: `python -m paper_2010_01545_b200 bench ...` and `... build`.

`bench` mirrors the reference harness `pwadvect bench` (cli.py:120-163): the
same row schema (BENCH_COLUMNS, cli.py:32-36), min/mean/all wall times over
--reps, per-run su/sv/sw checksums with a drift check across repetitions and
a cross-schedule agreement check, exit 1 on any failure, rows printed as a
table or written as CSV / JSON. Schedules are the GPU kernel variants
(engines.VARIANTS; the reference's FPGA schedule names are accepted and run
as the X-march). Wall time is device time of the kernels (CUDA events), the
fields already resident. The reference's model/sweep/calibrate/validate
commands evaluate FPGA cost models, which are out of scope here.
"""

from __future__ import annotations

import argparse
import csv
import json
import platform
import statistics
import sys
from pathlib import Path

BENCH_COLUMNS = ("schedule", "engines", "y_batch", "nx", "ny", "nz", "reps",
                 "wall_min_s", "wall_mean_s", "wall_all_s",
                 "checksum_su", "checksum_sv", "checksum_sw",
                 "external_reads", "external_writes", "local_reads", "local_writes",
                 "scratch_bytes_peak", "host", "gpoints_per_s")


def _grid(text: str):
    from .layout import make_grid
    try:
        nx, ny, nz = (int(p) for p in text.lower().split("x"))
        return make_grid(nx, ny, nz)
    except Exception as exc:  # noqa: BLE001
        raise argparse.ArgumentTypeError(f"bad grid {text!r} (want NXxNYxNZ): {exc}")


def _schedule(name: str) -> str:
    from .engines import VARIANTS
    key = name.lower().replace("-", "_")
    aliases = {"columnbuffered": "column_buffered", "ybatched": "y_batched", "xreordered": "x_reordered"}
    key = aliases.get(key.replace("_", ""), key)
    if key not in VARIANTS:
        raise argparse.ArgumentTypeError(f"unknown schedule {name!r}; choose from {VARIANTS}")
    return key


def _host() -> str:
    import torch
    gpu = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "no-gpu"
    return f"{platform.platform()} python{platform.python_version()} {gpu}"


def _cell(v) -> str:
    if isinstance(v, float):
        return f"{v:.6g}"
    return "" if v is None else str(v)


def write_rows(rows, columns, out, fmt) -> None:
    if out is None:
        widths = {c: max(len(c), *(len(_cell(r.get(c))) for r in rows)) for c in columns}
        print("  ".join(c.ljust(widths[c]) for c in columns))
        for r in rows:
            print("  ".join(_cell(r.get(c)).ljust(widths[c]) for c in columns))
        return
    path = Path(out)
    if fmt == "json":
        path.write_text(json.dumps([{c: r.get(c) for c in columns} for r in rows], indent=2) + "\n")
    else:
        with path.open("w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(columns)
            for r in rows:
                w.writerow([_cell(r.get(c)) for c in columns])
    print(f"wrote {len(rows)} row(s) to {path} ({fmt})")


def cmd_bench(args, parser) -> int:
    from . import engines, layout, stencil
    dims = args.grid
    gen = {"uniform": layout.GeneratorSpec.uniform(1.0, 1.1, 0.9), "trig": layout.GeneratorSpec.trig(),
           "random": layout.GeneratorSpec.random(args.seed),
           "baseline": layout.GeneratorSpec.baseline(args.seed)}[args.gen]
    fields = layout.fill_fields(dims, gen)
    coeffs = (stencil.baseline_coefficients(args.seed, dims.nz) if args.gen == "baseline"
              else stencil.default_coefficients(dims.nz))
    rows, failures = [], []
    host = _host()
    for variant in args.schedule:
        spec = engines.ScheduleSpec(variant, y_batch=min(args.y_batch, dims.ny), engines=args.engines)
        try:
            spec.validate(dims)
        except ValueError as exc:
            parser.error(str(exc))
        walls, sums, traffic = [], None, None
        for _ in range(args.reps):
            out, tc, wall = engines.run_schedule(fields, coeffs, spec)
            walls.append(wall)
            digest = tuple(layout.checksum(f) for f in (out.su, out.sv, out.sw))
            if sums is None:
                sums, traffic = digest, tc
            elif sums != digest:
                failures.append(f"{variant}: checksum changed between repetitions")
            elif traffic != tc:
                failures.append(f"{variant}: traffic counters changed between repetitions")
        rows.append({
            "schedule": variant, "engines": spec.engines, "y_batch": spec.y_batch,
            "nx": dims.nx, "ny": dims.ny, "nz": dims.nz, "reps": args.reps,
            "wall_min_s": min(walls), "wall_mean_s": statistics.fmean(walls),
            "wall_all_s": ";".join(f"{w:.6g}" for w in walls),
            "checksum_su": sums[0], "checksum_sv": sums[1], "checksum_sw": sums[2],
            "external_reads": traffic.external_reads, "external_writes": traffic.external_writes,
            "local_reads": traffic.local_reads, "local_writes": traffic.local_writes,
            "scratch_bytes_peak": traffic.scratch_bytes_peak, "host": host,
            "gpoints_per_s": dims.cells / min(walls) / 1e9,
        })
    if len({(r["checksum_su"], r["checksum_sv"], r["checksum_sw"]) for r in rows
            if not r["schedule"].endswith("_fma")}) > 1:
        failures.append("schedules disagree on output checksums")
    write_rows(rows, BENCH_COLUMNS, args.out, args.format)
    for msg in failures:
        print(f"FAIL {msg}", file=sys.stderr)
    return 1 if failures else 0


def cmd_build(args, parser) -> int:
    from .build import build
    print(build(force=True))
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_2010_01545_b200",
                                description=__doc__.splitlines()[0])
    subs = p.add_subparsers(dest="command", required=True)
    b = subs.add_parser("bench", help="run GPU schedules and report timings/traffic (reference row schema)")
    b.add_argument("--grid", type=_grid, required=True, metavar="NXxNYxNZ")
    b.add_argument("--schedule", action="append", type=_schedule, metavar="NAME",
                   help="repeatable; default xmarch")
    b.add_argument("--engines", type=int, default=1)
    b.add_argument("--y-batch", type=int, default=64, dest="y_batch")
    b.add_argument("--gen", choices=("uniform", "trig", "random", "baseline"), default="random")
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--out")
    b.add_argument("--format", choices=("csv", "json"), default="csv")
    b.set_defaults(func=cmd_bench)
    bl = subs.add_parser("build", help="compile libpwadv.so in-tree (nvcc, sm_100a)")
    bl.set_defaults(func=cmd_build)
    return p


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    if getattr(args, "schedule", "missing") is None:
        args.schedule = ["xmarch"]
    if getattr(args, "reps", 1) < 1:
        parser.error("--reps must be >= 1")
    return args.func(args, parser)
