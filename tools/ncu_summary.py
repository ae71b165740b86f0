"""Summarise ncu --set full captures of K1/K4 into profiles/ (raw CSV + ncu_traffic.json entry).

    python tools/ncu_summary.py [--round=r02] KEY REPORT.ncu-rep|RAW.csv [KEY REPORT ...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = {
    "duration_us": ("gpu__time_duration.sum", {"us": 1, "ms": 1e3, "ns": 1e-3}),
    "dram_read": ("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "dram_write": ("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", {"%": 1}),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", {"%": 1}),
    "registers": ("launch__registers_per_thread", {"register/thread": 1}),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", {"Ghz": 1, "Mhz": 1e-3}),
}


def summarise(key, rep, rnd="r02"):
    """rep: an .ncu-rep, or the raw CSV of one (`ncu -i X --page raw --csv`)."""
    if rep.endswith(".csv"):
        raw = Path(rep).read_text()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")][:80]}
    for name, (metric, scale) in METRICS.items():
        i = hdr.index(metric)
        out[name] = round(float(vals[i].replace(",", "")) * scale.get(units[i], 1), 4)
    out["bytes"] = int(out["dram_read"] + out["dram_write"])
    tag = key.replace(":", "_")
    dst = ROOT / "profiles" / f"{rnd}_ncu_full_{tag}_raw.csv"
    out["source"] = f"profiles/{dst.name} (ncu --set full, 1 launch, cold)"
    # the libpwadv.so the capture ran (shipped from this tree): bench.py uses
    # the entry only while the loaded library has the same hash
    sys.path.insert(0, str(ROOT))
    from paper_2010_01545_b200 import _lib
    out["build_id"] = _lib.build_id()
    dst.write_text(raw)
    return out


if __name__ == "__main__":
    p = ROOT / "profiles" / "ncu_traffic.json"
    table = json.loads(p.read_text()) if p.exists() else {}
    args = sys.argv[1:]
    rnd = "r02"
    if args and args[0].startswith("--round="):
        rnd = args.pop(0).split("=", 1)[1]
    for key, rep in zip(args[::2], args[1::2]):
        table[key] = summarise(key, rep, rnd)
        print(key, table[key])
    p.write_text(json.dumps(table, indent=1) + "\n")
