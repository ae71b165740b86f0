"""Live DRAM traffic of PW-advection launches from the hardware counters
(libpwadv_traffic.so, CUPTI range profiler).

The reference reports the element traffic of every run (TrafficReport,
pkg/src/pwadvect/schedules.py:99-114). `measure(fn)` runs `fn` — which
launches kernels — under the counters and returns the DRAM bytes those
launches read and wrote, their summed duration, and, given the plan's
bytes, the ratio measured / plan: traffic well above the plan means wasted
re-reads. L2 is flushed first (a write sweep, then a read sweep of another
buffer, so no dirty line of the sweep is written back inside the measured
kernels), matching ncu's cold-cache convention; `flush_l2=False` measures
with whatever the previous launches left in L2.

Diagnostic only — never inside a timed region (kernel replay serialises).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_LIB = Path(__file__).resolve().parent / "libpwadv_traffic.so"
_lib = None
_lock = threading.Lock()


class TrafficUnavailable(RuntimeError):
    """The counters cannot be read here (no library, no permission, no GPU)."""


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB.exists():
                raise TrafficUnavailable(f"{_LIB.name} not built (paper_2010_01545_b200/build.py)")
            L = ctypes.CDLL(str(_LIB))
            L.pwadv_traffic_begin.argtypes = [ctypes.c_int]
            L.pwadv_traffic_begin.restype = ctypes.c_int
            L.pwadv_traffic_end.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
            L.pwadv_traffic_end.restype = ctypes.c_int
            L.pwadv_traffic_last_error.argtypes = []
            L.pwadv_traffic_last_error.restype = ctypes.c_char_p
            L.pwadv_traffic_max_ranges.argtypes = []
            L.pwadv_traffic_max_ranges.restype = ctypes.c_int
            L.pwadv_traffic_num_values.argtypes = []
            L.pwadv_traffic_num_values.restype = ctypes.c_int
            _lib = L
        return _lib


def _err(L) -> str:
    return (L.pwadv_traffic_last_error() or b"").decode(errors="replace")


def flush_l2(device=None, nbytes: int = 512 << 20) -> None:
    """Evict L2 (126 MB on B200) with clean lines: write one buffer, then read
    another, both well above the L2 size."""
    import torch
    a = torch.empty(nbytes, dtype=torch.uint8, device=device)
    b = torch.ones(nbytes // 8, dtype=torch.float64, device=device)
    a.fill_(1)
    torch.cuda.synchronize(device)
    b.sum()
    torch.cuda.synchronize(device)
    del a, b


def measure(fn, *, plan_bytes: float | None = None, device: int | None = None,
            flush: bool = True) -> dict:
    """DRAM bytes read / written and kernel time of the launches `fn()` makes."""
    import torch
    L = lib()
    dev = torch.cuda.current_device() if device is None else int(device)
    with torch.cuda.device(dev):
        torch.cuda.synchronize()
        if flush:
            flush_l2(dev)
        if L.pwadv_traffic_begin(dev) != 0:
            raise TrafficUnavailable(_err(L))
        try:
            fn()
            torch.cuda.synchronize()
        finally:
            vals = (ctypes.c_double * L.pwadv_traffic_num_values())()
            n = ctypes.c_int(0)
            rc = L.pwadv_traffic_end(vals, ctypes.byref(n))
        if rc != 0:
            raise TrafficUnavailable(_err(L))
    rd, wr, ns, fp64_pct, fp64_inst = (float(x) for x in vals[:5])
    out = {"dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
           "kernel_us": ns / 1e3, "kernels": int(n.value),
           "fp64_pipe_pct": fp64_pct, "fp64_warp_inst": fp64_inst,
           "l2": "flushed before the launches" if flush else "as left by previous launches",
           "source": "CUPTI range profiler (dram__bytes_read.sum + dram__bytes_write.sum; "
                     "fp64 pipe: sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, "
                     "sm__inst_executed_pipe_fp64.sum), libpwadv_traffic.so"}
    if plan_bytes:
        out["plan_bytes"] = float(plan_bytes)
        out["ratio_to_plan"] = (rd + wr) / float(plan_bytes)
    return out
