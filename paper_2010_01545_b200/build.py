"""Build libpwadv.so in-tree with nvcc for sm_100a (no JIT cache, travels with gpurun)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libpwadv.so"
TRAFFIC_LIB = PKG / "libpwadv_traffic.so"  # optional: live DRAM counters (CUPTI)
TRAFFIC_SRC = "pwadv_traffic.cpp"
# translation units, compiled in parallel (the kernel instantiations are split
# over the pwadv_k_* units so no single nvcc run dominates the build)
SOURCES = ["pwadv_k_small.cu", "pwadv_k_ct.cu", "pwadv_k_nzc2.cu", "pwadv_k_pull.cu", "pwadv_k_ws.cu",
           "pwadv_k_nzc0.cu", "pwadv_k_nzc1.cu", "pwadv_k_nzc3.cu", "pwadv_k_ctodd.cu", "pwadv_advect.cu", "pwadv_api.cu",
           "pwadv_aux.cu", "pwadv_roles.cu", "pwadv_sync.cu"]
HEADERS = ["pwadv_device.cuh", "pwadv_internal.h", "pwadv_xmarch.cuh", "pwadv_ctile.cuh", "pwadv_kernels.h"]
OBJ = PKG.parent / "build" / "obj"


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def nvcc_flags(verbose: bool = False) -> list[str]:
    flags = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
             # bit-exact build: no FMA contraction anywhere (the formulas use
             # explicit __d*_rn intrinsics as well; the FMA variant uses
             # explicit __fma_rn and is selected at run time)
             "--fmad=false",
             "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
             "-I", str(PKG.parent / "include")]
    if verbose:
        flags += ["-Xptxas", "-v"]
    return flags


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "pwadv.h"]
    return any(d.stat().st_mtime > t for d in deps)


def cuda_home() -> Path:
    return Path(nvcc_path()).resolve().parent.parent


def build_traffic(force: bool = False) -> Path | None:
    """libpwadv_traffic.so (CUPTI range profiler, host code only): g++ against
    the toolkit's cupti headers; None where the toolkit has no CUPTI."""
    # CUPTI must be the copy the host process loads: torch imports its bundled
    # libcupti.so.12 (nvidia-cuda-cupti wheel) first, and a second copy with
    # the same soname would bind to it with mismatched structs. Prefer the
    # bundled headers + library; the toolkit's otherwise.
    cu = cuda_home()
    inc, lib = cu / "include", cu / "lib64"
    try:
        import nvidia.cuda_cupti as bundled
        b = Path(list(bundled.__path__)[0])
        if (b / "include" / "cupti_range_profiler.h").exists() and (b / "lib" / "libcupti.so.12").exists():
            inc, lib = b / "include", b / "lib"
    except ImportError:
        pass
    if not (inc / "cupti_range_profiler.h").exists():
        return None
    src = CSRC / TRAFFIC_SRC
    hdr = PKG.parent / "include" / "pwadv_traffic.h"
    if (not force and TRAFFIC_LIB.exists()
            and TRAFFIC_LIB.stat().st_mtime > max(src.stat().st_mtime, hdr.stat().st_mtime)):
        return TRAFFIC_LIB
    tmp = TRAFFIC_LIB.with_suffix(".so.tmp")
    cupti = lib / "libcupti.so"
    if not cupti.exists():
        cupti = lib / "libcupti.so.12"
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", f"-I{inc}",
           f"-I{cu / 'include'}", str(src), "-o", str(tmp), str(cupti),
           f"-L{cu / 'lib64' / 'stubs'}", f"-Wl,-rpath,{lib}", "-lcuda"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stderr}")
    os.replace(tmp, TRAFFIC_LIB)
    return TRAFFIC_LIB


def _nvcc(cmd: list[str], verbose: bool) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)


def source_id(extra: list[str] | None = None) -> str:
    """16 hex digits of the sha256 over every source and header of libpwadv
    and the nvcc flags: compiled into the library (pwadv_source_id)."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted(SOURCES + HEADERS):
        h.update(f.encode())
        h.update((CSRC / f).read_bytes())
    h.update((PKG.parent / "include" / "pwadv.h").read_bytes())
    # the flags without the (checkout-dependent) include path
    flags = [f for f in nvcc_flags() if not f.startswith(str(PKG.parent))]
    h.update(" ".join(flags + list(extra or [])).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> Path:
    """Compile every translation unit for sm_100a (in parallel, `jobs` nvcc
    processes, default: the host's cores) and link libpwadv.so in-tree."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    OBJ.mkdir(parents=True, exist_ok=True)
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    flags = nvcc_flags(verbose) + [f'-DPWADV_SOURCE_ID="{source_id()}"']
    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as pool:
        for f in [pool.submit(_nvcc, [nvcc_path(), *flags, "-c", "-o", str(o), str(CSRC / s)], verbose)
                  for s, o in zip(SOURCES, objs)]:
            f.result()
    tmp = LIB.with_suffix(".so.tmp")
    _nvcc([nvcc_path(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
           *[str(o) for o in objs]], verbose)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    build_traffic(force="--force" in sys.argv)
    print(LIB)
