"""CPU oracle for the PW-advection hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the thing measured or shipped: only
`tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and
`--impl reference`) may import it. The product package
`paper_2010_01545_b200` never imports it and has no CPU fallback.

Two independent restatements of the reference algorithm live here:

* `liboracle.so` (oracle/pwadv_oracle.c, plain C, -ffp-contract=off) — the
  fast one, threaded over X slabs like `run_schedule`'s engines
  (reference pkg/src/pwadvect/schedules.py:65-75, 207-232).
* `advect_numpy` — a vectorised numpy transcription of `compute_block`
  (reference pkg/src/pwadvect/kernel.py:139-185), used to cross-check the C
  restatement.

Both are pinned against the reference's own golden digests
(reference pkg/tests/goldens.json) and against fixtures produced by importing
the reference (tests/golden/make_golden.py → tests/golden/*.json, *.npz).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def build() -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, no FMA)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.oracle_advect.argtypes = [_D, _D, _D, _D, _D, _D, _I64, _I64, _I64,
                                    ctypes.c_double, ctypes.c_double, _D, _D, ctypes.c_int]
        L.oracle_advect.restype = ctypes.c_int
        L.oracle_advect_slab.argtypes = [_D, _D, _D, _D, _D, _D, _I64, _I64, _I64,
                                         ctypes.c_double, ctypes.c_double, _D, _D, _I64, _I64]
        L.oracle_advect_slab.restype = None
        L.oracle_wrap_halos.argtypes = [_D, _I64, _I64, _I64]
        L.oracle_wrap_halos.restype = None
        L.oracle_lcg_doubles.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _I64, _D]
        L.oracle_lcg_doubles.restype = None
        L.oracle_fill_random.argtypes = [_D, _D, _D, _I64, _I64, _I64, ctypes.c_uint64, ctypes.c_int]
        L.oracle_fill_random.restype = None
        L.oracle_baseline_coefficients.argtypes = [ctypes.c_uint64, _I64, _D, _D, _D, _D]
        L.oracle_baseline_coefficients.restype = None
        L.oracle_step.argtypes = [_D, _D, _D, _D, _I64, _I64, _I64, ctypes.c_double,
                                  ctypes.c_double, _D, _D, ctypes.c_double, ctypes.c_int]
        L.oracle_step.restype = ctypes.c_int
        L.oracle_step_open.argtypes = L.oracle_step.argtypes
        L.oracle_step_open.restype = ctypes.c_int
        L.oracle_fill_box.argtypes = [_D, _D, _D, _I64, _I64, _I64, ctypes.c_uint64, ctypes.c_int,
                                      _I64, _I64, _I64, _I64]
        L.oracle_fill_box.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# generation (reference grid.py:164-239 + BASELINE mapping)

def lcg_doubles(seed: int, count: int, start: int = 0) -> np.ndarray:
    out = np.empty(count)
    if count:
        lib().oracle_lcg_doubles(seed & (2**64 - 1), start, count, _p(out))
    return out


def fill_random(nx: int, ny: int, nz: int, seed: int, baseline: bool = False):
    """(u, v, w) padded arrays: reference random fill, optionally BASELINE-mapped."""
    shape = (nx + 2, ny + 2, nz)
    u, v, w = (np.empty(shape) for _ in range(3))
    lib().oracle_fill_random(_p(u), _p(v), _p(w), nx, ny, nz, seed & (2**64 - 1),
                             1 if baseline else 0)
    return u, v, w


def fill_box(gnx: int, gny: int, nz: int, seed: int, i0: int, j0: int, bnx: int, bny: int,
             baseline: bool = False):
    """(u, v, w) boxes of shape (bnx, bny, nz): global padded cells
    (i0.., j0.., :) of fill_random(gnx, gny, nz, seed), taken periodically."""
    u, v, w = (np.empty((bnx, bny, nz)) for _ in range(3))
    lib().oracle_fill_box(_p(u), _p(v), _p(w), gnx, gny, nz, seed & (2**64 - 1),
                          1 if baseline else 0, i0, j0, bnx, bny)
    return u, v, w


def baseline_coefficients(seed: int, nz: int) -> dict:
    """tcx=tcy=0.25/50, tzc1/tzc2 (+ recorded tzd1/tzd2) in [1e-3, 5e-3)."""
    arrs = [np.empty(nz) for _ in range(4)]
    lib().oracle_baseline_coefficients(seed & (2**64 - 1), nz, *(_p(a) for a in arrs))
    return {"tcx": 0.25 / 50.0, "tcy": 0.25 / 50.0, "tzc1": arrs[0], "tzc2": arrs[1],
            "tzd1": arrs[2], "tzd2": arrs[3]}


def wrap_halos(a: np.ndarray) -> None:
    nx, ny, nz = a.shape[0] - 2, a.shape[1] - 2, a.shape[2]
    lib().oracle_wrap_halos(_p(a), nx, ny, nz)


# --------------------------------------------------------------------------
# the stencil

def advect(u, v, w, tcx, tcy, tzc1, tzc2, engines: int = 1):
    """C restatement of run_reference (kernel.py:175-185); returns padded su, sv, sw."""
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    tzc1 = np.ascontiguousarray(tzc1, dtype=np.float64)
    tzc2 = np.ascontiguousarray(tzc2, dtype=np.float64)
    if tzc1.shape != (nz,) or tzc2.shape != (nz,):
        raise ValueError(f"coefficient length {tzc1.shape} != nz {nz}")
    outs = [np.zeros_like(u) for _ in range(3)]
    rc = lib().oracle_advect(_p(u), _p(v), _p(w), *(_p(o) for o in outs), nx, ny, nz,
                             float(tcx), float(tcy), _p(tzc1), _p(tzc2), int(engines))
    if rc:
        raise ValueError("oracle_advect: bad arguments")
    return tuple(outs)


def advect_into(u, v, w, su, sv, sw, tcx, tcy, tzc1, tzc2, engines: int = 1) -> None:
    """As `advect`, writing into caller-provided (pre-zeroed) outputs."""
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    rc = lib().oracle_advect(_p(u), _p(v), _p(w), _p(su), _p(sv), _p(sw), nx, ny, nz,
                             float(tcx), float(tcy), _p(tzc1), _p(tzc2), int(engines))
    if rc:
        raise ValueError("oracle_advect: bad arguments")


def advect_numpy(u, v, w, tcx, tcy, tzc1, tzc2):
    """Vectorised numpy transcription of compute_block/run_reference (kernel.py:139-185)."""
    with np.errstate(invalid="ignore", over="ignore"):  # non-finite inputs propagate, as numpy's
        return _advect_numpy(u, v, w, tcx, tcy, tzc1, tzc2)


def _advect_numpy(u, v, w, tcx, tcy, tzc1, tzc2):
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    tzc1 = np.asarray(tzc1, dtype=np.float64)
    tzc2 = np.asarray(tzc2, dtype=np.float64)
    F = {"u": u, "v": v, "w": w}

    def r(f, dx, dy, k):
        return F[f][1 + dx:nx + 1 + dx, 1 + dy:ny + 1 + dy, k]

    outs = []
    mid = slice(1, nz - 1)
    km1 = slice(0, nz - 2)
    kp1 = slice(2, nz)
    t = nz - 1
    for name in ("su", "sv", "sw"):
        s = np.zeros((nx, ny, nz))
        for ks, kd, kp, top in ((mid, km1, kp1, False), (t, t - 1, t, True)):
            if not top and nz <= 2:
                continue
            c1 = tzc1[ks]
            c2 = tzc2[ks]
            if name == "su":
                X = tcx * (r("u", -1, 0, ks) * (r("u", 0, 0, ks) + r("u", -1, 0, ks))
                           - r("u", 1, 0, ks) * (r("u", 0, 0, ks) + r("u", 1, 0, ks)))
                Y = tcy * (r("u", 0, -1, ks) * (r("v", 0, -1, ks) + r("v", 1, -1, ks))
                           - r("u", 0, 1, ks) * (r("v", 0, 0, ks) + r("v", 1, 0, ks)))
                A = c1 * r("u", 0, 0, kd) * (r("w", 0, 0, kd) + r("w", 1, 0, kd))
                if not top:
                    B = c2 * r("u", 0, 0, kp) * (r("w", 0, 0, ks) + r("w", 1, 0, ks))
            elif name == "sv":
                X = tcx * (r("v", -1, 0, ks) * (r("u", -1, 0, ks) + r("u", -1, 1, ks))
                           - r("v", 1, 0, ks) * (r("u", 0, 0, ks) + r("u", 0, 1, ks)))
                Y = tcy * (r("v", 0, -1, ks) * (r("v", 0, 0, ks) + r("v", 0, -1, ks))
                           - r("v", 0, 1, ks) * (r("v", 0, 0, ks) + r("v", 0, 1, ks)))
                A = c1 * r("v", 0, 0, kd) * (r("w", 0, 0, kd) + r("w", 0, 1, kd))
                if not top:
                    B = c2 * r("v", 0, 0, kp) * (r("w", 0, 0, ks) + r("w", 0, 1, ks))
            else:
                X = tcx * (r("w", -1, 0, ks) * (r("u", -1, 0, kd) + r("u", -1, 0, ks))
                           - r("w", 1, 0, ks) * (r("u", 0, 0, kd) + r("u", 0, 0, ks)))
                Y = tcy * (r("w", 0, -1, ks) * (r("v", 0, -1, kd) + r("v", 0, -1, ks))
                           - r("w", 0, 1, ks) * (r("v", 0, 0, kd) + r("v", 0, 0, ks)))
                A = c1 * r("w", 0, 0, kd) * (r("w", 0, 0, ks) + r("w", 0, 0, kd))
                if not top:
                    B = c2 * r("w", 0, 0, kp) * (r("w", 0, 0, ks) + r("w", 0, 0, kp))
            s[..., ks] = (X + Y) + A if top else (X + Y) + (A - B)
        full = np.zeros_like(u)
        full[1:-1, 1:-1, 1:] = s[..., 1:]
        outs.append(full)
    return tuple(outs)


# array-level API restated (reference kernel.py:73-162)

ROLES = (("u", -1, 0), ("u", -1, 1), ("u", 0, -1), ("u", 0, 0), ("u", 0, 1), ("u", 1, 0),
         ("v", -1, 0), ("v", 0, -1), ("v", 0, 0), ("v", 0, 1), ("v", 1, -1), ("v", 1, 0),
         ("w", -1, 0), ("w", 0, -1), ("w", 0, 0), ("w", 0, 1), ("w", 1, 0))
# (role index, k offset) of each formula operand, kernel.py:117-128
WIRING = (
    ((3, 0), (0, 0), (5, 0), (2, 0), (4, 0), (3, -1), (3, 1), (7, 0), (10, 0), (8, 0), (11, 0),
     (14, -1), (16, -1), (14, 0), (16, 0)),
    ((8, 0), (6, 0), (11, 0), (7, 0), (9, 0), (8, -1), (8, 1), (0, 0), (1, 0), (3, 0), (4, 0),
     (14, -1), (15, -1), (14, 0), (15, 0)),
    ((14, 0), (12, 0), (16, 0), (13, 0), (15, 0), (14, -1), (14, 1), (0, -1), (0, 0), (3, -1),
     (3, 0), (7, -1), (7, 0), (8, -1), (8, 0)),
)


def formula_numpy(which: int, args, top: bool = False):
    """su/sv/sw_formula (kernel.py:73-112) as one generic expression: the three
    formulas differ only in which operands fill the X, Y and Z slots."""
    tcx, tcy, c1, c2 = args[:4]
    o = args[4:]
    # (x1, x2, x3, x4, x5, x6, y1..y6, z1..z6) positions in the operand list
    slots = (
        (1, 0, 1, 2, 0, 2, 3, 7, 8, 4, 9, 10, 5, 11, 12, 6, 13, 14),   # su
        (1, 7, 8, 2, 9, 10, 3, 0, 3, 4, 0, 4, 5, 11, 12, 6, 13, 14),   # sv
        (1, 7, 8, 2, 9, 10, 3, 11, 12, 4, 13, 14, 5, 0, 5, 6, 0, 6),   # sw
    )[which]
    x1, x2, x3, x4, x5, x6, y1, y2, y3, y4, y5, y6, z1, z2, z3, z4, z5, z6 = (o[i] for i in slots)
    s = tcx * (x1 * (x2 + x3) - x4 * (x5 + x6))
    s = s + tcy * (y1 * (y2 + y3) - y4 * (y5 + y6))
    if top:
        return s + c1 * z1 * (z2 + z3)
    return s + (c1 * z1 * (z2 + z3) - c2 * z4 * (z5 + z6))


def compute_block_numpy(tcx, tcy, tzc1, tzc2, roles):
    """compute_block (kernel.py:139-162) over role arrays listed in ROLES order."""
    nz = roles[3].shape[-1]
    t = nz - 1
    outs = []
    for which in range(3):
        s = np.zeros_like(roles[3])
        if nz > 2:
            ops = [roles[r][..., 1 + dk:nz - 1 + dk] for r, dk in WIRING[which]]
            s[..., 1:nz - 1] = formula_numpy(which, [tcx, tcy, tzc1[1:nz - 1], tzc2[1:nz - 1]] + ops)
        ops = [roles[r][..., t - 1 if dk == -1 else t] for r, dk in WIRING[which]]
        s[..., t] = formula_numpy(which, [tcx, tcy, float(tzc1[t]), float(tzc2[t])] + ops, top=True)
        outs.append(s)
    return tuple(outs)


def run_schedule_numpy(u, v, w, tcx, tcy, tzc1, tzc2, engines: int = 1, outs=None):
    """The reference's own CPU path as written: run_schedule(..., "reference",
    engines) (schedules.py:207-232) — balanced X slabs (partition_domain,
    schedules.py:65-75), each engine thread evaluating compute_block on its
    slab's grid_roles views (schedules.py:131-135, kernel.py:139-172) with
    numpy ufuncs and scattering into the zeroed padded outputs. Same
    arithmetic form and speed as the reference (4.06 vs 4.04 Mpts/s on one
    thread in this container); bitwise equal to `advect`. `outs` (pre-zeroed
    padded arrays) may be passed to reuse them."""
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    engines = max(1, min(int(engines), nx))
    tzc1 = np.asarray(tzc1, dtype=np.float64)
    tzc2 = np.asarray(tzc2, dtype=np.float64)
    if outs is None:
        outs = tuple(np.zeros_like(u) for _ in range(3))
    F = {"u": u, "v": v, "w": w}
    base, rem = divmod(nx, engines)
    slabs, x = [], 1
    for e in range(engines):
        wd = base + (1 if e < rem else 0)
        slabs.append((x, x + wd))
        x += wd

    def slab(xb, xe):
        roles = [F[f][xb + dx:xe + dx, 1 + dy:ny + 1 + dy, :] for f, dx, dy in ROLES]
        with np.errstate(invalid="ignore", over="ignore"):
            blocks = compute_block_numpy(tcx, tcy, tzc1, tzc2, roles)
        for o, b in zip(outs, blocks):
            o[xb:xe, 1:ny + 1, 1:] = b[..., 1:]

    if engines == 1:
        slab(*slabs[0])
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=engines) as pool:
            for f in [pool.submit(slab, xb, xe) for xb, xe in slabs]:
                f.result()
    return tuple(outs)


def step(u, v, w, tcx, tcy, tzc1, tzc2, dt: float, steps: int, engines: int = 1):
    """Composed forward-Euler oracle: in place on u, v, w."""
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    scratch = np.zeros((3,) + u.shape)
    tzc1 = np.ascontiguousarray(tzc1, dtype=np.float64)
    tzc2 = np.ascontiguousarray(tzc2, dtype=np.float64)
    for _ in range(steps):
        rc = lib().oracle_step(_p(u), _p(v), _p(w), _p(scratch), nx, ny, nz, float(tcx),
                               float(tcy), _p(tzc1), _p(tzc2), float(dt), int(engines))
        if rc:
            raise ValueError("oracle_step: bad arguments")


def step_open(u, v, w, tcx, tcy, tzc1, tzc2, dt: float, steps: int, engines: int = 1):
    """As step(), but the halo ring is never refreshed: after n steps only the
    cells at distance >= n from the box edge are valid (light-cone check)."""
    nx, ny, nz = u.shape[0] - 2, u.shape[1] - 2, u.shape[2]
    scratch = np.zeros((3,) + u.shape)
    tzc1 = np.ascontiguousarray(tzc1, dtype=np.float64)
    tzc2 = np.ascontiguousarray(tzc2, dtype=np.float64)
    for _ in range(steps):
        rc = lib().oracle_step_open(_p(u), _p(v), _p(w), _p(scratch), nx, ny, nz, float(tcx),
                                    float(tcy), _p(tzc1), _p(tzc2), float(dt), int(engines))
        if rc:
            raise ValueError("oracle_step_open: bad arguments")


def lightcone_tile(gnx: int, gny: int, nz: int, seed: int, coeffs: dict, dt: float, steps: int,
                   i0: int, j0: int, ti: int, tj: int, engines: int = 1):
    """Interior rows i0..i0+ti-1, columns j0..j0+tj-1 (1-based, periodic) of
    (u, v, w) after `steps` forward steps of the BASELINE fill, computed from
    the (ti+2*steps) x (tj+2*steps) neighbourhood only."""
    r = steps
    fs = fill_box(gnx, gny, nz, seed, i0 - r, j0 - r, ti + 2 * r, tj + 2 * r, baseline=True)
    for _ in range(steps):
        step_open(*fs, coeffs["tcx"], coeffs["tcy"], coeffs["tzc1"], coeffs["tzc2"], dt, 1, engines)
        # only the interior is valid now: it is the next step's padded box
        fs = tuple(np.ascontiguousarray(f[1:-1, 1:-1]) for f in fs)
    return fs


# --------------------------------------------------------------------------
# digests and comparison (reference grid.py:242-249, schedules.py:235-272)

def checksum(padded: np.ndarray) -> str:
    interior = np.ascontiguousarray(padded[1:-1, 1:-1, :], dtype="<f8")
    return hashlib.blake2b(interior.tobytes(), digest_size=8).hexdigest()


def _ordered_bits(arr):
    bits = np.ascontiguousarray(arr).reshape(-1).view(np.int64)
    return np.where(bits >= 0, bits, np.int64(-(2**63)) - bits)


def max_ulp(a, b) -> int:
    oa, ob = _ordered_bits(a), _ordered_bits(b)
    same = (oa >= 0) == (ob >= 0)
    worst = 0
    if same.any():
        worst = int(np.abs(oa[same] - ob[same]).max())
    if (~same).any():
        ua = np.abs(oa[~same]).astype(np.uint64)
        ub = np.abs(ob[~same]).astype(np.uint64)
        worst = max(worst, int((ua + ub).max()))
    return worst


def compare(a, b) -> dict:
    """compare_outputs semantics over full padded arrays (schedules.py:261-272)."""
    pairs = list(zip(a, b))
    bitwise = all(np.array_equal(np.ascontiguousarray(x).view(np.int64),
                                 np.ascontiguousarray(y).view(np.int64)) for x, y in pairs)
    if bitwise:
        return {"bitwise_equal": True, "max_abs_diff": 0.0, "max_ulp_diff": 0, "normwise_rel": 0.0}
    max_abs = max(float(np.abs(x - y).max()) for x, y in pairs)
    ref_max = max(float(np.abs(x).max()) for x, _ in pairs) or 1.0
    mu = max(max_ulp(x, y) for x, y in pairs)
    return {"bitwise_equal": False, "max_abs_diff": max_abs, "max_ulp_diff": max(mu, 1),
            "normwise_rel": max_abs / ref_max}


def _host(a) -> np.ndarray:
    """numpy view/copy of a host array or a torch tensor (device or host)."""
    if hasattr(a, "detach"):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def compare_streamed(fields, outs, tcx, tcy, tzc1, tzc2, *, dt=None, slab: int = 64,
                     engines: int = 0) -> dict:
    """Every plane of a result against the C oracle, X-slab by X-slab.

    `fields` (u, v, w) and `outs` (su, sv, sw — or, with `dt`, the stepped
    u', v', w') are padded (nx+2, ny+2, nz) arrays or torch tensors on any
    device. Output planes [x0, x1) need input planes [x0-1, x1+1] only, so
    each slab of `slab` planes is copied to the host with one halo plane on
    each side and evaluated by the C restatement of run_reference
    (kernel.py:175-185), threaded over all host cores; memory stays bounded
    at full config sizes. Evaluations compare the whole padded output planes
    (halo columns and level 0 must be +0.0, as in zeros_sources); steps
    compare the interior columns against f + dt*s (mul then add), the
    composed oracle of SURVEY.md §8f1. Returns compare()'s record plus the
    planes checked and the first mismatching plane."""
    nx = int(fields[0].shape[0]) - 2
    engines = engines or host_threads()
    tz1 = np.ascontiguousarray(_host(tzc1), dtype=np.float64)
    tz2 = np.ascontiguousarray(_host(tzc2), dtype=np.float64)
    res = {"bitwise_equal": True, "max_abs_diff": 0.0, "max_ulp_diff": 0, "normwise_rel": 0.0}
    first_bad = None
    planes = 0
    for x0 in range(1, nx + 1, slab):
        x1 = min(x0 + slab, nx + 1)
        ins = [np.ascontiguousarray(_host(f[x0 - 1:x1 + 1]), dtype=np.float64) for f in fields]
        want = advect(*ins, tcx, tcy, tz1, tz2, engines=max(1, min(engines, x1 - x0)))
        got = [_host(o[x0:x1]) for o in outs]
        if dt is None:
            want = [wv[1:-1] for wv in want]
        else:
            want = [(f[1:-1] + float(dt) * s)[:, 1:-1] for f, s in zip(ins, (wv[1:-1] for wv in want))]
            got = [g[:, 1:-1] for g in got]
        c = compare(got, want)
        planes += x1 - x0
        if not c["bitwise_equal"]:
            if first_bad is None:
                first_bad = x0
            res["bitwise_equal"] = False
            res["max_abs_diff"] = max(res["max_abs_diff"], c["max_abs_diff"])
            res["max_ulp_diff"] = max(res["max_ulp_diff"], c["max_ulp_diff"])
            res["normwise_rel"] = max(res["normwise_rel"], c["normwise_rel"])
    res["planes_checked"] = planes
    res["first_bad_slab"] = first_bad
    return res
