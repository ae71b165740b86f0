"""Loader for the committed golden fixtures (tests/golden/, made by make_golden.py)."""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def _unhex(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


@lru_cache(maxsize=1)
def _raw():
    return json.loads((GOLDEN / "cases.json").read_text())


@lru_cache(maxsize=1)
def small_arrays():
    with np.load(GOLDEN / "small.npz") as z:
        return {k: z[k] for k in z.files}


def reference_goldens():
    return _raw()["reference_goldens_json"]


def load_cases():
    out = []
    for c in _raw()["cases"]:
        c = dict(c)
        c["tcx"] = float.fromhex(c["tcx"])
        c["tcy"] = float.fromhex(c["tcy"])
        c["tzc1"] = _unhex(c["tzc1"])
        c["tzc2"] = _unhex(c["tzc2"])
        out.append(c)
    return out


def step_cases():
    return json.loads((GOLDEN / "steps.json").read_text())["cases"]


def case_inputs(case):
    """Padded (u, v, w) for a golden case, regenerated (or loaded for test aids)."""
    from oracle import oracle
    nx, ny, nz = case["nx"], case["ny"], case["nz"]
    gen = case["generator"]
    if case["arrays"] and gen["mode"] in ("trig", "nonfinite"):
        arrs = small_arrays()
        return tuple(arrs[f"{case['name']}/{k}"].copy() for k in "uvw")
    if gen["mode"] == "uniform":
        shape = (nx + 2, ny + 2, nz)
        return np.full(shape, gen["a"]), np.full(shape, gen["b"]), np.full(shape, gen["c"])
    if gen["mode"] == "random":
        return oracle.fill_random(nx, ny, nz, gen["seed"], baseline=False)
    if gen["mode"] == "baseline":
        return oracle.fill_random(nx, ny, nz, gen["seed"], baseline=True)
    raise ValueError(gen)


@lru_cache(maxsize=1)
def array_api_fixtures():
    """arrays.npz: the reference's compute_block / grid_roles / *_formula outputs."""
    with np.load(GOLDEN / "arrays.npz") as z:
        return {k: z[k] for k in z.files}


def compute_block_cases():
    z = array_api_fixtures()
    out = []
    n = 0
    while f"cb{n}/coeffs" in z:
        roles = [z[f"cb{n}/role{m}"] for m in range(17)]
        nz = roles[0].shape[-1]
        c = z[f"cb{n}/coeffs"]
        out.append({"tcx": float(c[0]), "tcy": float(c[1]), "tzc1": c[2:2 + nz],
                    "tzc2": c[2 + nz:], "roles": roles,
                    "want": tuple(z[f"cb{n}/{k}"] for k in ("su", "sv", "sw"))})
        n += 1
    return out


def formula_cases():
    z = array_api_fixtures()
    out = []
    for which in range(3):
        for top in (0, 1):
            key = f"f{which}{top}"
            args = [z[f"{key}/arg{m}"] for m in range(19)]
            args = [float(a) if a.ndim == 0 else a for a in args]
            out.append({"which": which, "top": bool(top), "args": args, "want": z[f"{key}/out"]})
    return out
