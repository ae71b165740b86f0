"""ctypes binding of libpwadv.so (the C ABI declared in include/pwadv.h).

The library is built in-tree by `paper_2010_01545_b200/build.py` (nvcc,
sm_100a). There is no CPU fallback: if the shared library is missing or a
call fails, this module raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
import os as _os

# PWADV_LIB overrides the library (A/B builds of the same ABI for profiling)
LIB_PATH = Path(_os.environ["PWADV_LIB"]) if _os.environ.get("PWADV_LIB") else _PKG / "libpwadv.so"

_lock = threading.Lock()
_lib = None

c_double_p = ctypes.c_void_p  # device or host pointers are passed as raw addresses
_I64 = ctypes.c_int64
_D = ctypes.c_double
_P = ctypes.c_void_p

PWADV_OK = 0
PWADV_E_DIMS = -1
PWADV_E_NULL = -2
PWADV_E_RANGE = -3
PWADV_E_CUDA = -4
PWADV_E_ARG = -5
PWADV_E_ALIGN = -6

FLAG_FMA = 1
FLAG_SIMPLE = 2
FLAG_MARCH = 4
FLAG_UNALIGNED = 8
FLAG_RIM = 16
FLAG_GENERIC = 32
FLAG_L2_UNIT_HEAD = 64
FLAG_NO_PDL = 128
FLAG_NO_SPARE_TAIL = 0x1000
FLAG_SPARE_TAIL = 0x2000
FLAG_CTILE = 0x4000
FLAG_NO_CTILE = 0x8000
ABI_VERSION = 2


class Opts(ctypes.Structure):
    """pwadv_opts (include/pwadv.h)."""

    _fields_ = [("flags", ctypes.c_uint32), ("tile_j", ctypes.c_int32),
                ("stages", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("max_threads", ctypes.c_int32), ("chunks", ctypes.c_int32),
                ("trace", ctypes.c_void_p)]


class PlanInfo(ctypes.Structure):
    """pwadv_plan_info (include/pwadv.h)."""

    _fields_ = [("kernel", ctypes.c_int32), ("tile_j", ctypes.c_int32),
                ("threads_per_column", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int64), ("strips", ctypes.c_int64),
                ("chunks", ctypes.c_int32), ("long_strips", ctypes.c_int32),
                ("spare_ctas", ctypes.c_int32), ("main_chunk_planes", ctypes.c_int32)]


class Peers(ctypes.Structure):
    """pwadv_peers (include/pwadv.h): neighbour d's new u, v, w and extents."""

    _fields_ = [("u", ctypes.c_void_p * 8), ("v", ctypes.c_void_p * 8), ("w", ctypes.c_void_p * 8),
                ("nx", ctypes.c_int64 * 8), ("ny", ctypes.c_int64 * 8)]


NB_XM, NB_XP, NB_YM, NB_YP, NB_XMYM, NB_XMYP, NB_XPYM, NB_XPYP = range(8)


# name -> (restype, argtypes); every symbol include/pwadv.h declares
SIGNATURES = {
    "pwadv_abi_version": (ctypes.c_int, []),
    "pwadv_source_id": (ctypes.c_char_p, []),
    "pwadv_last_error": (ctypes.c_char_p, []),
    "pwadv_launch_count": (ctypes.c_uint64, []),
    "pwadv_reset_launch_count": (None, []),
    "pwadv_advect_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P, _P, _P]),
    "pwadv_advect_box_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P]
                             + [_I64] * 4 + [_P, _P]),
    "pwadv_step_box_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P, _D]
                           + [_I64] * 4 + [_P, _P]),
    "pwadv_describe_plan": (ctypes.c_int, [_I64] * 7 + [_P, ctypes.c_int, _P]),
    "pwadv_step_push_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P, _D, _P, _P, _P]),
    "pwadv_advect_pull_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P, _P, _P, _P]),
    "pwadv_step_pull_f64": (ctypes.c_int, [_P] * 6 + [_I64] * 3 + [_D, _D, _P, _P, _D, _P, _P, _P]),
    "pwadv_pull_halos_f64": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, _P, _P]),
    "pwadv_ipc_export": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_uint64)]),
    "pwadv_ipc_open": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.POINTER(_P)]),
    "pwadv_ipc_close": (ctypes.c_int, [_P, ctypes.c_uint64]),
    "pwadv_handshake_caps": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int)]),
    "pwadv_signal_peers": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_uint64, _P]),
    "pwadv_wait_peers": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_uint64, _P]),
    "pwadv_handshake": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.POINTER(_P),
                                       ctypes.c_int, ctypes.c_uint64, _P]),
    "pwadv_handshake_kernel": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.POINTER(_P),
                                              ctypes.c_int, ctypes.c_uint64, _P, ctypes.c_uint64, _P]),
    "pwadv_compute_block_f64": (ctypes.c_int, [_P] * 4 + [_I64, _I64, _D, _D, _P, _P,
                                                           ctypes.c_uint32, _P]),
    "pwadv_formula_f64": (ctypes.c_int, [ctypes.c_int32, _P, _P, _I64, ctypes.c_int32, _P,
                                         ctypes.c_uint32, _P]),
    "pwadv_pack_faces3_f64": (ctypes.c_int, [_P] * 5 + [_I64] * 3 + [ctypes.c_int32, _P]),
    "pwadv_unpack_faces3_f64": (ctypes.c_int, [_P] * 5 + [_I64] * 3 + [ctypes.c_int32, _P]),
    "pwadv_wrap_halos_f64": (ctypes.c_int, [_P, _I64, _I64, _I64, _P]),
    "pwadv_wrap_halos3_f64": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "pwadv_wrap_axis3_f64": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, ctypes.c_int32, _P]),
    "pwadv_fill_f64": (ctypes.c_int, [_P, _P, _P, _I64, _I64, _I64, ctypes.c_int32,
                                      ctypes.c_uint64, _D, _D, _D, _P]),
    "pwadv_fill_box_f64": (ctypes.c_int, [_P, _P, _P] + [_I64] * 7 + [ctypes.c_int32, ctypes.c_uint64,
                                                                      _D, _D, _D, _P]),
    "pwadv_pack_yface3_f64": (ctypes.c_int, [_P] * 4 + [_I64] * 4 + [_P]),
    "pwadv_unpack_yface3_f64": (ctypes.c_int, [_P] * 4 + [_I64] * 4 + [_P]),
    "pwadv_pack_xface3_f64": (ctypes.c_int, [_P] * 4 + [_I64] * 4 + [_P]),
    "pwadv_unpack_xface3_f64": (ctypes.c_int, [_P] * 4 + [_I64] * 4 + [_P]),
    "pwadv_ctx_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, _I64, _I64, _I64]),
    "pwadv_ctx_destroy": (ctypes.c_int, [_P]),
    "pwadv_ctx_advect_host": (ctypes.c_int, [_P] * 7 + [_D, _D, _P, _P, ctypes.c_int32, _P]),
    "pwadv_ctx_submit_host": (ctypes.c_int, [_P] * 7 + [_D, _D, _P, _P, ctypes.c_int32, _P]),
    "pwadv_ctx_sync": (ctypes.c_int, [_P]),
    "pwadv_ctx_last_bytes": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64),
                                            ctypes.POINTER(ctypes.c_uint64)]),
}


class PwadvError(RuntimeError):
    """A nonzero return code from libpwadv (message from pwadv_last_error)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libpwadv error {code}: {message}")
        self.code = code


def lib():
    """Load libpwadv.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2010_01545_b200.build` "
                    "(nvcc, sm_100a). The PW-advection path has no CPU fallback.")
            L = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            abi = L.pwadv_abi_version()
            if abi != ABI_VERSION:
                raise ImportError(f"libpwadv ABI {abi} != {ABI_VERSION}")
            _lib = L
    return _lib


_build_id = None


def build_id() -> str:
    """The source id compiled into the libpwadv.so this process loads
    (pwadv_source_id: sha256 over its sources, headers and nvcc flags, see
    build.source_id): stamps profiles (profiles/ncu_traffic.json) to the build
    they were taken with. Not a hash of the binary — nvcc output differs from
    build to build of the same sources (per-compilation module ids)."""
    global _build_id
    if _build_id is None:
        _build_id = lib().pwadv_source_id().decode()
    return _build_id


def check(rc: int) -> None:
    if rc != PWADV_OK:
        msg = lib().pwadv_last_error().decode(errors="replace")
        raise PwadvError(rc, msg)


def launch_count() -> int:
    return int(lib().pwadv_launch_count())


def reset_launch_count() -> None:
    lib().pwadv_reset_launch_count()


def opts_ptr(opts: "Opts | None"):
    return ctypes.byref(opts) if opts is not None else None
