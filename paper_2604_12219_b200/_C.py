"""ctypes binding of libpasa.so (include/pasa.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind this library; this
module only mirrors the C structs and loads the in-tree shared object.  It
fails loudly if the library is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PASA_LIB") or os.path.join(_HERE, "lib", "libpasa.so")   # override: A/B builds

PASA_OK, PASA_EINVAL, PASA_ESHAPE, PASA_EDTYPE, PASA_EUNSUPPORTED = 0, 1, 2, 3, 4
PASA_EDEGENERATE, PASA_ECUDA, PASA_ENOSPACE = 5, 6, 7
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ESHAPE", 3: "EDTYPE", 4: "EUNSUPPORTED",
                5: "EDEGENERATE", 6: "ECUDA", 7: "ENOSPACE"}
PASA_BF16, PASA_F32 = 0, 1
PASA_IN_LATENT, PASA_IN_VELOCITY = 0, 1
COMP = {"grouped": 0, "zeroth": 1, "none": 2}
PASA_ATTN_FORCE_SIMT = 1
PASA_ATTN_STATS_ONLY = 2
PASA_ATTN_REUSE_STATS = 4
PASA_ATTN_CTA_PAIR = 8
PRIOR = {"none": 0, "global": 1, "group": 2}

# every symbol include/pasa.h declares (tests check the library exports them all)
EXPORTS = [
    "pasa_budget_workspace_bytes", "pasa_route_workspace_bytes", "pasa_budget_init",
    "pasa_route_init", "pasa_budget_fini", "pasa_route_fini", "pasa_budget", "pasa_route",
    "pasa_attn", "pasa_attn_ex", "pasa_layer_seed", "pasa_budget_read", "pasa_route_read",
    "pasa_route_pooled_read", "pasa_route_dims", "pasa_last_launch_count", "pasa_last_error",
    "pasa_version", "pasa_debug_trace", "pasa_debug_flags", "pasa_attn_stats_read",
    "pasa_route_v", "pasa_route_het_read", "pasa_calibrate", "pasa_copy2d",
    "pasa_budget_local_sum", "pasa_budget_from_sums", "pasa_route_zc", "pasa_attn_zc",
]


class PasaTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("B", ctypes.c_int64), ("S", ctypes.c_int64), ("H", ctypes.c_int64),
                ("D", ctypes.c_int64), ("sB", ctypes.c_int64), ("sS", ctypes.c_int64),
                ("sH", ctypes.c_int64)]


class PasaLatent(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("numel", ctypes.c_int64)]


class PasaSchedule(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("step", ctypes.c_int32), ("rho", ctypes.c_double),
                ("dense_frac", ctypes.c_double), ("l1_mean", ctypes.c_double),
                ("h_t", ctypes.c_double), ("h_tm1", ctypes.c_double),
                ("rho_max", ctypes.c_double), ("rho_table", ctypes.POINTER(ctypes.c_double)),
                ("kind", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class PasaRouteCfg(ctypes.Structure):
    _fields_ = [("Bq", ctypes.c_int32), ("Bk", ctypes.c_int32), ("G", ctypes.c_int32),
                ("comp", ctypes.c_int32), ("beta", ctypes.c_double),
                ("H_total", ctypes.c_int64), ("head_offset", ctypes.c_int64),
                ("prior", ctypes.c_int32), ("_pad", ctypes.c_int32), ("eps", ctypes.c_double),
                ("qb_begin", ctypes.c_int32), ("qb_end", ctypes.c_int32),
                ("qk_fp8", ctypes.c_int32), ("_pad2", ctypes.c_int32)]


class PasaShards(ctypes.Structure):
    """pasa_shards: a [1, S, H, D] bf16 tensor as P sequence shards (include/pasa.h)."""
    _fields_ = [("dtype", ctypes.c_int32), ("nshards", ctypes.c_int32),
                ("S", ctypes.c_int64), ("H", ctypes.c_int64), ("D", ctypes.c_int64),
                ("sS", ctypes.c_int64), ("sH", ctypes.c_int64),
                ("start", ctypes.c_int64 * 9), ("data", ctypes.c_void_p * 8)]


class PasaError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: PASA_{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libpasa.so (built by paper_2604_12219_b200.build); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2604_12219_b200.build` "
                           "(there is no fallback path)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                            ctypes.c_size_t)
    T = ctypes.POINTER(PasaTensor)
    LT = ctypes.POINTER(PasaLatent)
    L.pasa_budget_workspace_bytes.restype = SZ
    L.pasa_budget_workspace_bytes.argtypes = []
    L.pasa_route_workspace_bytes.restype = SZ
    L.pasa_route_workspace_bytes.argtypes = [ctypes.POINTER(PasaRouteCfg), I64, I64, I64, I64]
    L.pasa_budget_init.argtypes = [P, SZ, ctypes.POINTER(P)]
    L.pasa_route_init.argtypes = [P, SZ, ctypes.POINTER(PasaRouteCfg), I64, I64, I64, I64,
                                  ctypes.POINTER(P)]
    L.pasa_budget_fini.argtypes = [P]
    L.pasa_budget_fini.restype = None
    L.pasa_route_fini.argtypes = [P]
    L.pasa_route_fini.restype = None
    L.pasa_budget.argtypes = [LT, LT, LT, ctypes.POINTER(PasaSchedule), P, P]
    L.pasa_budget_local_sum.argtypes = [LT, LT, LT, ctypes.POINTER(PasaSchedule), P, P, P]
    L.pasa_budget_from_sums.argtypes = [P, I32, I64, ctypes.POINTER(PasaSchedule), P, P]
    L.pasa_route.argtypes = [T, T, P, U64, I32, P, P]
    L.pasa_route_v.argtypes = [T, T, T, P, U64, I32, P, P]
    L.pasa_route_het_read.argtypes = [P, P, P]
    L.pasa_copy2d.argtypes = [P, SZ, P, SZ, SZ, SZ, I32, P]
    L.pasa_calibrate.argtypes = [P, I32, I32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                 P, P, P, P]
    L.pasa_attn.argtypes = [T, T, T, P, T, P]
    L.pasa_attn_ex.argtypes = [T, T, T, P, T, ctypes.c_uint32, P]
    SH = ctypes.POINTER(PasaShards)
    L.pasa_route_zc.argtypes = [SH, SH, SH, P, U64, I32, P, T, T, T, P]
    L.pasa_attn_zc.argtypes = [T, T, T, P, SH, P]
    L.pasa_layer_seed.argtypes = [U64, I32]
    L.pasa_layer_seed.restype = U64
    L.pasa_budget_read.argtypes = [P, ctypes.POINTER(ctypes.c_double), P]
    L.pasa_route_read.argtypes = [P, P, P, P, P, P]
    L.pasa_route_pooled_read.argtypes = [P, P, P, P]
    L.pasa_route_dims.argtypes = [P, ctypes.POINTER(ctypes.c_int64)]
    L.pasa_attn_stats_read.argtypes = [P, P, P, P, I32, P]
    L.pasa_attn_stats_read.restype = ctypes.c_int
    L.pasa_last_launch_count.restype = I32
    L.pasa_last_launch_count.argtypes = []
    L.pasa_last_error.restype = ctypes.c_char_p
    L.pasa_last_error.argtypes = []
    L.pasa_version.restype = ctypes.c_char_p
    L.pasa_version.argtypes = []
    L.pasa_debug_trace.restype = ctypes.c_int
    L.pasa_debug_trace.argtypes = [P, ctypes.c_int, ctypes.c_int]
    L.pasa_debug_flags.restype = ctypes.c_int
    L.pasa_debug_flags.argtypes = [ctypes.c_int]
    for name in ("pasa_budget_init", "pasa_route_init", "pasa_budget", "pasa_route",
                 "pasa_budget_local_sum", "pasa_budget_from_sums",
                 "pasa_attn", "pasa_attn_ex", "pasa_budget_read", "pasa_route_read",
                 "pasa_route_pooled_read", "pasa_route_dims", "pasa_route_zc", "pasa_attn_zc"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status != PASA_OK:
        raise PasaError(status, where, lib().pasa_last_error().decode())
