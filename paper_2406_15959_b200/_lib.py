"""ctypes binding of libelmddm.so: argument marshalling only (names = include/elmddm.h).

Every step of the hot path runs in the library's CUDA kernels; this module only converts torch
tensors to device pointers and streams.  There is no CPU fallback: if the library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ELMDDM_LIB selects an instrumented build of the same library (tools/chol_prof.py)
LIB_PATH = os.environ.get("ELMDDM_LIB", os.path.join(HERE, "libelmddm.so"))


class ElmddmError(RuntimeError):
    pass


class Config(C.Structure):
    _fields_ = [
        ("P", C.c_int32), ("M", C.c_int32), ("p", C.c_int32), ("q", C.c_int32),
        ("problem", C.c_int32), ("init_scheme", C.c_int32),
        ("init_c", C.c_double), ("r_over_diam", C.c_double), ("seed", C.c_uint64),
        ("s_begin", C.c_int32), ("s_end", C.c_int32), ("interface_mode", C.c_int32), ("layout", C.c_int32),
        ("tikhonov", C.c_double),
    ]


class Sizes(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "N", "S", "m", "ld", "ncols", "kaug", "G", "faces", "kaug_elems", "at_elems", "tau_elems",
        "pbuf_ld", "pbuf_elems", "sbuf_ld", "sbuf_elems", "work_elems", "band_ld", "band_nbw", "band_elems",
        "G_pad", "halfband", "chol_tasks", "chol_flops", "chol_n", "chol_blocks", "chol_ordering",
        "e_impl_begin", "e_impl_end", "ne", "na", "n_eq")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


STATUS = {0: "ELMDDM_OK", 1: "ELMDDM_EINVAL", 2: "ELMDDM_ENUMERIC", 3: "ELMDDM_ECUDA", 4: "ELMDDM_ENOMEM",
          100: "ELMDDM_WRANK"}
WRANK = 100


class RankWarning(UserWarning):
    """ELMDDM_WRANK: a subdomain's K^s is numerically rank deficient (min |R11_ii| < 1e-14 max
    |R11_ii|); the results are still computed (include/elmddm.h)."""

# every exported entry point of include/elmddm.h
EXPORTS = [
    "elmddm_create", "elmddm_destroy", "elmddm_last_error", "elmddm_sizes", "elmddm_sync",
    "elmddm_interface_points", "elmddm_band_index", "elmddm_chol_plan", "elmddm_interface_cg", "elmddm_init_hidden", "elmddm_assemble",
    "elmddm_set_coefficient", "elmddm_plan_query", "elmddm_dist_export", "elmddm_dist_import", "elmddm_dist_pool", "elmddm_dist_handshake",
    "elmddm_debug_dist_emulate",
    "elmddm_local_factor", "elmddm_schur_accumulate", "elmddm_interface_assemble",
    "elmddm_interface_factor_solve", "elmddm_interface_solve", "elmddm_back_solve", "elmddm_evaluate",
    "elmddm_set_timing", "elmddm_timing", "elmddm_dmma_probe",
]

KCLASSES = ["init", "assemble", "panel", "gemm_qr", "trsm", "gemm_schur", "iface", "chol", "gemm_chol", "trsv",
            "back", "eval"]


class Timing(C.Structure):
    _fields_ = [("launches", C.c_int64), ("count", C.c_int64 * 12), ("ms", C.c_double * 12)]

_lib = None


def load():
    """Load libelmddm.so (built by paper_2406_15959_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_2406_15959_b200/build.py` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, st = C.c_void_p, C.c_int64, C.c_int
    ctxp = C.c_void_p
    L.elmddm_create.argtypes = [C.POINTER(Config), C.c_int, C.POINTER(C.c_void_p)]
    L.elmddm_destroy.argtypes = [ctxp]
    L.elmddm_destroy.restype = None
    L.elmddm_last_error.argtypes = [ctxp]
    L.elmddm_last_error.restype = C.c_char_p
    L.elmddm_sizes.argtypes = [ctxp, C.POINTER(Sizes)]
    L.elmddm_sync.argtypes = [ctxp, vp]
    L.elmddm_interface_points.argtypes = [ctxp, vp]
    L.elmddm_band_index.argtypes = [ctxp, i64, i64]
    L.elmddm_band_index.restype = i64
    L.elmddm_chol_plan.argtypes = [ctxp, vp, vp, vp]
    L.elmddm_interface_cg.argtypes = [ctxp, vp, vp, vp, vp, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_double), vp]
    L.elmddm_init_hidden.argtypes = [ctxp, vp, vp, vp, vp]
    L.elmddm_assemble.argtypes = [ctxp, vp, vp, vp, vp, vp]
    L.elmddm_set_coefficient.argtypes = [ctxp, vp, C.c_int32]
    L.elmddm_plan_query.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp]
    L.elmddm_dist_export.argtypes = [ctxp, vp]
    L.elmddm_dist_import.argtypes = [ctxp, C.c_int32, C.c_int32, vp]
    L.elmddm_dist_pool.argtypes = [ctxp, C.POINTER(C.c_void_p)]
    L.elmddm_dist_handshake.argtypes = [ctxp, C.c_int32, C.POINTER(C.c_int32)]
    L.elmddm_debug_dist_emulate.argtypes = [ctxp, C.c_int32, vp, vp, vp, vp, C.POINTER(C.c_int64), vp]
    L.elmddm_local_factor.argtypes = [ctxp, vp, vp, vp, vp]
    L.elmddm_schur_accumulate.argtypes = [ctxp, vp, vp, vp, vp, vp, vp]
    L.elmddm_interface_assemble.argtypes = [ctxp, vp, vp, vp, vp, vp, vp]
    L.elmddm_interface_factor_solve.argtypes = [ctxp, vp, vp, vp, vp, vp]
    L.elmddm_interface_solve.argtypes = [ctxp, vp, vp, vp, vp, vp, vp, vp]
    L.elmddm_back_solve.argtypes = [ctxp, vp, vp, vp, vp, vp, vp]
    L.elmddm_evaluate.argtypes = [ctxp, vp, vp, vp, vp, i64, vp, vp]
    L.elmddm_set_timing.argtypes = [ctxp, C.c_int]
    L.elmddm_timing.argtypes = [ctxp, C.POINTER(Timing), C.c_int]
    L.elmddm_dmma_probe.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double)]
    for name in EXPORTS:
        f = getattr(L, name)
        if f.restype is C.c_int or name in ("elmddm_create",):
            f.restype = st
    for name in ["elmddm_create", "elmddm_sizes", "elmddm_sync", "elmddm_interface_points", "elmddm_chol_plan",
                 "elmddm_interface_cg",
                 "elmddm_init_hidden",
                 "elmddm_assemble", "elmddm_local_factor", "elmddm_schur_accumulate", "elmddm_interface_assemble",
                 "elmddm_interface_factor_solve", "elmddm_interface_solve", "elmddm_back_solve", "elmddm_evaluate",
                 "elmddm_set_timing", "elmddm_timing", "elmddm_dmma_probe"]:
        getattr(L, name).restype = st
    _lib = L
    return L
