"""ctypes binding of the plain-C fp64 oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs are the only callers.  The product package
``paper_2406_15959_b200`` never imports this module (tests/test_boundary.py checks that).
Every function documents the PAPER.md passage it follows in oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (fp-contract off so the RNG matches bit for bit)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-pthread", _SRC, "-lm", "-o", _LIB]
        )
    return _LIB


class Cfg(C.Structure):
    _fields_ = [
        ("P", C.c_int32), ("M", C.c_int32), ("p", C.c_int32), ("q", C.c_int32),
        ("problem", C.c_int32), ("init_scheme", C.c_int32),
        ("init_c", C.c_double), ("r_over_diam", C.c_double), ("seed", C.c_uint64),
        ("tikhonov", C.c_double), ("layout", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
        P = C.POINTER(Cfg)
        _lib.orc_problem.argtypes = [C.c_int, d, d, C.POINTER(d), C.POINTER(d)]
        _lib.orc_set_grf.argtypes = [vp, C.c_int]
        _lib.orc_rho.argtypes = [d, d, C.POINTER(d), C.POINTER(d), C.POINTER(d)]
        _lib.orc_geometry.argtypes = [P, vp]
        _lib.orc_rows.argtypes = [P, C.c_int, vp, vp, vp]
        _lib.orc_init_hidden.argtypes = [P, vp, vp, vp, vp]
        _lib.orc_assemble.argtypes = [P, C.c_int, vp, vp, vp, vp, vp]
        _lib.orc_qr.argtypes = [C.c_int, C.c_int, vp, C.c_int, vp]
        _lib.orc_apply_qt.argtypes = [C.c_int, C.c_int, vp, C.c_int, vp, vp]
        _lib.orc_apply_q.argtypes = [C.c_int, C.c_int, vp, C.c_int, vp, vp]
        _lib.orc_evaluate.argtypes = [P, vp, vp, vp, vp, i64, vp]
        _lib.orc_cholesky.argtypes = [vp, i64, C.c_int]
        _lib.orc_cholesky.restype = C.c_int
        _lib.orc_chol_solve.argtypes = [vp, i64, vp]
        _lib.orc_solve.argtypes = [P, vp, vp, C.c_int, vp, vp, vp, vp, i64, vp, vp, vp, vp, C.c_int]
        _lib.orc_band_cholesky.argtypes = [vp, i64, i64, C.c_int]
        _lib.orc_band_cholesky.restype = C.c_int
        _lib.orc_band_chol_solve.argtypes = [vp, i64, i64, vp]
        _lib.orc_solve.restype = C.c_int
        _lib.orc_local_pieces.argtypes = [P, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        _lib.orc_flux_eq.argtypes = [P, C.c_int, C.c_int]
        _lib.orc_flux_eq.restype = C.c_int
        _lib.orc_local_pieces.restype = C.c_int
        _lib.orc_sample_local.argtypes = [P, vp, vp, vp, vp, C.c_int, C.c_int, vp]
        _lib.orc_sample_local.restype = C.c_double
        del i32
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cfg(P, M, p, q, problem=0, init_scheme=0, init_c=0.125, r_over_diam=0.5, seed=0, tikhonov=0.0,
        layout=0) -> Cfg:
    """layout 0: face points (reading R1); 1: the paper's shared lattice with cross points (R32,
    p == q).  tikhonov < 0: the fixed rule lambda_s = eps max(m, M) ||K^s||_F (R33)."""
    return Cfg(P, M, p, q, problem, init_scheme, init_c, r_over_diam, seed, tikhonov, layout)


def set_grf(params) -> None:
    """Coefficient field of problem 6 (eqn:varpoisson): params [n][4] = (a_i, w_ix,
    w_iy, b_i) of eqn:grf; empty / None clears it (oracle.c orc_set_grf)."""
    if params is None or len(params) == 0:
        lib().orc_set_grf(None, 0)
        return
    p = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 4)
    lib().orc_set_grf(p.ctypes.data_as(C.c_void_p), int(p.shape[0]))


def rho(x: float, y: float):
    """(rho, d rho/dx, d rho/dy) of problem 6 at (x, y) (oracle.c orc_rho)."""
    r, rx, ry = C.c_double(), C.c_double(), C.c_double()
    lib().orc_rho(x, y, C.byref(r), C.byref(rx), C.byref(ry))
    return r.value, rx.value, ry.value


def problem(pid: int, x: float, y: float):
    u, f = C.c_double(), C.c_double()
    lib().orc_problem(pid, x, y, C.byref(u), C.byref(f))
    return u.value, f.value


def geometry(c: Cfg) -> dict:
    out = np.zeros(6, np.int64)
    lib().orc_geometry(C.byref(c), _p(out))
    return {"m": int(out[0]), "G": int(out[1]), "faces": int(out[2]), "N": int(out[3]), "NE": int(out[4]),
            "na": int(out[5])}


def flux_eq(c: Cfg, s: int):
    """Global flux equation of every flux row of A^s (oracle.c orc_flux_eq; -1 = none)."""
    na = geometry(c)["na"]
    return np.array([lib().orc_flux_eq(C.byref(c), s, a) for a in range(na)], dtype=np.int64)


def rows(c: Cfg, s: int):
    m = geometry(c)["m"]
    xy = np.zeros((m, 2))
    edge = np.zeros(m, np.int32)
    gidx = np.zeros(m, np.int32)
    lib().orc_rows(C.byref(c), s, _p(xy), _p(edge), _p(gidx))
    return xy, edge, gidx


def init_hidden(c: Cfg):
    N = c.P * c.P
    W = np.zeros((N, c.M, 2))
    b = np.zeros((N, c.M))
    xi = np.zeros((N, c.M, 2))
    tries = np.zeros((N, c.M), np.int32)
    lib().orc_init_hidden(C.byref(c), _p(W), _p(b), _p(xi), _p(tries))
    return W, b, xi, tries


def assemble(c: Cfg, s: int, W, b):
    """K^s (m x M), F^s (m), A (na x M: flux row e*q+k, then two per corner in layout 1; zero
    where there is no interface)."""
    geo = geometry(c)
    m = geo["m"]
    K = np.zeros((c.M, m))  # column-major storage == row-major (M, m)
    F = np.zeros(m)
    A = np.zeros((c.M, geo["na"]))
    lib().orc_assemble(C.byref(c), s, _p(np.ascontiguousarray(W)), _p(np.ascontiguousarray(b)), _p(K), _p(F), _p(A))
    return K.T.copy(), F, A.T.copy()


def qr(A: np.ndarray):
    """Unblocked Householder QR (oracle). Returns (factored column-major array (n, m), tau)."""
    m, n = A.shape
    Af = np.asfortranarray(A, dtype=np.float64).copy(order="F")
    tau = np.zeros(min(m, n))
    lib().orc_qr(m, n, Af.ctypes.data_as(C.c_void_p), m, _p(tau))
    return Af, tau


def apply_qt(Af, tau, v):
    m = Af.shape[0]
    v = np.array(v, dtype=np.float64, copy=True)
    lib().orc_apply_qt(m, len(tau), Af.ctypes.data_as(C.c_void_p), m, _p(tau), _p(v))
    return v


def apply_q(Af, tau, v):
    m = Af.shape[0]
    v = np.array(v, dtype=np.float64, copy=True)
    lib().orc_apply_q(m, len(tau), Af.ctypes.data_as(C.c_void_p), m, _p(tau), _p(v))
    return v


def cholesky(Mat: np.ndarray, nthreads: int = 1):
    L = np.array(Mat, dtype=np.float64, copy=True, order="C")
    rc = lib().orc_cholesky(_p(L), L.shape[0], nthreads)
    return np.tril(L), rc


def chol_solve(L: np.ndarray, g):
    Lc = np.ascontiguousarray(L)
    x = np.array(g, dtype=np.float64, copy=True)
    lib().orc_chol_solve(_p(Lc), Lc.shape[0], _p(x))
    return x


def band_cholesky(Bnd: np.ndarray, nthreads: int = 1):
    """Plain banded Cholesky (oracle.c orc_band_cholesky) of the lower band Bnd[i, k - i + bw]
    (row i holds columns i - bw .. i).  Returns (factor band, rc)."""
    B = np.array(Bnd, dtype=np.float64, copy=True, order="C")
    rc = lib().orc_band_cholesky(_p(B), B.shape[0], B.shape[1] - 1, nthreads)
    return B, rc


def band_chol_solve(B: np.ndarray, g):
    Bc = np.ascontiguousarray(B)
    x = np.array(g, dtype=np.float64, copy=True)
    lib().orc_band_chol_solve(_p(Bc), Bc.shape[0], Bc.shape[1] - 1, _p(x))
    return x


def evaluate(c: Cfg, W, b, coef, xy):
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    u = np.zeros(xy.shape[0])
    lib().orc_evaluate(C.byref(c), _p(np.ascontiguousarray(W)), _p(np.ascontiguousarray(b)),
                       _p(np.ascontiguousarray(coef)), _p(xy), xy.shape[0], u.ctypes.data_as(C.c_void_p))
    return u


def solve(c: Cfg, W, b, xy_eval=None, nthreads: int | None = None, want_system: bool = False, band: int = 0):
    """Algorithm 1 with the oracle's literal eqn:schur route.  band: interface
    Cholesky 0 auto (banded in strip order when G > 20000), 1 dense, 2 banded (want_system:
    dense route only)."""
    geo = geometry(c)
    G, N = geo["G"], geo["N"]
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    uG = np.zeros(max(G, 1))
    coef = np.zeros((N, c.M))
    resid = np.zeros(N)
    times = np.zeros(8)
    n_eval = 0 if xy_eval is None else xy_eval.shape[0]
    xy_eval = None if xy_eval is None else np.ascontiguousarray(xy_eval, dtype=np.float64)
    u = np.zeros(max(n_eval, 1))
    if want_system and band == 2:
        raise ValueError("want_system needs the dense route")
    Mout = np.zeros((G, G)) if (want_system and G > 0) else None
    gout = np.zeros(G) if (want_system and G > 0) else None
    rc = lib().orc_solve(C.byref(c), _p(np.ascontiguousarray(W)), _p(np.ascontiguousarray(b)), nthreads,
                         _p(uG), _p(coef), _p(resid), _p(xy_eval), n_eval, _p(u), _p(Mout), _p(gout), _p(times),
                         int(band))
    if rc != 0:
        raise RuntimeError(f"oracle solve failed rc={rc}")
    out = {"uG": uG[:G], "coef": coef, "resid": resid, "u": u[:n_eval],
           "times": dict(zip(["local", "iface_assemble", "iface_solve", "back", "eval"], times[:5].tolist()))}
    if want_system:
        out["M"], out["g"] = Mout, gout
    return out


def local_pieces(c: Cfg, s: int, W, b, uG=None):
    q = c.q
    mgmax = 4 * q + 4
    mamax = geometry(c)["na"]
    S1 = np.zeros((mgmax, mgmax))
    g1 = np.zeros(mgmax)
    PB = np.zeros((mamax, mgmax))
    pF = np.zeros(mamax)
    ig = np.zeros(mgmax, np.int32)
    aeq = np.zeros(mamax, np.int32)
    ma = np.zeros(1, np.int32)
    coef = np.zeros(c.M)
    resid = np.zeros(1)
    uGa = None if uG is None else np.ascontiguousarray(uG, dtype=np.float64)
    mg = lib().orc_local_pieces(C.byref(c), s, _p(np.ascontiguousarray(W)), _p(np.ascontiguousarray(b)), _p(uGa),
                                _p(S1), _p(g1), _p(PB), _p(pF), _p(ig), _p(coef), _p(resid), _p(aeq), _p(ma))
    na = int(ma[0])
    S1 = S1.reshape(-1)[: mg * mg].reshape(mg, mg)
    PB = PB.reshape(-1)[: na * mg].reshape(na, mg)
    out = {"mg": mg, "ma": na, "S1": S1, "g1": g1[:mg], "PB": PB, "pF": pF[:na], "ig": ig[:mg], "aeq": aeq[:na]}
    if uG is not None:
        out["coef"], out["resid"] = coef, float(resid[0])
    return out


def sample_local(c: Cfg, W, b, s_list, uG=None, nthreads: int | None = None) -> float:
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    s_arr = np.ascontiguousarray(s_list, dtype=np.int32)
    sink = np.zeros(len(s_arr))
    uGa = None if uG is None else np.ascontiguousarray(uG, dtype=np.float64)
    return lib().orc_sample_local(C.byref(c), _p(np.ascontiguousarray(W)), _p(np.ascontiguousarray(b)), _p(uGa),
                                  _p(s_arr), len(s_arr), nthreads, _p(sink))
