"""Pins of the CPU oracle (oracle/oracle.c) against what the paper and the mathematics fix.

CPU only (no GPU marker).  Each test names the passage or closed form it checks and is chosen so
that a plausible mistake (dropped term, wrong sign or index, transposed operand) fails it.
Independent arithmetic here is plain numpy (np.tanh, np.linalg.pinv / lstsq, finite differences),
never the oracle's own routines re-called.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import workloads as WL

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


def mkcfg(k=None, **kw):
    if k is not None:
        c = WL.config(k)
        c.update(kw)
    else:
        c = dict(P=2, M=16, p=6, q=5, problem=0, seed=7, init_scheme=0, init_c=0.125, r_over_diam=0.5)
        c.update(kw)
    return O.cfg(c["P"], c["M"], c["p"], c["q"], c["problem"], c.get("init_scheme", 0),
                 c.get("init_c", 0.125), c.get("r_over_diam", 0.5), c["seed"], c.get("tikhonov", 0.0),
                 c.get("layout", 0))


# ------------------------------------------------------------------------------------------------
# geometry (readings R1, R14)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("k", range(5))
def test_geometry_counts(k):
    g = O.geometry(mkcfg(k))
    assert g["m"] == GOLD["geometry"]["m"][k]
    assert g["G"] == GOLD["geometry"]["G"][k]


def test_shared_interface_points_bitwise_and_opposite_normals():
    """A face's points are the same in both neighbours (bit for bit, same global index) and the
    two neighbours see it through opposite edges, i.e. opposite outward normals."""
    c = mkcfg(P=3, M=8, p=4, q=5)
    P, q = 3, 5
    seen = {}
    for s in range(P * P):
        xy, edge, gidx = O.rows(c, s)
        for r in np.where(gidx >= 0)[0]:
            seen.setdefault(int(gidx[r]), []).append((s, int(edge[r]), tuple(xy[r])))
    G = O.geometry(c)["G"]
    assert sorted(seen) == list(range(G))
    opposite = {0: 1, 1: 0, 2: 3, 3: 2}
    for gi, lst in seen.items():
        assert len(lst) == 2
        (s1, e1, p1), (s2, e2, p2) = lst
        assert p1 == p2                       # bitwise identical coordinates
        assert opposite[e1] == e2             # opposite outward normals
    # points strictly inside the face (endpoints excluded, reading R1)
    xy, edge, gidx = O.rows(c, 4)
    h = 1.0 / P
    for e in range(4):
        pts = xy[edge == e]
        along = pts[:, 1] if e < 2 else pts[:, 0]
        lo = (4 // P if e < 2 else 4 % P) * h
        assert np.all(along > lo) and np.all(along < lo + h)
        assert np.all(np.diff(along) > 0)      # increasing coordinate
    assert (edge == -1).sum() == 16 and len(edge) == 16 + 4 * q


# ------------------------------------------------------------------------------------------------
# initialisation eqn:init
# ------------------------------------------------------------------------------------------------
def test_init_l_from_paper_table1():
    """n = 2^16 and c = 1/8 give l = 32 (Table 1 P:564 'sqrt(n/64)')."""
    g = GOLD["init_l_paper_table1"]
    c = mkcfg(P=4, M=4096, p=2, q=2, init_c=g["c"])   # N*M = 65536
    W, b, xi, tries = O.init_hidden(c)
    l = g["l"]
    assert np.abs(W).max() <= l
    assert np.abs(W).max() > 0.999 * l                    # U([-l,l]^2) fills the box
    assert abs(np.mean(W)) < 0.01 * l
    assert abs(np.var(W) - l * l / 3) < 0.02 * l * l / 3    # variance of U(-l,l)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_init_l_configs(k):
    W, b, xi, tries = O.init_hidden(mkcfg(k))
    l = GOLD["init_l_configs"]["l"][k]
    assert np.abs(W).max() <= l and np.abs(W).max() > 0.99 * l


def test_init_bias_centres_and_collar():
    """b = -w.xi so phi_j(xi_j) = sigma(0) = 0 (eqn:init); dist(xi, Omega_s) <= r with
    r = diam/2; rejection acceptance = area ratio (closed form in golden/pins.json)."""
    c = mkcfg(P=4, M=4000, p=2, q=2, seed=11)
    W, b, xi, tries = O.init_hidden(c)
    z = W[..., 0] * xi[..., 0] + W[..., 1] * xi[..., 1] + b
    scale = np.abs(W[..., 0] * xi[..., 0]) + np.abs(W[..., 1] * xi[..., 1])
    assert np.all(np.abs(z) <= 4 * np.finfo(float).eps * (scale + 1e-300))
    P = 4
    h = 1.0 / P
    r = 0.5 * math.sqrt(2) * h
    for s in range(P * P):
        i, j = s % P, s // P
        dx = np.maximum(np.maximum(i * h - xi[s, :, 0], xi[s, :, 0] - (i + 1) * h), 0)
        dy = np.maximum(np.maximum(j * h - xi[s, :, 1], xi[s, :, 1] - (j + 1) * h), 0)
        assert np.all(dx * dx + dy * dy <= r * r * (1 + 1e-12))
    acc = tries.size / tries.sum()
    p = GOLD["collar_acceptance"]["value"]
    se = math.sqrt(p * (1 - p) / tries.sum())
    assert abs(acc - p) < 4 * se
    # the sampled xi fill the collar: some lie outside Omega_s, some near the rounded corners
    s = 5
    i, j = s % P, s // P
    out = (xi[s, :, 0] < i * h) | (xi[s, :, 0] > (i + 1) * h)
    assert 0.2 < out.mean() < 0.6


def test_init_he_and_manual():
    W, b, xi, _ = O.init_hidden(mkcfg(P=2, M=500, init_scheme=2))
    assert np.all(b == 0.0)
    l = math.sqrt(2.0 / 500)
    assert np.abs(W).max() <= l and np.abs(W).max() > 0.98 * l
    W, b, xi, _ = O.init_hidden(mkcfg(P=2, M=500, init_scheme=1))
    assert np.abs(W).max() <= 1.0 and np.abs(W).max() > 0.98
    z = W[..., 0] * xi[..., 0] + W[..., 1] * xi[..., 1] + b
    assert np.abs(z).max() < 1e-15


def test_init_deterministic_and_seed_dependent():
    a = O.init_hidden(mkcfg(seed=3))
    b_ = O.init_hidden(mkcfg(seed=3))
    c = O.init_hidden(mkcfg(seed=4))
    assert np.array_equal(a[0], b_[0]) and np.array_equal(a[1], b_[1])
    assert not np.array_equal(a[0], c[0])


# ------------------------------------------------------------------------------------------------
# manufactured problems and assembly (eqn:nonoverlap_discrete P:231-280)
# ------------------------------------------------------------------------------------------------
def test_rhs_pinned_value():
    g = GOLD["poisson_rhs_problem1"]
    u, f = O.problem(1, g["x"], g["y"])
    assert abs(f - g["f"]) < 1e-12 * abs(g["f"])


@pytest.mark.parametrize("pid", [0, 1, 2, 3, 4])
def test_rhs_is_minus_laplacian(pid):
    rng = np.random.default_rng(pid)
    h = 1e-4
    for x, y in rng.uniform(0.05, 0.95, size=(20, 2)):
        U = lambda a, b: WL.exact(pid, np.array([[a, b]]))[0]
        lap = (U(x + h, y) + U(x - h, y) + U(x, y + h) + U(x, y - h) - 4 * U(x, y)) / h**2
        u, f = O.problem(pid, x, y)
        assert abs(u - U(x, y)) < 1e-13 * (1 + abs(u))
        assert abs(f + lap) < 2e-5 * (1 + abs(f))
    assert O.problem(5, 0.3, 0.7) == (0.0, 0.0)


def test_tanh_derivatives_at_zero_in_rows():
    """Place a neuron so that z = 0 exactly at chosen rows: value rows give sigma(0) = 0,
    interior rows -|w|^2 sigma''(0) = 0 and flux rows (w.n) sigma'(0) = w.n."""
    c = mkcfg(P=2, M=3, p=3, q=3)
    xy, edge, gidx = O.rows(c, 3)  # subdomain (1,1): left and bottom edges are interface
    N = 4
    W = np.zeros((N, 3, 2))
    b = np.zeros((N, 3))
    rl = np.where(edge == 0)[0][1]      # a left-edge (interface) point
    ri = 4                              # an interior point
    W[3, 0] = (2.0, 1.0)
    b[3, 0] = -(2.0 * xy[rl, 0] + 1.0 * xy[rl, 1])
    W[3, 1] = (-3.0, 0.5)
    b[3, 1] = -(-3.0 * xy[ri, 0] + 0.5 * xy[ri, 1])
    K, F, A = O.assemble(c, 3, W, b)
    gold = GOLD["tanh_derivatives_at_0"]
    assert K[rl, 0] == gold["sigma"]
    ar = rl - 9                          # flux row index e*q + k
    assert A[ar, 0] == -2.0 * gold["sigma1"]      # n = (-1, 0) on the left edge
    assert K[ri, 1] == -(9.0 + 0.25) * gold["sigma2"]
    # a zero neuron (w = 0, b = 0) gives sigma = 0 everywhere and no flux
    assert np.all(K[:, 2] == 0.0) and np.all(A[:, 2] == 0.0)


@pytest.mark.parametrize("s", [0, 3])
def test_assembly_rows_vs_finite_differences(s):
    """Interior rows = -Lap phi, value rows = phi, flux rows = d phi / d n_s, checked against
    np.tanh and central differences (1e-6 relative); F = [f; g; 0]."""
    c = mkcfg(P=2, M=24, p=5, q=4, problem=1, seed=5)
    W, b, xi, _ = O.init_hidden(c)
    K, F, A = O.assemble(c, s, W, b)
    xy, edge, gidx = O.rows(c, s)
    w = W[s]
    bb = b[s]
    phi = lambda p: np.tanh(w[:, 0] * p[0] + w[:, 1] * p[1] + bb)
    h = 1e-4
    normals = {0: (-1, 0), 1: (1, 0), 2: (0, -1), 3: (0, 1)}
    q = 4
    for r in range(len(edge)):
        p = xy[r]
        if edge[r] < 0:
            lap = (phi(p + [h, 0]) + phi(p - [h, 0]) + phi(p + [0, h]) + phi(p - [0, h]) - 4 * phi(p)) / h**2
            assert np.allclose(K[r], -lap, rtol=0, atol=1e-6 * np.abs(lap).max())
            u, f = O.problem(1, p[0], p[1])
            assert F[r] == f
        else:
            assert np.allclose(K[r], phi(p), rtol=0, atol=2e-15)
            e = edge[r]
            ar = r - 25
            assert ar // q == e
            n = np.array(normals[e], float)
            d = (phi(p + h * n) - phi(p - h * n)) / (2 * h)
            if gidx[r] >= 0:
                assert np.allclose(A[ar], d, rtol=0, atol=1e-7 * np.abs(d).max())
                assert F[r] == 0.0
            else:
                assert np.all(A[ar] == 0.0)
                assert F[r] == WL.exact(1, p[None])[0] or abs(F[r] - WL.exact(1, p[None])[0]) < 1e-14


# ------------------------------------------------------------------------------------------------
# Householder QR (reading R11/R20)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (50, 10), (200, 120), (37, 37)])
def test_qr_reconstruction_and_orthogonality(shape):
    rng = np.random.default_rng(sum(shape))
    A = rng.standard_normal(shape)
    Af, tau = O.qr(A)
    m, n = shape
    R = np.triu(Af[: min(m, n), :])
    QR = np.stack([O.apply_q(Af, tau, np.concatenate([R[:, j], np.zeros(m - R.shape[0])])) for j in range(n)], 1)
    assert np.linalg.norm(QR - A) <= 1e-12 * np.linalg.norm(A)
    v = rng.standard_normal(m)
    assert np.allclose(O.apply_qt(Af, tau, O.apply_q(Af, tau, v)), v, atol=1e-13 * np.linalg.norm(v))
    # |R| diagonal = |numpy R| diagonal (QR unique up to signs)
    Rn = np.linalg.qr(A, mode="r")
    assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(Rn)), rtol=1e-10)


def test_qr_zero_column_and_lstsq_mean():
    A = np.zeros((4, 2))
    A[:, 1] = [1, 2, 3, 4]
    Af, tau = O.qr(A)
    assert tau[0] == 0.0
    g = GOLD["lstsq_mean"]
    K = np.array(g["K"])
    Af, tau = O.qr(K)
    y = O.apply_qt(Af, tau, np.array(g["rhs"]))
    c = y[:1] / Af[0, 0]
    assert np.allclose(c, g["c"], rtol=1e-15)
    # least-squares optimality K^T (K c - rhs) = 0 on a random tall system
    rng = np.random.default_rng(1)
    K = rng.standard_normal((50, 10))
    rhs = rng.standard_normal(50)
    Af, tau = O.qr(K)
    y = O.apply_qt(Af, tau, rhs)
    c = np.linalg.solve(np.triu(Af[:10, :10]), y[:10])
    assert np.linalg.norm(K.T @ (K @ c - rhs)) < 1e-12 * np.linalg.norm(K) * np.linalg.norm(rhs)


def test_cholesky_pins():
    g = GOLD["spd_2x2"]
    L, rc = O.cholesky(np.array(g["A"]))
    assert rc == 0
    assert np.allclose(O.chol_solve(L, g["b"]), g["x"], rtol=1e-15)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((300, 200))
    S = X.T @ X + np.eye(200)
    L, rc = O.cholesky(S, nthreads=4)
    assert rc == 0 and np.allclose(L @ L.T, S, atol=1e-10 * np.abs(S).max())
    bb = rng.standard_normal(200)
    assert np.allclose(O.chol_solve(L, bb), np.linalg.solve(S, bb), rtol=1e-9)
    S[5, 5] = -1.0
    _, rc = O.cholesky(S)
    assert rc == 6                        # 1 + column of the first non-positive pivot


def _to_band(S, bw):
    n = S.shape[0]
    B = np.zeros((n, bw + 1))
    for i in range(n):
        lo = max(0, i - bw)
        B[i, lo - i + bw:] = S[i, lo:i + 1]
    return B


def test_band_cholesky_pins():
    """Banded Cholesky against numpy's dense Cholesky and solve on a random
    SPD band matrix; a non-positive pivot is reported by its column; threads do not change it."""
    rng = np.random.default_rng(11)
    n, bw = 240, 17
    X = rng.standard_normal((n, n))
    S = np.triu(np.tril(X @ X.T, bw), -bw) + 4.0 * bw * np.eye(n)     # banded, diagonally dominant
    B, rc = O.band_cholesky(_to_band(S, bw), nthreads=3)
    assert rc == 0
    Lref = np.linalg.cholesky(S)
    assert np.allclose(_to_band(Lref, bw), B, rtol=0, atol=1e-12 * np.abs(Lref).max())
    bb = rng.standard_normal(n)
    assert np.allclose(O.band_chol_solve(B, bb), np.linalg.solve(S, bb), rtol=1e-10)
    B1, _ = O.band_cholesky(_to_band(S, bw), nthreads=1)
    assert np.array_equal(B1, B)
    S2 = S.copy()
    S2[37, 37] = -1.0
    _, rc = O.band_cholesky(_to_band(S2, bw), nthreads=4)
    assert rc == 38


@pytest.mark.parametrize("P,q", [(3, 4), (4, 3), (5, 2)])
def test_strip_order_half_bandwidth(P, q):
    """Reading R14: in strip order the interface matrix M of eqn:schur has half-bandwidth
    (4P-1)q-1 -- the band the oracle's banded route stores (a narrower band would drop entries).
    It is attained from P = 4 on (the flux rows of a horizontal face H(i, j) couple H(i, j-1) with
    H(i, j+1), two strips apart, which needs 1 <= j <= P-3); below, it is an upper bound."""
    c = mkcfg(P=P, M=24, p=6, q=q, problem=2)
    W, b, _, _ = O.init_hidden(c)
    r = O.solve(c, W, b, want_system=True, band=1)
    i, j = np.nonzero(r["M"])
    hbw = int(np.abs(i - j).max())
    assert hbw == (4 * P - 1) * q - 1 if P >= 4 else hbw <= (4 * P - 1) * q - 1


@pytest.mark.parametrize("kw", [dict(k=1), dict(P=3, M=40, p=8, q=6, problem=1), dict(P=5, M=24, p=6, q=3, problem=2)])
def test_band_route_equals_dense_route(kw):
    """The banded interface route (used for configs 3-4) gives bit-identical u_Gamma, c, r_s and u
    to the dense route on the same problem: M's entries are summed in the same order and the
    terms the band leaves out of the Cholesky sums are exact zeros."""
    c = mkcfg(**kw)
    W, b, _, _ = O.init_hidden(c)
    xy = WL.eval_grid(21)
    r1 = O.solve(c, W, b, xy, band=1)
    r2 = O.solve(c, W, b, xy, band=2)
    for key in ("uG", "coef", "resid", "u"):
        assert np.array_equal(r1[key], r2[key]), key


# ------------------------------------------------------------------------------------------------
# Schur system (eqn:eliminated P:351-373, LS_system P:398-406, eqn:schur P:407-410)
# ------------------------------------------------------------------------------------------------
def _global_blocks(c, W, b):
    """Dense K (block diag), B (stacked -E), A (flux rows, globally indexed), F, from the oracle's
    assembly; numpy builds everything else."""
    geo = O.geometry(c)
    N, G, M, NE = geo["N"], geo["G"], c.M, geo["NE"]
    Ks, Fs, Bs, As = [], [], [], []
    for s in range(N):
        K, F, A4 = O.assemble(c, s, W, b)
        xy, edge, gidx = O.rows(c, s)
        m = len(edge)  # collocation rows, then (tikhonov != 0) the M damping rows
        B = np.zeros((m, G))
        Ag = np.zeros((NE, M))
        for r in np.where(gidx >= 0)[0]:
            B[r, gidx[r]] = -1.0
        for ar, eq in enumerate(O.flux_eq(c, s)):  # A = [A^1 ... A^N] by global flux equation
            if eq >= 0:
                Ag[eq] += A4[ar]
        Ks.append(K)
        Fs.append(F)
        Bs.append(B)
        As.append(Ag)
    from scipy.linalg import block_diag

    return block_diag(*Ks), np.vstack(Bs), np.hstack(As), np.concatenate(Fs)


def _tiny_cfg(P=2, **kw):
    # well-conditioned tiny instance: few neurons, many points, larger l (init_c = 1)
    base = dict(P=P, M=10, p=7, q=6, problem=0, seed=2, init_c=1.0)
    base.update(kw)
    return mkcfg(**base)


@pytest.mark.parametrize("P,layout", [(2, 0), (3, 0), (2, 1), (3, 1)])
def test_schur_matches_literal_eqn_schur(P, layout):
    """Oracle M, g == B^T (I + K^{+T} A^T A K^+ - K K^+) B and ... F with np.linalg.pinv;
    layout 1: the shared lattice with cross points and the corner flux rows (R32)."""
    c = _tiny_cfg(P, layout=layout, q=7)
    W, b, _, _ = O.init_hidden(c)
    K, B, A, F = _global_blocks(c, W, b)
    assert np.linalg.cond(K) < 1e8
    Kp = np.linalg.pinv(K)
    I = np.eye(K.shape[0])
    Op = I + Kp.T @ A.T @ A @ Kp - K @ Kp
    M_lit = B.T @ Op @ B
    g_lit = B.T @ Op @ F
    r = O.solve(c, W, b, want_system=True)
    assert np.abs(r["M"] - M_lit).max() <= 1e-10 * np.abs(M_lit).max()
    assert np.abs(r["g"] - g_lit).max() <= 1e-10 * np.abs(g_lit).max()
    assert np.array_equal(r["M"], r["M"].T) or np.abs(r["M"] - r["M"].T).max() < 1e-14 * np.abs(r["M"]).max()
    assert np.linalg.eigvalsh(r["M"]).min() > 0      # SPD


@pytest.mark.parametrize("P,lam,layout", [(2, 0.0, 0), (3, 0.0, 0), (2, 0.05, 0), (3, 0.3, 0), (2, 0.0, 1),
                                          (3, 0.0, 1), (3, 0.3, 1)])
def test_schur_solution_equals_monolithic_lstsq_of_eliminated_system(P, lam, layout):
    """Central equivalence: (c, u_Gamma) of the Schur route == the least-squares solution of the
    monolithic eqn:eliminated system [[K, B], [0, -AK^+B]] [c; u] = [F; -AK^+F].
    With Tikhonov damping (reading R29) K is the stacked [K; lam I] of every subdomain, B and F
    zero on the damping rows: the same identity then pins the damped route."""
    c = _tiny_cfg(P, tikhonov=lam, layout=layout, q=7 if layout else 6)
    W, b, _, _ = O.init_hidden(c)
    K, B, A, F = _global_blocks(c, W, b)
    Kp = np.linalg.pinv(K)
    top = np.hstack([K, B])
    bot = np.hstack([np.zeros((A.shape[0], K.shape[1])), -A @ Kp @ B])
    sol = np.linalg.lstsq(np.vstack([top, bot]), np.concatenate([F, -A @ Kp @ F]), rcond=None)[0]
    n = K.shape[1]
    r = O.solve(c, W, b)
    assert np.allclose(r["uG"], sol[n:], rtol=0, atol=1e-8 * np.abs(sol[n:]).max())
    assert np.allclose(r["coef"].ravel(), sol[:n], rtol=0, atol=1e-8 * np.abs(sol[:n]).max())
    # ... and it is NOT the LS solution of the uneliminated eqn:nonoverlap_discrete (reading R10)
    full = np.vstack([np.hstack([K, B]), np.hstack([A, np.zeros((A.shape[0], B.shape[1]))])])
    sol2 = np.linalg.lstsq(full, np.concatenate([F, np.zeros(A.shape[0])]), rcond=None)[0]
    assert np.abs(sol2[n:] - sol[n:]).max() > 1e-6 * np.abs(sol[n:]).max()


def test_single_subdomain_is_classical_elm():
    """P = 1: no interface (G = 0) and c = argmin ||K c - F||."""
    c = mkcfg(P=1, M=30, p=12, q=8, problem=4, seed=9, init_c=0.125)
    W, b, _, _ = O.init_hidden(c)
    K, F, _ = O.assemble(c, 0, W, b)
    assert O.geometry(c)["G"] == 0
    r = O.solve(c, W, b)
    ref = np.linalg.lstsq(K, F, rcond=None)[0]
    assert np.allclose(K @ r["coef"][0], K @ ref, rtol=0, atol=1e-10 * np.abs(F).max())
    assert abs(r["resid"][0] - np.linalg.norm(K @ ref - F)) < 1e-10 * np.linalg.norm(F)


def test_homogeneous_problem_gives_zero():
    c = mkcfg(P=3, M=20, p=6, q=5, problem=5)
    W, b, _, _ = O.init_hidden(c)
    r = O.solve(c, W, b, WL.eval_grid(11))
    assert np.all(r["uG"] == 0) and np.all(r["coef"] == 0) and np.all(r["u"] == 0)


# ------------------------------------------------------------------------------------------------
# properties of the solution at a BASELINE geometry
# ------------------------------------------------------------------------------------------------
def _u_local(W, b, coef, s, pts):
    w = W[s]
    return np.tanh(pts @ w.T + b[s]) @ coef[s]


@pytest.mark.parametrize("k", [0, 1])
def test_interface_continuity_bound(k):
    """|u_s(x_k) - u_Gamma,k| <= r_s (value row of the local residual), hence
    |u_s - u_t| <= r_s + r_t at every interface point."""
    c = mkcfg(k)
    W, b, _, _ = O.init_hidden(c)
    r = O.solve(c, W, b, want_system=True)
    N = O.geometry(c)["N"]
    vals = {}
    for s in range(N):
        xy, edge, gidx = O.rows(c, s)
        sel = gidx >= 0
        us = _u_local(W, b, r["coef"], s, xy[sel])
        dev = np.abs(us - r["uG"][gidx[sel]])
        assert np.all(dev <= r["resid"][s] * (1 + 1e-6) + 1e-13)
        for gi, v in zip(gidx[sel], us):
            vals.setdefault(int(gi), []).append((s, v))
    for gi, lst in vals.items():
        (s1, v1), (s2, v2) = lst
        assert abs(v1 - v2) <= (r["resid"][s1] + r["resid"][s2]) * (1 + 1e-6) + 1e-13
    # the interface system is solved to rounding (eqn:schur)
    M, g, u = r["M"], r["g"], r["uG"]
    assert np.linalg.norm(M @ u - g) <= 1e-12 * np.linalg.norm(g)


def test_error_falls_as_neurons_are_added():
    """Reading R21 ladder at config-0 geometry (P:75 observation, valid while M << m)."""
    errs = []
    xy = WL.eval_grid(41)
    ue = WL.exact(0, xy)
    for M in [8, 16, 32, 64, 128]:
        c = mkcfg(0, M=M)
        W, b, _, _ = O.init_hidden(c)
        r = O.solve(c, W, b, xy)
        errs.append(np.linalg.norm(r["u"] - ue) / np.linalg.norm(ue))
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6


def test_config1_accuracy_vs_exact():
    """Config 1 reaches rounding-level accuracy vs the exact solution (SURVEY scratch 2.5e-13);
    this fails if the flux term is formed as A (K^+ B) column by column (reading R23)."""
    c = mkcfg(1)
    W, b, _, _ = O.init_hidden(c)
    xy = WL.eval_grid()
    r = O.solve(c, W, b, xy)
    ue = WL.exact(0, xy)
    assert np.linalg.norm(r["u"] - ue) / np.linalg.norm(ue) < 1e-10


def test_init_study_direction_oracle():
    """PAPER.md Table 1: He initialisation (l = sqrt(2/n_N), b = 0) gives an
    interface RMSE orders of magnitude above the suggested eqn:init one (8.4e-3 vs
    2.9e-10 at 2x2).  Small 3x3 geometry; the oracle solves both."""
    rmse = {}
    for sch in (0, 2):
        c = O.cfg(3, 96, 12, 12, 0, sch, 0.125, 0.5, 11)
        W, b, _, _ = O.init_hidden(c)
        r = O.solve(c, W, b)
        pts = np.zeros((len(r["uG"]), 2))
        for s in range(9):
            xy, edge, gidx = O.rows(c, s)
            pts[gidx[gidx >= 0]] = xy[gidx >= 0]
        ue = np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
        rmse[sch] = float(np.sqrt(np.mean((r["uG"] - ue) ** 2)))
    assert rmse[0] < 1e-3 * rmse[2], rmse


# ------------------------------------------------------------------------------------------------
# variable coefficient (problem 6): eqn:varpoisson, rho = tanh(grf) + 1.1, eqn:grf
# (P:611-615); SURVEY §8(f) NEXT-4
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("alpha", [16.0, 32.0])
def test_varcoef_rho_range_and_gradient(alpha):
    """rho varies in [0.1, 2.1]; its analytic gradient matches central differences of
    rho itself (grad rho analytic, not differenced)."""
    O.set_grf(WL.grf_params(alpha, 11))
    rng = np.random.default_rng(3)
    vals = [O.rho(x, y)[0] for x, y in rng.uniform(0, 1, (2000, 2))]
    assert 0.1 <= min(vals) and max(vals) <= 2.1  # saturates: tanh(grf) = +-1 where |grf| is large
    assert min(vals) < 0.3 and max(vals) > 1.9  # the field really spans the range
    h = 1e-7
    for x, y in rng.uniform(0.1, 0.9, (20, 2)):
        r, rx, ry = O.rho(x, y)
        fx = (O.rho(x + h, y)[0] - O.rho(x - h, y)[0]) / (2 * h)
        fy = (O.rho(x, y + h)[0] - O.rho(x, y - h)[0]) / (2 * h)
        scale = max(1.0, abs(rx), abs(ry))
        assert abs(rx - fx) <= 1e-5 * scale and abs(ry - fy) <= 1e-5 * scale
    O.set_grf(None)


def test_varcoef_grf_statistics():
    """The draws of eqn:grf: a ~ N(0, alpha^4/256) for the paper's 256 terms (variance alpha^4 /
    nterms in general), w ~ N(0, alpha^2 I), b ~ U(0, 2 pi)."""
    assert WL.grf_params(16.0, 0).shape == (256, 4)
    n = 200000
    p = WL.grf_params(16.0, 0, nterms=n)
    assert abs(p[:, 0].std() - 16.0**2 / np.sqrt(n)) < 0.01 * 16.0**2 / np.sqrt(n)
    assert abs(p[:, 1].std() - 16.0) < 0.1 and abs(p[:, 2].std() - 16.0) < 0.1
    assert p[:, 3].min() >= 0 and p[:, 3].max() < 2 * np.pi and abs(p[:, 3].mean() - np.pi) < 0.02


def test_varcoef_interior_rows_are_minus_div_rho_grad_phi():
    """Interior rows of problem 6 = -div(rho grad phi), checked against central differences of
    the flux rho grad phi (np.tanh; rho from the oracle); value / flux rows and F = [1; 0; 0]."""
    grf = WL.grf_params(4.0, 5)
    O.set_grf(grf)
    c = O.cfg(2, 24, 5, 4, 6, 0, 0.125, 0.5, 5)
    W, b, _, _ = O.init_hidden(c)
    s = 1
    K, F, A = O.assemble(c, s, W, b)
    xy, edge, gidx = O.rows(c, s)
    w, bb = W[s], b[s]
    phi = lambda p: np.tanh(w[:, 0] * p[0] + w[:, 1] * p[1] + bb)
    h = 1e-4

    def flux(p, axis):
        e = np.array([h, 0.0]) if axis == 0 else np.array([0.0, h])
        dphi = (phi(p + e) - phi(p - e)) / (2 * h)
        return O.rho(p[0], p[1])[0] * dphi

    for r in range(len(edge)):
        p = xy[r]
        if edge[r] < 0:
            ex, ey = np.array([h, 0.0]), np.array([0.0, h])
            div = (flux(p + ex, 0) - flux(p - ex, 0)) / (2 * h) + (flux(p + ey, 1) - flux(p - ey, 1)) / (2 * h)
            assert np.allclose(K[r], -div, rtol=0, atol=2e-5 * max(1.0, np.abs(div).max()))
            assert F[r] == 1.0
        else:
            assert np.allclose(K[r], phi(p), rtol=0, atol=2e-15)
            assert F[r] == 0.0
    O.set_grf(None)


def test_varcoef_zero_field_is_scaled_poisson():
    """grf = 0 (all a_i = 0): rho = 1.1, grad rho = 0, so the interior rows are 1.1 x the
    constant-coefficient rows of -Lap (a special case that reduces to problem 0's operator)."""
    grf = WL.grf_params(8.0, 2)
    grf[:, 0] = 0.0
    O.set_grf(grf)
    c6 = O.cfg(2, 16, 5, 4, 6, 0, 0.125, 0.5, 9)
    c0 = O.cfg(2, 16, 5, 4, 0, 0, 0.125, 0.5, 9)
    W, b, _, _ = O.init_hidden(c6)
    K6, F6, A6 = O.assemble(c6, 2, W, b)
    K0, F0, A0 = O.assemble(c0, 2, W, b)
    _, edge, _ = O.rows(c6, 2)
    inn = edge < 0
    assert np.allclose(K6[inn], 1.1 * K0[inn], rtol=4e-16 * 4, atol=0)
    assert np.array_equal(K6[~inn], K0[~inn]) and np.array_equal(A6, A0)
    O.set_grf(None)


# ------------------------------------------------------------------------------------------------
# Kirchhoff plate (problem 7): Lap^2 u = q/D, u = Lap u = 0 on the boundary, two traces
# and two fluxes per interface point (reading R28); SURVEY §8(f) NEXT-4
# ------------------------------------------------------------------------------------------------
PLATE_D = 1e7 * 1e-9 / (12.0 * (1.0 - 0.3 * 0.3))


def test_plate_rhs_and_exact_solution():
    """f = q/D with q = sin(pi x) sin(pi y), and u = q / (4 pi^4 D) satisfies Lap^2 u = f (FD of
    the oracle's own u)."""
    assert abs(PLATE_D - 1e-2 / 10.92) < 1e-15
    x, y, h = 0.31, 0.62, 2e-3
    u = lambda a, b: O.problem(7, a, b)[0]
    lap = lambda a, b: (u(a + h, b) + u(a - h, b) + u(a, b + h) + u(a, b - h) - 4 * u(a, b)) / h**2
    bih = (lap(x + h, y) + lap(x - h, y) + lap(x, y + h) + lap(x, y - h) - 4 * lap(x, y)) / h**2
    f = O.problem(7, x, y)[1]
    assert abs(f - math.sin(math.pi * x) * math.sin(math.pi * y) / PLATE_D) < 1e-12 * abs(f)
    assert abs(bih - f) < 1e-3 * abs(f)
    assert abs(u(x, y) - math.sin(math.pi * x) * math.sin(math.pi * y) / (4 * math.pi**4 * PLATE_D)) < 1e-12


def test_plate_rows_vs_finite_differences():
    """Interior rows Lap^2 phi, u-trace rows phi, Lap-trace rows Lap phi, flux rows d phi/dn and
    d Lap phi / dn, against central differences of np.tanh; the edge block layout [u traces |
    Lap u traces] with both traces at the same points."""
    c = O.cfg(2, 12, 5, 8, 7, 0, 1.0 / 16, 0.5, 4)
    W, b, _, _ = O.init_hidden(c)
    s = 0
    K, F, A = O.assemble(c, s, W, b)
    xy, edge, gidx = O.rows(c, s)
    w, bb = W[s], b[s]
    phi = lambda p: np.tanh(w[:, 0] * p[0] + w[:, 1] * p[1] + bb)
    h = 1e-3

    def lap(fn, p):
        return (fn(p + [h, 0]) + fn(p - [h, 0]) + fn(p + [0, h]) + fn(p - [0, h]) - 4 * fn(p)) / h**2

    q, npts, pp = 8, 4, 25
    normals = {0: (-1, 0), 1: (1, 0), 2: (0, -1), 3: (0, 1)}
    for r in range(len(edge)):
        p = xy[r]
        if edge[r] < 0:
            bih = lap(lambda z: lap(phi, z), p)
            assert np.allclose(K[r], bih, rtol=0, atol=2e-3 * max(1.0, np.abs(bih).max()))
            continue
        e, k = edge[r], (r - pp) % q
        assert (r - pp) // q == e
        twin = pp + e * q + (k + npts) % q          # the other trace at the same point
        assert np.array_equal(xy[twin], p)
        n = np.array(normals[e], float)
        if k < npts:
            assert np.allclose(K[r], phi(p), rtol=0, atol=2e-15)
            d = (phi(p + h * n) - phi(p - h * n)) / (2 * h)
        else:
            lp = lap(phi, p)
            assert np.allclose(K[r], lp, rtol=0, atol=1e-5 * max(1.0, np.abs(lp).max()))
            d = (lap(phi, p + h * n) - lap(phi, p - h * n)) / (2 * h)
        if gidx[r] >= 0:
            assert np.allclose(A[r - pp], d, rtol=0, atol=1e-4 * max(1.0, np.abs(d).max()))
            assert F[r] == 0.0
        else:
            assert np.all(A[r - pp] == 0.0)


def test_plate_solution_accuracy():
    """The DDM solution of the plate problem (c = 1/16 of P:545) on 2 x 2 subdomains
    converges to the exact u: relative L2 error < 1e-9 (the paper's Table tab:platebending: 1e-8
    at 2 x 2 with n = 2^16; the SPEC acceptance bound is 1e-4)."""
    c = O.cfg(2, 256, 18, 24, 7, 0, 1.0 / 16, 0.5, 3)
    W, b, _, _ = O.init_hidden(c)
    xy = WL.eval_grid(41)
    r = O.solve(c, W, b, xy)
    ex = WL.exact(7, xy)
    assert np.linalg.norm(r["u"] - ex) / np.linalg.norm(ex) < 1e-9


# ------------------------------------------------------------------------------------------------
# Tikhonov damping of the local LS (reading R29)
# ------------------------------------------------------------------------------------------------
def test_tikhonov_rows_pinned():
    """lambda > 0 appends exactly lambda I (and zero right-hand side, no interface unknown, no
    flux) below the unchanged collocation rows."""
    lam = 0.37
    c0 = mkcfg(P=2, M=16, p=6, q=4, problem=2, seed=3)
    c1 = mkcfg(P=2, M=16, p=6, q=4, problem=2, seed=3, tikhonov=lam)
    W, b, _, _ = O.init_hidden(c0)
    m0 = 6 * 6 + 4 * 4
    assert O.geometry(c1)["m"] == m0 + 16 and O.geometry(c0)["m"] == m0
    for s in range(4):
        K0, F0, A0 = O.assemble(c0, s, W, b)
        K1, F1, A1 = O.assemble(c1, s, W, b)
        assert np.array_equal(K1[:m0], K0) and np.array_equal(F1[:m0], F0) and np.array_equal(A1, A0)
        assert np.array_equal(K1[m0:], lam * np.eye(16)) and not F1[m0:].any()
        _, edge, gidx = O.rows(c1, s)
        assert (edge[m0:] == -2).all() and (gidx[m0:] == -1).all()


def test_tikhonov_single_subdomain_closed_form():
    """P = 1: c = (K^T K + lambda^2 I)^{-1} K^T F (ridge regression), r = sqrt(||Kc - F||^2 +
    lambda^2 ||c||^2): closed forms from the normal equations, independent of the QR route."""
    c0 = mkcfg(P=1, M=30, p=12, q=8, problem=4, seed=9, init_c=0.125)
    W, b, _, _ = O.init_hidden(c0)
    K, F, _ = O.assemble(c0, 0, W, b)
    lam = 1e-3 * np.linalg.norm(K, 2)
    c1 = mkcfg(P=1, M=30, p=12, q=8, problem=4, seed=9, init_c=0.125, tikhonov=lam)
    r = O.solve(c1, W, b)
    ref = np.linalg.solve(K.T @ K + lam * lam * np.eye(30), K.T @ F)
    assert np.allclose(r["coef"][0], ref, rtol=0, atol=1e-9 * np.abs(ref).max())
    rr = np.sqrt(np.linalg.norm(K @ ref - F) ** 2 + lam * lam * np.linalg.norm(ref) ** 2)
    assert abs(r["resid"][0] - rr) <= 1e-9 * rr


# ------------------------------------------------------------------------------------------------
# the paper's shared lattice with cross points (readings R32, R33)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("P,n", [(2, 4), (3, 5), (4, 3)])
def test_lattice_geometry(P, n):
    """Layout 1: the rows of all subdomains are exactly the (P n + 1)^2 points of the global
    lattice ("distributed to each subdomain"), (n+1)^2 per subdomain; face points are shared
    by 2 subdomains and cross points (interior subdomain corners) by 4, each one interface unknown
    (G = 2P(P-1)(n-1) + (P-1)^2); every flux equation (one per face point, and per cross point one
    per incident face: the corner remark) has exactly two contributors whose normals
    are opposite (continuity of the flux)."""
    c = mkcfg(P=P, M=8, p=n - 1, q=n - 1, problem=0, seed=1, layout=1)
    geo = O.geometry(c)
    q = n - 1
    assert geo["m"] == (n + 1) ** 2
    assert geo["G"] == 2 * P * (P - 1) * q + (P - 1) ** 2
    assert geo["NE"] == 2 * P * (P - 1) * q + 4 * (P - 1) ** 2
    pts = {}
    owners = {}
    for s in range(P * P):
        xy, edge, gidx = O.rows(c, s)
        for (x, y), g in zip(xy, gidx):
            key = (round(x * P * n), round(y * P * n))
            assert abs(x * P * n - key[0]) < 1e-9 and abs(y * P * n - key[1]) < 1e-9
            pts.setdefault(key, set()).add(g)
            if g >= 0:
                owners.setdefault(g, []).append(s)
    assert set(pts) == {(a, b) for a in range(P * n + 1) for b in range(P * n + 1)}
    assert all(len(v) == 1 for v in pts.values())          # one unknown per shared point
    cnt = [len(owners[g]) for g in sorted(owners)]
    assert sorted(owners) == list(range(geo["G"]))
    assert cnt == [2] * (geo["G"] - (P - 1) ** 2) + [4] * (P - 1) ** 2
    W, b, _, _ = O.init_hidden(c)
    contrib = {}
    for s in range(P * P):
        _, _, A = O.assemble(c, s, W, b)
        for ar, eq in enumerate(O.flux_eq(c, s)):
            if eq >= 0:
                contrib.setdefault(int(eq), []).append(A[ar])
    assert sorted(contrib) == list(range(geo["NE"]))
    assert all(len(rows) == 2 for rows in contrib.values())  # (opposite normals: next test)


def test_lattice_corner_flux_rows():
    """Corner remark: a cross point gets one flux row per edge through the corner,
    with that edge's outward normal; each row equals the central difference of np.tanh(w.x + b)
    along the normal.  Corners on the boundary are Dirichlet value rows (g = u_exact) with no flux
    rows.  The two rows of every cross-point equation use opposite normals."""
    P, n = 3, 4
    c = mkcfg(P=P, M=6, p=n - 1, q=n - 1, problem=0, seed=3, layout=1)
    W, b, _, _ = O.init_hidden(c)
    q, pp = n - 1, (n - 1) ** 2
    normals = {}
    for s in range(P * P):
        i, j = s % P, s // P
        K, F, A = O.assemble(c, s, W, b)
        xy, edge, gidx = O.rows(c, s)
        eqs = O.flux_eq(c, s)
        for cc in range(4):
            r = pp + 4 * q + cc
            ci, cj = cc & 1, cc >> 1
            x, y = xy[r]
            assert (x, y) == ((i + ci) / P, (j + cj) / P)
            phi = lambda xx, yy: np.tanh(W[s][:, 0] * xx + W[s][:, 1] * yy + b[s])  # noqa: E731
            assert np.allclose(K[r], phi(x, y), rtol=0, atol=1e-15)
            interior = 0 < i + ci < P and 0 < j + cj < P
            assert (gidx[r] >= 0) == interior
            for d in range(2):
                ar = 4 * q + 2 * cc + d
                nrm = ((1.0 if ci else -1.0), 0.0) if d == 0 else (0.0, (1.0 if cj else -1.0))
                if not interior:
                    assert eqs[ar] == -1 and np.all(A[ar] == 0.0)
                    continue
                h = 1e-6
                fd = (phi(x + h * nrm[0], y + h * nrm[1]) - phi(x - h * nrm[0], y - h * nrm[1])) / (2 * h)
                assert np.allclose(A[ar], fd, rtol=1e-6, atol=1e-8)
                normals.setdefault(int(eqs[ar]), []).append(nrm)
            if not interior:
                u, _ = O.problem(0, x, y)
                assert F[r] == u
    assert len(normals) == 4 * (P - 1) ** 2
    for nr in normals.values():
        assert len(nr) == 2 and nr[0][0] == -nr[1][0] and nr[0][1] == -nr[1][1]


def test_lattice_single_subdomain_is_classical_elm():
    """P = 1 on the lattice: all (n+1)^2 points, corners included, are collocation rows; no
    interface, and c = argmin ||K c - F|| (the paper's N = 1 x 1 row of Table 2)."""
    c = mkcfg(P=1, M=30, p=9, q=9, problem=4, seed=9, init_c=0.125, layout=1)
    W, b, _, _ = O.init_hidden(c)
    K, F, _ = O.assemble(c, 0, W, b)
    assert K.shape[0] == 11 * 11 and O.geometry(c)["G"] == 0
    r = O.solve(c, W, b)
    ref = np.linalg.lstsq(K, F, rcond=None)[0]
    assert np.allclose(K @ r["coef"][0], K @ ref, rtol=0, atol=1e-9 * np.abs(F).max())


def test_damping_rule_eps_frobenius():
    """Reading R33: tikhonov < 0 selects lambda_s = eps max(m, M) ||K^s||_F (the collocation rows) in
    every subdomain -- the Tikhonov analogue of the numerical-rank cut rcond = eps max(m, n) that
    PyTorch's least squares (the paper's tool) applies by default."""
    c = mkcfg(P=2, M=20, p=5, q=5, problem=4, seed=2, layout=1, tikhonov=-1.0)
    W, b, _, _ = O.init_hidden(c)
    m = (5 + 1 + 1) ** 2
    for s in range(4):
        K, F, _ = O.assemble(c, s, W, b)
        assert K.shape[0] == m + 20
        lam = np.sqrt(np.sum(K[:m] ** 2)) * np.finfo(float).eps * max(m, 20)
        assert np.allclose(np.diag(K[m:]), lam, rtol=1e-14, atol=0)
        assert np.all(K[m:] - np.diag(np.diag(K[m:])) == 0.0) and np.all(F[m:] == 0.0)
