"""Study (CPU, numpy): the paper's Table 2 workloads (workloads.py configs 5, 6) with K^{s+} realised
by a truncated pseudo-inverse (numpy pinv, relative cutoff rtol) instead of the unpivoted QR of
reading R11 -- literal eqn:schur, dense interface solve, error vs the exact solution on a grid.
A negative rtol selects Tikhonov damping instead: K^+ = (K^T K + lam^2 I)^{-1} K^T with
lam = |rtol| sigma_max(K^s) (what a QR of [K^s; lam I] realises).
usage: python tools/pinv_study.py [config] [rtol ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import workloads as WL  # noqa: E402
from helpers import ocfg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rtols = [float(x) for x in sys.argv[2:]] or [1e-15, 1e-13, 1e-11, 1e-9]
c = WL.config(k)
oc = ocfg(c)
W, b, _, _ = O.init_hidden(oc)
geo = O.geometry(oc)
G, N, P, q, p = geo["G"], geo["N"], c["P"], c["q"], c["p"]
pp = p * p
xy = WL.eval_grid(51)
ue = WL.exact(c["problem"], xy)
loc = []
for s in range(N):
    K, F, A = O.assemble(oc, s, W, b)
    _, _, gidx = O.rows(oc, s)
    loc.append((K, F, A, gidx))
sv = np.linalg.svd(loc[N // 2][0], compute_uv=False)
print(f"{c['name']}: P={P} M={c['M']} m={pp + 4 * q} G={G}; interior subdomain sigma_max {sv[0]:.3e}, "
      f"sigma_min/sigma_max {sv[-1] / sv[0]:.2e}, #sigma > 1e-12 sigma_max: {(sv > 1e-12 * sv[0]).sum()}")
for rtol in rtols:
    Mg = np.zeros((G, G))
    g = np.zeros(G)
    Q = np.zeros((G, G))
    qv = np.zeros(G)
    Kps = []
    for s, (K, F, A, gidx) in enumerate(loc):
        if rtol > 0:
            Kp = np.linalg.pinv(K, rtol=rtol)
        else:
            lam = -rtol * np.linalg.norm(K, 2)
            Ka = np.vstack([K, lam * np.eye(K.shape[1])])
            Qa, Ra = np.linalg.qr(Ka)
            Kp = np.linalg.solve(Ra, Qa[: K.shape[0]].T)
        Kps.append(Kp)
        vr = np.nonzero(gidx >= 0)[0]           # interface value rows of s
        gi = gidx[vr]
        Pm = np.eye(K.shape[0]) - K @ Kp        # I - K K^+
        E = np.zeros((K.shape[0], len(vr)))
        E[vr, np.arange(len(vr))] = 1.0
        PE = Pm @ E
        Mg[np.ix_(gi, gi)] += E.T @ PE          # B^T (I - K K^+) B  (B = -E)
        g[gi] -= E.T @ (Pm @ F)                 # -B^T(I-KK^+)F sign: F - B u = F + E u
        Wf = A @ Kp                             # flux of c = K^+ (F + E u)
        fr = np.arange(A.shape[0])
        fg = gidx[pp + fr]                      # flux row e*q+k <-> the value row of the same point
        ok = fg >= 0
        Q[np.ix_(fg[ok], gi)] += (Wf @ E)[ok]
        qv[fg[ok]] += (Wf @ F)[ok]
    Mg += Q.T @ Q
    g -= Q.T @ qv
    u = np.linalg.solve(Mg, g)
    coef = np.zeros((N, c["M"]))
    for s, (K, F, A, gidx) in enumerate(loc):
        rhs = F.copy()
        rhs[gidx >= 0] += u[gidx[gidx >= 0]]
        coef[s] = Kps[s] @ rhs
    uh = O.evaluate(oc, W, b, coef, xy)
    err = np.linalg.norm(uh - ue) / np.linalg.norm(ue)
    print(f"  {'rtol' if rtol > 0 else 'tikhonov lam/sigma_max'} {abs(rtol):.0e}: rel L2 error vs exact {err:.3e}   (paper Table 2: {WL.PAPER_TABLE2[k][0]:.2e})")
