"""Accuracy-gap study (reading R24): where does the CUDA path's
larger error vs the exact solution come from -- the assembly (separable exponentials) or the
factorisation / elimination / interface path?

Cells (relative L2 error of u on the 101^2 grid vs the exact solution, and vs the oracle's u):
  oracle  K + oracle pipeline            (oracle.solve)
  CUDA    K + CUDA pipeline              (the product path)
  oracle  K + CUDA pipeline              (oracle-assembled K_aug / A^T uploaded in place of
                                          elmddm_assemble's output, then the CUDA path as usual)
  CUDA    K + LAPACK pipeline            (numpy: Householder QR = LAPACK dgeqrf, the same
  oracle  K + LAPACK pipeline             elimination as the oracle, dense solve)
This is a study tool: its numbers go to DESIGN.md, never into a test's expected values.
usage (GPU box): python tools/accuracy_study.py [k ...]   (default 2)
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import scipy.linalg as sla  # noqa: E402

import oracle as O  # noqa: E402
import workloads as WL  # noqa: E402
from helpers import gpu_ctx, ocfg  # noqa: E402


def lapack_pipeline(c, Ks, Fs, As, irows, igs, W, b, xy):
    """The oracle's route with LAPACK's QR and numpy: K^+ by Householder QR, the
    flux operator A R^{-1} formed once (reading R23), M u = g dense."""
    N = len(Ks)
    G = 2 * c["P"] * (c["P"] - 1) * c["q"]
    Mm = np.zeros((G, G))
    g = np.zeros(G)
    Qg = np.zeros((G, G))
    qg = np.zeros(G)
    facs = []
    for s in range(N):
        K, F, A, ir, ig = Ks[s], Fs[s], As[s], irows[s], igs[s]
        Q1, R = np.linalg.qr(K, mode="reduced")
        T = Q1[ir, :]
        yF = Q1.T @ F
        S1 = np.eye(len(ir)) - T @ T.T
        g1 = T @ yF - F[ir]
        Wr = sla.solve_triangular(R, A.T, trans="T").T
        PB = -Wr @ T.T
        pF = Wr @ yF
        Mm[np.ix_(ig, ig)] += S1
        g[ig] += g1
        Qg[np.ix_(ig, ig)] += PB
        qg[ig] += pF
        facs.append((Q1, R))
    Mm += Qg.T @ Qg
    g += Qg.T @ qg
    uG = np.linalg.solve(Mm, g)
    coef = np.zeros((N, c["M"]))
    for s in range(N):
        Q1, R = facs[s]
        rhs = Fs[s].copy()
        rhs[irows[s]] += uG[igs[s]]
        coef[s] = sla.solve_triangular(R, Q1.T @ rhs)
    P = c["P"]
    own = np.minimum((xy * P).astype(int), P - 1)
    owner = own[:, 1] * P + own[:, 0]
    u = np.einsum("pj,pj->p", coef[owner], np.tanh(np.einsum("pjd,pd->pj", W[owner], xy) + b[owner]))
    return u


def study(k):
    import torch

    c = WL.config(k)
    M, q = c["M"], c["q"]
    oc = ocfg(c)
    xy = WL.eval_grid()
    ue = WL.exact(c["problem"], xy)
    err = lambda u: float(np.linalg.norm(u - ue) / np.linalg.norm(ue))  # noqa: E731
    W, b, _, _ = O.init_hidden(oc)
    orc = O.solve(oc, W, b, xy, nthreads=len(os.sched_getaffinity(0)))
    vs = lambda u: float(np.linalg.norm(u - orc["u"]) / np.linalg.norm(orc["u"]))  # noqa: E731
    N = c["P"] ** 2
    # oracle assembly, per subdomain, plus the GPU layouts
    ctx, buf = gpu_ctx(c)
    z = ctx.sizes
    ld, ncols = z["ld"], z["ncols"]
    Ko, Fo, Ao, irows, igs = [], [], [], [], []
    for s in range(N):
        K, F, A = O.assemble(oc, s, W, b)
        _, _, gidx = O.rows(oc, s)
        m = len(gidx)
        ir = np.where(gidx >= 0)[0]
        Ko.append(K)
        Fo.append(F)
        Ao.append(A[ir - (m - 4 * q)])
        irows.append(ir)
        igs.append(gidx[ir])
    xy_t = torch.as_tensor(xy.reshape(-1), device="cuda")
    u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
    # (1) the product path
    ctx.run(buf, xy_t, u)
    torch.cuda.synchronize()
    u_gpu = u.cpu().numpy().copy()
    # (2) CUDA K for the LAPACK pipeline
    ctx.init_hidden(buf["W"], buf["b"])
    ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
    torch.cuda.synchronize()
    Kg_all = buf["Kaug"].view(z["S"], ncols, ld).cpu().numpy()
    At_all = buf["At"].view(-1, 4 * q, M).cpu().numpy()
    Kg, Fg, Ag = [], [], []
    for s in range(N):
        m = len(Fo[s])
        Kg.append(Kg_all[s, :M, :m].T.copy())
        Fg.append(Kg_all[s, M + 4 * q, :m].copy())
        Ag.append(At_all[s][irows[s] - (m - 4 * q)])
    dK = max(float(np.abs(Kg[s] - Ko[s]).max() / np.abs(Ko[s]).max()) for s in range(N))
    # (3) oracle K_aug / A^T uploaded, then the CUDA path from local_factor on
    Kaug = np.zeros((N, ncols, ld))
    At = np.zeros((N, 4 * q, M))
    for s in range(N):
        m = len(Fo[s])
        Kaug[s, :M, :m] = Ko[s].T
        for t, r in enumerate(irows[s]):
            Kaug[s, M + (r - (m - 4 * q)), r] = 1.0
        Kaug[s, M + 4 * q, :m] = Fo[s]
        _, _, A4 = O.assemble(oc, s, W, b)
        At[s] = A4
    buf["Kaug"].copy_(torch.as_tensor(Kaug.reshape(-1)))
    buf["At"].copy_(torch.as_tensor(At.reshape(-1)))
    ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
    ctx.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"])
    ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
    ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
    ctx.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"])
    u.zero_()
    ctx.evaluate(buf["W"], buf["b"], buf["coef"], xy_t, u)
    ctx.sync()
    u_gpu_on_orcK = u.cpu().numpy().copy()
    out = {"config": k, "max_rel_dK_gpu_vs_oracle": dK,
           "oracle_K+oracle": {"vs_exact": err(orc["u"])},
           "cuda_K+cuda": {"vs_exact": err(u_gpu), "vs_oracle": vs(u_gpu)},
           "oracle_K+cuda": {"vs_exact": err(u_gpu_on_orcK), "vs_oracle": vs(u_gpu_on_orcK)}}
    if k <= 2:
        u_l_g = lapack_pipeline(c, Kg, Fg, Ag, irows, igs, W, b, xy)
        u_l_o = lapack_pipeline(c, Ko, Fo, Ao, irows, igs, W, b, xy)
        out["cuda_K+lapack"] = {"vs_exact": err(u_l_g), "vs_oracle": vs(u_l_g)}
        out["oracle_K+lapack"] = {"vs_exact": err(u_l_o), "vs_oracle": vs(u_l_o)}
    return out


def eval_separable(c, W, b, coef, xy):
    """u on the points with the SAME floating-point form of sigma as the assembly kernel
    (separable exponentials about the owner subdomain's centre) instead of tanh."""
    P = c["P"]
    own = np.minimum((xy * P).astype(int), P - 1)
    owner = own[:, 1] * P + own[:, 0]
    cx = (2 * own[:, 0] + 1) / (2.0 * P)
    cy = (2 * own[:, 1] + 1) / (2.0 * P)
    wx, wy = W[owner, :, 0], W[owner, :, 1]
    bt = b[owner] + wx * cx[:, None] + wy * cy[:, None]
    Ex = np.exp(2.0 * (wx * (xy[:, :1] - cx[:, None]) + bt))
    Ey = np.exp(2.0 * wy * (xy[:, 1:] - cy[:, None]))
    phi = 1.0 - 2.0 / (1.0 + Ex * Ey)
    return np.einsum("pj,pj->p", coef[owner], phi)


def evalform(k):
    """The product path's coefficients evaluated with tanh (k_evaluate) and with the separable form."""
    import torch

    c = WL.config(k)
    oc = ocfg(c)
    xy = WL.eval_grid()
    ue = WL.exact(c["problem"], xy)
    err = lambda u: float(np.linalg.norm(u - ue) / np.linalg.norm(ue))  # noqa: E731
    W, b, _, _ = O.init_hidden(oc)
    ctx, buf = gpu_ctx(c)
    xy_t = torch.as_tensor(xy.reshape(-1), device="cuda")
    u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
    ctx.run(buf, xy_t, u)
    coef = buf["coef"].view(-1, c["M"]).cpu().numpy()
    return {"config": k, "tanh (k_evaluate)": err(u.cpu().numpy()),
            "separable form (numpy)": err(eval_separable(c, W, b, coef, xy)),
            "coef_norm_max": float(np.abs(coef).max())}


def rowswap(k):
    """Which rows of the CUDA-assembled K^s carry the gap (config k): interior (Laplacian) vs edge
    (value) rows swapped between the CUDA and the oracle assembly, and numpy assemblies with
    sigma' = 1 - sigma^2 (the oracle's form) or sigma' = sech^2 z (no cancellation), all through
    the CUDA pipeline."""
    import torch

    c = WL.config(k)
    M, q, p = c["M"], c["q"], c["p"]
    pp = p * p
    oc = ocfg(c)
    xy = WL.eval_grid()
    ue = WL.exact(c["problem"], xy)
    err = lambda u: float(np.linalg.norm(u - ue) / np.linalg.norm(ue))  # noqa: E731
    W, b, _, _ = O.init_hidden(oc)
    N = c["P"] ** 2
    xy_t = torch.as_tensor(xy.reshape(-1), device="cuda")

    def fresh():
        ctx, buf = gpu_ctx(c)
        ctx.init_hidden(buf["W"], buf["b"])
        ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
        torch.cuda.synchronize()
        return ctx, buf

    def finish(ctx, buf):
        ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
        ctx.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"])
        ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
        ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
        ctx.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"])
        u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
        ctx.evaluate(buf["W"], buf["b"], buf["coef"], xy_t, u)
        ctx.sync()
        return err(u.cpu().numpy())

    ctx, buf = fresh()
    z = ctx.sizes
    ld, ncols = z["ld"], z["ncols"]
    Kg = buf["Kaug"].view(N, ncols, ld).clone()
    Ko = torch.zeros_like(Kg)
    Kn1 = torch.zeros_like(Kg)
    Kn2 = torch.zeros_like(Kg)
    for s in range(N):
        K, F, _ = O.assemble(oc, s, W, b)
        xs, edge, _ = O.rows(oc, s)
        m = K.shape[0]
        Ko[s, :M, :m] = torch.as_tensor(K.T)
        zz = xs @ W[s].T + b[s][None, :]                       # direct z = w . x + b
        sg = np.tanh(zz)
        w2 = (W[s] ** 2).sum(1)[None, :]
        for Kn, s1 in ((Kn1, 1.0 - sg * sg), (Kn2, 1.0 / np.cosh(zz) ** 2)):
            Kk = np.where(edge[:, None] < 0, -w2 * (-2.0 * sg * s1), sg)   # -|w|^2 sigma''
            Kn[s, :M, :m] = torch.as_tensor(Kk.T)
    out = {"config": k, "cuda": finish(ctx, buf)}
    for name, rows_from_gpu in (("interior rows cuda, edge rows oracle", "int"),
                                ("interior rows oracle, edge rows cuda", "edge")):
        ctx, buf = fresh()
        Kv = buf["Kaug"].view(N, ncols, ld)
        if rows_from_gpu == "int":
            Kv[:, :M, pp:] = Ko[:, :M, pp:]
        else:
            Kv[:, :M, :pp] = Ko[:, :M, :pp]
        out[name] = finish(ctx, buf)
    for name, Kn in (("numpy direct z, sigma' = 1 - sigma^2", Kn1), ("numpy direct z, sigma' = sech^2", Kn2)):
        ctx, buf = fresh()
        buf["Kaug"].view(N, ncols, ld)[:, :M, :] = Kn[:, :M, :]
        out[name] = finish(ctx, buf)
    return out


def swaps(k):
    """Component swaps inside the CUDA pipeline (config k): which input or phase carries the gap."""
    import torch

    from helpers import band_to_dense

    c = WL.config(k)
    M, q = c["M"], c["q"]
    oc = ocfg(c)
    xy = WL.eval_grid()
    ue = WL.exact(c["problem"], xy)
    err = lambda u: float(np.linalg.norm(u - ue) / np.linalg.norm(ue))  # noqa: E731
    W, b, _, _ = O.init_hidden(oc)
    N = c["P"] ** 2
    out = {"config": k}
    xy_t = torch.as_tensor(xy.reshape(-1), device="cuda")

    def pipeline(ctx, buf, host_iface=False, refine=0):
        ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
        ctx.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"])
        ctx.interface_assemble(buf["Pbuf"], buf["Sbuf"], buf["Mband"], buf["g"], buf["work"])
        G = ctx.sizes["G"]
        if refine:
            # iterative refinement of the interface solve, emulated by refactoring a copy of M:
            # u <- u + M^{-1} (g - M u), the residual with the assembled (unfactored) M
            from test_gpu_parity import _band_matvec

            M0 = buf["Mband"].clone()
            g0 = buf["g"].clone()
            ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
            for _ in range(refine):
                r = g0.clone()
                r[:G] -= _band_matvec(ctx, M0, buf["uG"][:G])
                Mr = M0.clone()
                d = torch.zeros_like(buf["uG"])
                ctx.interface_factor_solve(Mr, r, d, buf["work"])
                buf["uG"] += d
        elif host_iface:
            Md = band_to_dense(ctx, buf["Mband"])
            gd = buf["g"][:G].cpu().numpy()
            buf["uG"][:G] = torch.as_tensor(np.linalg.solve(Md, gd), device="cuda")
        else:
            ctx.interface_factor_solve(buf["Mband"], buf["g"], buf["uG"], buf["work"])
        ctx.back_solve(buf["Kaug"], buf["uG"], buf["coef"], buf["resid"], buf["work"])
        u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
        ctx.evaluate(buf["W"], buf["b"], buf["coef"], xy_t, u)
        ctx.sync()
        return err(u.cpu().numpy())

    def fresh(**over):
        ctx, buf = gpu_ctx(dict(c, **over))
        ctx.init_hidden(buf["W"], buf["b"])
        ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
        torch.cuda.synchronize()
        return ctx, buf

    ctx, buf = fresh()
    z = ctx.sizes
    Kg = buf["Kaug"].clone()
    Ag = buf["At"].clone()
    ld, ncols = z["ld"], z["ncols"]
    Ko = np.zeros((N, ncols, ld))
    Ao = np.zeros((N, 4 * q, M))
    for s in range(N):
        K, F, A4 = O.assemble(oc, s, W, b)
        _, _, gidx = O.rows(oc, s)
        m = len(gidx)
        Ko[s, :M, :m] = K.T
        for r in np.where(gidx >= 0)[0]:
            Ko[s, M + (r - (m - 4 * q)), r] = 1.0
        Ko[s, M + 4 * q, :m] = F
        Ao[s] = A4
    Ko_t = torch.as_tensor(Ko.reshape(-1), device="cuda")
    Ao_t = torch.as_tensor(Ao.reshape(-1), device="cuda")
    out["gpuK+gpuA"] = pipeline(ctx, buf)
    ctx, buf = fresh()
    out["gpu + 1 interface refinement step"] = pipeline(ctx, buf, refine=1)
    ctx, buf = fresh()
    out["gpu + 2 interface refinement steps"] = pipeline(ctx, buf, refine=2)
    ctx, buf = fresh(); buf["Kaug"].copy_(Kg); buf["At"].copy_(Ao_t)
    out["gpuK+orcA"] = pipeline(ctx, buf)
    ctx, buf = fresh(); buf["Kaug"].copy_(Ko_t); buf["At"].copy_(Ag)
    out["orcK+gpuA"] = pipeline(ctx, buf)
    ctx, buf = fresh(); buf["Kaug"].copy_(Ko_t); buf["At"].copy_(Ao_t)
    out["orcK+orcA"] = pipeline(ctx, buf)
    # K part from the GPU, E and F columns from the oracle
    Kmix = Kg.view(N, ncols, ld).clone()
    Kmix[:, M:, :] = Ko_t.view(N, ncols, ld)[:, M:, :]
    ctx, buf = fresh(); buf["Kaug"].copy_(Kmix.reshape(-1)); buf["At"].copy_(Ag)
    out["gpuKpart+orcEF+gpuA"] = pipeline(ctx, buf)
    if ctx.sizes["G"] <= 8000:
        ctx, buf = fresh()
        out["gpu, host dense interface solve"] = pipeline(ctx, buf, host_iface=True)
        ctx, buf = fresh(); buf["Kaug"].copy_(Ko_t); buf["At"].copy_(Ao_t)
        out["orcK+orcA, host dense interface solve"] = pipeline(ctx, buf, host_iface=True)
    for mode in (2, 3):
        ctx, buf = fresh(interface_mode=mode)
        out[f"gpu, interface_mode {mode}"] = pipeline(ctx, buf)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "rowswap":
        print(json.dumps([rowswap(int(a)) for a in args[1:]], indent=1))
    elif args and args[0] == "evalform":
        print(json.dumps([evalform(int(a)) for a in args[1:]], indent=1))
    elif args and args[0] == "swaps":
        print(json.dumps([swaps(int(a)) for a in args[1:]] or [swaps(2)], indent=1))
    else:
        ks = [int(a) for a in args] or [2]
        res = [study(k) for k in ks]
        print(json.dumps(res, indent=1))
