"""Shared test helpers: run the CUDA path phase by phase and map its layouts onto the oracle's."""
from __future__ import annotations

import numpy as np

import oracle as O
import workloads as WL

EPS = np.finfo(float).eps


def ocfg(c: dict):
    O.set_grf(c.get("grf"))  # problem 6 coefficient (None clears it)
    return O.cfg(c["P"], c["M"], c["p"], c["q"], c["problem"], c.get("init_scheme", 0), c.get("init_c", 0.125),
                 c.get("r_over_diam", 0.5), c["seed"], c.get("tikhonov", 0.0), c.get("layout", 0))


def small(**kw):
    base = dict(P=2, M=16, p=6, q=4, problem=0, seed=7, init_scheme=0, init_c=0.125, r_over_diam=0.5)
    base.update(kw)
    if base["problem"] == 6 and base.get("grf") is None:
        base["grf"] = WL.grf_params(base.get("alpha", 4.0), base["seed"])
    return base


def gpu_ctx(c: dict, s_begin=0, s_end=None):
    import paper_2406_15959_b200 as E

    pr = E.Problem.from_config(c)
    ctx = E.Context(pr, s_begin, s_end)
    return ctx, ctx.alloc()


def run_gpu(c: dict, xy=None, upto="all"):
    """Run the hot path on cuda:0 for config dict c; returns (ctx, buf, u or None)."""
    import torch

    ctx, buf = gpu_ctx(c)
    xy_t = u = None
    if xy is not None:
        xy_t = torch.as_tensor(np.ascontiguousarray(xy), dtype=torch.float64, device="cuda").reshape(-1)
        u = torch.zeros(xy.shape[0], dtype=torch.float64, device="cuda")
    if upto == "all":
        ctx.run(buf, xy_t, u)
    else:
        ctx.init_hidden(buf["W"], buf["b"], buf["xi"])
        ctx.assemble(buf["W"], buf["b"], buf["Kaug"], buf["At"])
        if upto in ("factor", "schur"):
            ctx.local_factor(buf["Kaug"], buf["tau"], buf["work"])
        if upto == "schur":
            ctx.schur_accumulate(buf["Kaug"], buf["At"], buf["Pbuf"], buf["Sbuf"], buf["work"])
    torch.cuda.synchronize()
    return ctx, buf, u


def kaug_np(ctx, buf, sl):
    z = ctx.sizes
    K = buf["Kaug"].view(z["S"], z["ncols"], z["ld"])[sl].cpu().numpy()
    return K.T  # (ld, ncols)


def kaug_assembled_np(ctx, buf, sl, c: dict):
    """K_aug of local subdomain sl as elmddm_assemble defines it: the implicit E_Gamma columns
    [e_impl_begin, e_impl_end) (include/elmddm.h: not written, synthesised by the QR) filled with
    their definition -- a one at row p^2 + t of column M + t when edge t // q is an interface edge."""
    K = kaug_np(ctx, buf, sl).copy()
    z = ctx.sizes
    M, q, P, pp = c["M"], c["q"], c["P"], c["p"] ** 2
    s = ctx.s_begin + sl
    i, j = s % P, s // P
    iface = [i > 0, i < P - 1, j > 0, j < P - 1]
    iface += [0 < i + (cc & 1) < P and 0 < j + (cc >> 1) < P for cc in range(4)]  # lattice corners
    for col in range(z["e_impl_begin"], z["e_impl_end"]):
        t = col - M
        K[:, col] = 0.0
        if iface[t // q if t < 4 * q else 4 + t - 4 * q]:
            K[pp + t, col] = 1.0
    return K


def at_np(ctx, buf, sl, M, q):
    return buf["At"].view(-1, ctx.sizes["na"], M)[sl].cpu().numpy()  # (na, M) = A rows


def local_iface_index(c: dict, s: int):
    """GPU local index (e*q + k) of the oracle's interface points, in the oracle's row order."""
    xy, edge, gidx = O.rows(ocfg(c), s)
    m = len(edge)
    rows = np.where(gidx >= 0)[0]
    return rows - (m - 4 * c["q"]), gidx[rows]


def pbuf_np(ctx, buf, s, q):
    z = ctx.sizes
    return buf["Pbuf"].view(z["N"], z["kaug"], z["pbuf_ld"])[s].cpu().numpy().T  # (4q, kaug)


def sbuf_np(ctx, buf, s):
    """Gram block of subdomain s, symmetrised from its stored lower triangle (kaug, kaug)."""
    z = ctx.sizes
    S = buf["Sbuf"].view(z["N"], z["kaug"], z["sbuf_ld"])[s].cpu().numpy().T[: z["kaug"], :]
    return np.tril(S) + np.tril(S, -1).T


def band_offsets(ctx, i, j):
    """Offsets of Schur-matrix elements (i, j) (strip order, either triangle) in the packed tile
    storage (include/elmddm.h elmddm_band_index, vectorised): renumber into the factorisation
    order, take the lower element, look its tile up."""
    newidx, tmap, _ = ctx.chol_plan()
    a, b = newidx[np.asarray(i)], newidx[np.asarray(j)]
    a, b = np.maximum(a, b).astype(np.int64), np.minimum(a, b).astype(np.int64)
    tile = tmap[a // 64, b // 64].astype(np.int64)
    tld = ctx.sizes["band_ld"]
    return np.where(tile >= 0, tile * 64 * tld + a % 64 + (b % 64) * tld, -1)


def band_to_dense(ctx, Mband):
    """Full symmetric G x G matrix from the packed tile storage (host; small G only)."""
    G = ctx.sizes["G"]
    Mb = Mband.cpu().numpy()
    ii, jj = np.meshgrid(np.arange(G), np.arange(G), indexing="ij")
    off = band_offsets(ctx, ii.ravel(), jj.ravel())
    return np.where(off >= 0, Mb[np.maximum(off, 0)], 0.0).reshape(G, G)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))
