// elmddm.cu -- the C ABI (include/elmddm.h): context, geometry / face tables, argument
// validation, error reporting and the per-call launch sequences.
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "internal.h"

// NVTX range per C-ABI phase call (host-side enqueue span; names = the C-ABI entry points), so
// an nsys / ncu --nvtx timeline groups the kernels by the step of Algorithm 1 that launched them
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

namespace {

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

elmddm_status cuda_fail(elmddm_ctx* c, cudaError_t e, const char* where) {
    if (c) c->err = std::string(where) + ": " + cudaGetErrorString(e);
    return ELMDDM_ECUDA;
}

// face of edge e (0 L, 1 R, 2 B, 3 T) of subdomain (i, j); strip order (reading R14):
// strip j = [V(0..P-2, j) | H(0..P-1, j)], V between (i,j)-(i+1,j), H between (i,j)-(i,j+1).
int face_id(int P, int i, int j, int e) {
    const int strip = 2 * P - 1;
    if (e == 0) return i > 0 ? j * strip + (i - 1) : -1;
    if (e == 1) return i < P - 1 ? j * strip + i : -1;
    if (e == 2) return j > 0 ? (j - 1) * strip + (P - 1) + i : -1;
    return j < P - 1 ? j * strip + (P - 1) + i : -1;
}

template <typename T>
cudaError_t upload(T** dptr, const std::vector<T>& v) {
    size_t n = std::max<size_t>(v.size(), 1);
    cudaError_t e = cudaMalloc((void**)dptr, n * sizeof(T));
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

bool validate(const elmddm_config* cfg, std::string& why) {
    if (!cfg) return why = "null config", false;
    if (cfg->P < 1 || cfg->P > 1024) return why = "P out of range", false;
    if (cfg->M < 8 || cfg->M % 8 != 0) return why = "M must be a positive multiple of 8", false;
    if (cfg->p < 1) return why = "p must be >= 1", false;
    if (cfg->layout < 0 || cfg->layout > 1) return why = "layout must be 0 (face points) or 1 (lattice)", false;
    if (cfg->layout == 0 && (cfg->q < 2 || cfg->q % 2 != 0)) return why = "q must be even and >= 2", false;
    if (cfg->layout == 1 && (cfg->q < 1 || cfg->p != cfg->q)) return why = "lattice layout: need p == q >= 1", false;
    if (cfg->layout == 1 && cfg->problem == 7) return why = "lattice layout: plate bending not supported", false;
    int64_t m = (int64_t)cfg->p * cfg->p + 4 * cfg->q + (cfg->layout == 1 ? 4 : 0);
    if (m < cfg->M && cfg->tikhonov == 0.0)
        return why = "need m >= M (overdetermined local LS, P:288-292) or damping rows", false;
    if (!(cfg->tikhonov == cfg->tikhonov) || !(cfg->tikhonov < 1e300) || !(cfg->tikhonov > -1e300))
        return why = "tikhonov must be finite", false;
    if (cfg->tikhonov != 0.0) m += cfg->M;  // reading R29: M damping rows below the collocation rows
    // ld <= 3008: every panel variant; taller (up to ~9.6k rows): the 4-CTA cluster block panel;
    // taller still: the cooperative grid panel, which needs every subdomain's CTAs co-resident
    if (round_up(m, 32) > 3008 && panel_cl_stage(round_up(m, 32), 227 * 1024) == 0 &&
        (int64_t)(cfg->s_end - cfg->s_begin) > 64)
        return why = "very tall local problems (ld > ~9600 rows) need <= 64 subdomains per context", false;
    if (cfg->problem < 0 || cfg->problem > 7) return why = "unknown problem id", false;
    if (cfg->init_scheme < 0 || cfg->init_scheme > 2) return why = "unknown init_scheme", false;
    if (!(cfg->init_c > 0) || !(cfg->r_over_diam >= 0)) return why = "init_c must be > 0, r_over_diam >= 0", false;
    int64_t N = (int64_t)cfg->P * cfg->P;
    if (cfg->s_begin < 0 || cfg->s_end > N || cfg->s_begin >= cfg->s_end) return why = "bad [s_begin, s_end)", false;
    if (cfg->interface_mode < 0 || cfg->interface_mode > 3) return why = "bad interface_mode", false;
    if (cfg->q > 256) return why = "q too large", false;
    if (cfg->layout == 1 && (int64_t)(cfg->P - 1) * (cfg->P - 1) + 2LL * cfg->P * (cfg->P - 1) * cfg->q > 16384)
        return why = "lattice layout: dense interface limited to G <= 16384 unknowns", false;
    return true;
}

elmddm_status finish_tables(elmddm_ctx* c, const std::vector<int>& qsrc, const std::vector<int>& pptr,
                            const std::vector<int>& pbc, const std::vector<FaceTerm>& terms,
                            const std::vector<int>& gptr, const std::vector<FaceTerm>& gterms);

// Layout 1 (the paper's lattice, reading R32): interface unknowns G = faces q + (P-1)^2, flux
// equations n_eq = faces q + 4 (P-1)^2 (one per face point; per cross point one per incident face,
// the corner remark P:282-286), each with two contributors (subdomain, local flux row) kept in
// ascending subdomain order.  The interface system is assembled densely (Q of n_eq x (G+1), its
// Gram) and factored by the tile Cholesky on a dense plan: "faces" of 64 consecutive unknowns in
// natural order, every tile pair coupled.
elmddm_status build_tables_lattice(elmddm_ctx* c, const std::vector<int>& umap) {
    const int P = c->cfg.P, q = c->cfg.q, N = P * P, F = c->faces;
    const int64_t Gf = (int64_t)F * q, X = (int64_t)(P - 1) * (P - 1), G = Gf + X, NE = Gf + 4 * X;
    const int na = (int)c->sz.na;
    // unknown -> its (subdomain, local column) pairs, ascending s (2 for a face point, 4 for a
    // cross point): the S1 gather of k_lat_mfill
    std::vector<int> rmap((size_t)std::max<int64_t>(G, 1) * 8, -1);
    {
        const int ne = (int)c->sz.ne;
        std::vector<int> fill((size_t)std::max<int64_t>(G, 1), 0);
        for (int s = 0; s < N; ++s)
            for (int t = 0; t < ne; ++t) {
                const int u = umap[(size_t)s * ne + t];
                if (u < 0) continue;
                if (fill[u] >= 4) {
                    c->err = "internal: an interface unknown in more than four subdomains";
                    return ELMDDM_EINVAL;
                }
                rmap[(size_t)u * 8 + 2 * fill[u]] = s;
                rmap[(size_t)u * 8 + 2 * fill[u] + 1] = t;
                ++fill[u];
            }
    }
    // flux row ar of subdomain s -> equation (as orc_flux_eq of the oracle's layout 1; its own
    // numbering, re-derived here): face points f*q + k; cross point x, incident face t at Gf + 4x + t
    std::vector<int> eqsrc((size_t)std::max<int64_t>(NE, 1) * 4, -1);  // [eq][(s, ar) x 2]
    for (int s = 0; s < N; ++s) {  // ascending s: slot 0 gets the smaller subdomain
        int i = s % P, j = s / P;
        for (int ar = 0; ar < na; ++ar) {
            int64_t eq = -1;
            if (ar < 4 * q) {
                int f = c->sub_face[s * 4 + ar / q];
                if (f >= 0) eq = (int64_t)f * q + ar % q;
            } else {
                int cc = (ar - 4 * q) / 2, d = (ar - 4 * q) % 2, ci = cc & 1, cj = cc >> 1;
                int Xi = i + ci, Yj = j + cj;
                if (Xi > 0 && Xi < P && Yj > 0 && Yj < P) {
                    int x = (Yj - 1) * (P - 1) + (Xi - 1);
                    int t = d == 0 ? (cj == 1 ? 0 : 1) : (ci == 1 ? 2 : 3);
                    eq = Gf + 4LL * x + t;
                }
            }
            if (eq < 0) continue;
            int slot = eqsrc[eq * 4] < 0 ? 0 : 1;
            if (slot == 1 && eqsrc[eq * 4 + 2] >= 0) {
                c->err = "internal: a flux equation with more than two contributors";
                return ELMDDM_EINVAL;
            }
            eqsrc[eq * 4 + 2 * slot] = s;
            eqsrc[eq * 4 + 2 * slot + 1] = ar;
        }
    }
    c->sz.G = G;
    c->sz.faces = F;
    c->sz.n_eq = NE;
    c->sz.G_pad = round_up(std::max<int64_t>(G, 1), ELM_NB);
    c->sz.halfband = G > 0 ? G - 1 : 0;
    // dense plan: pseudo-faces of 64 unknowns, all pairs (b >= c)
    const int Fd = (int)((G + ELM_NB - 1) / ELM_NB);
    std::vector<std::pair<int, int>> allp;
    for (int b = 0; b < Fd; ++b)
        for (int cc = 0; cc <= b; ++cc) allp.push_back({b, cc});
    build_chol_plan(P, ELM_NB, Fd, allp, 0, c->crit_band, c->plan, chol_split_min());
    if (c->chol_sched) c->chol_sim_us = schedule_chol_tasks(c->plan, 2 * c->nsm);
    c->plan_q = ELM_NB;
    c->ld_q = round_up(std::max<int64_t>(NE, 1), 32);
    // face equation blocks: face f's q point equations, then the (<= 2) cross-point equations of its
    // endpoints, all contributed by the same two subdomains (s1 < s2); Q_f's columns are
    // [s1's ne local columns | s2's | rhs], its Gram G_f = Q_f^T Q_f.  flist[u]: the (face,
    // column) copies of unknown u (every face of every subdomain holding u), ascending face.
    const int ne = (int)c->sz.ne, nrow = q + 2;
    std::vector<int> feq((size_t)std::max(F, 1) * nrow, -1), fpair((size_t)std::max(F, 1) * 2, -1);
    std::vector<int> fcnt((size_t)std::max(F, 1), 0);
    for (int64_t eq = 0; eq < NE; ++eq) {
        const int s1 = eqsrc[eq * 4], a1 = eqsrc[eq * 4 + 1];
        // the face: for a face point f*q + k; for a cross-point equation the face holding the
        // contributors' shared edge (found from s1's flux row: its edge through the corner)
        int f;
        if (eq < Gf) {
            f = (int)(eq / q);
        } else {
            const int cc = (a1 - 4 * q) / 2, d = (a1 - 4 * q) % 2;
            const int e = d == 0 ? ((cc & 1) ? 1 : 0) : ((cc >> 1) ? 3 : 2);  // right/left, top/bottom
            f = c->sub_face[s1 * 4 + e];
        }
        if (f < 0 || fcnt[f] >= nrow) {
            c->err = "internal: flux equation outside its face block";
            return ELMDDM_EINVAL;
        }
        feq[(size_t)f * nrow + fcnt[f]++] = (int)eq;
        fpair[(size_t)f * 2] = std::min(s1, eqsrc[eq * 4 + 2]);
        fpair[(size_t)f * 2 + 1] = std::max(s1, eqsrc[eq * 4 + 2]);
    }
    const int FL = 16;
    std::vector<int> flist((size_t)std::max<int64_t>(G, 1) * FL * 2, -1), fn((size_t)std::max<int64_t>(G, 1), 0);
    for (int f = 0; f < F; ++f)
        for (int slot = 0; slot < 2; ++slot) {
            const int s = fpair[(size_t)f * 2 + slot];
            if (s < 0) continue;
            for (int t = 0; t < ne; ++t) {
                const int u = umap[(size_t)s * ne + t];
                if (u < 0) continue;
                if (fn[u] >= FL) {
                    c->err = "internal: an unknown in more than 16 face blocks";
                    return ELMDDM_EINVAL;
                }
                flist[((size_t)u * FL + fn[u]) * 2] = f;
                flist[((size_t)u * FL + fn[u]) * 2 + 1] = slot * ne + t;
                ++fn[u];
            }
        }
    c->lat_nrow = nrow;
    std::vector<int> tI(std::max(c->plan.ntiles, 1), 0), tJ(std::max(c->plan.ntiles, 1), 0);
    for (int I = 0; I < c->plan.nblk; ++I)
        for (int J = 0; J <= I; ++J) {
            const int t = c->plan.tile_map[(size_t)I * c->plan.nblk + J];
            if (t >= 0) {
                tI[t] = I;
                tJ[t] = J;
            }
        }
    cudaError_t e;
    if ((e = upload(&c->d_feq, feq)) != cudaSuccess || (e = upload(&c->d_fpair, fpair)) != cudaSuccess ||
        (e = upload(&c->d_flist, flist)) != cudaSuccess)
        return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_eqsrc, eqsrc)) != cudaSuccess || (e = upload(&c->d_rmap, rmap)) != cudaSuccess ||
        (e = upload(&c->d_tile_I, tI)) != cudaSuccess || (e = upload(&c->d_tile_J, tJ)) != cudaSuccess)
        return cuda_fail(c, e, "upload");
    c->npairs = c->nterms = c->ngterms = 0;
    return finish_tables(c, std::vector<int>(), std::vector<int>(1, 0), std::vector<int>(), std::vector<FaceTerm>(),
                         std::vector<int>(1, 0), std::vector<FaceTerm>());
}

elmddm_status build_tables(elmddm_ctx* c) {
    const int P = c->cfg.P, q = c->cfg.q, N = P * P;
    const int F = 2 * P * (P - 1);
    c->faces = F;
    c->sub_face.assign((size_t)N * 4, -1);
    c->face_sub.assign((size_t)F * 2, -1);
    c->face_edge.assign((size_t)F * 2, -1);
    for (int s = 0; s < N; ++s) {
        int i = s % P, j = s / P;
        for (int e = 0; e < 4; ++e) {
            int f = face_id(P, i, j, e);
            c->sub_face[s * 4 + e] = f;
            if (f < 0) continue;
            // slot 0 = left/lower subdomain (edges R or T), slot 1 = right/upper (edges L or B)
            int slot = (e == 1 || e == 3) ? 0 : 1;
            c->face_sub[f * 2 + slot] = s;
            c->face_edge[f * 2 + slot] = e;
        }
    }
    // local interface column t of subdomain s -> global unknown (strip-order face unknown f*q + k,
    // layout 1: then the cross points row-major), -1 on the boundary (the back-solve gather)
    const int lat = c->cfg.layout == 1;
    const int64_t Gf = (int64_t)F * q;
    const int ne = 4 * q + (lat ? 4 : 0), na = 4 * q + (lat ? 8 : 0);
    std::vector<int> umap((size_t)N * ne, -1);
    for (int s = 0; s < N; ++s) {
        int i = s % P, j = s / P;
        for (int t = 0; t < 4 * q; ++t) {
            int f = c->sub_face[s * 4 + t / q];
            umap[(size_t)s * ne + t] = f >= 0 ? f * q + t % q : -1;
        }
        for (int cc = 0; cc < ne - 4 * q; ++cc) {
            int Xi = i + (cc & 1), Yj = j + (cc >> 1);
            if (Xi > 0 && Xi < P && Yj > 0 && Yj < P)
                umap[(size_t)s * ne + 4 * q + cc] = (int)(Gf + (Yj - 1) * (P - 1) + (Xi - 1));
        }
    }
    c->sz.ne = ne;
    c->sz.na = na;
    cudaError_t e0 = upload(&c->d_umap, umap);
    if (e0 != cudaSuccess) return cuda_fail(c, e0, "upload");
    if (lat) return build_tables_lattice(c, umap);
    // neighbour slots of each flux face a: [a, other faces of sub 0, other faces of sub 1]
    c->nbr.assign((size_t)F * 7, -1);
    std::vector<int> qsrc((size_t)F * 8 * 6, -1);
    for (int a = 0; a < F; ++a) {
        int n = 0;
        c->nbr[a * 7 + n++] = a;
        for (int k = 0; k < 2; ++k) {
            int s = c->face_sub[a * 2 + k];
            for (int e = 0; e < 4; ++e) {
                int f = c->sub_face[s * 4 + e];
                if (f < 0 || f == a) continue;
                c->nbr[a * 7 + n++] = f;
            }
        }
        for (int t = 0; t < 8; ++t) {
            for (int k = 0; k < 2; ++k) {
                int s = c->face_sub[a * 2 + k];
                int er = c->face_edge[a * 2 + k];
                int ec = -1;
                if (t < 7) {
                    int b = c->nbr[a * 7 + t];
                    if (b < 0) continue;
                    for (int e = 0; e < 4; ++e)
                        if (c->sub_face[s * 4 + e] == b) ec = e;
                    if (ec < 0) continue;
                } else {
                    ec = 4;
                }
                int* d = &qsrc[((size_t)a * 8 + t) * 6 + k * 3];
                d[0] = s;
                d[1] = er;
                d[2] = ec;
            }
        }
    }
    // face-block pattern of M (b >= c) and its contributions, in a fixed order
    std::map<std::pair<int, int>, std::vector<FaceTerm>> pairs;
    for (int s = 0; s < N; ++s)
        for (int e1 = 0; e1 < 4; ++e1)
            for (int e2 = 0; e2 < 4; ++e2) {
                int b = c->sub_face[s * 4 + e1], cc = c->sub_face[s * 4 + e2];
                if (b < 0 || cc < 0 || b < cc) continue;
                pairs[{b, cc}].push_back(FaceTerm{0, s, e1 * q, e2 * q});
            }
    for (int a = 0; a < F; ++a)
        for (int t1 = 0; t1 < 7; ++t1)
            for (int t2 = 0; t2 < 7; ++t2) {
                int b = c->nbr[a * 7 + t1], cc = c->nbr[a * 7 + t2];
                if (b < 0 || cc < 0 || b < cc) continue;
                pairs[{b, cc}].push_back(FaceTerm{1, a, t1 * q, t2 * q});
            }
    std::vector<int> pptr, pbc;
    std::vector<FaceTerm> terms;
    int64_t hb = 0;
    pptr.push_back(0);
    for (auto& kv : pairs) {
        pbc.push_back(kv.first.first);
        pbc.push_back(kv.first.second);
        for (auto& t : kv.second) terms.push_back(t);
        pptr.push_back((int)terms.size());
        hb = std::max<int64_t>(hb, (int64_t)(kv.first.first - kv.first.second) * q + q - 1);
    }
    c->npairs = (int)pairs.size();
    c->nterms = (int)terms.size();
    // g terms per face b
    std::vector<int> gptr(1, 0);
    std::vector<FaceTerm> gterms;
    for (int b = 0; b < F; ++b) {
        for (int k = 0; k < 2; ++k) {
            int s = c->face_sub[b * 2 + k];
            if (s < 0) continue;
        }
        // ascending s
        int s0 = c->face_sub[b * 2 + 0], s1 = c->face_sub[b * 2 + 1];
        int sa = std::min(s0, s1), sb = std::max(s0, s1);
        for (int s : {sa, sb}) {
            int eb = -1;
            for (int e = 0; e < 4; ++e)
                if (c->sub_face[s * 4 + e] == b) eb = e;
            gterms.push_back(FaceTerm{0, s, eb * q, 4 * q});
        }
        for (int a = 0; a < F; ++a) {
            // only faces within reach can contain b; scan the 7 slots
            for (int t = 0; t < 7; ++t)
                if (c->nbr[a * 7 + t] == b) gterms.push_back(FaceTerm{1, a, t * q, 7 * q});
        }
        gptr.push_back((int)gterms.size());
    }
    c->ngterms = (int)gterms.size();

    const int64_t G = (int64_t)F * q;
    c->sz.G = G;
    c->sz.n_eq = G;
    c->sz.faces = F;
    c->sz.G_pad = round_up(std::max<int64_t>(G, 1), ELM_NB);
    c->sz.halfband = F > 0 ? hb : 0;
    // ordering + symbolic factorisation of the Schur matrix (plan.cu): interface_mode 0 picks the
    // ordering with less factorisation work, 1 / 2 the strip (envelope) order, 3 nested dissection
    std::vector<std::pair<int, int>> fpairs;
    interface_face_pairs(P, fpairs);  // the planner's pattern must be exactly the assembled one
    {
        bool same = fpairs.size() == pairs.size();
        size_t k = 0;
        for (auto it = pairs.begin(); same && it != pairs.end(); ++it, ++k) same = it->first == fpairs[k];
        if (!same) {
            c->err = "internal: interface pattern of the planner differs from the assembly's";
            return ELMDDM_EINVAL;
        }
    }
    const int mode = c->cfg.interface_mode;
    const int split = chol_split_min();
    if (mode == 3) {
        build_chol_plan(P, q, F, fpairs, 1, c->crit_band, c->plan, split);
    } else {
        build_chol_plan(P, q, F, fpairs, 0, c->crit_band, c->plan, split);
        if (mode == 0 && P >= 3) {
            CholPlan nd;
            build_chol_plan(P, q, F, fpairs, 1, c->crit_band, nd, split);
            if (nd.nupd < c->plan.nupd) c->plan = std::move(nd);
        }
    }
    if (c->chol_sched) c->chol_sim_us = schedule_chol_tasks(c->plan, 2 * c->nsm);
    c->plan_q = q;
    return finish_tables(c, qsrc, pptr, pbc, terms, gptr, gterms);
}

// plan sizes, device tables and flags (both layouts)
elmddm_status finish_tables(elmddm_ctx* c, const std::vector<int>& qsrc, const std::vector<int>& pptr,
                            const std::vector<int>& pbc, const std::vector<FaceTerm>& terms,
                            const std::vector<int>& gptr, const std::vector<FaceTerm>& gterms) {
    const int q = c->cfg.q;
    const CholPlan& pl = c->plan;
    const int nblk = pl.nblk;
    c->sz.band_ld = ELM_TLD;
    c->sz.band_nbw = nblk - 1;
    c->sz.band_elems = (int64_t)pl.ntiles * ELM_TS;
    c->sz.chol_n = pl.n;
    c->sz.chol_blocks = nblk;
    c->sz.chol_ordering = pl.ordering;
    {
        int eb = 0, ee = 0;
        if (c->implicit_e) elm_e_implicit_range(c->cfg.M, (int)c->sz.ne, &eb, &ee);
        c->sz.e_impl_begin = eb;
        c->sz.e_impl_end = ee;
    }
    c->ncrit = pl.ncrit;
    c->chol_flops = pl.nupd * 2 * (int64_t)ELM_NB * ELM_NB * ELM_NB;
    c->sz.chol_tasks = (int64_t)pl.tasks.size();
    c->sz.chol_flops = c->chol_flops;

    c->qrow_ld = q;
    c->qrow_cols = 7 * q + 1;
    c->ga_ld = 7 * q + 2;

    cudaError_t e;
    if ((e = upload(&c->d_sub_face, c->sub_face)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_qsrc, qsrc)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_pair_ptr, pptr)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_pair_bc, pbc)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_terms, terms)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_gterm_ptr, gptr)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_gterms, gterms)) != cudaSuccess) return cuda_fail(c, e, "upload");
    if ((e = upload(&c->d_fbase, pl.fbase)) != cudaSuccess || (e = upload(&c->d_pad, pl.pad)) != cudaSuccess ||
        (e = upload(&c->d_tile_map, pl.tile_map)) != cudaSuccess || (e = upload(&c->d_tasks, pl.tasks)) != cudaSuccess ||
        (e = upload(&c->d_klist, pl.klist)) != cudaSuccess || (e = upload(&c->d_diag_tid, pl.diag_tid)) != cudaSuccess ||
        (e = upload(&c->d_fwd_ptr, pl.fwd_ptr)) != cudaSuccess || (e = upload(&c->d_fwd, pl.fwd)) != cudaSuccess ||
        (e = upload(&c->d_bwd_ptr, pl.bwd_ptr)) != cudaSuccess || (e = upload(&c->d_bwd, pl.bwd)) != cudaSuccess ||
        (e = upload(&c->d_ntc, pl.ntc)) != cudaSuccess || (e = upload(&c->d_mrow_ptr, pl.mrow_ptr)) != cudaSuccess ||
        (e = upload(&c->d_tile_m, pl.tile_m)) != cudaSuccess ||
        (e = upload(&c->d_mrow, pl.mrow)) != cudaSuccess || (e = upload(&c->d_mcol_ptr, pl.mcol_ptr)) != cudaSuccess ||
        (e = upload(&c->d_mcol, pl.mcol)) != cudaSuccess)
        return cuda_fail(c, e, "upload");
    {
        // triangular-solve task lists (heavy block rows split into chunks, plan.cu)
        int nslots = 0;
        for (int dir = 0; dir < 2; ++dir) {
            std::vector<int4> svt;
            std::vector<int> rs;
            nslots = std::max(nslots, build_trsv_tasks(pl, dir, c->trsv_chunk, svt, rs));
            c->sv_ntasks[dir] = (int)svt.size();
            if ((e = upload(&c->d_sv_tasks[dir], svt)) != cudaSuccess || (e = upload(&c->d_sv_slot[dir], rs)) != cudaSuccess)
                return cuda_fail(c, e, "upload");
        }
        nslots = std::max(nslots, 1);
        if ((e = cudaMalloc((void**)&c->d_pflags, sizeof(int) * nslots)) != cudaSuccess ||
            (e = cudaMemset(c->d_pflags, 0, sizeof(int) * nslots)) != cudaSuccess ||
            (e = cudaMalloc((void**)&c->d_ppart, sizeof(double) * ELM_NB * nslots)) != cudaSuccess)
            return cuda_fail(c, e, "trsv slots");
    }
    if ((e = cudaMalloc((void**)&c->d_colcnt, sizeof(int) * nblk)) != cudaSuccess ||
        (e = cudaMemset(c->d_colcnt, 0, sizeof(int) * nblk)) != cudaSuccess ||
        (e = cudaMalloc((void**)&c->d_cready, sizeof(int) * nblk)) != cudaSuccess ||
        (e = cudaMalloc((void**)&c->d_chol_next, sizeof(int) * 4)) != cudaSuccess ||
        (e = cudaMemset(c->d_cready, 0, sizeof(int) * nblk)) != cudaSuccess ||
        (e = cudaMalloc((void**)&c->d_cflags, sizeof(int) * std::max(pl.ntiles, 1))) != cudaSuccess ||
        (e = cudaMemset(c->d_cflags, 0, sizeof(int) * std::max(pl.ntiles, 1))) != cudaSuccess)
        return cuda_fail(c, e, "flags");
    return ELMDDM_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

#define CHECK_CTX(c)                   \
    do {                               \
        if (!(c)) return ELMDDM_EINVAL; \
    } while (0)
#define CHECK_PTR(c, p)                                                                         \
    do {                                                                                        \
        if (!(p) || ((uintptr_t)(p) & 15)) {                                                    \
            (c)->err = std::string("null or misaligned (needs 16 B) pointer argument: ") + #p; \
            return ELMDDM_EINVAL;                                                               \
        }                                                                                       \
    } while (0)

}  // namespace

extern "C" {

elmddm_status elmddm_create(const elmddm_config* cfg, int device, elmddm_ctx** out) {
    if (!out) return ELMDDM_EINVAL;
    *out = nullptr;
    std::string why;
    if (!validate(cfg, why)) return ELMDDM_EINVAL;
    elmddm_ctx* c = new (std::nothrow) elmddm_ctx();
    if (!c) return ELMDDM_ENOMEM;
    c->cfg = *cfg;
    c->device = device;
    DeviceGuard dg(device);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete c;
        return ELMDDM_ECUDA;
    }
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) == cudaSuccess) c->nsm = nsm;
    {
        // subdomain groups for the QR streams (ELMDDM_QR_GROUPS overrides; 1 disables)
        const int64_t S = cfg->s_end - cfg->s_begin;
        // measured (tools/rank_slab.py, config 3 slabs of 256/128/64/32 subdomains): 8 groups is
        // best or within noise everywhere once there are at least 4 subdomains per group
        int g = (int)std::min<int64_t>(8, std::max<int64_t>(1, S / 4));
        if (const char* env = getenv("ELMDDM_QR_GROUPS")) g = atoi(env);
        c->qr_groups = g < 1 ? 1 : g;
        if (const char* env = getenv("ELMDDM_TMA")) c->use_tma = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_WY_REV3")) c->wy_rev3 = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_WY_HINT3")) c->wy_hint3 = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_IMPLICIT_E")) c->implicit_e = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_IFACE_REFINE")) c->iface_refine = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL_GRID")) c->panel_grid = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL_PAIR")) c->panel_pair = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_TRSM_CLUSTER")) c->trsm_cluster = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_GEMM_TMA")) c->gemm_tma = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_TRSM_WIDE")) c->trsm_wide = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_TRSV_CHUNK")) c->trsv_chunk = atoi(env);
        if (const char* env = getenv("ELMDDM_TRSV_INV")) c->trsv_inv = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_CHOL_TRSM_REFINE")) c->chol_trsm_refine = atoi(env) != 0;
        if (c->chol_trsm_refine < 0) c->chol_trsm_refine = !c->iface_refine;
        c->implicit_e = c->implicit_e && c->use_tma;
        // 4-CTA cluster panels cut the per-subdomain latency chain of the QR but spend more SM
        // time: they win for the small per-rank slabs of multi-GPU runs (config 3: 32 subdomains
        // 38.9 -> 28.0 ms, 16: 30.9 -> 18.9 ms) and lose for large ones (256: 174 -> 211 ms)
        c->panel_cluster = S <= 48;
        if (const char* env = getenv("ELMDDM_PANEL_CLUSTER")) c->panel_cluster = atoi(env) != 0;
        // on-chip 8-CTA cluster panels (whole panel in distributed shared memory, right-looking):
        // shortest per-subdomain chain, most SM time per panel -- the choice for small slabs
        // (config 3, 32 subdomains: QR 27.8 -> 26.6 ms, 16: 18.7 -> 14.9 ms; 256: 174 -> 203 ms)
        c->panel8 = S <= 48;
        if (const char* env = getenv("ELMDDM_CHOL_CRITBAND")) c->crit_band = std::max(1, atoi(env));
        if (const char* env = getenv("ELMDDM_CHOL_SCHED")) c->chol_sched = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL8")) c->panel8 = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL_MERGED")) c->panel_merged = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL_TMEM")) c->panel_tmem = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL8_TMEM")) c->panel8_tmem = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_PANEL_PRIO")) c->panel_prio = atoi(env) != 0;
        if (const char* env = getenv("ELMDDM_SCHUR_SIDE")) c->schur_side = atoi(env) != 0;
    }
    elmddm_sizes_t& z = c->sz;
    std::memset(&z, 0, sizeof(z));
    const int64_t P = cfg->P, M = cfg->M, q = cfg->q;
    z.N = P * P;
    z.S = cfg->s_end - cfg->s_begin;
    const int lat = cfg->layout == 1;
    z.ne = 4 * q + (lat ? 4 : 0);  // E_Gamma columns: edge points (+ the 4 corners, layout 1)
    z.na = 4 * q + (lat ? 8 : 0);  // flux rows: edge points (+ 2 per corner, layout 1)
    z.m = (int64_t)cfg->p * cfg->p + 4 * q + (lat ? 4 : 0);
    z.ld = round_up(z.m + (cfg->tikhonov != 0.0 ? cfg->M : 0), 32);
    z.kaug = z.ne + 1;
    z.ncols = M + z.kaug;
    z.kaug_elems = z.S * z.ld * z.ncols;
    z.at_elems = z.S * M * z.na;
    z.tau_elems = z.S * M;
    z.pbuf_ld = z.na;
    z.pbuf_elems = z.N * z.pbuf_ld * z.kaug;
    z.sbuf_ld = z.kaug + 1;
    z.sbuf_elems = z.N * z.sbuf_ld * z.kaug;
    elmddm_status st = build_tables(c);
    if (st != ELMDDM_OK) {
        elmddm_destroy(c);
        return st;
    }
    // V, T of the current panel; the grid panel's partial sums (<= 2 CTAs / SM) and counters
    c->work_factor = z.S * (ELM_NB * z.ld + ELM_NB * ELM_NB) + 2LL * c->nsm * (ELM_NB * (ELM_NB + 1) / 2) + z.S + 16;
    c->work_iface = std::max<int64_t>((int64_t)c->faces * ((int64_t)c->qrow_ld * c->qrow_cols +
                                                          (int64_t)c->ga_ld * c->qrow_cols),
                                      5 * z.chol_n + 2 * z.chol_blocks * (int64_t)ELM_TS + z.chol_n / 1024 + 16 +
                                          (c->iface_refine ? z.band_elems + 2 * z.chol_n : 0));
    if (lat)  // face equation blocks Q_f [q + 2][2 ne + 1] and their Grams [2 ne + 2][2 ne + 1]
        c->work_iface = std::max(c->work_iface, (int64_t)c->faces * ((int64_t)(c->lat_nrow + 3) / 4 * 4 * (2 * z.ne + 1) +
                                                                     (2 * z.ne + 2) * (2 * z.ne + 1)) + 64);
    c->work_back = z.S * z.ld + z.S + 8;  // z, and the grid back-substitution's counters
    z.work_elems = std::max(c->work_factor, std::max(c->work_iface, c->work_back));
    if ((e = cudaMalloc((void**)&c->d_status, sizeof(ElmStatus))) != cudaSuccess ||
        (e = cudaMemset(c->d_status, 0, sizeof(ElmStatus))) != cudaSuccess ||
        (e = cudaMalloc((void**)&c->d_flags, sizeof(int) * (z.chol_blocks + 1))) != cudaSuccess ||
        (e = cudaMemset(c->d_flags, 0, sizeof(int) * (z.chol_blocks + 1))) != cudaSuccess ||
        (e = cudaMalloc((void**)&c->d_epoch, sizeof(int) * 2)) != cudaSuccess ||
        (e = cudaMemset(c->d_epoch, 0, sizeof(int) * 2)) != cudaSuccess) {
        elmddm_destroy(c);
        return ELMDDM_ECUDA;
    }
    *out = c;
    return ELMDDM_OK;
}

void elmddm_destroy(elmddm_ctx* c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto s : c->gstreams) cudaStreamDestroy(s);
    for (auto e : c->ev_join) cudaEventDestroy(e);
    for (auto s : c->pstreams) cudaStreamDestroy(s);
    for (auto e : c->ev_panel) cudaEventDestroy(e);
    for (auto e : c->ev_wy) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (auto& p : c->ev_pending) {
        cudaEventDestroy(p.second.first);
        cudaEventDestroy(p.second.second);
    }
    cudaFree(c->d_status);
    cudaFree(c->d_flags);
    cudaFree(c->d_epoch);
    cudaFree(c->d_sub_face);
    cudaFree(c->d_qsrc);
    cudaFree(c->d_umap);
    cudaFree(c->d_eqsrc);
    cudaFree(c->d_rmap);
    cudaFree(c->d_tile_I);
    cudaFree(c->d_tile_J);
    cudaFree(c->d_feq);
    cudaFree(c->d_fpair);
    cudaFree(c->d_flist);
    cudaFree(c->d_pair_ptr);
    cudaFree(c->d_pair_bc);
    cudaFree(c->d_terms);
    cudaFree(c->d_gterm_ptr);
    cudaFree(c->d_gterms);
    cudaFree(c->d_fbase);
    cudaFree(c->d_pad);
    cudaFree(c->d_tile_map);
    cudaFree(c->d_klist);
    cudaFree(c->d_diag_tid);
    for (int dir = 0; dir < 2; ++dir) {
        cudaFree(c->d_sv_tasks[dir]);
        cudaFree(c->d_sv_slot[dir]);
    }
    cudaFree(c->d_pflags);
    cudaFree(c->d_ppart);
    cudaFree(c->d_tile_m);
    cudaFree(c->d_mrow_ptr);
    cudaFree(c->d_mrow);
    cudaFree(c->d_mcol_ptr);
    cudaFree(c->d_mcol);
    cudaFree(c->d_fwd_ptr);
    cudaFree(c->d_fwd);
    cudaFree(c->d_bwd_ptr);
    cudaFree(c->d_bwd);
    cudaFree(c->d_tasks);
    cudaFree(c->d_cflags);
    cudaFree(c->d_colcnt);
    cudaFree(c->d_cready);
    cudaFree(c->d_chol_next);
    cudaFree(c->d_grf);
    cudaFree(c->d_coef);
    for (void* pr : c->dist.opened) cudaIpcCloseMemHandle(pr);
    cudaFree(c->dist.region);
    cudaFree(c->dist.d_reps);
    cudaFree(c->d_ntc);
    delete c;
}

const char* elmddm_last_error(const elmddm_ctx* c) { return c ? c->err.c_str() : "null context"; }

elmddm_status elmddm_sizes(const elmddm_ctx* c, elmddm_sizes_t* out) {
    CHECK_CTX(c);
    if (!out) return ELMDDM_EINVAL;
    *out = c->sz;
    return ELMDDM_OK;
}

elmddm_status elmddm_chol_plan(const elmddm_ctx* c, int32_t* newidx, int32_t* tile_map, int32_t* tasks) {
    CHECK_CTX(c);
    const CholPlan& pl = c->plan;
    if (newidx)  // factorisation-order index of every interface unknown (strip order)
        for (int64_t x = 0; x < c->sz.G; ++x) newidx[x] = pl.fbase[x / c->plan_q] + (int)(x % c->plan_q);
    if (tile_map) std::copy(pl.tile_map.begin(), pl.tile_map.end(), tile_map);
    if (tasks) export_tasks(pl, tasks);
    return ELMDDM_OK;
}

elmddm_status elmddm_plan_query(int32_t P, int32_t q, int32_t ordering, int32_t workers, int64_t* stats,
                                int32_t* newidx, int32_t* tile_map, int32_t* tasks) {
    if (P < 2 || P > 1024 || q < 1 || q > 4096 || ordering < 0 || ordering > 1 || !stats) return ELMDDM_EINVAL;
    std::vector<std::pair<int, int>> fp;
    interface_face_pairs(P, fp);
    const int F = 2 * P * (P - 1);
    CholPlan pl;
    build_chol_plan(P, q, F, fp, ordering, 3, pl, chol_split_min());
    const double sim = workers > 0 ? schedule_chol_tasks(pl, workers) : 0.0;
    stats[0] = pl.n;
    stats[1] = pl.nblk;
    stats[2] = pl.ntiles;
    stats[3] = pl.nupd;
    stats[4] = (int64_t)pl.tasks.size();
    stats[5] = (int64_t)(sim * 1000.0);  // simulated makespan, ns
    if (newidx)
        for (int f = 0; f < F; ++f)
            for (int k = 0; k < q; ++k) newidx[(int64_t)f * q + k] = pl.fbase[f] + k;
    if (tile_map) std::copy(pl.tile_map.begin(), pl.tile_map.end(), tile_map);
    if (tasks) export_tasks(pl, tasks);
    return ELMDDM_OK;
}

// ---- multi-rank interface factorisation (replicated tile pools, CUDA IPC) -------------------
namespace {
struct RegionLayout {
    size_t pool, ybuf, cbuf, flags, cready, counter, hshake, bytes;
};
RegionLayout region_layout(const elmddm_ctx* c) {
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const CholPlan& pl = c->plan;
    RegionLayout L{};
    size_t o = 0;
    L.pool = o;
    o = up(o + sizeof(double) * (size_t)pl.ntiles * ELM_TS);
    L.ybuf = o;
    o = up(o + sizeof(double) * (size_t)pl.nblk * ELM_TS);
    L.cbuf = o;
    o = up(o + sizeof(double) * (size_t)pl.nblk * ELM_TS);
    L.flags = o;
    o = up(o + sizeof(int) * (size_t)pl.ntiles);
    L.cready = o;
    o = up(o + sizeof(int) * (size_t)pl.nblk);
    L.counter = o;
    o = up(o + sizeof(int) * 2);
    L.hshake = o;  // [0..63]: one word per peer rank, [64]: atomic counter (rank 0's region)
    o = up(o + sizeof(int) * 65);
    L.bytes = o;
    return L;
}
CholRep region_rep(void* base, const RegionLayout& L) {
    char* b = static_cast<char*>(base);
    return CholRep{reinterpret_cast<double*>(b + L.pool), reinterpret_cast<double*>(b + L.ybuf),
                   reinterpret_cast<double*>(b + L.cbuf), reinterpret_cast<int*>(b + L.flags),
                   reinterpret_cast<int*>(b + L.cready)};
}
cudaError_t alloc_region(const RegionLayout& L, void** out) {
    cudaError_t e = cudaMalloc(out, L.bytes);
    if (e != cudaSuccess) return e;
    return cudaMemset(static_cast<char*>(*out) + L.flags, 0, L.bytes - L.flags);  // flags, cready, counter
}
}  // namespace

elmddm_status elmddm_dist_export(elmddm_ctx* c, void* handle) {
    CHECK_CTX(c);
    if (!handle) return ELMDDM_EINVAL;
    DeviceGuard dg(c->device);
    const RegionLayout L = region_layout(c);
    cudaError_t e = cudaSuccess;
    if (!c->dist.region) {
        if ((e = alloc_region(L, &c->dist.region)) != cudaSuccess) return cuda_fail(c, e, "elmddm_dist_export");
        c->dist.region_bytes = L.bytes;
    }
    cudaIpcMemHandle_t h;
    if ((e = cudaIpcGetMemHandle(&h, c->dist.region)) != cudaSuccess) return cuda_fail(c, e, "elmddm_dist_export");
    std::memcpy(handle, &h, sizeof(h));
    return ELMDDM_OK;
}

elmddm_status elmddm_dist_import(elmddm_ctx* c, int32_t rank, int32_t world, const void* handles) {
    CHECK_CTX(c);
    if (world == 1) {  // back to the single-rank path
        DeviceGuard dg(c->device);
        for (void* pr : c->dist.opened) cudaIpcCloseMemHandle(pr);
        cudaFree(c->dist.d_reps);
        c->dist.opened.clear();
        c->dist.d_reps = nullptr;
        c->dist.reps.clear();
        c->dist.nrep = 1;
        c->dist.rank = 0;
        c->dist.counter = nullptr;
        return ELMDDM_OK;
    }
    if (world < 2 || world > 64 || rank < 0 || rank >= world || !handles || !c->dist.region) {
        c->err = "elmddm_dist_import: need 2 <= world <= 64, 0 <= rank < world, handles, and elmddm_dist_export first";
        return ELMDDM_EINVAL;
    }
    DeviceGuard dg(c->device);
    const RegionLayout L = region_layout(c);
    std::vector<CholRep> reps(world);
    std::vector<void*> opened;
    cudaError_t e = cudaSuccess;
    void* rank0 = nullptr;
    for (int r = 0; r < world; ++r) {
        void* base = c->dist.region;
        if (r != rank) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
            if ((e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess) {
                for (void* pr : opened) cudaIpcCloseMemHandle(pr);
                return cuda_fail(c, e, "elmddm_dist_import (cudaIpcOpenMemHandle)");
            }
            opened.push_back(base);
        }
        if (r == 0) rank0 = base;
        reps[r] = region_rep(base, L);
    }
    CholRep* d = nullptr;
    if ((e = cudaMalloc((void**)&d, sizeof(CholRep) * world)) != cudaSuccess ||
        (e = cudaMemcpy(d, reps.data(), sizeof(CholRep) * world, cudaMemcpyHostToDevice)) != cudaSuccess) {
        for (void* pr : opened) cudaIpcCloseMemHandle(pr);
        cudaFree(d);
        return cuda_fail(c, e, "elmddm_dist_import");
    }
    // the task order: list-scheduled for the CTAs of all ranks (every rank computes the same
    // order from the same plan, so the shared counter deals one list)
    if (c->chol_sched) {
        c->chol_sim_us = schedule_chol_tasks(c->plan, 2 * c->nsm * world);
        if ((e = cudaMemcpy(c->d_tasks, c->plan.tasks.data(), sizeof(TaskDesc) * c->plan.tasks.size(),
                            cudaMemcpyHostToDevice)) != cudaSuccess) {
            for (void* pr : opened) cudaIpcCloseMemHandle(pr);
            cudaFree(d);
            return cuda_fail(c, e, "elmddm_dist_import");
        }
    }
    // every rank starts the shared protocol from the same state: epoch 0 and cleared tile flags,
    // column counters and task counters in its own region (each rank clears its own; the
    // collective handshake that follows import orders this before any peer's first push)
    if ((e = cudaMemset(static_cast<char*>(c->dist.region) + L.flags, 0, L.hshake - L.flags)) != cudaSuccess) {
        for (void* pr : opened) cudaIpcCloseMemHandle(pr);
        cudaFree(d);
        return cuda_fail(c, e, "elmddm_dist_import");
    }
    c->dist.epoch = 0;
    for (void* pr : c->dist.opened) cudaIpcCloseMemHandle(pr);
    cudaFree(c->dist.d_reps);
    c->dist.opened = opened;
    c->dist.d_reps = d;
    c->dist.reps = reps;
    c->dist.nrep = world;
    c->dist.rank = rank;
    c->dist.emulate = false;
    c->dist.counter = reinterpret_cast<int*>(static_cast<char*>(rank0) + L.counter);
    return ELMDDM_OK;
}

// IPC sanity check before the factorisation relies on it: phase 0 writes a word into every
// peer's region (system-scope release) and adds 1 to rank 0's handshake counter (system-scope
// atomic); after a host barrier, phase 1 checks that every peer's word arrived and (rank 0)
// that the counter reads world - 1 + its previous value.
__global__ void k_dist_hshake(int phase, int rank, int world, int* const* hs, int magic, int* ok) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (phase == 0) {
        for (int r = 0; r < world; ++r)
            if (r != rank) asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(hs[r] + rank), "r"(magic) : "memory");
        if (rank != 0) atomicAdd_system(hs[0] + 64, 1);
        __threadfence_system();
        return;
    }
    int good = 1;
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;
        int v;
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(hs[rank] + r) : "memory");
        good &= v == magic;
    }
    if (rank == 0) {
        int v;
        asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(hs[0] + 64) : "memory");
        good &= v % (world - 1) == 0 && v > 0;
    }
    *ok = good;
}

elmddm_status elmddm_dist_handshake(elmddm_ctx* c, int32_t phase, int32_t* ok) {
    CHECK_CTX(c);
    if (c->dist.nrep < 2 || c->dist.emulate || (phase != 0 && phase != 1) || !ok) return ELMDDM_EINVAL;
    DeviceGuard dg(c->device);
    const RegionLayout L = region_layout(c);
    const int world = c->dist.nrep;
    // region bases of every rank (own and opened)
    std::vector<int*> hs(world);
    for (int r = 0; r < world; ++r)
        hs[r] = reinterpret_cast<int*>(reinterpret_cast<char*>(c->dist.reps[r].Mb) - L.pool + L.hshake);
    int** dhs = nullptr;
    int* dok = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc((void**)&dhs, sizeof(int*) * world)) != cudaSuccess ||
        (e = cudaMemcpy(dhs, hs.data(), sizeof(int*) * world, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMalloc((void**)&dok, sizeof(int))) != cudaSuccess || (e = cudaMemset(dok, 0, sizeof(int))) != cudaSuccess) {
        cudaFree(dhs);
        cudaFree(dok);
        return cuda_fail(c, e, "elmddm_dist_handshake");
    }
    k_dist_hshake<<<1, 32>>>(phase, c->dist.rank, world, dhs, 0x5a5a0000 + world, dok);
    e = cudaDeviceSynchronize();
    int h = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&h, dok, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(dhs);
    cudaFree(dok);
    if (e != cudaSuccess) return cuda_fail(c, e, "elmddm_dist_handshake");
    *ok = phase == 0 ? 1 : h;
    return ELMDDM_OK;
}

elmddm_status elmddm_dist_pool(const elmddm_ctx* c, double** pool) {
    CHECK_CTX(c);
    if (!pool || !c->dist.region) return ELMDDM_EINVAL;
    *pool = region_rep(c->dist.region, region_layout(c)).Mb;
    return ELMDDM_OK;
}

elmddm_status elmddm_debug_dist_emulate(elmddm_ctx* c, int32_t nrep, const double* Mband, const double* g, double* uG,
                                        double* work, int64_t* ndiff, void* stream) {
    CHECK_CTX(c);
    if (nrep < 2 || nrep > 8 || !Mband || !g || !uG || !work || !ndiff || c->dist.nrep > 1) return ELMDDM_EINVAL;
    DeviceGuard dg(c->device);
    cudaStream_t st = (cudaStream_t)stream;
    const RegionLayout L = region_layout(c);
    std::vector<void*> regs(nrep, nullptr);
    std::vector<CholRep> reps(nrep);
    cudaError_t e = cudaSuccess;
    CholRep* d = nullptr;
    unsigned long long* dcnt = nullptr;
    unsigned long long hcnt = 0;
    const DistState saved = c->dist;
    for (int r = 0; r < nrep && e == cudaSuccess; ++r) {
        if ((e = alloc_region(L, &regs[r])) != cudaSuccess) break;
        reps[r] = region_rep(regs[r], L);
        e = cudaMemcpyAsync(reps[r].Mb, Mband, sizeof(double) * (size_t)c->plan.ntiles * ELM_TS, cudaMemcpyDeviceToDevice,
                            st);
    }
    if (e == cudaSuccess && (e = cudaMalloc((void**)&d, sizeof(CholRep) * nrep)) == cudaSuccess &&
        (e = cudaMemcpy(d, reps.data(), sizeof(CholRep) * nrep, cudaMemcpyHostToDevice)) == cudaSuccess &&
        (e = cudaMalloc((void**)&dcnt, sizeof(unsigned long long))) == cudaSuccess &&
        (e = cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long), st)) == cudaSuccess) {
        c->dist.nrep = nrep;
        c->dist.rank = 0;
        c->dist.emulate = true;
        c->dist.reps = reps;
        c->dist.d_reps = d;
        c->dist.counter = reinterpret_cast<int*>(static_cast<char*>(regs[0]) + L.counter);
        e = run_cholesky_solve(c, reps[0].Mb, g, uG, work, st);
        for (int r = 1; r < nrep && e == cudaSuccess; ++r)
            e = dist_count_diff(reps[0].Mb, reps[r].Mb, (int64_t)c->plan.ntiles * ELM_TS, dcnt, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&hcnt, dcnt, sizeof(hcnt), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    c->dist = saved;
    for (void* r : regs) cudaFree(r);
    cudaFree(d);
    cudaFree(dcnt);
    if (e != cudaSuccess) return cuda_fail(c, e, "elmddm_debug_dist_emulate");
    *ndiff = (int64_t)hcnt;
    return elmddm_sync(c, stream);
}

int64_t elmddm_band_index(const elmddm_ctx* c, int64_t i, int64_t j) {
    if (!c || i < 0 || j < 0 || i >= c->sz.G || j >= c->sz.G) return -1;
    const CholPlan& pl = c->plan;
    const int q = c->plan_q;
    int64_t a = pl.fbase[i / q] + i % q, b = pl.fbase[j / q] + j % q;
    if (a < b) std::swap(a, b);
    const int t = pl.tile_map[(size_t)(a / ELM_NB) * pl.nblk + b / ELM_NB];
    if (t < 0) return -1;
    return (int64_t)t * ELM_TS + a % ELM_NB + (b % ELM_NB) * (int64_t)ELM_TLD;
}

elmddm_status elmddm_sync(elmddm_ctx* c, void* stream) {
    NvtxRange nvtx_("elmddm_sync");
    CHECK_CTX(c);
    DeviceGuard dg(c->device);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "elmddm_sync");
    ElmStatus h{0, 0, 0, 0};
    if ((e = cudaMemcpy(&h, c->d_status, sizeof(h), cudaMemcpyDeviceToHost)) != cudaSuccess)
        return cuda_fail(c, e, "elmddm_sync");
    if (h.code != 0) {
        cudaMemset(c->d_status, 0, sizeof(ElmStatus));
        if (h.info >= 0)
            c->err = "non-positive pivot in the interface Cholesky at row " + std::to_string(h.info);
        else if (h.info <= ELM_INFO_NONFINITE_QR)
            c->err = "non-finite value in the QR of subdomain " + std::to_string(ELM_INFO_NONFINITE_QR - h.info);
        else
            c->err = "interface factorisation / solve: block " + std::to_string(-1 - h.info) + " never completed";
        return (elmddm_status)h.code;
    }
    if (h.wcode != 0) {  // a warning: reported once, results valid
        cudaMemset(c->d_status, 0, sizeof(ElmStatus));
        c->err = "numerically rank-deficient K^s: min |R11_ii| < 1e-14 max |R11_ii| in subdomain " +
                 std::to_string(h.winfo) + " (and possibly others); results computed";
        return (elmddm_status)h.wcode;
    }
    return ELMDDM_OK;
}

elmddm_status elmddm_interface_points(const elmddm_ctx* c, double* xy) {
    CHECK_CTX(c);
    if (!xy) return ELMDDM_EINVAL;
    const int P = c->cfg.P, q = c->cfg.q;
    const int np = c->cfg.problem == 7 ? q / 2 : q;  // plate: unknowns k and k + np share a point
    for (int f = 0; f < c->faces; ++f) {
        int s = c->face_sub[f * 2], e = c->face_edge[f * 2];
        int i = s % P, j = s / P;
        for (int k = 0; k < q; ++k) {
            double t_along, fixed;
            const int kp = k % np;
            if (e == 1) {  // vertical face at x = (i+1)/P
                fixed = (double)(i + 1) / (double)P;
                t_along = (double)(j * (np + 1) + kp + 1) / (double)(P * (np + 1));
                xy[2 * ((int64_t)f * q + k)] = fixed;
                xy[2 * ((int64_t)f * q + k) + 1] = t_along;
            } else {  // horizontal face at y = (j+1)/P
                fixed = (double)(j + 1) / (double)P;
                t_along = (double)(i * (np + 1) + kp + 1) / (double)(P * (np + 1));
                xy[2 * ((int64_t)f * q + k)] = t_along;
                xy[2 * ((int64_t)f * q + k) + 1] = fixed;
            }
        }
    }
    if (c->cfg.layout == 1)  // the cross points, row-major, after the face unknowns
        for (int Y = 1; Y < P; ++Y)
            for (int X = 1; X < P; ++X) {
                const int64_t u = (int64_t)c->faces * q + (int64_t)(Y - 1) * (P - 1) + (X - 1);
                xy[2 * u] = (double)X / (double)P;
                xy[2 * u + 1] = (double)Y / (double)P;
            }
    return ELMDDM_OK;
}

elmddm_status elmddm_init_hidden(elmddm_ctx* c, double* W, double* b, double* xi, void* stream) {
    NvtxRange nvtx_("elmddm_init_hidden");
    CHECK_CTX(c);
    CHECK_PTR(c, W);
    CHECK_PTR(c, b);
    DeviceGuard dg(c->device);
    cudaError_t e = launch_init_hidden(c, W, b, xi, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_init_hidden");
}

elmddm_status elmddm_assemble(elmddm_ctx* c, const double* W, const double* b, double* Kaug, double* At,
                              void* stream) {
    NvtxRange nvtx_("elmddm_assemble");
    CHECK_CTX(c);
    CHECK_PTR(c, W);
    CHECK_PTR(c, b);
    CHECK_PTR(c, Kaug);
    CHECK_PTR(c, At);
    if (c->cfg.problem == 6 && !c->d_grf) {
        c->err = "problem 6 needs elmddm_set_coefficient before elmddm_assemble";
        return ELMDDM_EINVAL;
    }
    DeviceGuard dg(c->device);
    cudaError_t e = launch_assemble(c, W, b, Kaug, At, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_assemble");
}

elmddm_status elmddm_set_coefficient(elmddm_ctx* c, const double* params, int32_t nterms) {
    CHECK_CTX(c);
    if (c->cfg.problem != 6) {
        c->err = "elmddm_set_coefficient: only problem 6 has a coefficient field";
        return ELMDDM_EINVAL;
    }
    if (nterms < 1 || nterms > 65536 || !params) {
        c->err = "elmddm_set_coefficient: need 1 <= nterms <= 65536 and a host parameter array";
        return ELMDDM_EINVAL;
    }
    DeviceGuard dg(c->device);
    cudaError_t e = cudaSuccess;
    if (nterms != c->ngrf) {
        cudaFree(c->d_grf);
        c->d_grf = nullptr;
        c->ngrf = 0;
        if ((e = cudaMalloc((void**)&c->d_grf, sizeof(double) * 4 * (size_t)nterms)) != cudaSuccess)
            return cuda_fail(c, e, "elmddm_set_coefficient");
        c->ngrf = nterms;
    }
    if (!c->d_coef &&
        (e = cudaMalloc((void**)&c->d_coef, sizeof(double) * 4 * (size_t)c->sz.S * c->cfg.p * c->cfg.p)) != cudaSuccess)
        return cuda_fail(c, e, "elmddm_set_coefficient");
    e = cudaMemcpy(c->d_grf, params, sizeof(double) * 4 * (size_t)nterms, cudaMemcpyHostToDevice);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_set_coefficient");
}

elmddm_status elmddm_local_factor(elmddm_ctx* c, double* Kaug, double* tau, double* work, void* stream) {
    NvtxRange nvtx_("elmddm_local_factor");
    CHECK_CTX(c);
    CHECK_PTR(c, Kaug);
    CHECK_PTR(c, tau);
    CHECK_PTR(c, work);
    DeviceGuard dg(c->device);
    cudaError_t e = run_local_factor(c, Kaug, tau, work, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_local_factor");
}

elmddm_status elmddm_schur_accumulate(elmddm_ctx* c, double* Kaug, double* At, double* Pbuf, double* Sbuf,
                                      double* work, void* stream) {
    NvtxRange nvtx_("elmddm_schur_accumulate");
    CHECK_CTX(c);
    CHECK_PTR(c, Kaug);
    CHECK_PTR(c, At);
    CHECK_PTR(c, Pbuf);
    CHECK_PTR(c, Sbuf);
    DeviceGuard dg(c->device);
    cudaError_t e = run_schur_accumulate(c, Kaug, At, Pbuf, Sbuf, work, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_schur_accumulate");
}

elmddm_status elmddm_interface_assemble(elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband,
                                        double* g, double* work, void* stream) {
    NvtxRange nvtx_("elmddm_interface_assemble");
    CHECK_CTX(c);
    CHECK_PTR(c, Pbuf);
    CHECK_PTR(c, Sbuf);
    CHECK_PTR(c, Mband);
    CHECK_PTR(c, g);
    CHECK_PTR(c, work);
    DeviceGuard dg(c->device);
    cudaError_t e = run_interface_assemble(c, Pbuf, Sbuf, Mband, g, work, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_interface_assemble");
}

elmddm_status elmddm_interface_factor_solve(elmddm_ctx* c, double* Mband, const double* g, double* uG, double* work,
                                            void* stream) {
    NvtxRange nvtx_("elmddm_interface_factor_solve");
    CHECK_CTX(c);
    CHECK_PTR(c, Mband);
    CHECK_PTR(c, g);
    CHECK_PTR(c, uG);
    CHECK_PTR(c, work);
    DeviceGuard dg(c->device);
    cudaError_t e = run_cholesky_solve(c, Mband, g, uG, work, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_interface_factor_solve");
}

elmddm_status elmddm_interface_cg(elmddm_ctx* c, const double* Mband, const double* g, double* uG, double* work,
                                  double tol, int32_t maxit, int32_t* iters, double* relres, void* stream) {
    NvtxRange nvtx_("elmddm_interface_cg");
    CHECK_CTX(c);
    CHECK_PTR(c, Mband);
    CHECK_PTR(c, g);
    CHECK_PTR(c, uG);
    CHECK_PTR(c, work);
    if (!(tol > 0.0) || maxit < 1) {
        c->err = "elmddm_interface_cg: tol must be > 0 and maxit >= 1";
        return ELMDDM_EINVAL;
    }
    DeviceGuard dg(c->device);
    int it = 0;
    double rr = 0.0;
    cudaError_t e = run_interface_cg(c, Mband, g, uG, work, tol, maxit, &it, &rr, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "elmddm_interface_cg");
    if (iters) *iters = it;
    if (relres) *relres = rr;
    if (!(rr <= tol)) {
        c->err = "elmddm_interface_cg: no convergence in " + std::to_string(it) + " iterations (relative residual " +
                 std::to_string(rr) + ")";
        return ELMDDM_ENUMERIC;
    }
    return ELMDDM_OK;
}

elmddm_status elmddm_interface_solve(elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband, double* g,
                                     double* uG, double* work, void* stream) {
    elmddm_status s = elmddm_interface_assemble(c, Pbuf, Sbuf, Mband, g, work, stream);
    if (s != ELMDDM_OK) return s;
    s = elmddm_interface_factor_solve(c, Mband, g, uG, work, stream);
    if (s != ELMDDM_OK) return s;
    return elmddm_sync(c, stream);
}

elmddm_status elmddm_back_solve(elmddm_ctx* c, const double* Kaug, const double* uG, double* coef, double* resid,
                                double* work, void* stream) {
    NvtxRange nvtx_("elmddm_back_solve");
    CHECK_CTX(c);
    CHECK_PTR(c, Kaug);
    CHECK_PTR(c, uG);
    CHECK_PTR(c, coef);
    CHECK_PTR(c, resid);
    CHECK_PTR(c, work);
    DeviceGuard dg(c->device);
    cudaError_t e = run_back_solve(c, Kaug, uG, coef, resid, work, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_back_solve");
}

elmddm_status elmddm_evaluate(elmddm_ctx* c, const double* W, const double* b, const double* coef, const double* xy,
                              int64_t n, double* u, void* stream) {
    NvtxRange nvtx_("elmddm_evaluate");
    CHECK_CTX(c);
    if (n < 0) return ELMDDM_EINVAL;
    if (n == 0) return ELMDDM_OK;
    CHECK_PTR(c, W);
    CHECK_PTR(c, b);
    CHECK_PTR(c, coef);
    CHECK_PTR(c, xy);
    CHECK_PTR(c, u);
    DeviceGuard dg(c->device);
    cudaError_t e = launch_evaluate(c, W, b, coef, xy, n, u, (cudaStream_t)stream);
    return e == cudaSuccess ? ELMDDM_OK : cuda_fail(c, e, "elmddm_evaluate");
}

elmddm_status elmddm_set_timing(elmddm_ctx* c, int enable) {
    CHECK_CTX(c);
    c->timing = enable != 0;
    return ELMDDM_OK;
}

elmddm_status elmddm_timing(elmddm_ctx* c, elmddm_timing_t* out, int reset) {
    CHECK_CTX(c);
    DeviceGuard dg(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "elmddm_timing");
    for (auto& p : c->ev_pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, p.second.first, p.second.second) == cudaSuccess) c->cls_ms[p.first] += ms;
        c->ev_pool.push_back(p.second.first);
        c->ev_pool.push_back(p.second.second);
    }
    c->ev_pending.clear();
    if (out) {
        out->launches = c->launches;
        for (int k = 0; k < ELMDDM_NCLASS; ++k) {
            out->count[k] = c->cls_count[k];
            out->ms[k] = c->cls_ms[k];
        }
    }
    if (reset) {
        c->launches = 0;
        for (int k = 0; k < ELMDDM_NCLASS; ++k) {
            c->cls_count[k] = 0;
            c->cls_ms[k] = 0.0;
        }
    }
    return ELMDDM_OK;
}

}  // extern "C"
