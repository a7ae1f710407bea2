// schur.cu -- elimination of the output weights into the interface Schur system, the rank-0
// interface assembly, and the local back-solve.
//
//   W_s   = A^s R11^{-1}            (TRSM on At = (A^s)^T, in place; the flux operator formed once)
//   P_s   = W_s [R12 | y]           (flux of c^s(u) = q_s + P_s u_s)
//   S_s   = [T_E | t_F]^T [T_E | t_F]
//   M     = sum_s scatter(T_E^T T_E) + Q^T Q,   g = -sum_s scatter(T_E^T t_F) - Q^T q
//   c^s   = R11^{-1}(y + R12 u_s),  r_s = ||t_F + T_E u_s||
// (eqn:eliminated .. eqn:schur; readings R13 and R23 in DESIGN.md.)
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"
#include "tma.cuh"

namespace {

// ---- interface: Q row blocks ------------------------------------------------------------------
// Qrow[a] (q x (7q+1), ld qrow_ld): slot t (t < 7) = sum over the (<= 2) subdomains touching both
// face a and face nbr[a][t] of P_s[e_a rows, e_b cols]; slot 7 = sum_s q_s[e_a rows].
// qsrc[a][t][c][3] = (s, e_row, e_col) or s = -1.  grid (faces, 8).
__global__ void k_qrow(const double* __restrict__ Pbuf, int64_t pstride, int64_t pld, const int* __restrict__ qsrc,
                       int q, double* __restrict__ Qrow, int64_t qld, int64_t qstride) {
    const int a = blockIdx.x, t = blockIdx.y;
    const int* src = qsrc + ((int64_t)a * 8 + t) * 6;
    const int ncolblk = t < 7 ? q : 1;
    double* dst = Qrow + (int64_t)a * qstride + (int64_t)t * q * qld;
    for (int e = threadIdx.x; e < q * ncolblk; e += blockDim.x) {
        int i = e % q, j = e / q;
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            int s = src[c * 3];
            if (s >= 0) {
                int er = src[c * 3 + 1], ec = src[c * 3 + 2];
                int64_t col = t < 7 ? (int64_t)ec * q + j : 4 * (int64_t)q;
                v += Pbuf[(int64_t)s * pstride + (int64_t)er * q + i + col * pld];
            }
        }
        dst[i + (int64_t)j * qld] = v;
    }
}


// Ga = Qrow^T Qrow is symmetric and only its 64-tiles on and below the diagonal are computed
// (gemm lower_only): element (rr, cc) of an upper tile is read as (cc, rr)
__device__ __forceinline__ double ga_at(const double* __restrict__ Ga, int rr, int cc, int64_t gld) {
    return (rr >> 6) >= (cc >> 6) ? Ga[rr + (int64_t)cc * gld] : Ga[cc + (int64_t)rr * gld];
}

// M block (b, c) = sum of terms, written in the band storage (b == c: lower triangle only).
__global__ void k_massemble(const int* __restrict__ pair_ptr, const int* __restrict__ pair_bc,
                            const FaceTerm* __restrict__ terms, const double* __restrict__ Sbuf, int64_t sstride,
                            int64_t sld, const double* __restrict__ Ga, int64_t gstride, int64_t gld, int q,
                            double* __restrict__ Mband, const int* __restrict__ fbase,
                            const int* __restrict__ tile_map, int nblk) {
    const int p = blockIdx.x;
    const int b = pair_bc[2 * p], c = pair_bc[2 * p + 1];
    const int t0 = pair_ptr[p], t1 = pair_ptr[p + 1];
    for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
        int i = e % q, j = e / q;
        if (b == c && i < j) continue;
        double v = 0.0;
        for (int t = t0; t < t1; ++t) {
            FaceTerm ft = terms[t];
            if (ft.kind == 0) {  // S is symmetric and only its lower triangle is stored
                const int rr = ft.r0 + i, cc = ft.c0 + j;
                v += rr >= cc ? Sbuf[(int64_t)ft.src * sstride + rr + (int64_t)cc * sld]
                              : Sbuf[(int64_t)ft.src * sstride + cc + (int64_t)rr * sld];
            }
            else v += ga_at(Ga + (int64_t)ft.src * gstride, ft.r0 + i, ft.c0 + j, gld);
        }
        // element (b q + i, c q + j) at (a, d) of the factorisation order, lower triangle
        int a = fbase[b] + i, d = fbase[c] + j;
        if (a < d) {
            const int t = a;
            a = d;
            d = t;
        }
        const int tile = tile_map[(int64_t)(a / ELM_NB) * nblk + d / ELM_NB];
        Mband[(int64_t)tile * ELM_TS + a % ELM_NB + (d % ELM_NB) * ELM_TLD] = v;
    }
}

// g[b q + i] = -(sum of terms); grid faces.
__global__ void k_gassemble(const int* __restrict__ gptr, const FaceTerm* __restrict__ gterms,
                            const double* __restrict__ Sbuf, int64_t sstride, int64_t sld, const double* __restrict__ Ga,
                            int64_t gstride, int64_t gld, int q, double* __restrict__ g) {
    const int b = blockIdx.x;
    for (int i = threadIdx.x; i < q; i += blockDim.x) {
        double v = 0.0;
        for (int t = gptr[b]; t < gptr[b + 1]; ++t) {
            FaceTerm ft = gterms[t];
            if (ft.kind == 0) v += Sbuf[(int64_t)ft.src * sstride + ft.c0 + (int64_t)(ft.r0 + i) * sld];  // row 4q (lower)
            else v += ga_at(Ga + (int64_t)ft.src * gstride, ft.r0 + i, ft.c0, gld);
        }
        g[(int64_t)b * q + i] = -v;
    }
}

// padding unknowns of the factorisation order: unit diagonal; g beyond G (strip order): zero
__global__ void k_pad(double* Mband, const int* __restrict__ pad, int npad, const int* __restrict__ diag_tid,
                      double* g, int64_t G, int64_t G_pad) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < npad) {
        const int pidx = pad[x];
        Mband[(int64_t)diag_tid[pidx / ELM_NB] * ELM_TS + (pidx % ELM_NB) * (1 + ELM_TLD)] = 1.0;
    }
    if (G + x < G_pad) g[G + x] = 0.0;
}

// ---- back-solve -----------------------------------------------------------------------------
// z[s][r] = sum_t Kaug[s][r][M + t] v_t, v = [u_s ; 1].   grid (ceil(ld/256), S)
__global__ void __launch_bounds__(256) k_bs_gemv(elmddm_config cfg, const double* __restrict__ Kaug, int64_t ld,
                                                 int64_t ncols, const int* __restrict__ umap, int ne,
                                                 const double* __restrict__ uG, double* __restrict__ z) {
    extern __shared__ double v[];
    const int M = cfg.M, kaug = ne + 1;
    const int sl = blockIdx.y, s = cfg.s_begin + sl;
    for (int t = threadIdx.x; t < kaug; t += blockDim.x) {
        double val = 1.0;  // u_s gathered through the local -> global map, 0 on the boundary
        if (t < ne) {
            const int u = umap[(int64_t)s * ne + t];
            val = u >= 0 ? uG[u] : 0.0;
        }
        v[t] = val;
    }
    __syncthreads();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= ld) return;
    const double* A = Kaug + (int64_t)sl * ld * ncols + (int64_t)M * ld + r;
    double acc = 0.0;
    for (int t = 0; t < kaug; ++t) acc += A[(int64_t)t * ld] * v[t];
    z[(int64_t)sl * ld + r] = acc;
}

// per subdomain: resid = ||z[M:ld]||, coef = R11^{-1} z[0:M] (blocked column-oriented
// back substitution; 64-row diagonal blocks solved by warp 0).  grid S, BS_NT threads (the
// block-column GEMV updates are HBM-latency bound: more threads, more loads in flight).
constexpr int BS_NT = 1024;
__global__ void __launch_bounds__(BS_NT) k_bs_trsv(const double* __restrict__ Kaug, int64_t ld, int64_t ncols, int M,
                                                 double* __restrict__ z, double* __restrict__ coef,
                                                 double* __restrict__ resid) {
    __shared__ double Rs[64][65];
    __shared__ double cs[64];
    __shared__ double red[BS_NT / 32];
    __shared__ double rdg[64];
    const int sl = blockIdx.x;
    const double* A = Kaug + (int64_t)sl * ld * ncols;
    double* zs = z + (int64_t)sl * ld;
    // residual norm (deterministic)
    double ss = 0.0;
    for (int r = M + threadIdx.x; r < ld; r += blockDim.x) ss += zs[r] * zs[r];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        resid[sl] = sqrt(t);
    }
    const int nblk = (M + 63) / 64;
    for (int ib = nblk - 1; ib >= 0; --ib) {
        const int i0 = ib * 64, bi = min(64, M - i0);
        __syncthreads();
        for (int t = threadIdx.x; t < bi * bi; t += blockDim.x) {
            int r = t % bi, c = t / bi;
            Rs[r][c] = A[(int64_t)(i0 + c) * ld + i0 + r];
        }
        __syncthreads();
        if (threadIdx.x < bi) rdg[threadIdx.x] = 1.0 / Rs[threadIdx.x][threadIdx.x];
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            double z0 = lane < bi ? zs[i0 + lane] : 0.0;
            double z1 = lane + 32 < bi ? zs[i0 + lane + 32] : 0.0;
            for (int r = bi - 1; r >= 0; --r) {
                double cr;
                if (r >= 32) cr = __shfl_sync(0xffffffffu, z1, r - 32);
                else cr = __shfl_sync(0xffffffffu, z0, r);
                cr = cr * rdg[r];
                if (lane < r) z0 -= Rs[lane][r] * cr;
                if (lane + 32 < r) z1 -= Rs[lane + 32][r] * cr;
                if (lane == (r & 31)) {
                    if (r >= 32) z1 = cr;
                    else z0 = cr;
                }
            }
            if (lane < bi) cs[lane] = z0;
            if (lane + 32 < bi) cs[lane + 32] = z1;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < bi; t += blockDim.x) coef[(int64_t)sl * M + i0 + t] = cs[t];
        // z[0:i0] -= R[0:i0, i0:i0+bi] c_i
        for (int r = threadIdx.x; r < i0; r += blockDim.x) {
            double acc = 0.0;
            for (int k = 0; k < bi; ++k) acc += A[(int64_t)(i0 + k) * ld + r] * cs[k];
            zs[r] -= acc;
        }
    }
}

// ---- fused left-looking TRSM: W_s^T = R11^{-T} (A^s)^T, in place on At ---------------------------
// grid (ceil(4q/64), S), 256 threads.  CTA (cb, s) owns flux rows [64cb, 64cb+64) of At[s] and
// walks the 64-row neuron blocks i in order:
//     C_i = At_i - sum_{k<i} R_ki^T X_k        (DMMA; R_ki and X_k staged by TMA in 32-row chunks,
//                                               2-stage mbarrier pipeline; X_k = this CTA's
//                                               earlier output, L2-resident)
//     X_i = R_ii^{-T} C_i                       (forward substitution in shared memory: backward
//                                               stable, R11 is numerically rank deficient)
// Every output element is written once (the former 25 launches of rank-64 GEMM updates re-read
// and re-wrote At each step).
namespace trw {
using namespace elmtma;
constexpr int NT = 256;
constexpr int STAGE = 4 * BOX;           // R chunk (2 boxes) + X chunk (2 boxes)
constexpr int XP = 65;                   // padded stride of the diagonal-solve tiles
constexpr int SMEM_BODY = (2 * STAGE > 2 * 64 * XP + 64 ? 2 * STAGE : 2 * 64 * XP + 64);
constexpr int RSP = 4 * BOX;             // the diagonal block R_ii, TMA-prefetched (4 boxes of 16 rows)
constexpr int SMEM = (SMEM_BODY + RSP) * 8 + 64 + 1024;  // + mbarriers (<= 64 B)
}  // namespace trw

// Cluster version (launched with a cluster of gridDim.x CTAs, all flux-row tiles of one
// subdomain; nc = 1 without a cluster): the 4 (or nc) CTAs of a subdomain read the SAME chunks of
// R11, so the cluster's rank-0 CTA loads each R chunk once and multicasts it into every CTA's
// stage (cp.async.bulk.tensor ... .multicast::cluster; each CTA's full barrier expects the R and
// its own X bytes); before refilling a stage it waits on its cluster-wide empty barrier, which
// every warp of every CTA arrives on (remote mbarrier arrive) when done with the stage.  The
// diagonal solve reuses the stages as scratch, so the CTAs meet at a cluster barrier after every
// block.  Per-CTA arithmetic and order are unchanged (bit-identical to nc = 1).
__device__ __forceinline__ uint32_t trw_mapa(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void trw_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void trw_mbar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(elmtma::su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void trw_tma_load_mc(double* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                                uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;\n"
        ::"r"(elmtma::su32(dst)), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(c2), "r"(elmtma::su32(bar)), "h"(mask) : "memory");
}

__global__ void __launch_bounds__(trw::NT, 2) k_trsm_w(const __grid_constant__ CUtensorMap tmR,
                                                       const __grid_constant__ CUtensorMap tmA,
                                                       const double* __restrict__ Kaug, int64_t ld, int64_t ncols,
                                                       double* __restrict__ At, int M, int nat) {
    using namespace trw;
    extern __shared__ uint8_t raw[];
    double* base = reinterpret_cast<double*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
    double* stg = base;                                   // 2 stages x (R 2 boxes | X 2 boxes)
    double* RsP = base + SMEM_BODY;                       // R_ii prefetched by TMA (swizzled boxes)
    uint64_t* bar = reinterpret_cast<uint64_t*>(RsP + RSP);
    double* Cs = base;                                    // diagonal solve: C_i [c * XP + n]
    double* Rs = base + 64 * XP;                          // R_ii [r * XP + c]
    double* rinv = Rs + 64 * XP;                          // [64]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int s = blockIdx.y, n0 = blockIdx.x * 64;
    double* A = At + (int64_t)s * M * nat;
    uint32_t nc, crank;
    asm("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(nc));
    asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    const bool lead = crank == 0;
    const uint16_t mask = (uint16_t)((1u << nc) - 1u);
    // bar[0..1] full (local expect), bar[2..3] empty (this CTA's warps), bar[4..5] cluster empty
    // (the leader's: every warp of every CTA)
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], NT / 32);
        mbar_init(&bar[3], NT / 32);
        mbar_init(&bar[4], (int)(nc * (NT / 32)));
        mbar_init(&bar[5], (int)(nc * (NT / 32)));
        mbar_init(&bar[6], 1);  // R_ii landed
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (nc > 1) trw_cluster_sync();  // barriers initialised cluster-wide before any remote arrive
    const uint32_t cempty0 = trw_mapa(su32(&bar[4]), 0);  // the leader's cluster empty barriers (8 B apart)
    uint32_t gch = 0;  // chunks issued so far (stage = gch & 1, parity = (gch >> 1) & 1)
    const int nbk = (M + 63) / 64;
    for (int i = 0; i < nbk; ++i) {
        const int i0 = 64 * i, bi = min(64, M - i0);
        double acc[4][2][2];  // -C while the updates are added
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    acc[mt][nt][e] = (c < bi && n0 + n < nat) ? -A[(int64_t)(n0 + n) * M + i0 + c] : 0.0;
                }
        if (tid == 0) {  // R_ii behind the block's GEMM (RsP was last read before the previous block ended)
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect(&bar[6], 4 * BOX * 8);
#pragma unroll
            for (int h = 0; h < 4; ++h) tma_load(RsP + h * BOX, &tmR, i0 + 16 * h, i0, s, &bar[6]);
        }
        const int nch = 2 * i;  // k-blocks 0..i-1, two 32-row chunks each
        auto issue = [&](int ch, uint32_t g) {  // thread 0
            double* d = stg + (g & 1) * STAGE;
            const int r0 = 32 * ch;  // row of R11 / neuron index of X
            if (g >= 2) mbar_wait(&bar[2 + (g & 1)], ((g >> 1) - 1) & 1);  // this CTA consumed the stage
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect(&bar[g & 1], 4 * BOX * 8);  // R (multicast or own) + X (own)
            if (nc == 1) {
                tma_load(d, &tmR, r0, i0, s, &bar[g & 1]);
                tma_load(d + BOX, &tmR, r0 + 16, i0, s, &bar[g & 1]);
            } else if (lead) {
                if (g >= 2) trw_mbar_wait_cluster(&bar[4 + (g & 1)], ((g >> 1) - 1) & 1);  // every CTA did
                trw_tma_load_mc(d, &tmR, r0, i0, s, &bar[g & 1], mask);
                trw_tma_load_mc(d + BOX, &tmR, r0 + 16, i0, s, &bar[g & 1], mask);
            }
            tma_load(d + 2 * BOX, &tmA, r0, n0, s, &bar[g & 1]);
            tma_load(d + 3 * BOX, &tmA, r0 + 16, n0, s, &bar[g & 1]);
        };
        if (tid == 0 && nch > 0) issue(0, gch);
        for (int ch = 0; ch < nch; ++ch) {
            const uint32_t g = gch + ch;
            if (tid == 0 && ch + 1 < nch) issue(ch + 1, g + 1);
            mbar_wait(&bar[g & 1], (g >> 1) & 1);
            const double* Vs = stg + (g & 1) * STAGE;
            const double* Xs = Vs + 2 * BOX;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                double af[4], bf[2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = Vs[sw(kk, wm * 32 + mt * 8 + (lane >> 2))];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) bf[nt] = Xs[sw(kk, wn * 16 + nt * 8 + (lane >> 2))];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bar[2 + (g & 1)]);  // stage (g & 1) may be refilled (own X)
                if (nc > 1)                       // ... and, once every CTA is done, by the multicast R
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(
                                     cempty0 + 8u * (g & 1)) : "memory");
            }
        }
        gch += nch;
        __syncthreads();  // every warp is done with the stages: the diagonal solve reuses them
        // diagonal block: R_ii^T X = C
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    Cs[c * XP + n] = -acc[mt][nt][e];
                }
        mbar_wait(&bar[6], i & 1);
        for (int x = tid; x < 64 * 64; x += NT) {
            const int r = x & 63, c = x >> 6;
            Rs[r * XP + c] = (r <= c && c < bi) ? RsP[sw(r, c)] : 0.0;
        }
        __syncthreads();
        if (tid < bi) rinv[tid] = 1.0 / Rs[tid * XP + tid];
        __syncthreads();
        {
            // thread (n = tid >> 2, q = tid & 3) owns rows c = q + 4j of column n
            const int n = tid >> 2, q = tid & 3;
            double xv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) xv[j] = Cs[(q + 4 * j) * XP + n];
#pragma unroll
            for (int m = 0; m < 16; ++m) {
#pragma unroll
                for (int q0 = 0; q0 < 4; ++q0) {
                    const int c = 4 * m + q0;
                    if (q == q0) xv[m] *= rinv[c < bi ? c : 0];
                    const double xc = __shfl_sync(0xffffffffu, xv[m], (lane & ~3) | q0);
#pragma unroll
                    for (int j = m; j < 16; ++j)
                        if (j > m || q > q0) xv[j] = fma(-Rs[c * XP + q + 4 * j], xc, xv[j]);
                }
            }
            if (n0 + n < nat)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (q + 4 * j < bi) A[(int64_t)(n0 + n) * M + i0 + q + 4 * j] = xv[j];
        }
        // X_i is read back through the async proxy (TMA) by the later blocks of this CTA
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __syncthreads();
        // no CTA of the cluster may receive the next block's multicast chunks while another
        // still uses its stages as diagonal-solve scratch
        if (nc > 1) trw_cluster_sync();
    }
    if (nc > 1) trw_cluster_sync();  // no CTA exits while a multicast into it may be in flight
}


// 128 flux rows per CTA (512 threads, 16 warps of 32 x 16): each R11 chunk serves twice the
// columns, halving the R11 traffic of the 64-column version (config 4: 16.9 GB of DRAM reads for
// 4.3 GB of R11, the four CTAs of a subdomain drift apart and miss L2).  One CTA per SM (the
// 16 warps of two 64-column CTAs); per-element arithmetic and order as k_trsm_w (bit-identical).
namespace trw2 {
using namespace elmtma;
constexpr int NT = 512, NCOL = 128;
constexpr int STAGE = 6 * BOX;           // R chunk (2 boxes) + X chunk (2 x 2 boxes)
constexpr int XP = 65, CP = 129;         // padded strides: R_ii [r * XP + c], C_i [c * CP + n]
constexpr int DIAG = 64 * CP + 64 * XP + 64;
constexpr int SMEM_BODY = (2 * STAGE > DIAG ? 2 * STAGE : DIAG);
constexpr int SMEM = SMEM_BODY * 8 + 64 + 1024;
}  // namespace trw2

__global__ void __launch_bounds__(trw2::NT, 1) k_trsm_w2(const __grid_constant__ CUtensorMap tmR,
                                                         const __grid_constant__ CUtensorMap tmA,
                                                         const double* __restrict__ Kaug, int64_t ld, int64_t ncols,
                                                         double* __restrict__ At, int M, int nat) {
    using namespace trw2;
    extern __shared__ uint8_t raw[];
    double* base = reinterpret_cast<double*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
    double* stg = base;                                   // 2 stages x (R 2 boxes | X 4 boxes)
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + SMEM_BODY);
    double* Cs = base;                                    // diagonal solve: C_i [c * CP + n]
    double* Rs = base + 64 * CP;                          // R_ii [r * XP + c]
    double* rinv = Rs + 64 * XP;                          // [64]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;              // 2 x 8 warps of 32 rows x 16 columns
    const int s = blockIdx.y, n0 = blockIdx.x * NCOL;
    const double* R = Kaug + (int64_t)s * ld * ncols;
    double* A = At + (int64_t)s * M * nat;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], NT / 32);  // stage 0 / 1 released by every warp
        mbar_init(&bar[3], NT / 32);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    uint32_t gch = 0;  // chunks issued so far (stage = gch & 1, parity = (gch >> 1) & 1)
    const int nbk = (M + 63) / 64;
    for (int i = 0; i < nbk; ++i) {
        const int i0 = 64 * i, bi = min(64, M - i0);
        double acc[4][2][2];  // -C while the updates are added
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    acc[mt][nt][e] = (c < bi && n0 + n < nat) ? -A[(int64_t)(n0 + n) * M + i0 + c] : 0.0;
                }
        const int nch = 2 * i;  // k-blocks 0..i-1, two 32-row chunks each
        auto issue = [&](int ch, uint32_t g) {  // thread 0
            double* d = stg + (g & 1) * STAGE;
            const int r0 = 32 * ch;  // row of R11 / neuron index of X
            if (g >= 2) mbar_wait(&bar[2 + (g & 1)], ((g >> 1) - 1) & 1);  // previous chunk of the stage consumed
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect(&bar[g & 1], 6 * BOX * 8);
            tma_load(d, &tmR, r0, i0, s, &bar[g & 1]);
            tma_load(d + BOX, &tmR, r0 + 16, i0, s, &bar[g & 1]);
            tma_load(d + 2 * BOX, &tmA, r0, n0, s, &bar[g & 1]);
            tma_load(d + 3 * BOX, &tmA, r0 + 16, n0, s, &bar[g & 1]);
            tma_load(d + 4 * BOX, &tmA, r0, n0 + 64, s, &bar[g & 1]);
            tma_load(d + 5 * BOX, &tmA, r0 + 16, n0 + 64, s, &bar[g & 1]);
        };
        if (tid == 0 && nch > 0) issue(0, gch);
        for (int ch = 0; ch < nch; ++ch) {
            const uint32_t g = gch + ch;
            if (tid == 0 && ch + 1 < nch) issue(ch + 1, g + 1);
            mbar_wait(&bar[g & 1], (g >> 1) & 1);
            const double* Vs = stg + (g & 1) * STAGE;
            const double* Xs = Vs + 2 * BOX + (wn >> 2) * 2 * BOX;  // this warp's 64-column half
            const int wq = wn & 3;                                   // 16-column group in the half
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                double af[4], bf[2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = Vs[sw(kk, wm * 32 + mt * 8 + (lane >> 2))];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) bf[nt] = Xs[sw(kk, wq * 16 + nt * 8 + (lane >> 2))];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[2 + (g & 1)]);  // stage (g & 1) may be refilled
        }
        gch += nch;
        __syncthreads();  // every warp is done with the stages: the diagonal solve reuses them
        // diagonal block: R_ii^T X = C
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    Cs[c * CP + n] = -acc[mt][nt][e];
                }
        for (int x = tid; x < 64 * 64; x += NT) {
            const int r = x & 63, c = x >> 6;
            Rs[r * XP + c] = (r <= c && c < bi) ? R[(int64_t)(i0 + c) * ld + i0 + r] : 0.0;
        }
        __syncthreads();
        if (tid < bi) rinv[tid] = 1.0 / Rs[tid * XP + tid];
        __syncthreads();
        {
            // thread (n = tid >> 2, q = tid & 3) owns rows c = q + 4j of column n
            const int n = tid >> 2, q = tid & 3;
            double xv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) xv[j] = Cs[(q + 4 * j) * CP + n];
#pragma unroll
            for (int m = 0; m < 16; ++m) {
#pragma unroll
                for (int q0 = 0; q0 < 4; ++q0) {
                    const int c = 4 * m + q0;
                    if (q == q0) xv[m] *= rinv[c < bi ? c : 0];
                    const double xc = __shfl_sync(0xffffffffu, xv[m], (lane & ~3) | q0);
#pragma unroll
                    for (int j = m; j < 16; ++j)
                        if (j > m || q > q0) xv[j] = fma(-Rs[c * XP + q + 4 * j], xc, xv[j]);
                }
            }
            if (n0 + n < nat)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (q + 4 * j < bi) A[(int64_t)(n0 + n) * M + i0 + q + 4 * j] = xv[j];
        }
        // X_i is read back through the async proxy (TMA) by the later blocks of this CTA
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        __syncthreads();
    }
}


// Back substitution c = R11^{-1} z for very large M (the lattice's N <= 2 x 2: M = 16384 / 65536)
// with the CTAs of a cooperative launch split per subdomain (nper each): block row ib from the
// bottom, CTA 0 of the subdomain solves the 64 x 64 diagonal block (warp-level substitution as in
// k_bs_trsv), then every CTA updates its slice of z[0:i0] -= R[0:i0, i0:i0+64] c_i.  Two barriers
// per block; r_s = ||z[M:ld]|| by CTA 0 first.  Deterministic.
__device__ __forceinline__ unsigned bs_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bs_barrier(unsigned* cnt, unsigned nper, unsigned& gen) {
    __syncthreads();
    ++gen;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        while (bs_ld_acquire(cnt) < gen * nper) {
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_bs_trsv_grid(const double* __restrict__ Kaug, int64_t ld, int64_t ncols,
                                                      int M, double* __restrict__ z, double* __restrict__ coef,
                                                      double* __restrict__ resid, int nper, unsigned* __restrict__ cnt) {
    __shared__ double Rs[64][65];
    __shared__ double cs[64];
    __shared__ double red[8];
    __shared__ double rdg[64];
    const int sl = blockIdx.x / nper, cta = blockIdx.x % nper;
    const double* A = Kaug + (int64_t)sl * ld * ncols;
    double* zs = z + (int64_t)sl * ld;
    unsigned* C = cnt + sl;
    unsigned gen = 0;
    if (cta == 0) {
        double ss = 0.0;
        for (int64_t r = M + threadIdx.x; r < ld; r += blockDim.x) ss += zs[r] * zs[r];
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < 8; ++w) t += red[w];
            resid[sl] = sqrt(t);
        }
    }
    const int nblk = (M + 63) / 64;
    for (int ib = nblk - 1; ib >= 0; --ib) {
        const int i0 = ib * 64, bi = min(64, M - i0);
        if (cta == 0) {
            __syncthreads();
            for (int t = threadIdx.x; t < bi * bi; t += blockDim.x) {
                int r = t % bi, c = t / bi;
                Rs[r][c] = A[(int64_t)(i0 + c) * ld + i0 + r];
            }
            __syncthreads();
            if (threadIdx.x < bi) rdg[threadIdx.x] = 1.0 / Rs[threadIdx.x][threadIdx.x];
            __syncthreads();
            if (threadIdx.x < 32) {
                const int lane = threadIdx.x;
                double z0 = lane < bi ? zs[i0 + lane] : 0.0;
                double z1 = lane + 32 < bi ? zs[i0 + lane + 32] : 0.0;
                for (int r = bi - 1; r >= 0; --r) {
                    double cr = r >= 32 ? __shfl_sync(0xffffffffu, z1, r - 32) : __shfl_sync(0xffffffffu, z0, r);
                    cr = cr * rdg[r];
                    if (lane < r) z0 -= Rs[lane][r] * cr;
                    if (lane + 32 < r) z1 -= Rs[lane + 32][r] * cr;
                    if (lane == (r & 31)) {
                        if (r >= 32) z1 = cr;
                        else z0 = cr;
                    }
                }
                if (lane < bi) {
                    coef[(int64_t)sl * M + i0 + lane] = z0;
                    zs[i0 + lane] = z0;  // the solved block, read by every CTA after the barrier
                }
                if (lane + 32 < bi) {
                    coef[(int64_t)sl * M + i0 + lane + 32] = z1;
                    zs[i0 + lane + 32] = z1;
                }
            }
        }
        bs_barrier(C, nper, gen);
        if (i0 > 0) {
            if (threadIdx.x < bi) cs[threadIdx.x] = zs[i0 + threadIdx.x];
            __syncthreads();
            // z[0:i0] -= R[0:i0, i0:i0+bi] c_i over the own rows
            const int per = (i0 + nper - 1) / nper, ra = cta * per, rb = min(i0, ra + per);
            for (int r = ra + threadIdx.x; r < rb; r += blockDim.x) {
                double acc = 0.0;
                for (int k = 0; k < bi; ++k) acc += A[(int64_t)(i0 + k) * ld + r] * cs[k];
                zs[r] -= acc;
            }
            bs_barrier(C, nper, gen);
        }
    }
}

// ---- interface, layout 1 (the lattice with cross points, reading R32) ----------------------------
// Face equation blocks: Q_f[r][col] (column-major, ld nrow) for the (q + 2) flux equations of face
// f -- its point equations and the cross-point equations of its endpoints -- over the columns
// [s1's ne local columns | s2's ne | rhs]: each contributor (s, flux row ar) writes its own column
// range (no conflicts), the rhs q_e = P_s1[ar1, ne] + P_s2[ar2, ne] in ascending s.  The buffer is
// zero on entry.  grid F.
__global__ void k_qface(const double* __restrict__ Pbuf, int64_t pstride, int64_t pld, const int* __restrict__ eqsrc,
                        const int* __restrict__ feq, const int* __restrict__ fpair, int nrow, int ldr, int ne,
                        double* __restrict__ Qf, int64_t fstride) {
    const int f = blockIdx.x;
    double* Q = Qf + (int64_t)f * fstride;
    const int s1 = fpair[f * 2];
    for (int x = threadIdx.x; x < nrow * (2 * ne + 1); x += blockDim.x) {
        const int r = x % nrow, col = x / nrow;
        const int eq = feq[f * nrow + r];
        if (eq < 0) continue;
        double v = 0.0;
        if (col < 2 * ne) {
            const int slot = col / ne, t = col - slot * ne;
            for (int cc = 0; cc < 2; ++cc) {
                const int s = eqsrc[eq * 4 + 2 * cc], ar = eqsrc[eq * 4 + 2 * cc + 1];
                if (s >= 0 && (s == s1 ? 0 : 1) == slot) v = Pbuf[(int64_t)s * pstride + ar + (int64_t)t * pld];
            }
        } else {
            for (int cc = 0; cc < 2; ++cc) {
                const int s = eqsrc[eq * 4 + 2 * cc], ar = eqsrc[eq * 4 + 2 * cc + 1];
                if (s >= 0) v += Pbuf[(int64_t)s * pstride + ar + (int64_t)ne * pld];
            }
        }
        Q[r + (int64_t)col * ldr] = v;
    }
}

// symmetric matrices of which only the lower 64-tiles are stored (the batched GEMM's lower_only)
__device__ __forceinline__ double lower_at(const double* __restrict__ A, int64_t r, int64_t c, int64_t ld) {
    return (r >> 6) >= (c >> 6) ? A[r + c * ld] : A[c + r * ld];
}

// M = sum_s scatter(S1_s) + sum_f scatter(G_f) and g = -sum_s scatter(T_E^T t_F) - sum_f scatter(
// Q_f^T q_f) into the dense plan's packed tiles (natural order, every lower tile present).  Element
// (a, b): the S1 entries of the subdomains holding both unknowns (rmap: up to 4 (s, t) per unknown,
// ascending s) plus the Gram entries of every copy pair in the face blocks holding both (flist: up
// to 16 (face, column) per unknown, ascending face); unknowns >= G get a unit diagonal.
constexpr int LAT_FL = 16;
__global__ void k_lat_mfill(const double* __restrict__ Gf, int64_t gstride, int64_t gld, const int* __restrict__ flist,
                            const double* __restrict__ Sbuf, int64_t sstride, int64_t sld, const int* __restrict__ rmap,
                            int64_t G, const int* __restrict__ tile_I, const int* __restrict__ tile_J,
                            double* __restrict__ Mband) {
    const int t = blockIdx.x, I = tile_I[t], J = tile_J[t];
    double* T = Mband + (int64_t)t * ELM_TS;
    for (int x = threadIdx.x; x < ELM_NB * ELM_NB; x += blockDim.x) {
        const int r = x % ELM_NB, cc = x / ELM_NB;
        if (I == J && r < cc) continue;
        const int64_t a = (int64_t)I * ELM_NB + r, b = (int64_t)J * ELM_NB + cc;
        double v;
        if (a >= G || b >= G) {
            v = a == b ? 1.0 : 0.0;
        } else {
            v = 0.0;
            for (int ka = 0; ka < 4; ++ka) {
                const int sa = rmap[a * 8 + 2 * ka];
                if (sa < 0) break;
                for (int kb = 0; kb < 4; ++kb) {
                    const int sb = rmap[b * 8 + 2 * kb];
                    if (sb < 0) break;
                    if (sb == sa)
                        v += lower_at(Sbuf + (int64_t)sa * sstride, rmap[a * 8 + 2 * ka + 1], rmap[b * 8 + 2 * kb + 1], sld);
                }
            }
            const int* la = flist + a * LAT_FL * 2;
            const int* lb = flist + b * LAT_FL * 2;
            for (int ka = 0; ka < LAT_FL && la[2 * ka] >= 0; ++ka)
                for (int kb = 0; kb < LAT_FL && lb[2 * kb] >= 0; ++kb)
                    if (la[2 * ka] == lb[2 * kb])
                        v += lower_at(Gf + (int64_t)la[2 * ka] * gstride, la[2 * ka + 1], lb[2 * kb + 1], gld);
        }
        T[r + (int64_t)cc * ELM_TLD] = v;
    }
}

__global__ void k_lat_g(const double* __restrict__ Gf, int64_t gstride, int64_t gld, const int* __restrict__ flist,
                        const double* __restrict__ Sbuf, int64_t sstride, int64_t sld, const int* __restrict__ rmap,
                        int ne, int64_t G, int64_t G_pad, double* __restrict__ g) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= G_pad) return;
    if (a >= G) {
        g[a] = 0.0;
        return;
    }
    double v = 0.0;
    for (int k = 0; k < 4; ++k) {
        const int s = rmap[a * 8 + 2 * k];
        if (s < 0) break;
        v -= lower_at(Sbuf + (int64_t)s * sstride, rmap[a * 8 + 2 * k + 1], ne, sld);
    }
    const int* la = flist + a * LAT_FL * 2;
    for (int k = 0; k < LAT_FL && la[2 * k] >= 0; ++k)
        v -= lower_at(Gf + (int64_t)la[2 * k] * gstride, la[2 * k + 1], 2 * ne, gld);
    g[a] = v;
}

}  // namespace

cudaError_t run_interface_assemble_lattice(const elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband,
                                           double* g, double* work, cudaStream_t st) {
    const int64_t G = c->sz.G, F = c->faces, kaug = c->sz.kaug, ne = c->sz.ne, nrow = c->lat_nrow;
    const int64_t pstride = c->sz.pbuf_ld * kaug, sstride = c->sz.sbuf_ld * kaug;
    // (leading dimensions even: the GEMM stages 16-byte pairs of doubles)
    const int64_t ldr = (nrow + 3) / 4 * 4, ncol = 2 * ne + 1, fstride = ldr * ncol, gld = (ncol + 2) / 2 * 2,
                  gstride = gld * ncol;
    double* Qf = work;                // [F][ncol][nrow]
    double* Gf = Qf + F * fstride;    // [F][ncol][gld], lower tiles
    cudaError_t e;
    if (G <= 0) return cudaSuccess;
    if ((e = cudaMemsetAsync(Qf, 0, sizeof(double) * F * fstride, st)) != cudaSuccess) return e;
    {
        KTimer kt(c, ELMDDM_K_IFACE, st);
        k_qface<<<(unsigned)F, 256, 0, st>>>(Pbuf, pstride, c->sz.pbuf_ld, c->d_eqsrc, c->d_feq, c->d_fpair, (int)nrow,
                                             (int)ldr, (int)ne, Qf, fstride);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // G_f = Q_f^T Q_f (symmetric: lower 64-tiles only)
    GemmArgs gq{(int)ncol, (int)ncol, (int)nrow, Qf, ldr, fstride, Qf, ldr, fstride, Gf, gld, gstride, 1.0, 0.0, (int)F, 1};
    if ((e = gemm_launch(true, false, gq, st, c, ELMDDM_K_IFACE)) != cudaSuccess) return e;
    KTimer kt(c, ELMDDM_K_IFACE, st);
    k_lat_mfill<<<(unsigned)c->plan.ntiles, 256, 0, st>>>(Gf, gstride, gld, c->d_flist, Sbuf, sstride, c->sz.sbuf_ld,
                                                          c->d_rmap, G, c->d_tile_I, c->d_tile_J, Mband);
    k_lat_g<<<(unsigned)((c->sz.G_pad + 255) / 256), 256, 0, st>>>(Gf, gstride, gld, c->d_flist, Sbuf, sstride,
                                                                   c->sz.sbuf_ld, c->d_rmap, (int)ne, G, c->sz.G_pad, g);
    return cudaGetLastError();
}

// The F column of P_s = W_s [R12 | y] and the F row of S_s = [T_E | t_F]^T [T_E | t_F]
// (kaug = ne + 1: left to the 64-tiled GEMMs, the lone F column costs a whole tile row / column of
// CTAs, 20-33% of their work): per subdomain, warp-level dot products in a fixed order.
//   P[i, F] = sum_k W_s^T[k, i] y[k]          i < na      (W_s^T = At[s], [k + i M])
//   S[F, j] = sum_r T[r, j] t_F[r]            j <= F      (T = rows M.. of columns M.. of K_aug)
namespace {
__global__ void __launch_bounds__(256) k_fcol(const double* __restrict__ Kaug, int64_t ld, int64_t ncols, int M,
                                              int kaug, int Kt, const double* __restrict__ At, int nat,
                                              double* __restrict__ P, int64_t pld, int64_t pstride,
                                              double* __restrict__ Sg, int64_t sld, int64_t sstride) {
    const int64_t s = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int F = kaug - 1;
    const double* K = Kaug + s * ld * ncols;
    const double* y = K + (int64_t)(M + F) * ld;      // rows [0, M) of column M + F
    const double* tF = y + M;                        // rows [M, M + Kt)
    const double* W = At + s * (int64_t)M * nat;
    // (four independent partial sums per lane: four loads in flight per lane, fixed order)
    for (int i = w; i < nat; i += 8) {
        const double* wi = W + (int64_t)i * M;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int k = lane;
        for (; k + 96 < M; k += 128) {
            v0 += wi[k] * y[k];
            v1 += wi[k + 32] * y[k + 32];
            v2 += wi[k + 64] * y[k + 64];
            v3 += wi[k + 96] * y[k + 96];
        }
        for (; k < M; k += 32) v0 += wi[k] * y[k];
        double v = (v0 + v1) + (v2 + v3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) P[s * pstride + i + (int64_t)F * pld] = v;
    }
    for (int j = w; j <= F; j += 8) {
        const double* tj = K + M + (int64_t)(M + j) * ld;
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int r = lane;
        for (; r + 96 < Kt; r += 128) {
            v0 += tj[r] * tF[r];
            v1 += tj[r + 32] * tF[r + 32];
            v2 += tj[r + 64] * tF[r + 64];
            v3 += tj[r + 96] * tF[r + 96];
        }
        for (; r < Kt; r += 32) v0 += tj[r] * tF[r];
        double v = (v0 + v1) + (v2 + v3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {  // (both triangles: the consumers read diagonal 64-tiles in full)
            Sg[s * sstride + F + (int64_t)j * sld] = v;
            Sg[s * sstride + j + (int64_t)F * sld] = v;
        }
    }
}
}  // namespace

cudaError_t run_schur_accumulate(const elmddm_ctx* c, double* Kaug, double* At, double* Pbuf, double* Sbuf,
                                 double* work, cudaStream_t st) {
    (void)work;
    const int64_t S = c->sz.S, ld = c->sz.ld, ncols = c->sz.ncols, kaug = c->sz.kaug;
    const int M = c->cfg.M, nat = (int)c->sz.na;  // flux rows (4q, or 4q + 8 on the lattice)
    cudaError_t e;
    // S_s = [T_E | t_F]^T [T_E | t_F] does not depend on the TRSM: it runs on a side stream beside
    // it and fills the TRSM's last partial wave (serialised when per-class timing is on)
    const int Kt = (int)(ld - M);
    const int64_t s0 = c->cfg.s_begin;
    const int64_t pstride = c->sz.pbuf_ld * kaug, sstride = c->sz.sbuf_ld * kaug;
    const int ke = (int)kaug - 1;  // the 64-tiled GEMMs cover the E columns; k_fcol the F column / row
    GemmArgs gs{ke, ke, Kt, Kaug + M + (int64_t)M * ld, ld, ld * ncols, Kaug + M + (int64_t)M * ld, ld,
                ld * ncols, Sbuf + s0 * sstride, c->sz.sbuf_ld, sstride, 1.0, 0.0, (int)S, 1 /* lower tiles only */};
    const bool side = !c->timing && c->schur_side;
    cudaStream_t sst = st;
    if (side) {
        if ((e = c->ensure_streams(1)) != cudaSuccess) return e;
        sst = c->gstreams[0];
        cudaEventRecord(c->ev_fork, st);
        cudaStreamWaitEvent(sst, c->ev_fork, 0);
        if ((e = gemm_launch(true, false, gs, sst, c, ELMDDM_K_GEMM_SCHUR)) != cudaSuccess) return e;
    }
    // W_s^T = R11^{-T} A^T: one fused left-looking TRSM launch (in place on At)
    {
        CUtensorMap tmR, tmA;
        if (!elm_encode_tmap(&tmR, Kaug, ld, ncols, S, ld * ncols) || !elm_encode_tmap(&tmA, At, M, nat, S, (int64_t)M * nat))
            return cudaErrorInvalidValue;
        // (a per-device attribute: set on every call, a few microseconds of host time)
        if ((e = cudaFuncSetAttribute(k_trsm_w, cudaFuncAttributeMaxDynamicSharedMemorySize, trw::SMEM)) != cudaSuccess)
            return e;
        dim3 g((nat + 63) / 64, (unsigned)S);
        // the flux-row tiles of a subdomain form one cluster (R11 chunks multicast), up to 8
        const int ncl = (c->trsm_cluster && g.x >= 2 && g.x <= 8) ? (int)g.x : 1;
        KTimer kt(c, ELMDDM_K_TRSM, st);
        if (ncl == 1 && c->trsm_wide && nat > 64) {  // 128 flux rows per CTA
            if ((e = cudaFuncSetAttribute(k_trsm_w2, cudaFuncAttributeMaxDynamicSharedMemorySize, trw2::SMEM)) !=
                cudaSuccess)
                return e;
            dim3 g2((nat + 127) / 128, (unsigned)S);
            k_trsm_w2<<<g2, trw2::NT, trw2::SMEM, st>>>(tmR, tmA, Kaug, ld, ncols, At, M, nat);
        } else if (ncl > 1) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = g;
            cfg.blockDim = dim3(trw::NT);
            cfg.dynamicSmemBytes = trw::SMEM;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)ncl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if ((e = cudaLaunchKernelEx(&cfg, k_trsm_w, tmR, tmA, (const double*)Kaug, (int64_t)ld, (int64_t)ncols, At, M,
                                        nat)) != cudaSuccess)
                return e;
        } else {
            k_trsm_w<<<g, trw::NT, trw::SMEM, st>>>(tmR, tmA, Kaug, ld, ncols, At, M, nat);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // P_s = W_s [R12 | y]   (na x kaug)
    GemmArgs gp{nat, ke, M, At, M, (int64_t)M * nat, Kaug + (int64_t)M * ld, ld, ld * ncols,
                Pbuf + s0 * pstride, c->sz.pbuf_ld, pstride, 1.0, 0.0, (int)S, 0};
    if ((e = gemm_launch(true, false, gp, st, c, ELMDDM_K_GEMM_SCHUR)) != cudaSuccess) return e;
    {
        KTimer kt(c, ELMDDM_K_GEMM_SCHUR, st);
        k_fcol<<<(unsigned)S, 256, 0, st>>>(Kaug, ld, ncols, M, (int)kaug, Kt, At, nat, Pbuf + s0 * pstride,
                                             c->sz.pbuf_ld, pstride, Sbuf + s0 * sstride, c->sz.sbuf_ld, sstride);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (side) {
        cudaEventRecord(c->ev_join[0], sst);
        return cudaStreamWaitEvent(st, c->ev_join[0], 0);
    }
    return gemm_launch(true, false, gs, st, c, ELMDDM_K_GEMM_SCHUR);
}

cudaError_t run_interface_assemble(const elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband,
                                   double* g, double* work, cudaStream_t st) {
    if (c->cfg.layout == 1) return run_interface_assemble_lattice(c, Pbuf, Sbuf, Mband, g, work, st);
    const int q = c->cfg.q;
    const int64_t F = c->faces, kaug = c->sz.kaug;
    const int64_t pstride = c->sz.pbuf_ld * kaug, sstride = c->sz.sbuf_ld * kaug;
    const int64_t qstride = (int64_t)c->qrow_ld * c->qrow_cols;
    const int64_t gstride = (int64_t)c->ga_ld * c->qrow_cols;
    double* Qrow = work;
    double* Ga = Qrow + F * qstride;
    cudaError_t e;
    if ((e = cudaMemsetAsync(Mband, 0, sizeof(double) * c->sz.band_elems, st)) != cudaSuccess) return e;
    if (F > 0) {
        { KTimer kt(c, ELMDDM_K_IFACE, st);
        k_qrow<<<dim3((unsigned)F, 8), 256, 0, st>>>(Pbuf, pstride, c->sz.pbuf_ld, c->d_qsrc, q, Qrow, c->qrow_ld,
                                                      qstride); }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        // Ga[a] = Qrow[a]^T Qrow[a]  (symmetric: lower 64-tiles only, read through ga_at)
        GemmArgs gg{c->qrow_cols, c->qrow_cols, q, Qrow, c->qrow_ld, qstride, Qrow, c->qrow_ld, qstride, Ga, c->ga_ld,
                    gstride, 1.0, 0.0, (int)F, 1};
        if ((e = gemm_launch(true, false, gg, st, c, ELMDDM_K_IFACE)) != cudaSuccess) return e;
        { KTimer kt(c, ELMDDM_K_IFACE, st);
        k_massemble<<<(unsigned)c->npairs, 256, 0, st>>>(c->d_pair_ptr, c->d_pair_bc, c->d_terms, Sbuf, sstride,
                                                          c->sz.sbuf_ld, Ga, gstride, c->ga_ld, q, Mband,
                                                          c->d_fbase, c->d_tile_map, c->plan.nblk); }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        { KTimer kt(c, ELMDDM_K_IFACE, st);
        k_gassemble<<<(unsigned)F, 128, 0, st>>>(c->d_gterm_ptr, c->d_gterms, Sbuf, sstride, c->sz.sbuf_ld, Ga,
                                                  gstride, c->ga_ld, q, g); }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    const int64_t npad = std::max<int64_t>((int64_t)c->plan.pad.size(), c->sz.G_pad - c->sz.G);
    if (npad > 0) {
        KTimer kt(c, ELMDDM_K_IFACE, st);
        k_pad<<<(unsigned)((npad + 127) / 128), 128, 0, st>>>(Mband, c->d_pad, (int)c->plan.pad.size(), c->d_diag_tid, g,
                                                              c->sz.G, c->sz.G_pad);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t run_back_solve(const elmddm_ctx* c, const double* Kaug, const double* uG, double* coef, double* resid,
                           double* work, cudaStream_t st) {
    const int64_t S = c->sz.S, ld = c->sz.ld, ncols = c->sz.ncols;
    double* z = work;
    dim3 g1((unsigned)((ld + 255) / 256), (unsigned)S);
    { KTimer kt(c, ELMDDM_K_BACK, st);
    k_bs_gemv<<<g1, 256, sizeof(double) * c->sz.kaug, st>>>(c->cfg, Kaug, ld, ncols, c->d_umap, (int)c->sz.ne, uG,
                                                            z); }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    KTimer kt(c, ELMDDM_K_BACK, st);
    const int M = c->cfg.M;
    static const bool force_grid = [] {
        const char* env = getenv("ELMDDM_BS_GRID");
        return env && atoi(env) != 0;
    }();
    if ((M >= 8192 || force_grid) && S <= 64) {  // very large networks, few subdomains: all SMs' CTAs
        const int nper = (int)std::max<int64_t>(1, (2LL * c->nsm) / S);
        unsigned* cnt = reinterpret_cast<unsigned*>(z + S * ld);
        if ((e = cudaMemsetAsync(cnt, 0, sizeof(unsigned) * S, st)) != cudaSuccess) return e;
        int64_t ld_v = ld, nc_v = ncols;
        int M_v = M, per_v = nper;
        void* args[] = {(void*)&Kaug, (void*)&ld_v, (void*)&nc_v, (void*)&M_v, (void*)&z, (void*)&coef, (void*)&resid,
                        (void*)&per_v, (void*)&cnt};
        return cudaLaunchCooperativeKernel((void*)k_bs_trsv_grid, dim3((unsigned)(nper * S)), dim3(256), args, 0, st);
    }
    // all subdomains resident at 1024 threads (2 CTAs / SM): more loads in flight per subdomain
    // (config 3: 1.12 -> 0.83 ms); more subdomains than that: 512 threads, 4 CTAs / SM (config 4)
    const int nt = S <= 2 * (int64_t)c->nsm ? BS_NT : BS_NT / 2;
    k_bs_trsv<<<(unsigned)S, nt, 0, st>>>(Kaug, ld, ncols, M, z, coef, resid);
    return cudaGetLastError();
}
