// qr.cu -- batched blocked Householder QR of every K_aug[s] = [K^s | E_Gamma | F^s] (no pivoting).
//
// Blocking:
//   * panels of NB = 64 columns; inside a panel, base blocks of BB = 8 columns are factored
//     left-looking by ONE CTA per subdomain with the (ld - j0) x 8 block resident in shared
//     memory: previous reflectors of the panel are applied (W = Vp^T C, Z = T^T W, C -= Vp Z),
//     the 8 columns are factored with one deterministic block reduction per column (warp
//     shuffles + shared memory), the explicit V and the growing compact-WY factor T are written;
//   * after each panel, the trailing matrix (all remaining columns, including E_Gamma and F) is
//     updated with three batched DMMA GEMMs: W = V^T C, Z = T^T W, C <- C - V Z.
// Householder convention (reading R20): alpha = -sign(x0)||x|| (sign(0) = +1), v0 = 1,
// tau = (alpha - x0)/alpha, ||x|| = 0 -> tau = 0.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "tma.cuh"
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <vector>
#include <cstdio>

namespace {

constexpr int PNT = 512;           // threads of the panel-block kernel
constexpr int PNW = PNT / 32;      // warps

struct PanelArgs {
    double* Kaug;
    int64_t ld, ncols;
    double* tau;
    int M;
    double* Vbuf;  // [S][NB][ld]  explicit V of the current panel (absolute rows)
    double* Tbuf;  // [S][NB][NB]  compact-WY T of the current panel (column-major)
    int j0;        // panel start column
    int blk;       // base block index inside the panel
    int s_off;     // first local subdomain of this launch (subdomain groups on separate streams)
    int ring;      // doubles of the V_prev ring (k_panel_block)
    int tcols;     // k_panel_t: TMEM columns to allocate (0: 512; 256 lets two panel CTAs share an SM)
};

// block-wide deterministic sum of NV values per thread; result broadcast in tot[0..NV)
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* red, double* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) red[warp * NV + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < PNW; ++w) s += red[w * NV + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ void dmma8(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

constexpr int RED_ELEMS = 2 * 56 * 36; // minimum V_prev ring (also T staging / reduction scratch)
constexpr int VNS = 4;                  // ring stages (VNS - 1 chunks in flight)

// rows per staged chunk of V_prev for kp columns in a ring stage of sst doubles: as many 16-row
// groups as fit with the padded stride rch + 4 (== 4 mod 16: conflict-free fragments).  The ring
// takes whatever shared memory the resident block leaves (PanelArgs::ring), so late panels
// (short blocks) stream V_prev in large chunks with VNS - 1 of them in flight.
__device__ __forceinline__ int vp_rows(int kp, int sst) {
    const int r = ((sst / kp - 4) / 16) * 16;
    return r < 16 ? 16 : r;
}

// stage rows [c*rch, c*rch + nr) of V_prev columns [0, kp) into dst[col*(rch+4) + row] (16 B cp.async)
__device__ __forceinline__ void vp_chunk(double* dst, const double* __restrict__ Vp, int64_t ld, int kp, int rch,
                                         int c, int nr) {
    const int rcp = rch + 4, n = kp * (nr / 2);
    for (int t = threadIdx.x; t < n; t += PNT) {
        const int col = t / (nr / 2), r = (t % (nr / 2)) * 2;
        unsigned d = (unsigned)__cvta_generic_to_shared(dst + col * rcp + r);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(Vp + (int64_t)col * ld + c * rch + r));
    }
}

// Stream rows [0, R) of V_prev (kp columns) through the VNS-stage ring; consume(st, c, rch, nr)
// is called by every thread for each chunk once it is resident (stage layout st[col*(rch+4)+row]).
// One __syncthreads per chunk: it publishes chunk c and frees the stage chunk c + VNS - 1 refills.
template <class F>
__device__ __forceinline__ void vp_stream(const double* __restrict__ Vp, int64_t ld, int R, int kp, double* ring,
                                          int sst, F&& consume) {
    const int rch = vp_rows(kp, sst);
    const int nch = (R + rch - 1) / rch;
#pragma unroll
    for (int i = 0; i < VNS - 1; ++i) {
        if (i < nch) vp_chunk(ring + i * sst, Vp, ld, kp, rch, i, min(rch, R - i * rch));
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(VNS - 2));
        __syncthreads();
        const int cn = c + VNS - 1;
        if (cn < nch) vp_chunk(ring + (cn % VNS) * sst, Vp, ld, kp, rch, cn, min(rch, R - cn * rch));
        asm volatile("cp.async.commit_group;\n" ::);
        consume(ring + (c % VNS) * sst, c, rch, min(rch, R - c * rch));
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
}

// G (kp x 8, column-major ld kp) = Vp^T X on the FP64 tensor pipe, V_prev streamed through the
// ring.  Warp w owns m-tile w/2 (8 columns of V_prev) and the k-steps of parity w%2 in every
// chunk; the two parities are summed at the end (fixed order).
__device__ void vt_block(const double* __restrict__ Vp, int64_t ld, int R, int kp, const double* X, int RP, double* G,
                         double* ring, int sst, double* pairbuf) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mtiles = kp >> 3, t = warp >> 1, par = warp & 1;
    const int kr = lane & 3, cn = lane >> 2;
    double a0 = 0.0, a1 = 0.0;
    vp_stream(Vp, ld, R, kp, ring, sst, [&](const double* st, int c, int rch, int nr) {
        const int rcp = rch + 4, nq = nr / 8;
        if (t < mtiles) {
#pragma unroll 4
            for (int q = 0; q < nq; ++q) {
                const int kk = (2 * q + par) * 4 + kr;  // row inside the chunk
                dmma8(a0, a1, st[(t * 8 + cn) * rcp + kk], X[cn * RP + c * rch + kk]);
            }
        }
    });
    if (t < mtiles && par == 1) {
        pairbuf[t * 64 + lane * 2] = a0;
        pairbuf[t * 64 + lane * 2 + 1] = a1;
    }
    __syncthreads();
    if (t < mtiles && par == 0) {
        a0 += pairbuf[t * 64 + lane * 2];
        a1 += pairbuf[t * 64 + lane * 2 + 1];
        // fragment: row i = t*8 + lane/4 (V column), col c = 2*(lane%4) + e
        G[(2 * kr) * kp + t * 8 + cn] = a0;
        G[(2 * kr + 1) * kp + t * 8 + cn] = a1;
    }
}

__global__ void __launch_bounds__(PNT, 1) k_panel_block(PanelArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int sl = a.s_off + blockIdx.x;
    const int64_t ld = a.ld;
    const int j0 = a.j0, jb = j0 + ELM_BB * a.blk, kp = ELM_BB * a.blk;
    const int R = (int)(ld - j0);     // rows held: [j0, ld)  (multiple of 32)
    const int RP = R + 4;             // padded column stride (conflict-free DMMA fragments)
    const int d0 = jb - j0;           // local row of the block's first diagonal entry
    double* Cb = sm;                  // [8][RP]
    double* Wsm = Cb + 8 * RP;        // [8][kp]  (<= 8*56)
    double* Zsm = Wsm + 8 * 56;       // [8][kp]
    double* red = Zsm + 8 * 56;       // a.ring doubles: V_prev ring / T staging / reduction scratch
    double* tot = red + a.ring;       // [40]
    const int sst = (a.ring / VNS) & ~1;
    double* Tbb = tot + 40;           // [8][8]
    double* taus = Tbb + 64;          // [8]

    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    const double* Vp = V + j0;        // column c of Vp at Vp + c*ld, rows relative to j0
#ifdef ELM_PANEL_PROF
    long long pst[12];
    pst[0] = clock64();
#define PSTAMP(k) pst[k] = clock64()
#else
#define PSTAMP(k)
#endif

    // load the block: rows [j0, ld) of columns [jb, jb+8)
    for (int c = 0; c < 8; ++c) {
        const double* src = A + (int64_t)(jb + c) * ld + j0;
        for (int r2 = threadIdx.x; r2 < R / 2; r2 += PNT) {
            unsigned d = (unsigned)__cvta_generic_to_shared(Cb + c * RP + 2 * r2);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * r2));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    PSTAMP(1);

    if (kp > 0) {
        // W = Vp^T Cb
        vt_block(Vp, ld, R, kp, Cb, RP, Wsm, red, sst, Zsm);
        __syncthreads();
        PSTAMP(2);
        // T (kp x kp, upper) -> smem (reuse the reduction scratch), Z = T^T W
        double* Ts = red;
        for (int t = threadIdx.x; t < kp * kp; t += PNT) {
            int r = t % kp, c = t / kp;
            Ts[c * kp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int cp = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = 0; k <= cp; ++k) s += Ts[cp * kp + k] * Wsm[c * kp + k];
            Zsm[c * kp + cp] = s;
        }
        __syncthreads();
        PSTAMP(3);
        // Cb -= Vp Z on the FP64 tensor pipe: M = R rows (8-row tiles over the 16 warps),
        // N = 8 columns, K = kp; the B fragments (Z) are held in registers.
        {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            const int kr = lane & 3, rn = lane >> 2;
            const int ksteps = kp >> 2;
            double zb[14];
#pragma unroll
            for (int t = 0; t < 14; ++t) zb[t] = t < ksteps ? -Zsm[rn * kp + t * 4 + kr] : 0.0;
            // V_prev streamed through the ring; the 8-row m-tiles of a chunk are dealt to the warps
            vp_stream(Vp, ld, R, kp, red, sst, [&](const double* st, int c, int rch, int nr) {
                const int rcp = rch + 4, nmt = nr / 8;
                for (int mt = warp; mt < nmt; mt += PNW) {
                    const int r0 = c * rch + mt * 8;
                    double c0 = Cb[(2 * kr) * RP + r0 + rn], c1 = Cb[(2 * kr + 1) * RP + r0 + rn];
#pragma unroll
                    for (int t = 0; t < 14; ++t)
                        if (t < ksteps) dmma8(c0, c1, st[(t * 4 + kr) * rcp + mt * 8 + rn], zb[t]);
                    Cb[(2 * kr) * RP + r0 + rn] = c0;
                    Cb[(2 * kr + 1) * RP + r0 + rn] = c1;
                }
            });
        }
        __syncthreads();
        PSTAMP(4);
    }

    // factor the 8 columns: one block reduction per column
    for (int c = 0; c < 8; ++c) {
        const int d = d0 + c;
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.0;
        for (int r = d + 1 + threadIdx.x; r < R; r += PNT) {
            double x = Cb[c * RP + r];
            v[0] += x * x;
#pragma unroll
            for (int c2 = 1; c2 < 8; ++c2)
                if (c + c2 < 8) v[c2] += x * Cb[(c + c2) * RP + r];
        }
        block_sum<8>(v, red, tot);
        const double x0 = Cb[c * RP + d];
        const double nrm = sqrt(x0 * x0 + tot[0]);
        double alpha = x0, tau = 0.0, scale = 0.0;
        if (nrm != 0.0) {
            alpha = x0 >= 0.0 ? -nrm : nrm;
            scale = 1.0 / (x0 - alpha);
            tau = (alpha - x0) / alpha;
        }
        double w[8], yd[8];
#pragma unroll
        for (int c2 = 1; c2 < 8; ++c2) {
            yd[c2] = (c + c2 < 8) ? Cb[(c + c2) * RP + d] : 0.0;
            w[c2] = tau * (yd[c2] + scale * tot[c2]);
        }
        __syncthreads();  // row d read by everyone before it is rewritten
        if (tau != 0.0) {
            for (int r = d + 1 + threadIdx.x; r < R; r += PNT) {
                const double x = Cb[c * RP + r];
                const double vs = scale * x;
#pragma unroll
                for (int c2 = 1; c2 < 8; ++c2)
                    if (c + c2 < 8) Cb[(c + c2) * RP + r] -= w[c2] * vs;
                Cb[c * RP + r] = vs;
            }
        }
        if (threadIdx.x == 0) {
#pragma unroll
            for (int c2 = 1; c2 < 8; ++c2)
                if (c + c2 < 8) Cb[(c + c2) * RP + d] = yd[c2] - w[c2];
            Cb[c * RP + d] = alpha;
            taus[c] = tau;
        }
        __syncthreads();
        PSTAMP(5);
    }

    // write back R (upper) + V (below the diagonal) and tau
    for (int c = 0; c < 8; ++c) {
        double2* dst = reinterpret_cast<double2*>(A + (int64_t)(jb + c) * ld + j0);
        for (int r2 = threadIdx.x; r2 < R / 2; r2 += PNT) dst[r2] = make_double2(Cb[c * RP + 2 * r2], Cb[c * RP + 2 * r2 + 1]);
    }
    if (threadIdx.x < 8) a.tau[(int64_t)sl * a.M + jb + threadIdx.x] = taus[threadIdx.x];
    __syncthreads();
    PSTAMP(6);
    // explicit V of the block (zeros above, unit diagonal) -> smem and Vbuf
    for (int c = 0; c < 8; ++c) {
        const int d = d0 + c;
        double2* dst = reinterpret_cast<double2*>(V + (int64_t)(kp + c) * ld + j0);
        for (int r2 = threadIdx.x; r2 < R / 2; r2 += PNT) {
            double v2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int r = 2 * r2 + e;
                v2[e] = r < d ? 0.0 : (r == d ? 1.0 : Cb[c * RP + r]);
                Cb[c * RP + r] = v2[e];
            }
            dst[r2] = make_double2(v2[0], v2[1]);
        }
    }
    __syncthreads();
    PSTAMP(7);

    // T of the block: Tbb[i][i] = tau_i, Tbb[0:i, i] = -tau_i Tbb[0:i,0:i] (Vb^T v_i)[0:i]
    {
        double g[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) g[k] = 0.0;
        for (int r = d0 + threadIdx.x; r < R; r += PNT) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = Cb[c * RP + r];
            int k = 0;
#pragma unroll
            for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
                for (int c2 = c1 + 1; c2 < 8; ++c2) g[k++] += x[c1] * x[c2];
        }
        block_sum<28>(g, red, tot);
        if (threadIdx.x < 32) {
            // Tbb column i: Tbb[r][i] = -tau_i sum_{k=r}^{i-1} Tbb[r][k] G8[k][i]; lane r owns row r
            const int r = threadIdx.x & 7;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) {
                            const int gi = (k * (15 - k)) / 2 + (i - k - 1);  // packed index of G8[k][i]
                            s += trow[k] * tot[gi];
                        }
                    trow[i] = -taus[i] * s;
                }
            }
            if (threadIdx.x < 8)
#pragma unroll
                for (int i = 0; i < 8; ++i) Tbb[i * 8 + r] = trow[i];
        }
        __syncthreads();
        PSTAMP(8);
    }
    // T[0:kp+8, kp:kp+8]
    if (kp > 0) {
        vt_block(Vp, ld, R, kp, Cb, RP, Wsm, red, sst, Zsm);  // Gx = Vp^T Vb   (kp x 8)
        __syncthreads();
        PSTAMP(9);
        // Y = Gx Tbb (kp x 8)
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int r = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = 0; k <= c; ++k) s += Wsm[k * kp + r] * Tbb[c * 8 + k];
            Zsm[c * kp + r] = s;
        }
        __syncthreads();
        // T[0:kp, kp+c] = -T[0:kp,0:kp] Y   (T staged in smem)
        double* Ts = red;
        for (int t = threadIdx.x; t < kp * kp; t += PNT) {
            int r = t % kp, c = t / kp;
            Ts[c * kp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int r = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = r; k < kp; ++k) s += Ts[k * kp + r] * Zsm[c * kp + k];
            Wsm[c * kp + r] = -s;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int r = t % kp, c = t / kp;
            T[(kp + c) * ELM_NB + r] = Wsm[c * kp + r];
        }
    }
    for (int t = threadIdx.x; t < 64; t += PNT) {
        int r = t % 8, c = t / 8;
        T[(kp + c) * ELM_NB + kp + r] = Tbb[c * 8 + r];
    }
    {
        int c = threadIdx.x / ELM_NB, r = threadIdx.x % ELM_NB;  // 512 threads = 8 columns x 64 rows
        if (r >= kp + 8) T[(kp + c) * ELM_NB + r] = 0.0;
    }
#ifdef ELM_PANEL_PROF
    pst[10] = clock64();
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 200) && (a.blk == 4) && (a.j0 == 256 || a.j0 == 1024))
        printf("PANELPROF j0=%d blk=%d cta=%d load %lld vt1 %lld z %lld upd %lld fact %lld wb %lld vexp %lld tbb %lld vt2 %lld text %lld\n",
               a.j0, a.blk, blockIdx.x, pst[1] - pst[0], pst[2] - pst[1], pst[3] - pst[2], pst[4] - pst[3], pst[5] - pst[4],
               pst[6] - pst[5], pst[7] - pst[6], pst[8] - pst[7], pst[9] - pst[8], pst[10] - pst[9]);
#endif
}

// ------------------------------------------------------------------------------------------
// One launch per panel (k_panel_block's arithmetic, restructured): the CTA of a subdomain walks
// the panel's 8-column blocks left-looking with the block resident in shared memory.  The
// Gram product V_prev^T V_{b-1} that extends T by block b-1 is taken in the SAME streaming pass
// as block b's W = V_prev^T C_b (V_{b-1} is the last 8 columns of every staged chunk), so each
// block streams V_prev twice (W, then C -= V_prev Z) instead of three times; only the last block
// of the panel needs its own Gram pass.  The column factorisation owns rows by thread (rows t,
// t + 512, ...), reduces the 8 sums of a column with 9 shuffles, and needs one barrier per column.
// ------------------------------------------------------------------------------------------
constexpr int PANELP_FIXED = 3 * 8 * 56 + 2 * PNW * 8 + 40 + 64 + 8 + 64;  // Wsm, Zsm, Gp, red x2, tot, Tbb, taus, rowfix

// T[0:kpp, kpp:kpp+8] = -T[0:kpp,0:kpp] (G Tbb), G = V[:, 0:kpp]^T V_b (kpp x 8, G[c*kpp + r]),
// Tbb = T of the block (Tbb[c*8 + r]).  Ts, Ys: shared scratch.  Ends with a barrier.
__device__ void t_extend(double* T, int kpp, const double* G, const double* Tbb, double* Ts, double* Ys) {
    for (int t = threadIdx.x; t < kpp * 8; t += PNT) {
        const int r = t % kpp, c = t / kpp;
        double s = 0.0;
        for (int k = 0; k <= c; ++k) s += G[k * kpp + r] * Tbb[c * 8 + k];
        Ys[c * kpp + r] = s;
    }
    for (int t = threadIdx.x; t < kpp * kpp; t += PNT) {
        const int r = t % kpp, c = t / kpp;
        Ts[c * kpp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kpp * 8; t += PNT) {
        const int r = t % kpp, c = t / kpp;
        double s = 0.0;
        for (int k = r; k < kpp; ++k) s += Ts[k * kpp + r] * Ys[c * kpp + k];
        T[(kpp + c) * ELM_NB + r] = -s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(PNT, 1) k_panel_p(PanelArgs a, int nb) {
    extern __shared__ __align__(16) double sm[];
    const int sl = a.s_off + blockIdx.x;
    const int64_t ld = a.ld;
    const int j0 = a.j0;
    const int R = (int)(ld - j0);
    const int RP = R + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* Cb = sm;                  // [8][RP]
    double* Wsm = Cb + 8 * RP;        // [8][kp]
    double* Zsm = Wsm + 8 * 56;       // [8][kp]
    double* Gp = Zsm + 8 * 56;        // [8][kp-8]
    double* red = Gp + 8 * 56;        // [2][PNW][8] column sums (double-buffered)
    double* ring = red + 2 * PNW * 8; // a.ring doubles: V_prev ring / T staging / reduction scratch
    double* tot = ring + a.ring;      // [40]
    double* Tbb = tot + 40;           // [8][8]
    double* taus = Tbb + 64;          // [8]
    double* rowfix = taus + 8;        // [8][8] the diagonal rows' new values (written to Cb after the loop)
    const int sst = (a.ring / VNS) & ~1;
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    const double* Vp = V + j0;
    const int kr = lane & 3, cn = lane >> 2;

    for (int b = 0; b < nb / 8; ++b) {
        const int kp = 8 * b, jb = j0 + kp, d0 = kp;
        // A. the block: rows [j0, ld) of columns [jb, jb+8)
        for (int c = 0; c < 8; ++c) {
            const double* src = A + (int64_t)(jb + c) * ld + j0;
            for (int r2 = tid; r2 < R / 2; r2 += PNT) {
                unsigned d = (unsigned)__cvta_generic_to_shared(Cb + c * RP + 2 * r2);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * r2));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        if (kp > 0) {
            // B. one pass over V_prev: W = V_prev^T C_b and G = V_prev[:, 0:kp-8]^T V_{b-1}
            const int kpp = kp - 8;
            {
                const int mtiles = kp >> 3, t = warp >> 1, par = warp & 1;
                double a0 = 0.0, a1 = 0.0, g0 = 0.0, g1 = 0.0;
                vp_stream(Vp, ld, R, kp, ring, sst, [&](const double* st, int c, int rch, int nr) {
                    const int rcp = rch + 4, nq = nr / 8;
                    if (t < mtiles) {
                        const bool two = t < mtiles - 1;
#pragma unroll 4
                        for (int q = 0; q < nq; ++q) {
                            const int kk = (2 * q + par) * 4 + kr;
                            const double av = st[(t * 8 + cn) * rcp + kk];
                            dmma8(a0, a1, av, Cb[cn * RP + c * rch + kk]);
                            if (two) dmma8(g0, g1, av, st[(kpp + cn) * rcp + kk]);
                        }
                    }
                });
                double* pb = Zsm;  // pair-sum scratch: [mtiles][64] x 2 products <= 896 doubles
                if (t < mtiles && par == 1) {
                    pb[t * 64 + lane * 2] = a0;
                    pb[t * 64 + lane * 2 + 1] = a1;
                    ring[t * 64 + lane * 2] = g0;
                    ring[t * 64 + lane * 2 + 1] = g1;
                }
                __syncthreads();
                if (t < mtiles && par == 0) {
                    a0 += pb[t * 64 + lane * 2];
                    a1 += pb[t * 64 + lane * 2 + 1];
                    Wsm[(2 * kr) * kp + t * 8 + cn] = a0;
                    Wsm[(2 * kr + 1) * kp + t * 8 + cn] = a1;
                    if (t < mtiles - 1) {
                        g0 += ring[t * 64 + lane * 2];
                        g1 += ring[t * 64 + lane * 2 + 1];
                        Gp[(2 * kr) * kpp + t * 8 + cn] = g0;
                        Gp[(2 * kr + 1) * kpp + t * 8 + cn] = g1;
                    }
                }
                __syncthreads();
            }
            // C. T extension by block b-1 (Tbb still holds its T), then Z = T^T W
            if (kpp > 0) t_extend(T, kpp, Gp, Tbb, ring, ring + kpp * kpp);
            {
                double* Ts = ring;
                for (int t = tid; t < kp * kp; t += PNT) {
                    const int r = t % kp, c = t / kp;
                    Ts[c * kp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
                }
                __syncthreads();
                for (int t = tid; t < kp * 8; t += PNT) {
                    const int cp = t % kp, c = t / kp;
                    double s = 0.0;
                    for (int k = 0; k <= cp; ++k) s += Ts[cp * kp + k] * Wsm[c * kp + k];
                    Zsm[c * kp + cp] = s;
                }
                __syncthreads();
            }
            // D. C_b -= V_prev Z (DMMA, V_prev streamed again)
            {
                const int ksteps = kp >> 2;
                double zb[14];
#pragma unroll
                for (int t = 0; t < 14; ++t) zb[t] = t < ksteps ? -Zsm[cn * kp + t * 4 + kr] : 0.0;
                __syncthreads();  // Ts (ring) no longer read
                vp_stream(Vp, ld, R, kp, ring, sst, [&](const double* st, int c, int rch, int nr) {
                    const int rcp = rch + 4, nmt = nr / 8;
                    for (int mt = warp; mt < nmt; mt += PNW) {
                        const int r0 = c * rch + mt * 8;
                        double c0 = Cb[(2 * kr) * RP + r0 + cn], c1 = Cb[(2 * kr + 1) * RP + r0 + cn];
#pragma unroll
                        for (int t = 0; t < 14; ++t)
                            if (t < ksteps) dmma8(c0, c1, st[(t * 4 + kr) * rcp + mt * 8 + cn], zb[t]);
                        Cb[(2 * kr) * RP + r0 + cn] = c0;
                        Cb[(2 * kr + 1) * RP + r0 + cn] = c1;
                    }
                });
            }
        }

        // E. factor the 8 columns; thread t owns rows t, t + PNT, ... (no trailing barrier)
        for (int c = 0; c < 8; ++c) {
            const int d = d0 + c, nk = 8 - c;
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = 0.0;
            for (int r = tid; r < R; r += PNT) {
                if (r <= d) continue;
                const double x = Cb[c * RP + r];
                v[0] += x * x;
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) v[k] += x * Cb[(c + k) * RP + r];
            }
            double* rb = red + (c & 1) * PNW * 8;
            {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                double h4[4], h2[2], h1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double snd = b4 ? v[i] : v[i + 4];
                    h4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double snd = b3 ? h4[i] : h4[i + 2];
                    h2[i] = (b3 ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
                }
                {
                    const double snd = b2 ? h2[0] : h2[1];
                    h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, snd, 4);
                }
                h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
                h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
                if ((lane & 3) == 0) rb[warp * 8 + (lane >> 2)] = h1;
            }
            __syncthreads();
            // lane k < 8: the column sum k (fixed-order tree over the warps); lane 8 + k: y_k
            double mine = 0.0;
            if (lane < 8) {
                double p4[4];
#pragma unroll
                for (int w4 = 0; w4 < 4; ++w4)
                    p4[w4] = (rb[(4 * w4) * 8 + lane] + rb[(4 * w4 + 1) * 8 + lane]) +
                             (rb[(4 * w4 + 2) * 8 + lane] + rb[(4 * w4 + 3) * 8 + lane]);
                mine = (p4[0] + p4[1]) + (p4[2] + p4[3]);
            } else if (lane < 16) {
                mine = (lane - 8 < nk) ? Cb[(c + lane - 8) * RP + d] : 0.0;
            }
            const double ts0 = __shfl_sync(0xffffffffu, mine, 0);
            const double x0 = __shfl_sync(0xffffffffu, mine, 8);
            const double nrm = sqrt(x0 * x0 + ts0);
            double alpha = x0, tau = 0.0, scale = 0.0;
            if (nrm != 0.0) {
                alpha = x0 >= 0.0 ? -nrm : nrm;
                scale = 1.0 / (x0 - alpha);
                tau = (alpha - x0) / alpha;
            }
            const double ydl = __shfl_sync(0xffffffffu, mine, (lane & 7) + 8);
            const double wl = (lane >= 1 && lane < nk) ? tau * (ydl + scale * mine) : 0.0;
            double w[8], yd[8];
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                w[k] = __shfl_sync(0xffffffffu, wl, k);
                yd[k] = __shfl_sync(0xffffffffu, mine, k + 8);
            }
            if (tau != 0.0) {
                for (int r = tid; r < R; r += PNT) {
                    if (r <= d) continue;
                    const double x = Cb[c * RP + r];
                    const double vs = scale * x;
#pragma unroll
                    for (int k = 1; k < 8; ++k)
                        if (k < nk) Cb[(c + k) * RP + r] -= w[k] * vs;
                    Cb[c * RP + r] = vs;
                }
            }
            // the diagonal row's new values: other warps may still be reading row d (lanes 8..15
            // above), and no later column reads it, so they go to Cb after the loop
            if (tid == 0) {
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) rowfix[c * 8 + k] = yd[k] - w[k];
                rowfix[c * 8] = alpha;
                taus[c] = tau;
            }
        }
        __syncthreads();
        if (tid < 64) {
            const int c = tid >> 3, k = tid & 7;
            if (c + k < 8) Cb[(c + k) * RP + d0 + c] = rowfix[c * 8 + k];
        }
        __syncthreads();

        // F. write back R + V and tau; explicit V of the block -> smem and Vbuf
        for (int c = 0; c < 8; ++c) {
            const int d = d0 + c;
            double2* dst = reinterpret_cast<double2*>(A + (int64_t)(jb + c) * ld + j0);
            double2* dv = reinterpret_cast<double2*>(V + (int64_t)(kp + c) * ld + j0);
            for (int r2 = tid; r2 < R / 2; r2 += PNT) {
                const double x0 = Cb[c * RP + 2 * r2], x1 = Cb[c * RP + 2 * r2 + 1];
                dst[r2] = make_double2(x0, x1);
                const int r = 2 * r2;
                const double v0 = r < d ? 0.0 : (r == d ? 1.0 : x0);
                const double v1 = r + 1 < d ? 0.0 : (r + 1 == d ? 1.0 : x1);
                Cb[c * RP + r] = v0;
                Cb[c * RP + r + 1] = v1;
                dv[r2] = make_double2(v0, v1);
            }
        }
        if (tid < 8) a.tau[(int64_t)sl * a.M + jb + tid] = taus[tid];
        __syncthreads();
        // G. T of the block: Tbb[i][i] = tau_i, Tbb[0:i, i] = -tau_i Tbb[0:i,0:i] (Vb^T v_i)[0:i]
        {
            double g[28];
#pragma unroll
            for (int k = 0; k < 28; ++k) g[k] = 0.0;
            for (int r = d0 + tid; r < R; r += PNT) {
                double x[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) x[c] = Cb[c * RP + r];
                int k = 0;
#pragma unroll
                for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
                    for (int c2 = c1 + 1; c2 < 8; ++c2) g[k++] += x[c1] * x[c2];
            }
            block_sum<28>(g, ring, tot);
            if (tid < 32) {
                const int r = tid & 7;
                double trow[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[i] : 0.0;
#pragma unroll
                for (int i = 1; i < 8; ++i) {
                    if (r < i) {
                        double s = 0.0;
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if (k >= r && k < i) {
                                const int gi = (k * (15 - k)) / 2 + (i - k - 1);
                                s += trow[k] * tot[gi];
                            }
                        trow[i] = -taus[i] * s;
                    }
                }
                if (tid < 8)
#pragma unroll
                    for (int i = 0; i < 8; ++i) Tbb[i * 8 + r] = trow[i];
            }
            __syncthreads();
        }
        for (int t = tid; t < 64; t += PNT) {
            const int r = t % 8, c = t / 8;
            T[(kp + c) * ELM_NB + kp + r] = Tbb[c * 8 + r];
        }
        {
            const int c = tid / ELM_NB, r = tid % ELM_NB;  // 512 threads = 8 columns x 64 rows
            if (r >= kp + 8) T[(kp + c) * ELM_NB + r] = 0.0;
        }
        __syncthreads();
    }
    // H. the last block's T extension: its own Gram pass
    const int kpp = nb - 8;
    if (kpp > 0) {
        vt_block(Vp, ld, R, kpp, Cb, RP, Gp, ring, sst, Zsm);
        __syncthreads();
        t_extend(T, kpp, Gp, Tbb, ring, ring + kpp * kpp);
    }
}


// block-wide deterministic sum for NWARPS warps (k_panel_t): result broadcast in tot[0..NV)
template <int NV, int NWARPS>
__device__ __forceinline__ void block_sum_n(double (&v)[NV], double* red, double* tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) red[warp * NV + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double s = 0.0;
        for (int w = 0; w < NWARPS; ++w) s += red[w * NV + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
}

// t_extend for NTH threads
template <int NTH>
__device__ void t_extend_n(double* T, int kpp, const double* G, const double* Tbb, double* Ts, double* Ys) {
    for (int t = threadIdx.x; t < kpp * 8; t += NTH) {
        const int r = t % kpp, c = t / kpp;
        double s = 0.0;
        for (int k = 0; k <= c; ++k) s += G[k * kpp + r] * Tbb[c * 8 + k];
        Ys[c * kpp + r] = s;
    }
    for (int c = threadIdx.x >> 5; c < kpp; c += NTH / 32) {  // warp per column, coalesced
        const int lane = threadIdx.x & 31;
        double v0 = lane <= c ? T[c * ELM_NB + lane] : 0.0;
        double v1 = lane + 32 <= c && lane + 32 < kpp ? T[c * ELM_NB + lane + 32] : 0.0;
        if (lane < kpp) Ts[c * kpp + lane] = v0;
        if (lane + 32 < kpp) Ts[c * kpp + lane + 32] = v1;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kpp * 8; t += NTH) {
        const int r = t % kpp, c = t / kpp;
        double s = 0.0;
        for (int k = r; k < kpp; ++k) s += Ts[k * kpp + r] * Ys[c * kpp + k];
        T[(kpp + c) * ELM_NB + r] = -s;
    }
    __syncthreads();
}
// ------------------------------------------------------------------------------------------
// TMEM-resident panel (sm_100a): k_panel_p's arithmetic with the (ld - j0) x 8 block kept in
// tensor memory instead of shared memory, 256 threads and <= 128 registers, so that the panel
// CTA (~116 KB of shared memory: V_prev ring + a chunk staging buffer) shares its SM with one
// trailing-update CTA (108 KB): the latency-bound panel no longer takes a whole SM away from
// the DMMA-bound trailing updates (one k_wy_tma CTA alone keeps 83% of two CTAs' rate).
// TMEM layout (32-bit columns): row r of the block = 128 g + 32 q + lane lives in TMEM lane
// 32 q + lane, columns [16 g, 16 g + 16) (the 8 doubles of the row); warp w reaches lane quarter
// q = w % 4 and takes the row groups g = w / 4, w / 4 + 2, ...  The DMMA passes stage the rows of
// each V_prev chunk through shared memory; the column factorisation works on TMEM rows directly
// (thread = row, one tcgen05.ld / tcgen05.st of 16 columns per row), with the update of column c
// fused with the partial sums of column c + 1.
// ------------------------------------------------------------------------------------------
namespace pt {
constexpr int NT = 256, NW = 8;
constexpr int RCH_MAX = 256;                 // rows per staged chunk (Cs staging buffer)
constexpr int SMEM = 116 * 1024;             // > 228/2 KB: never two panel CTAs (TMEM) per SM;
                                             // + 108 KB trailing-update CTA fits
}  // namespace pt

__device__ __forceinline__ uint32_t tm_addr(uint32_t base, int quarter, int col) {
    return base + ((uint32_t)(32 * quarter) << 16) + (uint32_t)col;
}
__device__ __forceinline__ void tm_ld8(uint32_t addr, double (&v)[8]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = __hiloint2double((int)r[2 * c + 1], (int)r[2 * c]);
}
// issue a 16-column TMEM load without waiting (pair with tm_wait_ld + tm_unpack8)
__device__ __forceinline__ void tm_ld16(uint32_t addr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tm_unpack8(const uint32_t (&r)[16], double (&v)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = __hiloint2double((int)r[2 * c + 1], (int)r[2 * c]);
}
// store 8 doubles to TMEM without waiting (tm_wait_st before reloading the same columns)
__device__ __forceinline__ void tm_st8_nw(uint32_t addr, const double (&v)[8]) {
    uint32_t r[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        r[2 * c] = (uint32_t)__double2loint(v[c]);
        r[2 * c + 1] = (uint32_t)__double2hiint(v[c]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t addr, const double (&v)[8]) {
    uint32_t r[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        r[2 * c] = (uint32_t)__double2loint(v[c]);
        r[2 * c + 1] = (uint32_t)__double2hiint(v[c]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
        ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// stage rows [c*rch, c*rch + nr) of V_prev columns [0, kp) into dst[col*(rch+4) + row], NTH threads
template <int NTH>
__device__ __forceinline__ void vp_chunk_n(double* dst, const double* __restrict__ Vp, int64_t ld, int kp, int rch,
                                           int c, int nr) {
    const int rcp = rch + 4, n = kp * (nr / 2);
    for (int t = threadIdx.x; t < n; t += NTH) {
        const int col = t / (nr / 2), r = (t % (nr / 2)) * 2;
        unsigned d = (unsigned)__cvta_generic_to_shared(dst + col * rcp + r);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(Vp + (int64_t)col * ld + c * rch + r));
    }
}
template <int NTH, class F>
__device__ __forceinline__ void vp_stream_n(const double* __restrict__ Vp, int64_t ld, int R, int kp, double* ring,
                                            int sst, int rmax, F&& consume) {
    int rch = vp_rows(kp, sst);
    if (rch > rmax) rch = rmax;
    rch = 1 << (31 - __clz(rch));  // a power of two: chunks tile the staging windows of rmax rows
    const int nch = (R + rch - 1) / rch;
#pragma unroll
    for (int i = 0; i < VNS - 1; ++i) {
        if (i < nch) vp_chunk_n<NTH>(ring + i * sst, Vp, ld, kp, rch, i, min(rch, R - i * rch));
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(VNS - 2));
        __syncthreads();
        const int cn = c + VNS - 1;
        if (cn < nch) vp_chunk_n<NTH>(ring + (cn % VNS) * sst, Vp, ld, kp, rch, cn, min(rch, R - cn * rch));
        asm volatile("cp.async.commit_group;\n" ::);
        consume(ring + (c % VNS) * sst, c, rch, min(rch, R - c * rch));
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
}

constexpr int PANELT_FIXED = 3 * 8 * 56 + 8 * (pt::RCH_MAX + 4) + 2 * pt::NW * 8 + 40 + 64 + 8 + 16 + 8;

#ifdef ELM_QR_PROF
// per-CTA timeline of the QR phase (tools/qr_prof.py): t0, t1, smid | kind << 16, j0 << 20 | subdomain
__device__ unsigned long long g_qr_prof[1 << 20][4];
__device__ unsigned g_qr_n;
struct QrProf {
    unsigned long long t0, aux;
    int kind;
    __device__ QrProf(int k, unsigned long long x) : aux(x), kind(k) {
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    __device__ ~QrProf() {
        if (threadIdx.x != 0) return;
        unsigned long long t1;
        unsigned sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        const unsigned i = atomicAdd(&g_qr_n, 1u);
        if (i < (1u << 20)) {
            g_qr_prof[i][0] = t0;
            g_qr_prof[i][1] = t1;
            g_qr_prof[i][2] = sm | ((unsigned long long)kind << 16);
            g_qr_prof[i][3] = aux;
        }
    }
};
#define QR_PROF(k, x) QrProf qr_prof_(k, x)
#else
#define QR_PROF(k, x)
#endif
__global__ void __launch_bounds__(pt::NT, 2) k_panel_t(PanelArgs a, int nb) {
    QR_PROF(0, ((unsigned long long)a.j0 << 20) | (unsigned)(a.s_off + blockIdx.x));
    using namespace pt;
    const uint32_t tcols = a.tcols > 0 ? (uint32_t)a.tcols : 512u;
    extern __shared__ __align__(16) double sm[];
    __shared__ uint32_t s_tbase;
    const int sl = a.s_off + blockIdx.x;
    const int64_t ld = a.ld;
    const int j0 = a.j0;
    const int R = (int)(ld - j0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int quarter = warp & 3, gpar = warp >> 2;
    const int ngr = (R + 127) / 128;           // row groups
    double* Wsm = sm;                          // [8][kp]
    double* Zsm = Wsm + 8 * 56;                // [8][kp]
    double* Gp = Zsm + 8 * 56;                 // [8][kp-8]
    double* Cs = Gp + 8 * 56;                  // [8][RCH_MAX+4] staged block rows of a chunk
    double* red = Cs + 8 * (RCH_MAX + 4);      // [2][NW][8]
    double* tot = red + 2 * NW * 8;            // [40]
    double* Tbb = tot + 40;                    // [8][8]
    double* taus = Tbb + 64;                   // [8]
    double* drow = taus + 8;                   // [2][8] the current diagonal row (double-buffered)
    double* ring = drow + 16 + 8;              // a.ring doubles
    const int sst = (a.ring / VNS) & ~1;
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    const double* Vp = V + j0;
    const int kr = lane & 3, cn = lane >> 2;

    // TMEM: the whole 512 columns (one panel CTA per SM by construction)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tbase)), "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = s_tbase;
    auto row_of = [&](int g) { return 128 * g + 32 * quarter + lane; };
    auto taddr = [&](int g) { return tm_addr(tbase, quarter, 16 * g); };

#ifdef ELM_PANEL_PROF
    long long tq[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tq0 = clock64(), tqa, fq[4] = {0, 0, 0, 0}, fqa = 0;
#define TQ(i) do { const long long _n = clock64(); tq[i] += _n - tqa; tqa = _n; } while (0)
#else
#define TQ(i)
#endif
    for (int b = 0; b < nb / 8; ++b) {
        const int kp = 8 * b, jb = j0 + kp, d0 = kp;
#ifdef ELM_PANEL_PROF
        tqa = clock64();
#endif
        // A. the block -> TMEM (thread = row; rows >= R are zero)
        for (int g = gpar; g < ngr; g += 2) {
            const int r = row_of(g);
            double v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = r < R ? __ldcg(A + (int64_t)(jb + c) * ld + j0 + r) : 0.0;
            tm_st8(taddr(g), v);
        }
        __syncthreads();
        TQ(0);
        // stage rows [r0, r0 + nr) of the block into Cs (owner threads), then a barrier
        auto stage = [&](int r0, int nr, int rcp) {
            const int g0 = r0 / 128, g1 = (r0 + nr - 1) / 128;
            int g = g0 + ((g0 & 1) != gpar);
            for (; g + 2 <= g1; g += 4) {  // two row groups per wait (warp-uniform)
                uint32_t ra[16], rb[16];
                tm_ld16(taddr(g), ra);
                tm_ld16(taddr(g + 2), rb);
                tm_wait_ld();
                double va[8], vb[8];
                tm_unpack8(ra, va);
                tm_unpack8(rb, vb);
                const int r = row_of(g), s2 = row_of(g + 2);
                if (r >= r0 && r < r0 + nr)
#pragma unroll
                    for (int c = 0; c < 8; ++c) Cs[c * rcp + r - r0] = va[c];
                if (s2 >= r0 && s2 < r0 + nr)
#pragma unroll
                    for (int c = 0; c < 8; ++c) Cs[c * rcp + s2 - r0] = vb[c];
            }
            for (; g <= g1; g += 2) {
                double v[8];
                tm_ld8(taddr(g), v);
                const int r = row_of(g);
                if (r >= r0 && r < r0 + nr)
#pragma unroll
                    for (int c = 0; c < 8; ++c) Cs[c * rcp + r - r0] = v[c];
            }
            __syncthreads();
        };
        auto unstage = [&](int r0, int nr, int rcp) {
            // a lane writes its row only if the row is in the chunk: the other lanes of the warp
            // re-store the value they hold (loaded first; TMEM stores are warp-collective)
            const int g0 = r0 / 128, g1 = (r0 + nr - 1) / 128;
            for (int g = g0 + ((g0 & 1) != gpar); g <= g1; g += 2) {
                const int r = row_of(g);
                const bool in = r >= r0 && r < r0 + nr;
                double v[8];
                if (__all_sync(0xffffffffu, in)) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) v[c] = Cs[c * rcp + r - r0];
                } else {
                    tm_ld8(taddr(g), v);
                    if (in)
#pragma unroll
                        for (int c = 0; c < 8; ++c) v[c] = Cs[c * rcp + r - r0];
                }
                tm_st8_nw(taddr(g), v);
            }
            tm_wait_st();
        };
        if (kp > 0) {
            // B. one pass over V_prev: W = V_prev^T C_b and G = V_prev[:, 0:kp-8]^T V_{b-1}
            const int kpp = kp - 8, mtiles = kp >> 3;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
            vp_stream_n<NT>(Vp, ld, R, kp, ring, sst, RCH_MAX, [&](const double* st, int c, int rch, int nr) {
                const int rcp = rch + 4, nq = nr / 8;
                const int r0 = c * rch, w0 = r0 & ~(RCH_MAX - 1), off = r0 - w0;  // staging window
                if (off == 0) stage(w0, min(RCH_MAX, R - w0), RCH_MAX + 4);
                if (warp < mtiles) {
                    const bool two = warp < mtiles - 1;
                    const int t = warp;
#pragma unroll 2
                    for (int q = 0; q < nq; ++q) {
                        const int k0 = 8 * q + kr, k1 = k0 + 4;
                        const double av0 = st[(t * 8 + cn) * rcp + k0], av1 = st[(t * 8 + cn) * rcp + k1];
                        dmma8(a0, a1, av0, Cs[cn * (RCH_MAX + 4) + off + k0]);
                        dmma8(a2, a3, av1, Cs[cn * (RCH_MAX + 4) + off + k1]);
                        if (two) {
                            dmma8(g0, g1, av0, st[(kpp + cn) * rcp + k0]);
                            dmma8(g2, g3, av1, st[(kpp + cn) * rcp + k1]);
                        }
                    }
                }
            });
            if (warp < mtiles) {
                const int t = warp;
                Wsm[(2 * kr) * kp + t * 8 + cn] = a0 + a2;
                Wsm[(2 * kr + 1) * kp + t * 8 + cn] = a1 + a3;
                if (warp < mtiles - 1) {
                    Gp[(2 * kr) * kpp + t * 8 + cn] = g0 + g2;
                    Gp[(2 * kr + 1) * kpp + t * 8 + cn] = g1 + g3;
                }
            }
            __syncthreads();
            TQ(1);
            // C. T extension by block b-1, then Z = T^T W
            if (kpp > 0) t_extend_n<NT>(T, kpp, Gp, Tbb, ring, ring + kpp * kpp);
            {
                double* Ts = ring;
                // (warp per column, lanes over rows: coalesced, independent loads in flight)
                for (int c = warp; c < kp; c += NW) {
                    double v0 = lane <= c ? T[c * ELM_NB + lane] : 0.0;
                    double v1 = lane + 32 <= c && lane + 32 < kp ? T[c * ELM_NB + lane + 32] : 0.0;
                    if (lane < kp) Ts[c * kp + lane] = v0;
                    if (lane + 32 < kp) Ts[c * kp + lane + 32] = v1;
                }
                __syncthreads();
                for (int t = tid; t < kp * 8; t += NT) {
                    const int cp = t % kp, c = t / kp;
                    double s = 0.0;
                    for (int k = 0; k <= cp; ++k) s += Ts[cp * kp + k] * Wsm[c * kp + k];
                    Zsm[c * kp + cp] = s;
                }
                __syncthreads();
            }
            TQ(2);
            // D. C_b -= V_prev Z (DMMA on the staged rows, written back to TMEM)
            {
                const int ksteps = kp >> 2;
                double zb[14];
#pragma unroll
                for (int t = 0; t < 14; ++t) zb[t] = t < ksteps ? -Zsm[cn * kp + t * 4 + kr] : 0.0;
                __syncthreads();
                vp_stream_n<NT>(Vp, ld, R, kp, ring, sst, RCH_MAX, [&](const double* st, int c, int rch, int nr) {
                    const int rcp = rch + 4, nmt = nr / 8;
                    const int r0 = c * rch, w0 = r0 & ~(RCH_MAX - 1), off = r0 - w0, wn = min(RCH_MAX, R - w0);
                    constexpr int WCP = RCH_MAX + 4;
                    if (off == 0) stage(w0, wn, WCP);
                    for (int mt = warp; mt < nmt; mt += NW) {
                        const int rr = off + mt * 8 + cn;
                        double c0 = Cs[(2 * kr) * WCP + rr], c1 = Cs[(2 * kr + 1) * WCP + rr];
#pragma unroll
                        for (int t = 0; t < 14; ++t)
                            if (t < ksteps) dmma8(c0, c1, st[(t * 4 + kr) * rcp + mt * 8 + cn], zb[t]);
                        Cs[(2 * kr) * WCP + rr] = c0;
                        Cs[(2 * kr + 1) * WCP + rr] = c1;
                    }
                    if (off + nr == wn) {  // the window's last chunk: write the window back
                        __syncthreads();
                        unstage(w0, wn, WCP);
                    }
                });
            }
        }

        TQ(3);
        // E. factor the 8 columns on the TMEM rows.  Partial sums of column c are accumulated
        //    while column c-1 is applied; row d's owner publishes the diagonal row in drow.
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.0;
        for (int g = gpar; g < ngr; g += 2) {
            double x[8];
            tm_ld8(taddr(g), x);
            const int r = row_of(g);
            if (r < R && r > d0) {
                v[0] += x[0] * x[0];
#pragma unroll
                for (int k = 1; k < 8; ++k) v[k] += x[0] * x[k];
            }
            if (r == d0)
#pragma unroll
                for (int k = 0; k < 8; ++k) drow[k] = x[k];
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int d = d0 + c, nk = 8 - c;
            double* rb = red + (c & 1) * NW * 8;
#ifdef ELM_PANEL_PROF
            fqa = clock64();
#endif
            {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                double h4[4], h2[2], h1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double snd = b4 ? v[i] : v[i + 4];
                    h4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double snd = b3 ? h4[i] : h4[i + 2];
                    h2[i] = (b3 ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
                }
                {
                    const double snd = b2 ? h2[0] : h2[1];
                    h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, snd, 4);
                }
                h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
                h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
                if ((lane & 3) == 0) rb[warp * 8 + (lane >> 2)] = h1;
            }
            __syncthreads();
#ifdef ELM_PANEL_PROF
            { const long long _n = clock64(); fq[0] += _n - fqa; fqa = _n; }
#endif
            const double* dr = drow + (c & 1) * 8;   // diagonal row: columns c .. 7 at dr[c..7]
            double mine = 0.0;
            if (lane < 8) {
                mine = ((rb[0 * 8 + lane] + rb[1 * 8 + lane]) + (rb[2 * 8 + lane] + rb[3 * 8 + lane])) +
                       ((rb[4 * 8 + lane] + rb[5 * 8 + lane]) + (rb[6 * 8 + lane] + rb[7 * 8 + lane]));
            } else if (lane < 16) {
                mine = (lane - 8 < nk) ? dr[c + lane - 8] : 0.0;
            }
            const double ts0 = __shfl_sync(0xffffffffu, mine, 0);
            const double x0 = __shfl_sync(0xffffffffu, mine, 8);
            // (R20's alpha = -sign(x0) ||x||, tau = (alpha - x0) / alpha = 1 + |x0| / ||x||,
            // 1 / (x0 - alpha) = sign(x0) / (|x0| + ||x||): one rsqrt and one reciprocal on the
            // column's serial chain instead of a square root and two divisions)
            const double ss = fma(x0, x0, ts0);
            double alpha = x0, tau = 0.0, scale = 0.0;
            if (ss != 0.0) {
                const double rs = rsqrt(ss), nrm = ss * rs, ax = fabs(x0);
                alpha = x0 >= 0.0 ? -nrm : nrm;
                tau = fma(ax, rs, 1.0);
                scale = (x0 >= 0.0 ? 1.0 : -1.0) / (ax + nrm);
            }
            const double ydl = __shfl_sync(0xffffffffu, mine, (lane & 7) + 8);
            const double wl = (lane >= 1 && lane < nk) ? tau * (ydl + scale * mine) : 0.0;
            double w[8], yd[8];
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                w[k] = __shfl_sync(0xffffffffu, wl, k);
                yd[k] = __shfl_sync(0xffffffffu, mine, k + 8);
            }
            // apply column c to own rows (and the diagonal row's owner writes R's row d), and
            // accumulate the partial sums of column c + 1 on the updated rows
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = 0.0;
#ifdef ELM_PANEL_PROF
            { const long long _n = clock64(); fq[1] += _n - fqa; fqa = _n; }
#endif
            double* drn = drow + ((c + 1) & 1) * 8;
            auto body = [&](int g, double (&x)[8]) {
                const int r = row_of(g);
                const int rw = r - d;  // > 0: below the diagonal; 0: the diagonal row
                if (r < R && rw >= 0) {
                    if (rw == 0) {
#pragma unroll
                        for (int k = 1; k < 8; ++k)
                            if (c + k < 8) x[c + k] = yd[k] - w[k];
                        x[c] = alpha;
                    } else if (tau != 0.0) {
                        const double vs = scale * x[c];
#pragma unroll
                        for (int k = 1; k < 8; ++k)
                            if (c + k < 8) x[c + k] -= w[k] * vs;
                        x[c] = vs;
                    }
                    if (c < 7) {
                        if (rw == 1) {  // next column's diagonal row
#pragma unroll
                            for (int k = 0; k < 8; ++k) drn[k] = x[k];
                        } else if (rw > 1) {
                            const double xn = x[(c + 1) & 7];
                            v[0] += xn * xn;
#pragma unroll
                            for (int k = 1; k < 8; ++k)
                                if (c + 1 + k < 8) v[k] += xn * x[(c + 1 + k) & 7];
                        }
                    }
                }
            };
            int g = gpar;
            for (; g + 2 < ngr; g += 4) {  // two row groups per TMEM wait (warp-uniform)
                uint32_t ra[16], rb[16];
                tm_ld16(taddr(g), ra);
                tm_ld16(taddr(g + 2), rb);
                tm_wait_ld();
                double xa[8], xb[8];
                tm_unpack8(ra, xa);
                tm_unpack8(rb, xb);
                body(g, xa);
                body(g + 2, xb);
                tm_st8_nw(taddr(g), xa);  // warp-collective: every lane stores (unchanged rows too)
                tm_st8_nw(taddr(g + 2), xb);
            }
            for (; g < ngr; g += 2) {
                double x[8];
                tm_ld8(taddr(g), x);
                body(g, x);
                tm_st8_nw(taddr(g), x);
            }
            tm_wait_st();
#ifdef ELM_PANEL_PROF
            { const long long _n = clock64(); fq[2] += _n - fqa; fqa = _n; }
#endif
            if (tid == 0) taus[c] = tau;
        }
        __syncthreads();

        TQ(4);
        // F. write back R + V and tau; explicit V -> Vbuf; Gram of V_b for T_b
        double gq[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) gq[k] = 0.0;
        for (int g = gpar; g < ngr; g += 2) {
            const int r = row_of(g);
            double x[8];
            tm_ld8(taddr(g), x);
            if (r < R) {
                double vx[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    A[(int64_t)(jb + c) * ld + j0 + r] = x[c];
                    const int dc = d0 + c;
                    vx[c] = r < dc ? 0.0 : (r == dc ? 1.0 : x[c]);
                    V[(int64_t)(kp + c) * ld + j0 + r] = vx[c];
                }
                if (r >= d0) {
                    int k = 0;
#pragma unroll
                    for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
                        for (int c2 = c1 + 1; c2 < 8; ++c2) gq[k++] += vx[c1] * vx[c2];
                }
            }
        }
        if (tid < 8) a.tau[(int64_t)sl * a.M + jb + tid] = taus[tid];
        block_sum_n<28, NW>(gq, ring, tot);
        if (tid < 32) {
            const int r = tid & 7;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) {
                            const int gi = (k * (15 - k)) / 2 + (i - k - 1);
                            s += trow[k] * tot[gi];
                        }
                    trow[i] = -taus[i] * s;
                }
            }
            if (tid < 8)
#pragma unroll
                for (int i = 0; i < 8; ++i) Tbb[i * 8 + r] = trow[i];
        }
        __syncthreads();
        for (int t = tid; t < 64; t += NT) {
            const int r = t % 8, c = t / 8;
            T[(kp + c) * ELM_NB + kp + r] = Tbb[c * 8 + r];
        }
        for (int t = tid; t < 8 * ELM_NB; t += NT) {
            const int c = t / ELM_NB, r = t % ELM_NB;
            if (r >= kp + 8) T[(kp + c) * ELM_NB + r] = 0.0;
        }
        __syncthreads();  // Vbuf / T writes of this block before the next block reads them
        TQ(5);
    }
#ifdef ELM_PANEL_PROF
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 64) && (a.j0 == 0 || a.j0 == 256 || a.j0 == 512 || a.j0 == 1024))
        printf("PTPROF j0=%d total %lld load %lld wpass %lld z %lld upd %lld fact %lld wb %lld | red+sync %lld par %lld apply %lld\n", a.j0, clock64() - tq0,
               tq[0], tq[1], tq[2], tq[3], tq[4], tq[5], fq[0], fq[1], fq[2]);
#endif
#undef TQ
    // G. the last block's T extension: a Gram-only pass over [V_prev | V_last] (from Vbuf)
    const int kpp = nb - 8;
    if (kpp > 0) {
        const int kpl = nb, mtiles = kpp >> 3;
        double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
        vp_stream_n<NT>(Vp, ld, R, kpl, ring, sst, RCH_MAX, [&](const double* st, int c, int rch, int nr) {
            const int rcp = rch + 4, nq = nr / 8;
            if (warp < mtiles) {
                const int t = warp;
#pragma unroll 2
                for (int q = 0; q < nq; ++q) {
                    const int k0 = 8 * q + kr, k1 = k0 + 4;
                    dmma8(g0, g1, st[(t * 8 + cn) * rcp + k0], st[(kpp + cn) * rcp + k0]);
                    dmma8(g2, g3, st[(t * 8 + cn) * rcp + k1], st[(kpp + cn) * rcp + k1]);
                }
            }
        });
        if (warp < mtiles) {
            Gp[(2 * kr) * kpp + warp * 8 + cn] = g0 + g2;
            Gp[(2 * kr + 1) * kpp + warp * 8 + cn] = g1 + g3;
        }
        __syncthreads();
        t_extend_n<NT>(T, kpp, Gp, Tbb, ring, ring + kpp * kpp);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(tcols));
}

// ------------------------------------------------------------------------------------------
// Fused compact-WY trailing update for one 64-column block of one subdomain:
//     W = V^T C   (64 x 64, K = R rows)          phase 1, DMMA, 32-row chunks, 2-stage cp.async
//     Z = -T^T W  (64 x 64)                      phase 2, DMMA
//     C = C + V Z (R x 64)                       phase 3, DMMA, 32-row chunks, coalesced stores
// V columns >= nb and T entries outside nb x nb are treated as zero (last, narrower panel).
// grid (ceil(N/64), S), 256 threads (8 warps), ~108 KB dynamic shared memory -> 2 CTAs / SM.
// ------------------------------------------------------------------------------------------
namespace wy {
constexpr int NT = 256, CH = 32, PADC = CH + 4, PADZ = 64 + 4;
constexpr int STAGE = 2 * 64 * PADC;          // V chunk [64 cols][PADC] + C chunk [64 cols][PADC]
constexpr int SMEM = (2 * STAGE + 64 * PADZ) * 8;

__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// load rows [r0, r0+32) of 64 columns (col j at base + j*ld) into dst[j][k] (stride PADC);
// columns >= nvalid are zero-filled
__device__ __forceinline__ void load_chunk(double* dst, const double* base, int64_t ld, int nvalid, int tid) {
#pragma unroll
    for (int it = 0; it < (64 * CH / 2) / NT; ++it) {
        int ch = tid + it * NT;
        int j = ch / (CH / 2), k = (ch % (CH / 2)) * 2;
        bool ok = j < nvalid;
        cp16(dst + j * PADC + k, ok ? base + (int64_t)j * ld + k : base, ok ? 16 : 0);
    }
}
}  // namespace wy

__global__ void __launch_bounds__(wy::NT, 2) k_wy_update(const double* __restrict__ Vbuf, const double* __restrict__ Tbuf,
                                                         double* __restrict__ Kaug, int64_t ld, int64_t ncols, int j0,
                                                         int nb, int c0, int N, int s_off) {
    using namespace wy;
    extern __shared__ __align__(16) double sm[];
    double* st0 = sm;
    double* Zs = sm + 2 * STAGE;  // [64 n][PADZ]  W, then -Z
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = s_off + blockIdx.y, nblk = blockIdx.x;
    const int R = (int)(ld - j0);
    const int nch = R / CH;
    const int ncv = min(64, N - nblk * 64);
    const double* V = Vbuf + (int64_t)sl * ELM_NB * ld + j0;                 // V[r + j*ld]
    double* C = Kaug + (int64_t)sl * ld * ncols + j0 + (int64_t)(c0 + nblk * 64) * ld;  // C[r + n*ld]
    const double* T = Tbuf + (int64_t)sl * ELM_NB * ELM_NB;

    // ---------------- phase 1: W = V^T C ----------------
    const int wm = warp & 1, wn = warp >> 1;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    load_chunk(st0, V, ld, nb, tid);
    load_chunk(st0 + 64 * PADC, C, ld, ncv, tid);
    commit();
    for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) {
            double* nx = st0 + ((c + 1) & 1) * STAGE;
            load_chunk(nx, V + (c + 1) * CH, ld, nb, tid);
            load_chunk(nx + 64 * PADC, C + (c + 1) * CH, ld, ncv, tid);
        }
        commit();
        wait<1>();
        __syncthreads();
        const double* Vs = st0 + (c & 1) * STAGE;
        const double* Cs = Vs + 64 * PADC;
#pragma unroll
        for (int ks = 0; ks < CH / 4; ++ks) {
            const int kk = ks * 4 + (lane & 3);
            double af[4], bf[2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = Vs[(wm * 32 + mt * 8 + (lane >> 2)) * PADC + kk];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) bf[nt] = Cs[(wn * 16 + nt * 8 + (lane >> 2)) * PADC + kk];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
        __syncthreads();  // stage (c & 1) is overwritten by the load issued next iteration
    }
    wait<0>();
    // ---------------- phase 2: Z = -T^T W ----------------
    // W -> Zs[n][i]; T -> Ts[i][k] = T[k + 64 i] (masked to nb x nb)
    double* Ts = st0;  // [64 i][PADZ]
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int i = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                Zs[n * PADZ + i] = acc[mt][nt][e];
            }
    for (int t = tid; t < 64 * 64; t += NT) {
        int k = t & 63, i = t >> 6;
        Ts[i * PADZ + k] = (i < nb && k < nb) ? T[k + 64 * i] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int ks = 0; ks < 16; ++ks) {
        const int kk = ks * 4 + (lane & 3);
        double af[4], bf[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[mt] = Ts[(wm * 32 + mt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bf[nt] = Zs[(wn * 16 + nt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int i = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                Zs[n * PADZ + i] = -acc[mt][nt][e];   // B operand of phase 3: [n][k]
            }
    __syncthreads();
    // ---------------- phase 3: C += V (-Z), 32-row chunks ----------------
    const int wm3 = warp & 1, wn3 = warp >> 1;  // warp tile 16 rows x 16 cols
    load_chunk(st0, V, ld, nb, tid);
    load_chunk(st0 + 64 * PADC, C, ld, ncv, tid);
    commit();
    for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) {
            double* nx = st0 + ((c + 1) & 1) * STAGE;
            load_chunk(nx, V + (c + 1) * CH, ld, nb, tid);
            load_chunk(nx + 64 * PADC, C + (c + 1) * CH, ld, ncv, tid);
        }
        commit();
        wait<1>();
        __syncthreads();
        const double* Vs = st0 + (c & 1) * STAGE;  // [k = V col][r]
        double* Cs = (double*)Vs + 64 * PADC;      // [n][r]
        double a3[2][2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm3 * 16 + mt * 8 + (lane >> 2), n = wn3 * 16 + nt * 8 + 2 * (lane & 3) + e;
                    a3[mt][nt][e] = Cs[n * PADC + r];
                }
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
            const int kk = ks * 4 + (lane & 3);
            double af[2], bf[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) af[mt] = Vs[kk * PADC + wm3 * 16 + mt * 8 + (lane >> 2)];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) bf[nt] = Zs[(wn3 * 16 + nt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) dmma(a3[mt][nt][0], a3[mt][nt][1], af[mt], bf[nt]);
        }
        __syncthreads();  // all reads of Cs done before it is overwritten with results
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm3 * 16 + mt * 8 + (lane >> 2), n = wn3 * 16 + nt * 8 + 2 * (lane & 3) + e;
                    Cs[n * PADC + r] = a3[mt][nt][e];
                }
        __syncthreads();
        double* Cg = C + c * CH;
#pragma unroll
        for (int it = 0; it < (64 * CH / 2) / NT; ++it) {
            int ch = tid + it * NT;
            int j = ch / (CH / 2), k = (ch % (CH / 2)) * 2;
            if (j < ncv) *reinterpret_cast<double2*>(Cg + (int64_t)j * ld + k) = *reinterpret_cast<const double2*>(Cs + j * PADC + k);
        }
        __syncthreads();  // Cs of this stage is read by the stores before the next prefetch reuses it
    }
}

// ------------------------------------------------------------------------------------------
// TMA version of the fused compact-WY trailing update (operands staged by cp.async.bulk.tensor
// with 128B swizzle, mbarrier-tracked 2-stage pipeline; updated C chunks written back by TMA
// stores).  Same arithmetic as k_wy_update.  A 32-row chunk = 2 TMA boxes of 16 rows x 64 cols.
// ------------------------------------------------------------------------------------------
namespace wyt {
constexpr int NT = 256, CH = 32, PADZ = 64 + 4;
using elmtma::BOX;
constexpr int STAGE = 4 * BOX;            // V (2 boxes) + C (2 boxes)
constexpr int SMEM = (2 * STAGE + 64 * PADZ) * 8 + 64 + 1024;

using namespace elmtma;
#define ELM_SWIZZLE CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
}  // namespace wyt

// Implicit E_Gamma tiles (elm_e_implicit_range): in the first trailing update (j0 = 0) a 64-column
// tile inside [e_begin, e_end) is the unit matrix block [0; I; 0] restricted to its columns (a one
// at row pp + (col - M) when the column's edge is an interface edge, else a zero column).  Its
// chunks are written into shared memory instead of being loaded, and phase 1 (W = V^T C) visits
// only the chunks that hold its ones.
struct EsynArgs {
    int e_begin, e_end;   // implicit columns (empty: off)
    int M, q, pp, P, s_begin;
    int lattice;          // layout 1: columns M + 4q .. M + 4q + 3 are the corners (cross points)
};

__global__ void __launch_bounds__(wyt::NT, 2) k_wy_tma(const __grid_constant__ CUtensorMap tmV,
                                                       const __grid_constant__ CUtensorMap tmK,
                                                       const double* __restrict__ Tbuf, int64_t ld, int j0, int nb,
                                                       int c0, int N, int s_off, EsynArgs es, int rev3) {
    QR_PROF(1, ((unsigned long long)j0 << 20) | (unsigned)(s_off + blockIdx.y));
    using namespace wyt;
    extern __shared__ uint8_t raw[];
    // 1024-byte alignment for the swizzled TMA boxes; pointer arithmetic on `raw` keeps the
    // shared address space visible to the compiler (LDS, not generic LD)
    double* base = reinterpret_cast<double*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
    double* stg = base;                        // 2 stages x (V box0, V box1, C box0, C box1)
    double* Zs = base + 2 * STAGE;             // [64 n][PADZ]
    uint64_t* bar = reinterpret_cast<uint64_t*>(Zs + 64 * PADZ);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int sl = s_off + blockIdx.y;
    const int ncol0 = c0 + blockIdx.x * 64;
    const int R = (int)(ld - j0), nch = R / CH;
    const double* T = Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    if (tid == 0) {
        mbar_init(&bar[0], 1);  // [0..1] stage full (TMA)
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], NT / 32);  // [2..3] phase 1: every warp done with the stage
        mbar_init(&bar[3], NT / 32);
        mbar_init(&bar[4], NT / 32);  // [4..5] phase 3: every warp's C part written back into the stage
        mbar_init(&bar[5], NT / 32);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // T (nb x nb, zero outside) is fetched into the Z area while phase 1 runs (cp.async; the Z
    // area is free until phase 2, which then takes W into the stage area instead)
    for (int t = tid; t < 64 * 32; t += NT) {
        const int i = t >> 5, k2 = (t & 31) * 2;
        const int bytes = (i < nb && k2 < nb) ? (k2 + 1 < nb ? 16 : 8) : 0;
        const unsigned d = (unsigned)__cvta_generic_to_shared(Zs + i * PADZ + k2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(bytes ? T + k2 + 64 * i : T),
                     "r"(bytes));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    __syncthreads();
    // implicit E_Gamma tile (j0 = 0 only: the host passes an empty range otherwise)
    const bool syn = ncol0 >= es.e_begin && ncol0 + 64 <= es.e_end;
    int iface_mask = 0;
    if (syn) {
        const int s = es.s_begin + sl, si = s % es.P, sj = s / es.P;
        iface_mask = (si > 0) | ((si < es.P - 1) << 1) | ((sj > 0) << 2) | ((sj < es.P - 1) << 3);
        if (es.lattice)  // corner cc = (ci, cj) is a cross point iff it is inside the domain
            for (int cc = 0; cc < 4; ++cc) {
                const int X = si + (cc & 1), Y = sj + (cc >> 1);
                iface_mask |= (X > 0 && X < es.P && Y > 0 && Y < es.P) << (4 + cc);
            }
    }
    // the C part of a stage for chunk c of a synthetic tile: element (row, col) of the swizzled
    // 32 x 64 chunk is 1 iff row c*CH + row == pp + (ncol0 + col - M) on an interface edge
    auto fill = [&](double* Cs, int c) {
        for (int t = tid; t < 2 * BOX; t += NT) {
            const int bx = t / BOX, rem = t - bx * BOX, col = rem >> 4, x = rem & 15;
            const int row = bx * 16 + ((((x >> 2) ^ (col & 3))) << 2) + (x & 3);
            const int ecol = ncol0 + col - es.M;
            const int bit = ecol < 4 * es.q ? ecol / es.q : 4 + (ecol - 4 * es.q);
            Cs[t] = (c * CH + row == es.pp + ecol && ((iface_mask >> bit) & 1)) ? 1.0 : 0.0;
        }
    };
    uint32_t par0 = 0, par1 = 0;
    // (flags bit 1: phase 3's C chunks are last-use -- loaded and stored evict-first, so that L2
    // keeps the other CTAs' phase-1 chunks for their phase 3 instead)
    const bool hint3 = (rev3 & 2) != 0;
    const uint64_t pol = hint3 && tid == 0 ? l2_evict_first() : 0ull;
    auto issue = [&](int c, int st, bool last_use = false) {
        double* d = stg + st * STAGE;
        mbar_expect(&bar[st], (syn ? 2 : 4) * BOX * 8);
        tma_load(d, &tmV, j0 + c * CH, 0, sl, &bar[st]);
        tma_load(d + BOX, &tmV, j0 + c * CH + 16, 0, sl, &bar[st]);
        if (!syn) {
            if (last_use && hint3) {
                tma_load_hint(d + 2 * BOX, &tmK, j0 + c * CH, ncol0, sl, &bar[st], pol);
                tma_load_hint(d + 3 * BOX, &tmK, j0 + c * CH + 16, ncol0, sl, &bar[st], pol);
            } else {
                tma_load(d + 2 * BOX, &tmK, j0 + c * CH, ncol0, sl, &bar[st]);
                tma_load(d + 3 * BOX, &tmK, j0 + c * CH + 16, ncol0, sl, &bar[st]);
            }
        }
    };
    // phase-1 chunks: all, or for a synthetic tile the ones holding its ones (W = V^T C is zero
    // on the others)
    int cb = 0, n1 = nch;
    if (syn) {
        const int r_lo = es.pp + ncol0 - es.M, r_hi = r_lo + 63;
        cb = r_lo / CH;
        n1 = (iface_mask ? min(r_hi / CH, nch - 1) - cb + 1 : 0);
    }
    auto wait_stage = [&](int st) {
        if (st == 0) {
            mbar_wait(&bar[0], par0);
            par0 ^= 1;
        } else {
            mbar_wait(&bar[1], par1);
            par1 ^= 1;
        }
    };
    // ---------------- phase 1: W = V^T C ----------------
    const int wm = warp & 1, wn = warp >> 1;
    // valid columns of this tile: the last tile of every update holds only the F column (and any
    // rest of the E_Gamma block); warps whose 16 columns are all out of range skip their DMMAs
    const int ncv = N - (int)blockIdx.x * 64;
    const bool act = wn * 16 < ncv;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // Stage hand-off without CTA-wide barriers (except for synthesised E tiles): a warp arrives on
    // the stage's mbarrier when done with it, and only thread 0 waits there before refilling the
    // stage (phase 1) or before storing the written-back C chunk by TMA (phase 3).
    const bool mb = !syn;
    uint32_t epar = 0u, dpar = 0u;  // (thread 0) parity bits (bit s: stage s) of bar[2..3], bar[4..5]
    if (tid == 0 && n1 > 0) issue(cb, 0);
    for (int i1 = 0; i1 < n1; ++i1) {
        const int st = i1 & 1, c = cb + i1;
        if (tid == 0 && i1 + 1 < n1) {
            if (mb && i1 >= 1) {  // every warp is done with chunk i1 - 1 in stage st ^ 1
                mbar_wait(&bar[2 + (st ^ 1)], (epar >> (st ^ 1)) & 1u);
                epar ^= 1u << (st ^ 1);
            }
            issue(c + 1, st ^ 1);
        }
        wait_stage(st);
        const double* Vs = stg + st * STAGE;
        const double* Cs = Vs + 2 * BOX;
        if (syn) {
            fill(stg + st * STAGE + 2 * BOX, c);
            __syncthreads();
        }
#pragma unroll
        for (int ks = 0; ks < CH / 4; ++ks) {
            if (!act) break;
            const int kk = ks * 4 + (lane & 3);
            double af[4], bf[2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = Vs[sw(kk, wm * 32 + mt * 8 + (lane >> 2))];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) bf[nt] = Cs[sw(kk, wn * 16 + nt * 8 + (lane >> 2))];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
        if (mb) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[2 + st]);
        } else {
            __syncthreads();
        }
    }
    __syncthreads();  // every warp is done with the stages: phase 2 keeps W there
    // ---------------- phase 2: Z = -T^T W ----------------
    const double* Ts = Zs;  // [64 i][PADZ] (prefetched)
    double* Ws = stg;       // [64 n][PADZ]
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int i = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                Ws[n * PADZ + i] = acc[mt][nt][e];
            }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll 4
    for (int ks = 0; ks < 16; ++ks) {
        if (!act) break;
        const int kk = ks * 4 + (lane & 3);
        double af[4], bf[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[mt] = Ts[(wm * 32 + mt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bf[nt] = Ws[(wn * 16 + nt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
    __syncthreads();  // T read: the Z area takes Z
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int i = wm * 32 + mt * 8 + (lane >> 2), n = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                Zs[n * PADZ + i] = -acc[mt][nt][e];
            }
    __syncthreads();
    // ---------------- phase 3: C += V (-Z) ----------------
    // rev3: the chunks bottom-up, so that the first ones are those phase 1 read last and that
    // are still in L2 (each chunk is independent here: the same bits in either order)
    const int wm3 = warp & 1, wn3 = warp >> 1;
    auto chunk3 = [&](int i) { return (rev3 & 1) ? nch - 1 - i : i; };
    if (tid == 0) issue(chunk3(0), n1 & 1 ? 1 : 0, true);  // continue the stage rotation of phase 1
    const int sbase = n1 & 1;
    for (int i3 = 0; i3 < nch; ++i3) {
        const int st = (i3 + sbase) & 1, c = chunk3(i3);
        if (tid == 0 && i3 + 1 < nch) {
            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // stage st^1 stored?
            issue(chunk3(i3 + 1), st ^ 1, true);
        }
        wait_stage(st);
        const double* Vs = stg + st * STAGE;
        double* Cs = stg + st * STAGE + 2 * BOX;
        if (syn) {  // (the stage's previous TMA store finished reading it before the last issue)
            fill(Cs, c);
            __syncthreads();
        }
        double a3[2][2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm3 * 16 + mt * 8 + (lane >> 2), n = wn3 * 16 + nt * 8 + 2 * (lane & 3) + e;
                    a3[mt][nt][e] = Cs[sw(r, n)];
                }
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
            if (!act) break;  // (wn3 == wn: the same column group as in phase 1)
            const int kk = ks * 4 + (lane & 3);
            double af[2], bf[2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) af[mt] = Vs[sw(wm3 * 16 + mt * 8 + (lane >> 2), kk)];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) bf[nt] = Zs[(wn3 * 16 + nt * 8 + (lane >> 2)) * PADZ + kk];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) dmma(a3[mt][nt][0], a3[mt][nt][1], af[mt], bf[nt]);
        }
        // (a warp writes back exactly the C part it read: no barrier before the write-back)
        if (!mb) __syncthreads();  // all reads of this C stage done
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm3 * 16 + mt * 8 + (lane >> 2), n = wn3 * 16 + nt * 8 + 2 * (lane & 3) + e;
                    Cs[sw(r, n)] = a3[mt][nt][e];
                }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (mb) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[4 + st]);
            if (tid == 0) {  // every warp's part written (and its reads of the stage done)
                mbar_wait(&bar[4 + st], (dpar >> st) & 1u);
                dpar ^= 1u << st;
            }
        } else {
            __syncthreads();
        }
        if (tid == 0) {
            if (hint3) {
                tma_store_hint(&tmK, j0 + c * CH, ncol0, sl, Cs, pol);
                tma_store_hint(&tmK, j0 + c * CH + 16, ncol0, sl, Cs + BOX, pol);
            } else {
                tma_store(&tmK, j0 + c * CH, ncol0, sl, Cs);
                tma_store(&tmK, j0 + c * CH + 16, ncol0, sl, Cs + BOX);
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}



// ------------------------------------------------------------------------------------------
// Grid panel for very tall local problems (the paper's N = 1 x 1 / 2 x 2 lattice workloads:
// 33k / 132k damped rows, beyond the cluster panels).  One cooperative launch per panel: the
// CTAs of a subdomain split its rows [j0, ld) into contiguous slices, the 64-column panel stays
// in K_aug (L2-resident), and every column is one unblocked Householder step (reading R20) with
// two barriers among the subdomain's CTAs: (1) partial sums of the column's squares -> every CTA
// reduces them in the same fixed order and forms alpha, tau, v; (2) partial dot products of v
// with the panel's remaining columns -> the same fixed-order reduction -> rank-1 update of the
// own slice.  Then V (explicit, to Vbuf), tau, and T from the Gram V^T V (fixed-order partial
// sums) by the forward recurrence T[0:j, j] = -tau_j T[0:j, 0:j] (V^T v_j).  Deterministic.
// ------------------------------------------------------------------------------------------
namespace gp {
constexpr int NT = 256, NW = NT / 32;
constexpr int NG = ELM_NB * (ELM_NB + 1) / 2;  // Gram entries (upper triangle incl. diagonal)
}  // namespace gp

__device__ __forceinline__ unsigned gp_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// barrier among the nper CTAs of one subdomain (cooperative launch: all co-resident);
// a monotone counter zeroed before the launch
__device__ __forceinline__ void gp_barrier(unsigned* cnt, unsigned nper, unsigned& gen) {
    __syncthreads();
    ++gen;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        while (gp_ld_acquire(cnt) < gen * nper) {
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(gp::NT) k_panel_grid(PanelArgs a, int nb, int nper, double* __restrict__ part,
                                                       unsigned* __restrict__ cnt) {
    using namespace gp;
    extern __shared__ double dsm[];  // Gs [64][65] | Ts [64][65] | vs [64][33]
    double* Gs = dsm;
    double* Ts = Gs + ELM_NB * (ELM_NB + 1);
    double* vs = Ts + ELM_NB * (ELM_NB + 1);
    __shared__ double red[NW];
    __shared__ double wsh[ELM_NB];
    __shared__ double prm[4];  // alpha, tau, scale
    const int sd = blockIdx.x / nper, cta = blockIdx.x % nper;
    const int sl = a.s_off + sd;
    const int64_t ld = a.ld;
    const int j0 = a.j0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* Vb = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    double* P = part + (int64_t)sd * nper * NG;  // [cta][NG] partials of this subdomain
    unsigned* C = cnt + sd;
    unsigned gen = 0;
    const int64_t R = ld - j0, per = (R + nper - 1) / nper;
    const int64_t r0 = j0 + (int64_t)cta * per, r1 = (ld < r0 + per ? ld : r0 + per);  // own rows [r0, r1)
    for (int c = 0; c < nb; ++c) {
        const int64_t jc = j0 + c;
        const bool own_jc = jc >= r0 && jc < r1;
        double* x = A + jc * ld;
        const int64_t i0 = r0 > jc + 1 ? r0 : jc + 1;
        // (1) ||x[jc+1:]||^2 over the own rows
        double ss = 0.0;
        for (int64_t i = i0 + tid; i < r1; i += NT) ss = fma(x[i], x[i], ss);
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (lane == 0) red[warp] = ss;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NW; ++w) t += red[w];
            P[(int64_t)cta * NG] = t;
        }
        // row jc of the panel's later columns, published by its owner before anyone updates it
        // (one element per thread: by thread 0 alone, each strided load waited for the previous
        // store, ~60 L2 round trips on the owner CTA while every other CTA waited at the barrier)
        if (own_jc)
            for (int k = tid; k < nb - 1 - c; k += NT)
                P[(int64_t)cta * NG + ELM_NB * (1 + (c & 1)) + k] = A[(jc + 1 + k) * ld + jc];
        gp_barrier(C, nper, gen);
        if (tid == 0) {
            double t = 0.0;
            for (int k = 0; k < nper; ++k) t += P[(int64_t)k * NG];
            const int owner = (int)((jc - j0) / per);
            const double x0 = A[jc * ld + jc];
            const double nrm = sqrt(x0 * x0 + t);
            double alpha = x0, tau = 0.0, scale = 0.0;
            if (nrm != 0.0) {
                alpha = x0 >= 0.0 ? -nrm : nrm;
                scale = 1.0 / (x0 - alpha);
                tau = (alpha - x0) / alpha;
            }
            prm[0] = alpha;
            prm[1] = tau;
            prm[2] = scale;
            prm[3] = (double)owner;
        }
        __syncthreads();
        const double tau = prm[1], scale = prm[2];
        const int owner = (int)prm[3];
        // v = x / (x0 - alpha) below the diagonal (own rows)
        for (int64_t i = i0 + tid; i < r1; i += NT) x[i] *= scale;
        __syncthreads();
        // (2) partial sums_{i > jc} v_i A[i, k] for the remaining panel columns
        const int nk = nb - 1 - c;
        for (int k = warp; k < nk; k += NW) {
            const double* y = A + (jc + 1 + k) * ld;
            double d = 0.0;
            for (int64_t i = i0 + lane; i < r1; i += 32) d = fma(x[i], y[i], d);
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            if (lane == 0) P[(int64_t)cta * NG + 1 + k] = d;
        }
        gp_barrier(C, nper, gen);
        if (tid < nk) {  // w_k = tau (A[jc, k] + sum_i v_i A[i, k]), fixed order
            double d = P[(int64_t)owner * NG + ELM_NB * (1 + (c & 1)) + tid];
            for (int k2 = 0; k2 < nper; ++k2) d += P[(int64_t)k2 * NG + 1 + tid];
            wsh[tid] = tau * d;
        }
        __syncthreads();
        for (int k = warp; k < nk; k += NW) {
            double* y = A + (jc + 1 + k) * ld;
            const double w = wsh[k];
            // four rows per lane loaded before any store (the store to y[i] may alias, for the
            // compiler, the next rows' loads: one row at a time serialised every load on the
            // previous store -- ncu: 23% of the kernel's stall samples on this FMA)
            int64_t i = i0 + lane;
            for (; i + 96 < r1; i += 128) {
                const double x0 = x[i], x1 = x[i + 32], x2 = x[i + 64], x3 = x[i + 96];
                const double y0 = y[i], y1 = y[i + 32], y2 = y[i + 64], y3 = y[i + 96];
                y[i] = fma(-w, x0, y0);
                y[i + 32] = fma(-w, x1, y1);
                y[i + 64] = fma(-w, x2, y2);
                y[i + 96] = fma(-w, x3, y3);
            }
            for (; i < r1; i += 32) y[i] = fma(-w, x[i], y[i]);
            if (lane == 0 && own_jc) y[jc] -= w;  // row jc: v_jc = 1 (the owner)
        }
        if (tid == 0 && own_jc) {
            x[jc] = prm[0];  // R_jj
            a.tau[(int64_t)sl * a.M + jc] = tau;
        }
        // No grid barrier at the end of a column (a CTA barrier suffices: the next column's norm
        // reads the own rows other warps just updated): the next column's first grid barrier
        // already orders every CTA's update of its own rows (the next diagonal element included)
        // before anyone reads them, and the published diagonal row alternates between two slots
        // by column parity, so a CTA running ahead never overwrites the one a slower CTA still
        // reads.  After the last column the Gram partials below reuse every slot: a grid barrier.
        if (c == nb - 1)
            gp_barrier(C, nper, gen);
        else
            __syncthreads();
    }
    // explicit V (absolute rows, unit diagonal, zero above) of the own rows
    for (int c = 0; c < ELM_NB; ++c) {
        const int64_t jc = j0 + c;
        for (int64_t i = r0 + tid; i < r1; i += NT)
            Vb[(int64_t)c * ld + i] = c >= nb ? 0.0 : (i < jc ? 0.0 : (i == jc ? 1.0 : A[jc * ld + i]));
    }
    // partial Gram V^T V (upper, k <= l) over the own rows, 32-row chunks staged in shared memory
    double acc[(NG + NT - 1) / NT];
#pragma unroll
    for (int u = 0; u < (NG + NT - 1) / NT; ++u) acc[u] = 0.0;
    __syncthreads();
    for (int64_t b0 = r0; b0 < r1; b0 += 32) {
        const int nr = (int)(r1 - b0 < 32 ? r1 - b0 : 32);
        for (int e = tid; e < ELM_NB * 32; e += NT) {
            const int c = e / 32, r = e % 32;
            vs[c * 33 + r] = r < nr ? Vb[(int64_t)c * ld + b0 + r] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < (NG + NT - 1) / NT; ++u) {
            const int e = tid + u * NT;
            if (e < NG) {
                int k = 0, rem = e;
                while (rem >= ELM_NB - k) {
                    rem -= ELM_NB - k;
                    ++k;
                }
                const int l = k + rem;
                double sacc = acc[u];
                for (int r = 0; r < 32; ++r) sacc = fma(vs[k * 33 + r], vs[l * 33 + r], sacc);
                acc[u] = sacc;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < (NG + NT - 1) / NT; ++u)
        if (tid + u * NT < NG) P[(int64_t)cta * NG + tid + u * NT] = acc[u];
    gp_barrier(C, nper, gen);
    if (cta != 0) return;
    // T (64 x 64, column-major, upper) by the forward recurrence, one CTA per subdomain
    for (int e = tid; e < NG; e += NT) {
        int k = 0, rem = e;
        while (rem >= ELM_NB - k) {
            rem -= ELM_NB - k;
            ++k;
        }
        const int l = k + rem;
        double sacc = 0.0;
        for (int k2 = 0; k2 < nper; ++k2) sacc += P[(int64_t)k2 * NG + e];
        Gs[k * (ELM_NB + 1) + l] = sacc;
    }
    for (int e = tid; e < ELM_NB * (ELM_NB + 1); e += NT) Ts[e] = 0.0;
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        const double tj = a.tau[(int64_t)sl * a.M + j0 + j];
        if (tid < j) {  // T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]
            double sacc = 0.0;
            for (int k = tid; k < j; ++k) sacc += Ts[tid * (ELM_NB + 1) + k] * Gs[k * (ELM_NB + 1) + j];
            Ts[tid * (ELM_NB + 1) + j] = -tj * sacc;
        }
        if (tid == 0) Ts[j * (ELM_NB + 1) + j] = tj;
        __syncthreads();
    }
    for (int e = tid; e < ELM_NB * ELM_NB; e += NT) {
        const int r = e % ELM_NB, c = e / ELM_NB;
        T[(int64_t)c * ELM_NB + r] = (r < nb && c < nb) ? Ts[r * (ELM_NB + 1) + c] : 0.0;
    }
}

constexpr int GP_SMEM = (2 * ELM_NB * (ELM_NB + 1) + ELM_NB * 33) * 8;

// ------------------------------------------------------------------------------------------
// Cluster version of the panel base block: one subdomain's 8-column block is factored by a
// cluster of PCL CTAs (PCL SMs), CTA z holding the rows [z Rq, (z+1) Rq) of the panel range.
// With a quarter of the rows resident (<= 49 KB) each CTA streams its share of V_prev through a
// deep ring (chunks of up to 128 rows at kp = 56); the cross-CTA sums (W = V_prev^T C, the 8
// column reductions, the Gram of the block, V_prev^T V_b) are all-reduced through distributed
// shared memory: every CTA writes its partial into slot z of every CTA's buffer, one cluster
// barrier, then every CTA sums the slots in the same fixed order (deterministic, and every CTA
// computes identical alpha / tau / T).  DESIGN.md §5.2.
// ------------------------------------------------------------------------------------------
namespace pcl {
constexpr int CL = 4;                 // CTAs per subdomain
constexpr int STG = 56 * 132;         // doubles per ring stage (default; smaller for tall panels)
constexpr int STG_MIN = 56 * 36;      // >= 32 rows of a 56-column V chunk, and 2 stages hold T (56^2)
constexpr int XN = 448;               // doubles per exchange slot (kp * 8 <= 448)
}  // namespace pcl

__device__ __forceinline__ int vp_rows_cl(int kp, int stg) {
    const int r = ((stg / kp - 4) / 32) * 32;
    return r < 32 ? 32 : (r > 256 ? 256 : r);
}

// G (kp x 8, column-major ld kp) = Vp[0:nr]^T X[0:nr] (partial over this CTA's rows)
__device__ void vt_block_cl(const double* __restrict__ Vp, int64_t ld, int nr, int kp, const double* X, int RP,
                            double* G, double* ring, double* pairbuf, int stg) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int mtiles = kp >> 3, t = warp >> 1, par = warp & 1;
    const int kr = lane & 3, cn = lane >> 2;
    const int rch = vp_rows_cl(kp, stg), rcp = rch + 4;
    const int nch = (nr + rch - 1) / rch;
    double a0 = 0.0, a1 = 0.0;
    if (nch > 0) {
        vp_chunk(ring, Vp, ld, kp, rch, 0, min(rch, nr));
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) vp_chunk(ring + ((c + 1) & 1) * stg, Vp, ld, kp, rch, c + 1, min(rch, nr - (c + 1) * rch));
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);
        __syncthreads();
        const double* st = ring + (c & 1) * stg;
        const int nq = min(rch, nr - c * rch) / 8;
        if (t < mtiles) {
#pragma unroll 4
            for (int q = 0; q < nq; ++q) {
                const int kk = (2 * q + par) * 4 + kr;
                dmma8(a0, a1, st[(t * 8 + cn) * rcp + kk], X[cn * RP + c * rch + kk]);
            }
        }
        __syncthreads();
    }
    if (t < mtiles && par == 1) {
        pairbuf[t * 64 + lane * 2] = a0;
        pairbuf[t * 64 + lane * 2 + 1] = a1;
    }
    __syncthreads();
    if (t < mtiles && par == 0) {
        a0 += pairbuf[t * 64 + lane * 2];
        a1 += pairbuf[t * 64 + lane * 2 + 1];
        G[(2 * kr) * kp + t * 8 + cn] = a0;
        G[(2 * kr + 1) * kp + t * 8 + cn] = a1;
    }
}

size_t panel_cl_smem(int64_t Rq, int stg) {
    return (size_t)(8 * (Rq + 4) + 2 * stg + 2 * pcl::CL * pcl::XN + 2 * 8 * 56 + PNW * 28 + 40 + 64 + 8 + 16) * 8;
}
// ring stage of the cluster panel for a panel of ld rows: the default, or as much as fits next to
// the row block (tall panels, e.g. the damped local LS of reading R29); 0 if even STG_MIN does not fit
int cl_stage(int64_t ld, int smem_optin) {
    const int64_t Rq = ((ld + 32 * pcl::CL - 1) / (32 * pcl::CL)) * 32;
    if (panel_cl_smem(Rq, pcl::STG) <= (size_t)smem_optin) return pcl::STG;
    const int64_t avail = ((int64_t)smem_optin - (int64_t)panel_cl_smem(Rq, 0)) / 16;  // doubles per stage
    const int stg = (int)std::min<int64_t>(pcl::STG, avail & ~(int64_t)7);
    return stg >= pcl::STG_MIN ? stg : 0;
}

__global__ void __cluster_dims__(pcl::CL, 1, 1) __launch_bounds__(PNT, 1) k_panel_cl(PanelArgs a) {
    using namespace pcl;
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    extern __shared__ __align__(16) double sm[];
    const int z = (int)cl.block_rank();
    const int sl = a.s_off + (int)blockIdx.x / CL;
    const int64_t ld = a.ld;
    const int j0 = a.j0, jb = j0 + ELM_BB * a.blk, kp = ELM_BB * a.blk;
    const int R = (int)(ld - j0);
    const int Rq = ((R + 32 * CL - 1) / (32 * CL)) * 32;
    const int r0 = z * Rq, nr = max(0, min(Rq, R - r0));
    const int RP = Rq + 4;
    const int d0 = jb - j0;
    const int tid = threadIdx.x;
    double* Cb = sm;                      // [8][RP]  own rows
    const int stg = a.ring;               // doubles per ring stage (panel_cl_stage)
    double* ring = Cb + 8 * RP;           // [2][stg]
    double* xch = ring + 2 * stg;         // [2][CL][XN]
    double* Wsm = xch + 2 * CL * XN;      // [8][kp]
    double* Zsm = Wsm + 8 * 56;           // [8][kp]
    double* red = Zsm + 8 * 56;           // [PNW][28]
    double* tot = red + PNW * 28;         // [40]
    double* Tbb = tot + 40;               // [8][8]
    double* taus = Tbb + 64;              // [8]
    double* pay = taus + 8;               // [16]
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    const double* Vz = V + j0 + r0;       // own rows of V_prev: column c at Vz + c*ld
    int xpar = 0;
    // all-reduce: mine[0..n) -> slot z of every CTA's buffer; returns the local buffer ([CL][XN])
    auto exchange = [&](const double* mine, int n) -> const double* {
        double* buf = xch + xpar * CL * XN;
        for (int t = tid; t < CL * n; t += PNT) {
            const int dst = t / n, i = t % n;
            double* rb = cl.map_shared_rank(buf, dst);
            rb[z * XN + i] = mine[i];
        }
        cl.sync();
        xpar ^= 1;
        return buf;
    };

    // A. own rows of the block
    for (int c = 0; c < 8; ++c) {
        const double* src = A + (int64_t)(jb + c) * ld + j0 + r0;
        for (int r2 = tid; r2 < nr / 2; r2 += PNT) {
            unsigned d = (unsigned)__cvta_generic_to_shared(Cb + c * RP + 2 * r2);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * r2));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();

    if (kp > 0) {
        // B. W = V_prev^T C (all-reduced), Z = T^T W, C -= V_prev Z on own rows
        vt_block_cl(Vz, ld, nr, kp, Cb, RP, Wsm, ring, Zsm, stg);
        __syncthreads();
        const double* buf = exchange(Wsm, kp * 8);
        for (int i = tid; i < kp * 8; i += PNT) {
            double v = 0.0;
            for (int s = 0; s < CL; ++s) v += buf[s * XN + i];
            Wsm[i] = v;
        }
        double* Ts = ring;
        for (int t = tid; t < kp * kp; t += PNT) {
            const int r = t % kp, c = t / kp;
            Ts[c * kp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
        }
        __syncthreads();
        for (int t = tid; t < kp * 8; t += PNT) {
            const int cp = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = 0; k <= cp; ++k) s += Ts[cp * kp + k] * Wsm[c * kp + k];
            Zsm[c * kp + cp] = s;
        }
        __syncthreads();
        {
            const int lane = tid & 31, warp = tid >> 5;
            const int kr = lane & 3, rn = lane >> 2;
            const int ksteps = kp >> 2;
            double zb[14];
#pragma unroll
            for (int t = 0; t < 14; ++t) zb[t] = t < ksteps ? -Zsm[rn * kp + t * 4 + kr] : 0.0;
            __syncthreads();  // Ts (ring) no longer read
            const int rch = vp_rows_cl(kp, stg), rcp = rch + 4;
            const int nch = (nr + rch - 1) / rch;
            if (nch > 0) {
                vp_chunk(ring, Vz, ld, kp, rch, 0, min(rch, nr));
                asm volatile("cp.async.commit_group;\n" ::);
            }
            for (int c = 0; c < nch; ++c) {
                if (c + 1 < nch) vp_chunk(ring + ((c + 1) & 1) * stg, Vz, ld, kp, rch, c + 1, min(rch, nr - (c + 1) * rch));
                asm volatile("cp.async.commit_group;\n" ::);
                asm volatile("cp.async.wait_group 1;\n" ::);
                __syncthreads();
                const double* st = ring + (c & 1) * stg;
                const int nmt = min(rch, nr - c * rch) / 8;
                for (int mt = warp; mt < nmt; mt += PNW) {
                    const int rr = c * rch + mt * 8;
                    double c0 = Cb[(2 * kr) * RP + rr + rn], c1 = Cb[(2 * kr + 1) * RP + rr + rn];
#pragma unroll
                    for (int t = 0; t < 14; ++t)
                        if (t < ksteps) dmma8(c0, c1, st[(t * 4 + kr) * rcp + mt * 8 + rn], zb[t]);
                    Cb[(2 * kr) * RP + rr + rn] = c0;
                    Cb[(2 * kr + 1) * RP + rr + rn] = c1;
                }
                __syncthreads();
            }
        }
        __syncthreads();
    }

    // C. factor the 8 columns: one cluster-wide reduction per column
    for (int c = 0; c < 8; ++c) {
        const int d = d0 + c;                 // panel-relative row of the diagonal entry
        const int zo = d / Rq, dl = d - zo * Rq;
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.0;
        for (int r = max(0, d + 1 - r0) + tid; r < nr; r += PNT) {
            const double x = Cb[c * RP + r];
            v[0] += x * x;
#pragma unroll
            for (int c2 = 1; c2 < 8; ++c2)
                if (c + c2 < 8) v[c2] += x * Cb[(c + c2) * RP + r];
        }
        block_sum<8>(v, red, tot);
        if (tid < 16) {
            double p = 0.0;
            if (tid < 8) p = tot[tid];
            else if (z == zo) p = (tid == 8) ? Cb[c * RP + dl] : ((c + tid - 8 < 8) ? Cb[(c + tid - 8) * RP + dl] : 0.0);
            pay[tid] = p;
        }
        __syncthreads();
        const double* buf = exchange(pay, 16);
        double ts[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double s = 0.0;
            for (int q = 0; q < CL; ++q) s += buf[q * XN + k];
            ts[k] = s;
        }
        const double x0 = buf[zo * XN + 8];
        const double nrm = sqrt(x0 * x0 + ts[0]);
        double alpha = x0, tau = 0.0, scale = 0.0;
        if (nrm != 0.0) {
            alpha = x0 >= 0.0 ? -nrm : nrm;
            scale = 1.0 / (x0 - alpha);
            tau = (alpha - x0) / alpha;
        }
        double w[8], yd[8];
#pragma unroll
        for (int c2 = 1; c2 < 8; ++c2) {
            yd[c2] = (c + c2 < 8) ? buf[zo * XN + 8 + c2] : 0.0;
            w[c2] = tau * (yd[c2] + scale * ts[c2]);
        }
        if (tau != 0.0) {
            for (int r = max(0, d + 1 - r0) + tid; r < nr; r += PNT) {
                const double x = Cb[c * RP + r];
                const double vs = scale * x;
#pragma unroll
                for (int c2 = 1; c2 < 8; ++c2)
                    if (c + c2 < 8) Cb[(c + c2) * RP + r] -= w[c2] * vs;
                Cb[c * RP + r] = vs;
            }
        }
        if (tid == 0) {
            if (z == zo) {
#pragma unroll
                for (int c2 = 1; c2 < 8; ++c2)
                    if (c + c2 < 8) Cb[(c + c2) * RP + dl] = yd[c2] - w[c2];
                Cb[c * RP + dl] = alpha;
            }
            taus[c] = tau;
        }
        __syncthreads();
    }

    // D. write back R (upper) + V (below the diagonal) of own rows, and tau
    for (int c = 0; c < 8; ++c) {
        double2* dst = reinterpret_cast<double2*>(A + (int64_t)(jb + c) * ld + j0 + r0);
        for (int r2 = tid; r2 < nr / 2; r2 += PNT) dst[r2] = make_double2(Cb[c * RP + 2 * r2], Cb[c * RP + 2 * r2 + 1]);
    }
    if (z == 0 && tid < 8) a.tau[(int64_t)sl * a.M + jb + tid] = taus[tid];
    __syncthreads();
    // E. explicit V of the block (zeros above, unit diagonal) on own rows -> smem and Vbuf
    for (int c = 0; c < 8; ++c) {
        const int d = d0 + c;
        double2* dst = reinterpret_cast<double2*>(V + (int64_t)(kp + c) * ld + j0 + r0);
        for (int r2 = tid; r2 < nr / 2; r2 += PNT) {
            double v2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 2 * r2 + e, gr = r0 + r;
                v2[e] = gr < d ? 0.0 : (gr == d ? 1.0 : Cb[c * RP + r]);
                Cb[c * RP + r] = v2[e];
            }
            dst[r2] = make_double2(v2[0], v2[1]);
        }
    }
    __syncthreads();
    // F. T of the block from the (all-reduced) Gram of V_b
    {
        double g[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) g[k] = 0.0;
        for (int r = max(0, d0 - r0) + tid; r < nr; r += PNT) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = Cb[c * RP + r];
            int k = 0;
#pragma unroll
            for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
                for (int c2 = c1 + 1; c2 < 8; ++c2) g[k++] += x[c1] * x[c2];
        }
        block_sum<28>(g, red, tot);
        const double* buf = exchange(tot, 28);
        if (tid < 32) {
            const int r = tid & 7;
            double gs[28];
#pragma unroll
            for (int k = 0; k < 28; ++k) {
                double s = 0.0;
                for (int q = 0; q < CL; ++q) s += buf[q * XN + k];
                gs[k] = s;
            }
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) {
                            const int gi = (k * (15 - k)) / 2 + (i - k - 1);
                            s += trow[k] * gs[gi];
                        }
                    trow[i] = -taus[i] * s;
                }
            }
            if (tid < 8)
#pragma unroll
                for (int i = 0; i < 8; ++i) Tbb[i * 8 + r] = trow[i];
        }
        __syncthreads();
    }
    // G. T[0:kp, kp:kp+8] = -T Y, Y = (V_prev^T V_b) Tbb
    if (kp > 0) {
        vt_block_cl(Vz, ld, nr, kp, Cb, RP, Wsm, ring, Zsm, stg);
        __syncthreads();
        const double* buf = exchange(Wsm, kp * 8);
        for (int i = tid; i < kp * 8; i += PNT) {
            double v = 0.0;
            for (int s = 0; s < CL; ++s) v += buf[s * XN + i];
            Wsm[i] = v;
        }
        __syncthreads();
        if (z == 0) {
            for (int t = tid; t < kp * 8; t += PNT) {
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = 0; k <= c; ++k) s += Wsm[k * kp + r] * Tbb[c * 8 + k];
                Zsm[c * kp + r] = s;
            }
            double* Ts = ring;
            for (int t = tid; t < kp * kp; t += PNT) {
                const int r = t % kp, c = t / kp;
                Ts[c * kp + r] = r <= c ? T[c * ELM_NB + r] : 0.0;
            }
            __syncthreads();
            for (int t = tid; t < kp * 8; t += PNT) {
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = r; k < kp; ++k) s += Ts[k * kp + r] * Zsm[c * kp + k];
                T[(kp + c) * ELM_NB + r] = -s;
            }
        }
    }
    if (z == 0) {
        for (int t = tid; t < 64; t += PNT) {
            const int r = t % 8, c = t / 8;
            T[(kp + c) * ELM_NB + kp + r] = Tbb[c * 8 + r];
        }
        const int c = tid / ELM_NB, r = tid % ELM_NB;  // 512 threads = 8 columns x 64 rows
        if (r >= kp + 8) T[(kp + c) * ELM_NB + r] = 0.0;
    }
    cl.sync();  // no CTA leaves while others may still write into its shared memory
}

// ------------------------------------------------------------------------------------------
// On-chip panel factorisation: one panel (nb <= 64 columns) of one subdomain on a cluster of 8
// CTAs (8 SMs).  CTA z holds rows [z Rq, (z+1) Rq) of ALL panel columns in shared memory
// (<= 190 KB at config 3), so the panel is read from and written to HBM once and nothing is
// streamed.  Right-looking inside the panel by 8-column blocks:
//   * column j: partial sums (||x||^2 below the diagonal, x . y for the block columns to its
//     right) over own rows -> ONE cluster all-reduce through distributed shared memory (every CTA
//     writes its partial into slot z of every CTA's buffer, one cluster barrier, every CTA sums
//     the slots in the same fixed order: deterministic, and identical alpha / tau everywhere);
//     then the rank-1 update of the block columns on own rows;
//   * block b: G = V_b^T A_panel (8 x nb, DMMA over own rows) -> ONE all-reduce.  G holds the
//     Gram entries of V_b against every earlier reflector and itself (kept for T) and
//     W = V_b^T C_rest; the rest of the panel is updated locally: C_rest -= V_b (T_b^T W).
// At the end every CTA writes its rows of R / V (in place) and of the explicit V (Vbuf); CTA 0
// assembles T (nb x nb) from the Gram entries and the taus (column recurrence of the compact-WY
// factor, by 8-column blocks).  Same Householder convention and formulas as k_panel_block.
// DESIGN.md §5.2.
// ------------------------------------------------------------------------------------------
// remote (distributed shared memory) async stores that complete on the receiver's mbarrier:
// an all-reduce costs one store burst and one local mbarrier wait, no cluster-wide barrier
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async2(uint32_t raddr, double x, double y, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
                 "d"(x), "d"(y), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n}\n" ::"r"(elmtma::su32(b)), "r"(parity)
        : "memory");
}

namespace p8 {
constexpr int CL = 8;      // CTAs per subdomain
constexpr int NT = 256;    // threads per CTA
constexpr int NW = NT / 32;
constexpr int XC = 16;     // column exchange: 8 partial sums + the diagonal row's 8 values
constexpr int XB = 512;    // block exchange: G (8 x 64)
}  // namespace p8

// rows per CTA: multiple of 16 (padded column stride Rq + 4 == 4 mod 16: conflict-free fragments)
__host__ __device__ __forceinline__ int p8_rq(int64_t R) { return (int)((R + 16 * p8::CL - 1) / (16 * p8::CL)) * 16; }
constexpr int P8_TAIL = 2 * 64 * 64 + 64 * 8;  // CTA 0's T assembly reuses the panel region
size_t panel8_smem(int64_t R, int nb) {
    const int64_t Rq = p8_rq(R);
    return (size_t)(std::max<int64_t>(nb * (Rq + 4), P8_TAIL) + 2 * p8::CL * p8::XC + p8::CL * p8::XB + p8::NW * 8 + 64 +
                    64 + 64 + 4) * 8;
}

__global__ void __cluster_dims__(p8::CL, 1, 1) __launch_bounds__(p8::NT, 1) k_panel_c8(PanelArgs a, int nb) {
    using namespace p8;
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    extern __shared__ __align__(16) double sm[];
    const int z = (int)cl.block_rank();
    const int sl = a.s_off + (int)blockIdx.x / CL;
    const int64_t ld = a.ld;
    const int j0 = a.j0;
    const int R = (int)(ld - j0);
    const int Rq = p8_rq(R);
    const int r0 = z * Rq, nr = max(0, min(Rq, R - r0));
    const int RP = Rq + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* Ap = sm;                    // [nb][RP] the panel, own rows
    double* xc = Ap + max(nb * RP, P8_TAIL);  // [2][CL][XC] column exchange (double-buffered)
    double* xb = xc + 2 * CL * XC;      // [CL][XB] block exchange; after the sum: Gs = slot 0, Zs = slot 1
    double* red = xb + CL * XB;         // [NW][8]
    double* taus = red + NW * 8;        // [64]
    double* Tb = taus + 64;             // [8][8] T of the current block: Tb[i*8 + r] = T_b(r, i)
    double* Rsv = Tb + 64;              // [64] R part of the current diagonal block
    uint64_t* mbx = reinterpret_cast<uint64_t*>(Rsv + 64);  // [3] mbarriers: column exchange x2, block exchange
    double* Gs = xb;
    double* Zs = xb + XB;               // [8][68]
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;

    // A. own rows of the panel
    for (int c = 0; c < nb; ++c) {
        const double* src = A + (int64_t)(j0 + c) * ld + j0 + r0;
        for (int r2 = tid; r2 < nr / 2; r2 += NT) {
            unsigned d = (unsigned)__cvta_generic_to_shared(Ap + c * RP + 2 * r2);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * r2));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) elmtma::mbar_init(mbx + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cl.sync();  // every CTA of the cluster has started, its mbarriers are initialised
    const uint32_t xc_s = elmtma::su32(xc), xb_s = elmtma::su32(xb), mbx_s = elmtma::su32(mbx);

    int xcnt = 0;  // column exchanges so far (buffer / mbarrier xcnt & 1, phase xcnt >> 1)
#ifdef ELM_PANEL_PROF
    long long q_col = 0, q_xw = 0, q_g = 0, q_upd = 0, q_t0 = clock64(), q_a, q_b;
    long long q_p[6] = {0, 0, 0, 0, 0, 0}, q_c;
#define QS(v) v = clock64()
#define QA(acc, from) acc += clock64() - from
#else
#define QS(v)
#define QA(acc, from)
#endif
    for (int b = 0; b < nb / 8; ++b) {
        const int jb = 8 * b;
        // B. the 8 columns of the block, one cluster all-reduce each
        QS(q_a);
        for (int c = 0; c < 8; ++c) {
            const int j = jb + c;           // panel column == panel-relative row of its diagonal
            const int zo = j / Rq, dl = j - zo * Rq;
            const int nk = 8 - c;
            const int jl = j - r0;          // local row of the diagonal (rows > jl take part)
            QS(q_c);
            // partial sums over own rows below the diagonal; thread t owns rows t, t + NT, ...
            // for the whole panel, so the column loop needs no trailing barrier
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = 0.0;
            for (int r = tid; r < nr; r += NT) {
                if (r <= jl) continue;
                const double x = Ap[j * RP + r];
                v[0] += x * x;
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) v[k] += x * Ap[(j + k) * RP + r];
            }
            QA(q_p[0], q_c); QS(q_c);
            // warp sum of the 8 values by halving exchanges (9 shuffles): lanes 4k..4k+3 end
            // with the sum of value k
            {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                double h4[4], h2[2], h1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double snd = b4 ? v[i] : v[i + 4];
                    h4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double snd = b3 ? h4[i] : h4[i + 2];
                    h2[i] = (b3 ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
                }
                {
                    const double snd = b2 ? h2[0] : h2[1];
                    h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, snd, 4);
                }
                h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
                h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
                if ((lane & 3) == 0) red[warp * 8 + (lane >> 2)] = h1;
            }
            __syncthreads();
            QA(q_p[1], q_c); QS(q_c);
            const int xb_i = xcnt & 1;
            double* xcb = xc + xb_i * CL * XC;
            if (tid == 0) elmtma::mbar_expect(mbx + xb_i, CL * XC * 8);
            if (tid < CL * XC / 2) {
                const int dst = tid / (XC / 2), i = 2 * (tid % (XC / 2));
                double p[2] = {0.0, 0.0};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (i + e < 8) {
                        for (int w = 0; w < NW; ++w) p[e] += red[w * 8 + i + e];
                    } else if (z == zo && i + e - 8 < nk) {
                        p[e] = Ap[(j + i + e - 8) * RP + dl];
                    }
                }
                st_async2(mapa_u32(xc_s + (uint32_t)((xb_i * CL * XC + z * XC + i) * 8), dst), p[0], p[1],
                          mapa_u32(mbx_s + 8u * xb_i, dst));
            }
            QA(q_p[2], q_c);
            QS(q_b);
            mbar_wait_cluster(mbx + xb_i, (xcnt >> 1) & 1);
            QA(q_xw, q_b);
            ++xcnt;
            QS(q_c);
            // lane k < 8: sum of value k over the CTAs (fixed order); lane 8 + k: the diagonal
            // row's value in column j + k; then broadcast within the warp
            double mine = 0.0;
            if (lane < 8) {
                double s0 = xcb[0 * XC + lane] + xcb[1 * XC + lane], s1 = xcb[2 * XC + lane] + xcb[3 * XC + lane];
                double s2 = xcb[4 * XC + lane] + xcb[5 * XC + lane], s3 = xcb[6 * XC + lane] + xcb[7 * XC + lane];
                mine = (s0 + s1) + (s2 + s3);
            } else if (lane < 16) {
                mine = xcb[zo * XC + lane];
            }
            const double ts0 = __shfl_sync(0xffffffffu, mine, 0);
            const double x0 = __shfl_sync(0xffffffffu, mine, 8);
            const double nrm = sqrt(x0 * x0 + ts0);
            double alpha = x0, tau = 0.0, scale = 0.0;
            if (nrm != 0.0) {
                alpha = x0 >= 0.0 ? -nrm : nrm;
                scale = 1.0 / (x0 - alpha);
                tau = (alpha - x0) / alpha;
            }
            // lane k (1..7): w_k = tau (y_k + scale t_k), y_k from lane 8 + k
            const double ydl = __shfl_sync(0xffffffffu, mine, (lane & 7) + 8);
            const double wl = (lane >= 1 && lane < nk) ? tau * (ydl + scale * mine) : 0.0;
            double w[8], yd[8];
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                w[k] = __shfl_sync(0xffffffffu, wl, k);
                yd[k] = __shfl_sync(0xffffffffu, mine, k + 8);
            }
            QA(q_p[3], q_c); QS(q_c);
            if (tau != 0.0) {
                for (int r = tid; r < nr; r += NT) {
                    if (r <= jl) continue;
                    const double x = Ap[j * RP + r];
                    const double vs = scale * x;
#pragma unroll
                    for (int k = 1; k < 8; ++k)
                        if (k < nk) Ap[(j + k) * RP + r] -= w[k] * vs;
                    Ap[j * RP + r] = vs;
                }
            }
            if (z == zo && tid == dl % NT) {  // the owner of the diagonal row
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) Ap[(j + k) * RP + dl] = yd[k] - w[k];
                Ap[j * RP + dl] = alpha;
            }
            if (tid == 0) taus[j] = tau;
            QA(q_p[4], q_c);
        }
        __syncthreads();
        QA(q_col, q_a);
        QS(q_a);
        // C. explicit V_b in the diagonal block (unit diagonal, zeros above; R saved)
        const int zb = jb / Rq, db = jb - zb * Rq;
        if (z == zb && tid < 64) {
            const int r = tid & 7, i = tid >> 3;
            if (r <= i) {
                Rsv[tid] = Ap[(jb + i) * RP + db + r];
                Ap[(jb + i) * RP + db + r] = r == i ? 1.0 : 0.0;
            }
        }
        __syncthreads();
        // D. G = V_b^T A_panel over own rows >= jb (DMMA; warp w: columns [8w, 8w+8)), all-reduced
        const int kb0 = max(0, jb - r0);
        const int ntile = nb / 8;
        if (tid == 0) elmtma::mbar_expect(mbx + 2, CL * ntile * 64 * 8);
        if (warp < ntile) {
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
            const double* va = Ap + (jb + (lane >> 2)) * RP + (lane & 3);
            const double* vbp = Ap + (8 * warp + (lane >> 2)) * RP + (lane & 3);
            for (int k0 = kb0; k0 < nr; k0 += 8) {  // nr - kb0 is a multiple of 8
                dmma8(a0, a1, va[k0], vbp[k0]);
                dmma8(b0, b1, va[k0 + 4], vbp[k0 + 4]);
            }
            const int gi = (lane >> 2) * 64 + 8 * warp + 2 * (lane & 3);
#pragma unroll
            for (int dst = 0; dst < CL; ++dst)
                st_async2(mapa_u32(xb_s + (uint32_t)((z * XB + gi) * 8), dst), a0 + b0, a1 + b1, mapa_u32(mbx_s + 16u, dst));
        }
        mbar_wait_cluster(mbx + 2, b & 1);
        double gsum[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + h * NT;
            double s = 0.0;
            if ((e & 63) < nb)
                for (int q = 0; q < CL; ++q) s += xb[q * XB + e];
            gsum[h] = s;
        }
        __syncthreads();
        Gs[tid] = gsum[0];
        Gs[tid + NT] = gsum[1];
        __syncthreads();
        // E. T_b (8 x 8) from the block's Gram (Gs[k][jb + i], k < i) and its taus; CTA 0 keeps
        //    the Gram entries of V_b against all earlier reflectors for T (global scratch in Tbuf)
        if (tid < 8) {
            const int r = tid;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[jb + i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) s += trow[k] * Gs[k * 64 + jb + i];
                    trow[i] = -taus[jb + i] * s;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Tb[i * 8 + r] = trow[i];
        }
        if (z == 0)
            for (int t = tid; t < 8 * (jb + 8); t += NT) {
                const int i = t / (jb + 8), k = t % (jb + 8);
                if (k < jb + i) T[(jb + i) * ELM_NB + k] = Gs[i * 64 + k];  // S(k, jb+i) = v_k . v_{jb+i}
            }
        __syncthreads();
        QA(q_g, q_a);
        QS(q_a);
        // F. Z = T_b^T W on the columns right of the block; C_rest -= V_b Z on own rows >= jb
        const int c1 = jb + 8, ncr = nb - c1;
        if (ncr > 0) {
            for (int t = tid; t < 8 * ncr; t += NT) {
                const int i = t / ncr, col = c1 + t % ncr;
                double s = 0.0;
                for (int k = 0; k <= i; ++k) s += Tb[i * 8 + k] * Gs[k * 64 + col];
                Zs[i * 68 + col] = s;
            }
            __syncthreads();
            const int nmt = (nr - kb0) / 8, nnt = ncr / 8;
            const int kr = lane & 3, rn = lane >> 2;
            for (int it = warp; it < nmt * nnt; it += NW) {
                const int mt = it % nmt, nt = it / nmt;
                const int rb0 = kb0 + 8 * mt, cb = c1 + 8 * nt;
                double c0 = Ap[(cb + 2 * kr) * RP + rb0 + rn], c1v = Ap[(cb + 2 * kr + 1) * RP + rb0 + rn];
#pragma unroll
                for (int ks = 0; ks < 2; ++ks)
                    dmma8(c0, c1v, Ap[(jb + 4 * ks + kr) * RP + rb0 + rn], -Zs[(4 * ks + kr) * 68 + cb + rn]);
                Ap[(cb + 2 * kr) * RP + rb0 + rn] = c0;
                Ap[(cb + 2 * kr + 1) * RP + rb0 + rn] = c1v;
            }
            __syncthreads();
        }
        // G. restore R in the diagonal block
        if (z == zb && tid < 64) {
            const int r = tid & 7, i = tid >> 3;
            if (r <= i) Ap[(jb + i) * RP + db + r] = Rsv[tid];
        }
        __syncthreads();
        QA(q_upd, q_a);
    }
#ifdef ELM_PANEL_PROF
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 5) && (a.j0 == 256 || a.j0 == 1024))
        printf("P8PROF j0=%d cta=%d z=%d total %lld col %lld (xwait %lld) gblk %lld upd %lld | partial %lld shfl+sync %lld send %lld param %lld apply+sync %lld\n", a.j0, blockIdx.x, z,
               clock64() - q_t0, q_col, q_xw, q_g, q_upd, q_p[0], q_p[1], q_p[2], q_p[3], q_p[4]);
#endif

    // H. write back R + V (in place) and the explicit V of own rows; tau
    for (int c = 0; c < nb; ++c) {
        double2* dst = reinterpret_cast<double2*>(A + (int64_t)(j0 + c) * ld + j0 + r0);
        double2* dv = reinterpret_cast<double2*>(V + (int64_t)c * ld + j0 + r0);
        for (int r2 = tid; r2 < nr / 2; r2 += NT) {
            const double x0 = Ap[c * RP + 2 * r2], x1 = Ap[c * RP + 2 * r2 + 1];
            dst[r2] = make_double2(x0, x1);
            const int g0 = r0 + 2 * r2;
            dv[r2] = make_double2(g0 < c ? 0.0 : (g0 == c ? 1.0 : x0), g0 + 1 < c ? 0.0 : (g0 + 1 == c ? 1.0 : x1));
        }
    }
    if (z != 0) return;
    if (tid < nb) a.tau[(int64_t)sl * a.M + j0 + tid] = taus[tid];
    // I. CTA 0: T = compact-WY factor of the panel from S = strictly upper part of V^T V:
    //    T(i,i) = tau_i; by blocks, T[0:kp, kp:kp+8] = -T[0:kp,0:kp] S[0:kp, kp:kp+8] T_b
    __syncthreads();
    double* Ss = sm;                 // [64][64] column-major (panel smem is free now)
    double* Ts = sm + 64 * 64;       // [64][64]
    double* Ys = Ts + 64 * 64;       // [64][8]
    for (int t = tid; t < 64 * 64; t += NT) {
        const int r = t & 63, c = t >> 6;
        Ss[t] = (r < c && c < nb) ? T[t] : 0.0;
        Ts[t] = 0.0;
    }
    __syncthreads();
    for (int b = 0; b < nb / 8; ++b) {
        const int kp = 8 * b;
        if (tid < 8) {  // T_b
            const int r = tid;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[kp + i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) s += trow[k] * Ss[(kp + i) * 64 + kp + k];
                    trow[i] = -taus[kp + i] * s;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Ts[(kp + i) * 64 + kp + r] = trow[i];
        }
        __syncthreads();
        if (kp > 0) {
            for (int t = tid; t < kp * 8; t += NT) {  // Y = S[0:kp, kp:kp+8] T_b
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = 0; k <= c; ++k) s += Ss[(kp + k) * 64 + r] * Ts[(kp + c) * 64 + kp + k];
                Ys[c * 64 + r] = s;
            }
            __syncthreads();
            for (int t = tid; t < kp * 8; t += NT) {  // T[0:kp, kp+c] = -T[0:kp,0:kp] Y
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = r; k < kp; ++k) s += Ts[k * 64 + r] * Ys[c * 64 + k];
                Ts[(kp + c) * 64 + r] = -s;
            }
            __syncthreads();
        }
    }
    for (int t = tid; t < 64 * 64; t += NT) T[t] = Ts[t];
}


// ------------------------------------------------------------------------------------------
// k_panel_c8 with the panel in tensor memory (k_panel_c8t): the 8-CTA cluster panel of small
// slabs, each CTA's rows of all panel columns in TMEM (row r = 128 g + 32 q + lane -> TMEM lane
// 32 q + lane, columns [128 g, 128 g + 128): 64 doubles), so the CTA needs ~116 KB of shared
// memory and shares its SM with a trailing-update CTA, as k_panel_t does for large slabs.  The
// block being factored is staged in shared memory (the column steps are k_panel_c8's), G =
// V_b^T A_panel is computed on staged 64-row chunks, and C_rest -= V_b Z runs on the TMEM rows.
// ------------------------------------------------------------------------------------------
namespace p8t {
constexpr int SMEM = 116 * 1024;
constexpr int GCH = 64;      // rows per staged chunk of the G pass
constexpr int GLD = 68;      // its column stride
}  // namespace p8t

__global__ void __cluster_dims__(p8::CL, 1, 1) __launch_bounds__(p8::NT, 2) k_panel_c8t(PanelArgs a, int nb) {
    using namespace p8;
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ uint32_t s_tbase;
    const int z = (int)cl.block_rank();
    const int sl = a.s_off + (int)blockIdx.x / CL;
    const int64_t ld = a.ld;
    const int j0 = a.j0;
    const int R = (int)(ld - j0);
    const int Rq = p8_rq(R);
    const int r0 = z * Rq, nr = max(0, min(Rq, R - r0));
    const int RP = Rq + 4;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int quarter = warp & 3, gpar = warp >> 2;
    const int ngr = (nr + 127) / 128;
    double* Bp = sm;                            // [8][RP] the block being factored, own rows
    double* Gst = Bp + 8 * RP;                  // [64][GLD] staged rows of the G pass
    double* xc = Gst + 64 * p8t::GLD;           // [2][CL][XC]
    double* xb = xc + 2 * CL * XC;              // [CL][XB]; after the sum: Gs = slot 0, Zs = slot 1
    double* red = xb + CL * XB;                 // [NW][8]
    double* taus = red + NW * 8;                // [64]
    double* Tb = taus + 64;                     // [8][8]
    double* Rsv = Tb + 64;                      // [64]
    uint64_t* mbx = reinterpret_cast<uint64_t*>(Rsv + 64);
    double* Gs = xb;
    double* Zs = xb + XB;                       // [8][68]
    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = s_tbase;
    auto row_of = [&](int g) { return 128 * g + 32 * quarter + lane; };
    auto taddr = [&](int g, int cb) { return tm_addr(tbase, quarter, 128 * g + 16 * cb); };
    const int ncb = nb / 8;

    // A. own rows of the panel -> TMEM (rows >= nr zero)
    for (int g = gpar; g < ngr; g += 2) {
        const int r = row_of(g);
        for (int cb = 0; cb < ncb; ++cb) {
            double v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = r < nr ? __ldcg(A + (int64_t)(j0 + 8 * cb + c) * ld + j0 + r0 + r) : 0.0;
            tm_st8_nw(taddr(g, cb), v);
        }
        tm_wait_st();
    }
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) elmtma::mbar_init(mbx + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cl.sync();
    const uint32_t xc_s = elmtma::su32(xc), xb_s = elmtma::su32(xb), mbx_s = elmtma::su32(mbx);
    int xcnt = 0;

    for (int b = 0; b < ncb; ++b) {
        const int jb = 8 * b;
        // stage the block (own rows) from TMEM
        for (int g = gpar; g < ngr; g += 2) {
            double v[8];
            tm_ld8(taddr(g, b), v);
            const int r = row_of(g);
            if (r < Rq)
#pragma unroll
                for (int c = 0; c < 8; ++c) Bp[c * RP + r] = v[c];
        }
        __syncthreads();
        // B. the 8 columns of the block, one cluster all-reduce each
        
        for (int c = 0; c < 8; ++c) {
            const int j = jb + c;           // panel column == panel-relative row of its diagonal
            const int zo = j / Rq, dl = j - zo * Rq;
            const int nk = 8 - c;
            const int jl = j - r0;          // local row of the diagonal (rows > jl take part)
            
            // partial sums over own rows below the diagonal; thread t owns rows t, t + NT, ...
            // for the whole panel, so the column loop needs no trailing barrier
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = 0.0;
            for (int r = tid; r < nr; r += NT) {
                if (r <= jl) continue;
                const double x = Bp[c * RP + r];
                v[0] += x * x;
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) v[k] += x * Bp[(c + k) * RP + r];
            }
             
            // warp sum of the 8 values by halving exchanges (9 shuffles): lanes 4k..4k+3 end
            // with the sum of value k
            {
                const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
                double h4[4], h2[2], h1;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double snd = b4 ? v[i] : v[i + 4];
                    h4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, snd, 16);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double snd = b3 ? h4[i] : h4[i + 2];
                    h2[i] = (b3 ? h4[i + 2] : h4[i]) + __shfl_xor_sync(0xffffffffu, snd, 8);
                }
                {
                    const double snd = b2 ? h2[0] : h2[1];
                    h1 = (b2 ? h2[1] : h2[0]) + __shfl_xor_sync(0xffffffffu, snd, 4);
                }
                h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
                h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
                if ((lane & 3) == 0) red[warp * 8 + (lane >> 2)] = h1;
            }
            __syncthreads();
             
            const int xb_i = xcnt & 1;
            double* xcb = xc + xb_i * CL * XC;
            if (tid == 0) elmtma::mbar_expect(mbx + xb_i, CL * XC * 8);
            if (tid < CL * XC / 2) {
                const int dst = tid / (XC / 2), i = 2 * (tid % (XC / 2));
                double p[2] = {0.0, 0.0};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (i + e < 8) {
                        for (int w = 0; w < NW; ++w) p[e] += red[w * 8 + i + e];
                    } else if (z == zo && i + e - 8 < nk) {
                        p[e] = Bp[(c + i + e - 8) * RP + dl];
                    }
                }
                st_async2(mapa_u32(xc_s + (uint32_t)((xb_i * CL * XC + z * XC + i) * 8), dst), p[0], p[1],
                          mapa_u32(mbx_s + 8u * xb_i, dst));
            }
            
            
            mbar_wait_cluster(mbx + xb_i, (xcnt >> 1) & 1);
            
            ++xcnt;
            
            // lane k < 8: sum of value k over the CTAs (fixed order); lane 8 + k: the diagonal
            // row's value in column j + k; then broadcast within the warp
            double mine = 0.0;
            if (lane < 8) {
                double s0 = xcb[0 * XC + lane] + xcb[1 * XC + lane], s1 = xcb[2 * XC + lane] + xcb[3 * XC + lane];
                double s2 = xcb[4 * XC + lane] + xcb[5 * XC + lane], s3 = xcb[6 * XC + lane] + xcb[7 * XC + lane];
                mine = (s0 + s1) + (s2 + s3);
            } else if (lane < 16) {
                mine = xcb[zo * XC + lane];
            }
            const double ts0 = __shfl_sync(0xffffffffu, mine, 0);
            const double x0 = __shfl_sync(0xffffffffu, mine, 8);
            const double nrm = sqrt(x0 * x0 + ts0);
            double alpha = x0, tau = 0.0, scale = 0.0;
            if (nrm != 0.0) {
                alpha = x0 >= 0.0 ? -nrm : nrm;
                scale = 1.0 / (x0 - alpha);
                tau = (alpha - x0) / alpha;
            }
            // lane k (1..7): w_k = tau (y_k + scale t_k), y_k from lane 8 + k
            const double ydl = __shfl_sync(0xffffffffu, mine, (lane & 7) + 8);
            const double wl = (lane >= 1 && lane < nk) ? tau * (ydl + scale * mine) : 0.0;
            double w[8], yd[8];
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                w[k] = __shfl_sync(0xffffffffu, wl, k);
                yd[k] = __shfl_sync(0xffffffffu, mine, k + 8);
            }
             
            if (tau != 0.0) {
                for (int r = tid; r < nr; r += NT) {
                    if (r <= jl) continue;
                    const double x = Bp[c * RP + r];
                    const double vs = scale * x;
#pragma unroll
                    for (int k = 1; k < 8; ++k)
                        if (k < nk) Bp[(c + k) * RP + r] -= w[k] * vs;
                    Bp[c * RP + r] = vs;
                }
            }
            if (z == zo && tid == dl % NT) {  // the owner of the diagonal row
#pragma unroll
                for (int k = 1; k < 8; ++k)
                    if (k < nk) Bp[(c + k) * RP + dl] = yd[k] - w[k];
                Bp[c * RP + dl] = alpha;
            }
            if (tid == 0) taus[j] = tau;
            
        }
        __syncthreads();
        
        
        // C. explicit V_b in the diagonal block (unit diagonal, zeros above; R saved)

        // C. explicit V_b in the diagonal block of the staged block (R saved)
        const int zb = jb / Rq, db = jb - zb * Rq;
        if (z == zb && tid < 64) {
            const int r = tid & 7, i = tid >> 3;
            if (r <= i) {
                Rsv[tid] = Bp[i * RP + db + r];
                Bp[i * RP + db + r] = r == i ? 1.0 : 0.0;
            }
        }
        __syncthreads();
        // D. G = V_b^T A_panel over own rows >= jb: staged 64-row chunks (block b's columns from
        //    the staged block, the others from TMEM), DMMA, then the cluster all-reduce
        const int kb0 = max(0, jb - r0);
        const int ntile = ncb;
        if (tid == 0) elmtma::mbar_expect(mbx + 2, CL * ntile * 64 * 8);
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        for (int ck = kb0 & ~(p8t::GCH - 1); ck < nr; ck += p8t::GCH) {
            // owner threads of rows [ck, ck + GCH): groups g = ck / 128, quarters of that half
            const int g = ck / 128;
            if ((g & 1) == gpar) {
                const int r = row_of(g);
                const bool in = r >= ck && r < ck + p8t::GCH;
                for (int cb = 0; cb < ncb; ++cb) {
                    double v[8];
                    tm_ld8(taddr(g, cb), v);
                    if (in) {
                        if (cb == b)
#pragma unroll
                            for (int c = 0; c < 8; ++c) v[c] = Bp[c * RP + r];
#pragma unroll
                        for (int c = 0; c < 8; ++c) Gst[(8 * cb + c) * p8t::GLD + r - ck] = r < nr ? v[c] : 0.0;
                    }
                }
            }
            __syncthreads();
            if (warp < ntile) {
                const double* va = Gst + (jb + (lane >> 2)) * p8t::GLD + (lane & 3);
                const double* vbp = Gst + (8 * warp + (lane >> 2)) * p8t::GLD + (lane & 3);
                const int k1 = min(p8t::GCH, nr - ck);
                for (int k0 = max(0, kb0 - ck); k0 < k1; k0 += 8) {
                    dmma8(a0, a1, va[k0], vbp[k0]);
                    dmma8(b0, b1, va[k0 + 4], vbp[k0 + 4]);
                }
            }
            __syncthreads();
        }
        if (warp < ntile) {
            const int gi = (lane >> 2) * 64 + 8 * warp + 2 * (lane & 3);
#pragma unroll
            for (int dst = 0; dst < CL; ++dst)
                st_async2(mapa_u32(xb_s + (uint32_t)((z * XB + gi) * 8), dst), a0 + b0, a1 + b1, mapa_u32(mbx_s + 16u, dst));
        }
        mbar_wait_cluster(mbx + 2, b & 1);
        double gsum[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int e = tid + h * NT;
            double s = 0.0;
            if ((e & 63) < nb)
                for (int q = 0; q < CL; ++q) s += xb[q * XB + e];
            gsum[h] = s;
        }
        __syncthreads();
        Gs[tid] = gsum[0];
        Gs[tid + NT] = gsum[1];
        __syncthreads();
        // E. T_b and the Gram entries for T (as k_panel_c8)
        if (tid < 8) {
            const int r = tid;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[jb + i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) s += trow[k] * Gs[k * 64 + jb + i];
                    trow[i] = -taus[jb + i] * s;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Tb[i * 8 + r] = trow[i];
        }
        if (z == 0)
            for (int t = tid; t < 8 * (jb + 8); t += NT) {
                const int i = t / (jb + 8), k = t % (jb + 8);
                if (k < jb + i) T[(jb + i) * ELM_NB + k] = Gs[i * 64 + k];
            }
        __syncthreads();
        // F. Z = T_b^T W; C_rest -= V_b Z on the TMEM rows >= jb (thread = row)
        const int c1 = jb + 8, ncr = nb - c1;
        if (ncr > 0) {
            for (int t = tid; t < 8 * ncr; t += NT) {
                const int i = t / ncr, col = c1 + t % ncr;
                double s = 0.0;
                for (int k = 0; k <= i; ++k) s += Tb[i * 8 + k] * Gs[k * 64 + col];
                Zs[i * 68 + col] = s;
            }
            __syncthreads();
            for (int g = gpar; g < ngr; g += 2) {
                const int r = row_of(g);
                const bool act = r < nr && r >= kb0;
                double vb[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) vb[i] = act ? Bp[i * RP + r] : 0.0;
                for (int cb = b + 1; cb < ncb; ++cb) {
                    double x[8];
                    tm_ld8(taddr(g, cb), x);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) s += vb[i] * Zs[i * 68 + 8 * cb + c];
                        x[c] -= s;
                    }
                    tm_st8_nw(taddr(g, cb), x);
                }
                tm_wait_st();
            }
        }
        // G. restore R in the diagonal block; the factored block back to TMEM
        if (z == zb && tid < 64) {
            const int r = tid & 7, i = tid >> 3;
            if (r <= i) Bp[i * RP + db + r] = Rsv[tid];
        }
        __syncthreads();
        for (int g = gpar; g < ngr; g += 2) {
            const int r = row_of(g);
            double v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = r < nr ? Bp[c * RP + r] : 0.0;
            tm_st8(taddr(g, b), v);
        }
        __syncthreads();
    }

    // H. write back R + V (in place) and the explicit V of own rows; tau
    for (int g = gpar; g < ngr; g += 2) {
        const int r = row_of(g);
        for (int cb = 0; cb < ncb; ++cb) {
            double x[8];
            tm_ld8(taddr(g, cb), x);
            if (r < nr) {
                const int gr = r0 + r;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int col = 8 * cb + c;
                    A[(int64_t)(j0 + col) * ld + j0 + gr] = x[c];
                    V[(int64_t)col * ld + j0 + gr] = gr < col ? 0.0 : (gr == col ? 1.0 : x[c]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
    if (z != 0) return;
    if (tid < nb) a.tau[(int64_t)sl * a.M + j0 + tid] = taus[tid];
    // I. CTA 0: T = compact-WY factor of the panel from S = strictly upper part of V^T V:
    //    T(i,i) = tau_i; by blocks, T[0:kp, kp:kp+8] = -T[0:kp,0:kp] S[0:kp, kp:kp+8] T_b
    __syncthreads();
    double* Ss = sm;                 // [64][64] column-major (panel smem is free now)
    double* Ts = sm + 64 * 64;       // [64][64]
    double* Ys = Ts + 64 * 64;       // [64][8]
    for (int t = tid; t < 64 * 64; t += NT) {
        const int r = t & 63, c = t >> 6;
        Ss[t] = (r < c && c < nb) ? T[t] : 0.0;
        Ts[t] = 0.0;
    }
    __syncthreads();
    for (int b = 0; b < nb / 8; ++b) {
        const int kp = 8 * b;
        if (tid < 8) {  // T_b
            const int r = tid;
            double trow[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) trow[i] = (i == r) ? taus[kp + i] : 0.0;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                if (r < i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (k >= r && k < i) s += trow[k] * Ss[(kp + i) * 64 + kp + k];
                    trow[i] = -taus[kp + i] * s;
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) Ts[(kp + i) * 64 + kp + r] = trow[i];
        }
        __syncthreads();
        if (kp > 0) {
            for (int t = tid; t < kp * 8; t += NT) {  // Y = S[0:kp, kp:kp+8] T_b
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = 0; k <= c; ++k) s += Ss[(kp + k) * 64 + r] * Ts[(kp + c) * 64 + kp + k];
                Ys[c * 64 + r] = s;
            }
            __syncthreads();
            for (int t = tid; t < kp * 8; t += NT) {  // T[0:kp, kp+c] = -T[0:kp,0:kp] Y
                const int r = t % kp, c = t / kp;
                double s = 0.0;
                for (int k = r; k < kp; ++k) s += Ts[k * 64 + r] * Ys[c * 64 + k];
                Ts[(kp + c) * 64 + r] = -s;
            }
            __syncthreads();
        }
    }
    for (int t = tid; t < 64 * 64; t += NT) T[t] = Ts[t];

}

constexpr int PANEL_FIXED = 8 * 56 * 2 + 40 + 64 + 8;  // Wsm, Zsm, tot, Tbb, taus (doubles)
// V_prev ring of the panel-block kernel for R resident rows: all shared memory the block leaves
int panel_ring(int64_t R, int smem_optin) {
    const int64_t r = ((int64_t)smem_optin / 8 - 8 * (R + 4) - PANEL_FIXED) & ~(int64_t)(2 * VNS - 1);
    return (int)std::max<int64_t>(r, RED_ELEMS);
}
size_t panel_smem_bytes(int64_t R, int ring) { return (size_t)(8 * (R + 4) + PANEL_FIXED + ring) * 8; }
int panelp_ring(int64_t R, int smem_optin) {
    const int64_t r = ((int64_t)smem_optin / 8 - 8 * (R + 4) - PANELP_FIXED) & ~(int64_t)(2 * VNS - 1);
    return (int)std::max<int64_t>(r, RED_ELEMS);
}
size_t panelp_smem_bytes(int64_t R, int ring) { return (size_t)(8 * (R + 4) + PANELP_FIXED + ring) * 8; }
int panelt_ring(int smem = pt::SMEM) { return (smem / 8 - PANELT_FIXED) & ~(2 * VNS - 1); }
// panels of <= 2048 rows allocate 256 TMEM columns and 112 KB of shared memory, so that two panel
// CTAs can share an SM (ELMDDM_PANEL_PAIR=0: the whole TMEM and 116 KB, one per SM)
constexpr int PT_SMEM_PAIR = 112 * 1024;

}  // namespace

namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
}  // namespace

// 3-D fp64 tensor map {d0 rows (contiguous), d1 columns (stride d0*8 B), d2 batches (stride s2 elems)},
// box 16 x 64 x 1, 128B swizzle, out-of-bounds elements read as zero.
bool elm_encode_tmap_s(CUtensorMap* tm, const double* base, int64_t d0, int64_t d1, int64_t d2, int64_t s1,
                       int64_t s2) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (d0 < 1 || d1 < 1 || d2 < 1 || (s1 * 8) % 16 != 0 || (s2 * 8) % 16 != 0 || ((uintptr_t)base & 15) != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    cuuint64_t strides[2] = {(cuuint64_t)(s1 * 8), (cuuint64_t)(s2 * 8)};
    cuuint32_t box[3] = {16, 64, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, ELM_SWIZZLE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool elm_encode_tmap(CUtensorMap* tm, const double* base, int64_t d0, int64_t d1, int64_t d2, int64_t s2) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
    cuuint64_t strides[2] = {(cuuint64_t)(d0 * 8), (cuuint64_t)(s2 * 8)};
    cuuint32_t box[3] = {16, 64, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, ELM_SWIZZLE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// SPEC factorize_ls: "warns (not errors) when sigma_min/sigma_max < 1e-14".  |R11_ii| bound the
// singular values of K^s from inside (sigma_min <= min |R11_ii|, max |R11_ii| <= sigma_max), so
// min |R11_ii| < 1e-14 max |R11_ii| is a sufficient condition (no false warnings).  A non-finite
// diagonal (a NaN / Inf anywhere in K^s reaches it through the Householder norms) is an error
// (numerical breakdown on non-finite values): ELMDDM_ENUMERIC, info
// ELM_INFO_NONFINITE_QR - s.  grid S.
static __global__ void __launch_bounds__(256) k_rank_check(const double* __restrict__ Kaug, int64_t ld, int64_t ncols, int M,
                                                    int s_begin, ElmStatus* status) {
    __shared__ double smx[8], smn[8];
    const double* R = Kaug + (int64_t)blockIdx.x * ld * ncols;
    double mx = 0.0, mn = INFINITY;
    bool bad = false;
    for (int i = threadIdx.x; i < M; i += 256) {
        const double d = fabs(R[(int64_t)i * ld + i]);
        bad |= !isfinite(d);
        mx = fmax(mx, d);
        mn = fmin(mn, d);
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) elm_set_status(status, ELMDDM_ENUMERIC, ELM_INFO_NONFINITE_QR - (s_begin + (int)blockIdx.x));
        return;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smx[threadIdx.x >> 5] = mx;
        smn[threadIdx.x >> 5] = mn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            mx = fmax(mx, smx[w]);
            mn = fmin(mn, smn[w]);
        }
        if (!(mn > 1e-14 * mx)) elm_set_warning(status, ELMDDM_WRANK, s_begin + (int)blockIdx.x);
    }
}

cudaError_t run_local_factor(const elmddm_ctx* c, double* Kaug, double* tau, double* work, cudaStream_t st) {
    const int64_t S = c->sz.S, ld = c->sz.ld, ncols = c->sz.ncols;
    const int M = c->cfg.M;
    double* Vbuf = work;
    double* Tbuf = Vbuf + S * ELM_NB * ld;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    const size_t smax = panel_smem_bytes(ld, panel_ring(ld, optin));
    const bool blk_ok = smax <= (size_t)optin;  // the one-CTA block panel holds (ld - j0) x 8 in shared memory
    if (blk_ok &&
        (e = cudaFuncSetAttribute(k_panel_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax)) != cudaSuccess)
        return e;
    // 4-CTA cluster block panels: for small slabs (panel_cluster), and for panels too tall for one
    // CTA (the damped local LS of reading R29), with a ring stage sized to what fits
    // very tall local problems (the lattice's N <= 2 x 2): the cooperative grid panel
    const bool use_grid = c->panel_grid || (!blk_ok && cl_stage(ld, optin) == 0);
    const bool use_cl = !use_grid && (c->panel_cluster || !blk_ok);
    const int stg_cl = use_grid ? 0 : cl_stage(ld, optin);
    if (use_cl && stg_cl == 0) return cudaErrorInvalidValue;
    int gp_per = 0;
    if (use_grid) {
        if ((e = cudaFuncSetAttribute(k_panel_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, GP_SMEM)) != cudaSuccess)
            return e;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_panel_grid, gp::NT, GP_SMEM);
        const int64_t cap = std::min<int64_t>((int64_t)std::max(occ, 1) * c->nsm, 2LL * c->nsm);
        gp_per = (int)std::max<int64_t>(1, std::min<int64_t>(cap / S, (ld + 255) / 256));
        if (gp_per * S > cap) return cudaErrorInvalidValue;  // more subdomains than co-resident CTAs
    }
    const bool pp_ok = c->panel_merged && panelp_smem_bytes(ld, panelp_ring(ld, optin)) <= (size_t)optin;
    const bool pt_ok = c->panel_tmem && (ld + 127) / 128 * 16 <= 512;
    if (pt_ok && (e = cudaFuncSetAttribute(k_panel_t, cudaFuncAttributeMaxDynamicSharedMemorySize, pt::SMEM)) != cudaSuccess)
        return e;
    if (pp_ok && (e = cudaFuncSetAttribute(k_panel_p, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess)
        return e;
    if (stg_cl > 0 &&
        (e = cudaFuncSetAttribute(k_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)panel_cl_smem(((ld + 32 * pcl::CL - 1) / (32 * pcl::CL)) * 32, stg_cl))) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k_wy_update, cudaFuncAttributeMaxDynamicSharedMemorySize, wy::SMEM)) != cudaSuccess)
        return e;
    // (the TMEM variant of the cluster panel measured slower: config 3 slabs of 32 / 16
    // subdomains 26.6 -> 28.9 / 15.0 -> 16.6 ms; opt-in ELMDDM_PANEL8_TMEM=1)
    const bool p8t_ok = c->panel8 && c->panel8_tmem && p8_rq(ld) <= 512;
    const bool p8_ok = !p8t_ok && c->panel8 && panel8_smem(ld, std::min<int64_t>(M, ELM_NB)) <= (size_t)optin;
    if (p8t_ok &&
        (e = cudaFuncSetAttribute(k_panel_c8t, cudaFuncAttributeMaxDynamicSharedMemorySize, p8t::SMEM)) != cudaSuccess)
        return e;
    if (p8_ok && (e = cudaFuncSetAttribute(k_panel_c8, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess)
        return e;
    // (experiment hook) ELMDDM_WY_SMEM: dynamic shared memory of the trailing update, to force
    // one CTA per SM and measure the single-CTA throughput
    int wy_smem = wyt::SMEM;
    if (const char* env = getenv("ELMDDM_WY_SMEM")) wy_smem = std::max(wyt::SMEM, atoi(env));
    if ((e = cudaFuncSetAttribute(k_wy_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, wy_smem)) != cudaSuccess)
        return e;
    // TMA descriptors: K_aug {ld, ncols, S} and V {ld, nb, S} (columns >= nb read as zero), boxes 16 x 64
    CUtensorMap tmK, tmV64, tmVlast;
    const int nb_last = M % ELM_NB == 0 ? ELM_NB : M % ELM_NB;
    bool use_tma = c->use_tma && elm_encode_tmap(&tmK, Kaug, ld, ncols, S, ld * ncols) &&
                   elm_encode_tmap(&tmV64, Vbuf, ld, ELM_NB, S, ELM_NB * ld) &&
                   elm_encode_tmap(&tmVlast, Vbuf, ld, nb_last, S, ELM_NB * ld);
    // implicit E_Gamma tiles of the first trailing update (the assembly did not write them)
    const int pp_rows = (int)(c->cfg.p * c->cfg.p);
    const EsynArgs esyn{(int)c->sz.e_impl_begin, (int)c->sz.e_impl_end, M, (int)c->cfg.q, pp_rows, (int)c->cfg.P,
                        (int)c->cfg.s_begin, (int)(c->cfg.layout == 1)};
    const EsynArgs esyn_off{0, 0, M, (int)c->cfg.q, pp_rows, (int)c->cfg.P, (int)c->cfg.s_begin, 0};
    if (!use_tma && esyn.e_end > esyn.e_begin) return cudaErrorInvalidValue;  // create() ties implicit_e to use_tma
    // Subdomain groups on separate streams: the latency-bound panel factorisation of one group
    // overlaps the DMMA-bound trailing updates of the others (the factorisations of different
    // subdomains are independent).
    // (with timing enabled the groups are serialised so that per-class event times do not overlap)
    const int ngroups = (c->timing || use_grid) ? 1 : (int)std::min<int64_t>(c->qr_groups, S);
    std::vector<cudaStream_t> streams(ngroups, st), pstr(ngroups, st);
    const bool prio = ngroups > 1 && c->panel_prio && c->panel_tmem;
    if (ngroups > 1) {
        if ((e = c->ensure_streams(ngroups)) != cudaSuccess) return e;
        if (prio && (e = c->ensure_panel_streams(ngroups)) != cudaSuccess) return e;
        cudaEventRecord(c->ev_fork, st);
        for (int g = 0; g < ngroups; ++g) {
            streams[g] = c->gstreams[g];
            cudaStreamWaitEvent(streams[g], c->ev_fork, 0);
            pstr[g] = streams[g];
            if (prio) {
                pstr[g] = c->pstreams[g];
                cudaStreamWaitEvent(pstr[g], c->ev_fork, 0);
            }
        }
    }
    for (int j0 = 0; j0 < M; j0 += ELM_NB) {
        const int nb = (M - j0) < ELM_NB ? (M - j0) : ELM_NB;
        const int ring = panel_ring(ld - j0, optin);
        const size_t smem = panel_smem_bytes(ld - j0, ring);
        const size_t smem_cl = panel_cl_smem(((ld - j0 + 32 * pcl::CL - 1) / (32 * pcl::CL)) * 32, stg_cl);
        const int n_tr = (int)(ncols - (j0 + nb));
        for (int g = 0; g < ngroups; ++g) {
            const int g0 = (int)(S * g / ngroups), g1 = (int)(S * (g + 1) / ngroups);
            if (g1 <= g0) continue;
            PanelArgs pa{Kaug, ld, ncols, tau, M, Vbuf, Tbuf, j0, 0, g0, ring};
            if (use_grid) {
                double* part = Tbuf + S * ELM_NB * ELM_NB;
                unsigned* cnt = reinterpret_cast<unsigned*>(part + (int64_t)gp_per * S * gp::NG);
                if ((e = cudaMemsetAsync(cnt, 0, sizeof(unsigned) * S, streams[g])) != cudaSuccess) return e;
                int nb_v = nb, per_v = gp_per;
                void* args[] = {(void*)&pa, (void*)&nb_v, (void*)&per_v, (void*)&part, (void*)&cnt};
                KTimer kt(c, ELMDDM_K_PANEL, streams[g]);
                if ((e = cudaLaunchCooperativeKernel((void*)k_panel_grid, dim3((unsigned)(gp_per * (g1 - g0))),
                                                     dim3(gp::NT), args, GP_SMEM, streams[g])) != cudaSuccess)
                    return e;
            } else if (p8t_ok) {
                if (prio && j0 > 0) cudaStreamWaitEvent(pstr[g], c->ev_wy[g], 0);
                {
                    KTimer kt(c, ELMDDM_K_PANEL, pstr[g]);
                    k_panel_c8t<<<(unsigned)((g1 - g0) * p8::CL), p8::NT, p8t::SMEM, pstr[g]>>>(pa, nb);
                    if ((e = cudaGetLastError()) != cudaSuccess) return e;
                }
                if (prio) {
                    cudaEventRecord(c->ev_panel[g], pstr[g]);
                    cudaStreamWaitEvent(streams[g], c->ev_panel[g], 0);
                }
            } else if (p8_ok) {
                KTimer kt(c, ELMDDM_K_PANEL, streams[g]);
                k_panel_c8<<<(unsigned)((g1 - g0) * p8::CL), p8::NT, panel8_smem(ld - j0, nb), streams[g]>>>(pa, nb);
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            } else if (pt_ok && !use_cl) {
                // (prio: the panel runs on the group's high-priority stream after the group's
                // previous trailing update; the next trailing update waits for it)
                if (prio && j0 > 0) cudaStreamWaitEvent(pstr[g], c->ev_wy[g], 0);
                {
                    KTimer kt(c, ELMDDM_K_PANEL, pstr[g]);
                    PanelArgs pp = pa;
                    const bool pair = c->panel_pair && (ld + 127) / 128 * 16 <= 256;
                    pp.ring = panelt_ring(pair ? PT_SMEM_PAIR : pt::SMEM);
                    pp.tcols = pair ? 256 : 512;
                    k_panel_t<<<(unsigned)(g1 - g0), pt::NT, pair ? PT_SMEM_PAIR : pt::SMEM, pstr[g]>>>(pp, nb);
                    if ((e = cudaGetLastError()) != cudaSuccess) return e;
                }
                if (prio) {
                    cudaEventRecord(c->ev_panel[g], pstr[g]);
                    cudaStreamWaitEvent(streams[g], c->ev_panel[g], 0);
                }
            } else if (pp_ok && !use_cl) {
                KTimer kt(c, ELMDDM_K_PANEL, streams[g]);
                PanelArgs pp = pa;
                pp.ring = panelp_ring(ld - j0, optin);
                k_panel_p<<<(unsigned)(g1 - g0), PNT, panelp_smem_bytes(ld - j0, pp.ring), streams[g]>>>(pp, nb);
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            }
            for (int blk = 0; !use_grid && !p8_ok && !p8t_ok && !((pp_ok || pt_ok) && !use_cl) && blk < nb / ELM_BB; ++blk) {
                pa.blk = blk;
                KTimer kt(c, ELMDDM_K_PANEL, streams[g]);
                if (use_cl) {
                    PanelArgs pc = pa;
                    pc.ring = stg_cl;
                    k_panel_cl<<<(unsigned)((g1 - g0) * pcl::CL), PNT, smem_cl, streams[g]>>>(pc);
                } else
                    k_panel_block<<<(unsigned)(g1 - g0), PNT, smem, streams[g]>>>(pa);
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            }
            if (n_tr <= 0) continue;
            dim3 grid((unsigned)((n_tr + 63) / 64), (unsigned)(g1 - g0));
            KTimer kt(c, ELMDDM_K_GEMM_QR, streams[g]);
            if (use_tma)
                k_wy_tma<<<grid, wyt::NT, wy_smem, streams[g]>>>(nb == ELM_NB ? tmV64 : tmVlast, tmK, Tbuf, ld, j0, nb,
                                                                   j0 + nb, n_tr, g0, j0 == 0 ? esyn : esyn_off,
                                                                   c->wy_rev3 | (c->wy_hint3 << 1));
            else
                k_wy_update<<<grid, wy::NT, wy::SMEM, streams[g]>>>(Vbuf, Tbuf, Kaug, ld, ncols, j0, nb, j0 + nb, n_tr, g0);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            if (prio) cudaEventRecord(c->ev_wy[g], streams[g]);
        }
    }
    if (ngroups > 1) {
        for (int g = 0; g < ngroups; ++g) {
            if (prio) {  // the last panel may end after the group's last trailing update
                cudaEventRecord(c->ev_panel[g], pstr[g]);
                cudaStreamWaitEvent(streams[g], c->ev_panel[g], 0);
            }
            cudaEventRecord(c->ev_join[g], streams[g]);
            cudaStreamWaitEvent(st, c->ev_join[g], 0);
        }
    }
    // rank warning (ELMDDM_WRANK): min |R11_ii| < 1e-14 max |R11_ii| in some subdomain
    {
        KTimer kt(c, ELMDDM_K_PANEL, st);
        k_rank_check<<<(unsigned)S, 256, 0, st>>>(Kaug, ld, ncols, M, (int)c->cfg.s_begin, c->d_status);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int panel_cl_stage(int64_t ld, int smem_optin) { return cl_stage(ld, smem_optin); }

#ifdef ELM_QR_PROF
extern "C" int elmddm_debug_qr_prof(void* host, int n) {  // n records (host: [n][4] u64); returns the count
    unsigned cnt = 0;
    cudaMemcpyFromSymbol(&cnt, g_qr_n, sizeof(unsigned));
    if (host && n > 0) cudaMemcpyFromSymbol(host, g_qr_prof, sizeof(unsigned long long) * 4 * (size_t)n);
    return (int)cnt;
}
extern "C" int elmddm_debug_qr_prof_reset() {
    unsigned z = 0;
    return (int)cudaMemcpyToSymbol(g_qr_n, &z, sizeof(unsigned));
}
#endif
