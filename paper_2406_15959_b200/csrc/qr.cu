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

// G (kp x 8, smem, col-major ld kp) = Vp^T X, Vp = V columns [0, kp) rows [j0, ld) (global,
// explicit), X = 8 columns in smem (col-major, row stride R, rows relative to j0).
__device__ void vt_times_block(const double* __restrict__ Vp, int64_t ld, int R, int kp, const double* X, double* G) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ngroups = (kp + 3) / 4;
    for (int grp = warp; grp < ngroups; grp += PNW) {
        double acc[4][8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[a][c] = 0.0;
        const int cp0 = grp * 4;
        for (int r = lane; r < R; r += 32) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = X[c * R + r];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                if (cp0 + a < kp) {
                    double v = Vp[(int64_t)(cp0 + a) * ld + r];
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[a][c] += v * x[c];
                }
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double s = acc[a][c];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0 && cp0 + a < kp) G[c * kp + cp0 + a] = s;
            }
    }
}

__global__ void __launch_bounds__(PNT, 1) k_panel_block(PanelArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int sl = blockIdx.x;
    const int64_t ld = a.ld;
    const int j0 = a.j0, jb = j0 + ELM_BB * a.blk, kp = ELM_BB * a.blk;
    const int R = (int)(ld - j0);     // rows held: [j0, ld)
    const int d0 = jb - j0;           // local row of the block's first diagonal entry
    double* Cb = sm;                  // [8][R]
    double* Wsm = Cb + 8 * R;         // [8][kp]  (<= 8*56)
    double* Zsm = Wsm + 8 * 56;       // [8][kp]
    double* red = Zsm + 8 * 56;       // [PNW][36]
    double* tot = red + PNW * 36;     // [36]
    double* Tbb = tot + 40;           // [8][8]
    double* taus = Tbb + 64;          // [8]

    double* A = a.Kaug + (int64_t)sl * ld * a.ncols;
    double* V = a.Vbuf + (int64_t)sl * ELM_NB * ld;
    double* T = a.Tbuf + (int64_t)sl * ELM_NB * ELM_NB;
    const double* Vp = V + j0;        // column c of Vp at Vp + c*ld, rows relative to j0

    // load the block: rows [j0, ld) of columns [jb, jb+8)
    for (int c = 0; c < 8; ++c)
        for (int r = threadIdx.x; r < R; r += PNT) Cb[c * R + r] = A[(int64_t)(jb + c) * ld + j0 + r];
    __syncthreads();

    if (kp > 0) {
        // W = Vp^T Cb
        vt_times_block(Vp, ld, R, kp, Cb, Wsm);
        __syncthreads();
        // Z = T^T W  (T upper triangular kp x kp)
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int cp = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = 0; k <= cp; ++k) s += T[cp * ELM_NB + k] * Wsm[c * kp + k];
            Zsm[c * kp + cp] = s;
        }
        __syncthreads();
        // Cb -= Vp Z
        for (int r = threadIdx.x; r < R; r += PNT) {
            double acc[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = 0.0;
            for (int k = 0; k < kp; ++k) {
                double v = Vp[(int64_t)k * ld + r];
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[c] += v * Zsm[c * kp + k];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) Cb[c * R + r] -= acc[c];
        }
        __syncthreads();
    }

    // factor the 8 columns
    for (int c = 0; c < 8; ++c) {
        const int d = d0 + c;
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = 0.0;
        for (int r = d + 1 + threadIdx.x; r < R; r += PNT) {
            double x = Cb[c * R + r];
            v[0] += x * x;
#pragma unroll
            for (int c2 = 1; c2 < 8; ++c2)
                if (c + c2 < 8) v[c2] += x * Cb[(c + c2) * R + r];
        }
        block_sum<8>(v, red, tot);
        const double x0 = Cb[c * R + d];
        const double nrm = sqrt(x0 * x0 + tot[0]);
        double alpha = x0, tau = 0.0, scale = 0.0;
        if (nrm != 0.0) {
            alpha = x0 >= 0.0 ? -nrm : nrm;
            scale = 1.0 / (x0 - alpha);
            tau = (alpha - x0) / alpha;
        }
        // apply H = I - tau v v^T to the remaining columns of the block
        if (tau != 0.0) {
            for (int c2 = 1; c + c2 < 8; ++c2) {
                double yd = Cb[(c + c2) * R + d];
                double w = tau * (yd + scale * tot[c2]);
                for (int r = d + 1 + threadIdx.x; r < R; r += PNT) Cb[(c + c2) * R + r] -= w * scale * Cb[c * R + r];
                __syncthreads();  // all threads read yd before thread 0 writes it
                if (threadIdx.x == 0) Cb[(c + c2) * R + d] = yd - w;
            }
            for (int r = d + 1 + threadIdx.x; r < R; r += PNT) Cb[c * R + r] *= scale;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            Cb[c * R + d] = alpha;
            taus[c] = tau;
        }
        __syncthreads();
    }

    // write back R (upper) + V (below the diagonal) and tau
    for (int c = 0; c < 8; ++c)
        for (int r = threadIdx.x; r < R; r += PNT) A[(int64_t)(jb + c) * ld + j0 + r] = Cb[c * R + r];
    if (threadIdx.x < 8) a.tau[(int64_t)sl * a.M + jb + threadIdx.x] = taus[threadIdx.x];
    __syncthreads();
    // explicit V of the block (zeros above, unit diagonal) -> smem and Vbuf
    for (int c = 0; c < 8; ++c)
        for (int r = threadIdx.x; r < R; r += PNT) {
            const int d = d0 + c;
            double v = r < d ? 0.0 : (r == d ? 1.0 : Cb[c * R + r]);
            Cb[c * R + r] = v;
            V[(int64_t)(kp + c) * ld + j0 + r] = v;
        }
    __syncthreads();

    // T of the block: Tbb[i][i] = tau_i, Tbb[0:i, i] = -tau_i Tbb[0:i,0:i] (Vb^T v_i)[0:i]
    {
        double g[28];
#pragma unroll
        for (int k = 0; k < 28; ++k) g[k] = 0.0;
        for (int r = d0 + threadIdx.x; r < R; r += PNT) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = Cb[c * R + r];
            int k = 0;
#pragma unroll
            for (int c1 = 0; c1 < 8; ++c1)
#pragma unroll
                for (int c2 = c1 + 1; c2 < 8; ++c2) g[k++] += x[c1] * x[c2];
        }
        // reduce 28 values (reuse the 36-wide scratch)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int k = 0; k < 28; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) g[k] += __shfl_xor_sync(0xffffffffu, g[k], o);
        }
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 28; ++k) red[warp * 36 + k] = g[k];
        __syncthreads();
        if (threadIdx.x < 28) {
            double s = 0.0;
            for (int w = 0; w < PNW; ++w) s += red[w * 36 + threadIdx.x];
            tot[threadIdx.x] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double G8[8][8];
            int k = 0;
            for (int c1 = 0; c1 < 8; ++c1)
                for (int c2 = c1 + 1; c2 < 8; ++c2) G8[c1][c2] = tot[k++];
            for (int i = 0; i < 8; ++i) {
                for (int r = 0; r < 8; ++r) Tbb[i * 8 + r] = 0.0;
                Tbb[i * 8 + i] = taus[i];
                for (int r = 0; r < i; ++r) {
                    double s = 0.0;
                    for (int k2 = r; k2 < i; ++k2) s += Tbb[k2 * 8 + r] * G8[k2][i];
                    Tbb[i * 8 + r] = -taus[i] * s;
                }
            }
        }
        __syncthreads();
    }
    // T[0:kp+8, kp:kp+8]
    if (kp > 0) {
        vt_times_block(Vp, ld, R, kp, Cb, Wsm);  // Gx = Vp^T Vb   (kp x 8)
        __syncthreads();
        // Y = Gx Tbb (kp x 8)
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int r = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = 0; k <= c; ++k) s += Wsm[k * kp + r] * Tbb[c * 8 + k];
            Zsm[c * kp + r] = s;
        }
        __syncthreads();
        // T[0:kp, kp+c] = -T[0:kp,0:kp] Y
        for (int t = threadIdx.x; t < kp * 8; t += PNT) {
            int r = t % kp, c = t / kp;
            double s = 0.0;
            for (int k = r; k < kp; ++k) s += T[k * ELM_NB + r] * Zsm[c * kp + k];
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
        // zero below the diagonal block inside the panel's T (columns kp..kp+7, rows > kp+7)
    }
    if (threadIdx.x < 8 * ELM_NB) {
        int c = threadIdx.x / ELM_NB, r = threadIdx.x % ELM_NB;
        if (r >= kp + 8) T[(kp + c) * ELM_NB + r] = 0.0;
    }
}

size_t panel_smem_bytes(int64_t R) { return (size_t)(8 * R + 8 * 56 * 2 + PNW * 36 + 40 + 64 + 8) * 8; }

}  // namespace

cudaError_t run_local_factor(const elmddm_ctx* c, double* Kaug, double* tau, double* work, cudaStream_t st) {
    const int64_t S = c->sz.S, ld = c->sz.ld, ncols = c->sz.ncols;
    const int M = c->cfg.M;
    double* Vbuf = work;
    double* Tbuf = Vbuf + S * ELM_NB * ld;
    double* Wbuf = Tbuf + S * ELM_NB * ELM_NB;
    double* Zbuf = Wbuf + S * ELM_NB * ncols;
    const size_t smax = panel_smem_bytes(ld);
    cudaError_t e = cudaFuncSetAttribute(k_panel_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax);
    if (e != cudaSuccess) return e;
    for (int j0 = 0; j0 < M; j0 += ELM_NB) {
        const int nb = (M - j0) < ELM_NB ? (M - j0) : ELM_NB;
        PanelArgs pa{Kaug, ld, ncols, tau, M, Vbuf, Tbuf, j0, 0};
        const size_t smem = panel_smem_bytes(ld - j0);
        for (int blk = 0; blk < nb / ELM_BB; ++blk) {
            pa.blk = blk;
            KTimer kt(c, ELMDDM_K_PANEL, st);
            k_panel_block<<<(unsigned)S, PNT, smem, st>>>(pa);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        const int n_tr = (int)(ncols - (j0 + nb));
        if (n_tr <= 0) continue;
        const int R = (int)(ld - j0);
        // W = V^T C
        GemmArgs g1{nb, n_tr, R, Vbuf + j0, ld, ELM_NB * ld, Kaug + j0 + (int64_t)(j0 + nb) * ld, ld, ld * ncols,
                    Wbuf, ELM_NB, ELM_NB * ncols, 1.0, 0.0, (int)S, 0};
        if ((e = gemm_launch(true, false, g1, st, c, ELMDDM_K_GEMM_QR)) != cudaSuccess) return e;
        // Z = T^T W
        GemmArgs g2{nb, n_tr, nb, Tbuf, ELM_NB, ELM_NB * ELM_NB, Wbuf, ELM_NB, ELM_NB * ncols, Zbuf, ELM_NB,
                    ELM_NB * ncols, 1.0, 0.0, (int)S, 0};
        if ((e = gemm_launch(true, false, g2, st, c, ELMDDM_K_GEMM_QR)) != cudaSuccess) return e;
        // C -= V Z
        GemmArgs g3{R, n_tr, nb, Vbuf + j0, ld, ELM_NB * ld, Zbuf, ELM_NB, ELM_NB * ncols,
                    Kaug + j0 + (int64_t)(j0 + nb) * ld, ld, ld * ncols, -1.0, 1.0, (int)S, 0};
        if ((e = gemm_launch(false, false, g3, st, c, ELMDDM_K_GEMM_QR)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}
