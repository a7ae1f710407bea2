// chol.cu -- band-limited tiled Cholesky of the interface Schur matrix (eqn:schur is SPD,
// P:412; reading R12: direct Cholesky instead of the paper's CG) and the two triangular solves.
//
// Storage: element (i, j) of the lower band at Mband[i + j * LD] with LD = (nbw + 2) * 64 (or
// LD = G_pad when dense): 64 x 64 tiles of the band are plain column-major sub-matrices with
// leading dimension LD, so the SYRK updates run on the DMMA GEMM.  Only tiles (I, J) with
// 0 <= I - J <= nbw are ever touched (no aliasing).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace {

constexpr int NB = ELM_NB;

// Factor the diagonal tile A_kk (in smem, lower) in place, blocked by 8 columns:
// 8x8 diagonal block (thread 0) -> panel solve (one thread per row) -> rank-8 trailing update.
// 3 barriers per 8 columns.  Returns false on a non-positive pivot.
__device__ bool potrf_tile(double (*L)[NB + 1], int n) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    for (int j0 = 0; j0 < n; j0 += 8) {
        const int jw = min(8, n - j0);
        if (threadIdx.x == 0) {
            for (int c = j0; c < j0 + jw; ++c) {
                double d = L[c][c];
                for (int l = j0; l < c; ++l) d -= L[c][l] * L[c][l];
                if (!(d > 0.0) && bad < 0) bad = c;
                d = sqrt(fmax(d, 1e-300));
                L[c][c] = d;
                for (int i = c + 1; i < j0 + jw; ++i) {
                    double v = L[i][c];
                    for (int l = j0; l < c; ++l) v -= L[i][l] * L[c][l];
                    L[i][c] = v / d;
                }
            }
        }
        __syncthreads();
        for (int i = j0 + jw + threadIdx.x; i < n; i += blockDim.x) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = c < jw ? L[i][j0 + c] : 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (c < jw) {
                    double v = x[c];
#pragma unroll
                    for (int l = 0; l < 8; ++l)
                        if (l < c) v -= x[l] * L[j0 + c][j0 + l];
                    x[c] = v / L[j0 + c][j0 + c];
                }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < jw) L[i][j0 + c] = x[c];
        }
        __syncthreads();
        const int b0 = j0 + jw, m = n - b0;
        for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
            const int i = b0 + t % m, l = b0 + t / m;
            if (l <= i) {
                double v = L[i][l];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (c < jw) v -= L[i][j0 + c] * L[l][j0 + c];
                L[i][l] = v;
            }
        }
        __syncthreads();
    }
    return bad < 0;
}

// grid 1 + nsub.  CTA 0 writes L_kk; CTA t >= 1 solves L_{k+t,k} = A_{k+t,k} L_kk^{-T}.
__global__ void __launch_bounds__(256) k_potrf_trsm(double* __restrict__ Mb, int64_t LD, int k, int n,
                                                    ElmStatus* status) {
    __shared__ double L[NB][NB + 1];
    const int64_t k0 = (int64_t)k * NB;
    double* Akk = Mb + k0 + k0 * LD;
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        int i = t % NB, j = t / NB;
        L[i][j] = (i < n && j < n && i >= j) ? Akk[i + (int64_t)j * LD] : 0.0;
    }
    __syncthreads();
    bool ok = potrf_tile(L, n);
    if (blockIdx.x == 0) {
        if (!ok && threadIdx.x == 0) elm_set_status(status, ELMDDM_ENUMERIC, (int)k0);
        for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
            int i = t % NB, j = t / NB;
            if (i < n && j < n && i >= j) Akk[i + (int64_t)j * LD] = L[i][j];
        }
        return;
    }
    double* Ap = Mb + (k0 + (int64_t)blockIdx.x * NB) + k0 * LD;
    // row r: x L^T = a  <=>  L x^T = a^T; thread (r, part) owns columns l = part + 4u
    const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
    double xv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) xv[u] = Ap[r + (int64_t)(part + 4 * u) * LD];
    for (int cidx = 0; cidx < n; ++cidx) {
        const int owner = cidx & 3, uo = cidx >> 2;
        double xc = 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (u == uo) xc = xv[u];
        xc = __shfl_sync(0xffffffffu, xc, (threadIdx.x & 31 & ~3) | owner);
        xc = xc / L[cidx][cidx];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            int l = part + 4 * u;
            if (l > cidx && l < n) xv[u] -= xc * L[l][cidx];
            if (l == cidx) xv[u] = xc;
        }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) Ap[r + (int64_t)(part + 4 * u) * LD] = xv[u];
}

// forward step k: CTA 0 solves L_kk z_k = y_k; CTA t >= 1: y_{k+t} -= L_{k+t,k} z_k
__global__ void __launch_bounds__(128) k_fwd(const double* __restrict__ Mb, int64_t LD, int k, int n,
                                             double* __restrict__ y, double* __restrict__ z) {
    __shared__ double L[NB][NB + 1];
    __shared__ double xs[NB];
    const int64_t k0 = (int64_t)k * NB;
    const double* Akk = Mb + k0 + k0 * LD;
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        int i = t % NB, j = t / NB;
        L[i][j] = (i < n && j < n && i >= j) ? Akk[i + (int64_t)j * LD] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double z0 = lane < n ? y[k0 + lane] : 0.0, z1 = lane + 32 < n ? y[k0 + lane + 32] : 0.0;
        for (int c = 0; c < n; ++c) {
            double xc = __shfl_sync(0xffffffffu, c < 32 ? z0 : z1, c & 31);
            xc /= L[c][c];
            if (lane > c) z0 -= L[lane][c] * xc;
            if (lane + 32 > c) z1 -= L[lane + 32][c] * xc;
            if (lane == (c & 31)) {
                if (c < 32) z0 = xc;
                else z1 = xc;
            }
        }
        xs[lane] = z0;
        xs[lane + 32] = z1;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int t = threadIdx.x; t < n; t += blockDim.x) z[k0 + t] = xs[t];
        return;
    }
    const int64_t r0 = k0 + (int64_t)blockIdx.x * NB;
    const double* Ap = Mb + r0 + k0 * LD;
    for (int r = threadIdx.x; r < NB; r += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < n; ++c) acc += Ap[r + (int64_t)c * LD] * xs[c];
        y[r0 + r] -= acc;
    }
}

// backward step k: CTA 0 solves L_kk^T u_k = z_k; CTA t >= 1: z_{k-t} -= L_{k,k-t}^T u_k
__global__ void __launch_bounds__(128) k_bwd(const double* __restrict__ Mb, int64_t LD, int k, int n,
                                             double* __restrict__ z, double* __restrict__ u) {
    __shared__ double L[NB][NB + 1];
    __shared__ double xs[NB];
    const int64_t k0 = (int64_t)k * NB;
    const double* Akk = Mb + k0 + k0 * LD;
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        int i = t % NB, j = t / NB;
        L[i][j] = (i < n && j < n && i >= j) ? Akk[i + (int64_t)j * LD] : (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double z0 = lane < n ? z[k0 + lane] : 0.0, z1 = lane + 32 < n ? z[k0 + lane + 32] : 0.0;
        for (int c = n - 1; c >= 0; --c) {
            double xc = __shfl_sync(0xffffffffu, c < 32 ? z0 : z1, c & 31);
            xc /= L[c][c];
            // z_l -= L[c][l] x_c for l < c
            if (lane < c) z0 -= L[c][lane] * xc;
            if (lane + 32 < c) z1 -= L[c][lane + 32] * xc;
            if (lane == (c & 31)) {
                if (c < 32) z0 = xc;
                else z1 = xc;
            }
        }
        xs[lane] = z0;
        xs[lane + 32] = z1;
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int t = threadIdx.x; t < n; t += blockDim.x) u[k0 + t] = xs[t];
        return;
    }
    const int64_t c0 = k0 - (int64_t)blockIdx.x * NB;  // target block k - t
    const double* Ap = Mb + k0 + c0 * LD;              // tile (k, k-t): rows k0.., cols c0..
    for (int cc = threadIdx.x; cc < NB; cc += blockDim.x) {
        double acc = 0.0;
        for (int r = 0; r < n; ++r) acc += Ap[r + (int64_t)cc * LD] * xs[r];
        z[c0 + cc] -= acc;
    }
}

}  // namespace

cudaError_t run_cholesky_solve(const elmddm_ctx* c, double* Mband, const double* g, double* uG, double* work,
                               cudaStream_t st) {
    const int64_t Gp = c->sz.G_pad, LD = c->sz.band_ld;
    const int nblk = (int)(Gp / NB);
    const int nbw = (int)c->sz.band_nbw;
    double* y = work;
    double* z = y + Gp;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(y, g, sizeof(double) * Gp, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    for (int k = 0; k < nblk; ++k) {
        const int nsub = (nblk - 1 - k) < nbw ? (nblk - 1 - k) : nbw;
        { KTimer kt(c, ELMDDM_K_POTRF, st);
        k_potrf_trsm<<<1 + nsub, 256, 0, st>>>(Mband, LD, k, NB, c->d_status); }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (nsub > 0) {
            const int64_t r0 = (int64_t)(k + 1) * NB, k0 = (int64_t)k * NB;
            GemmArgs gs{nsub * NB, nsub * NB, NB, Mband + r0 + k0 * LD, LD, 0, Mband + r0 + k0 * LD, LD, 0,
                        Mband + r0 + r0 * LD, LD, 0, -1.0, 1.0, 1, 1};
            if ((e = gemm_launch(false, true, gs, st, c, ELMDDM_K_GEMM_CHOL)) != cudaSuccess) return e;
        }
    }
    for (int k = 0; k < nblk; ++k) {
        const int nsub = (nblk - 1 - k) < nbw ? (nblk - 1 - k) : nbw;
        KTimer kt(c, ELMDDM_K_TRSV, st);
        k_fwd<<<1 + nsub, 128, 0, st>>>(Mband, LD, k, NB, y, z);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    for (int k = nblk - 1; k >= 0; --k) {
        const int nsub = k < nbw ? k : nbw;
        KTimer kt(c, ELMDDM_K_TRSV, st);
        k_bwd<<<1 + nsub, 128, 0, st>>>(Mband, LD, k, NB, z, uG);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}
