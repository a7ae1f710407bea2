// cg.cu -- the paper's interface solver: conjugate gradients on eqn:schur to a
// relative residual tolerance (1e-9 in the paper), as an alternative to the direct
// envelope Cholesky of chol.cu (reading R12).  M is the packed-tile lower envelope written by
// elmddm_interface_assemble; every reduction is a fixed-order two-level sum (deterministic).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace {

constexpr int NB = ELM_NB;
constexpr int LP = ELM_TLD;

// y_I = sum_{J <= I} M(I,J) x_J + sum_{I' > I} M(I',I)^T x_I' in the factorisation order (one
// CTA per 64-row block I, 256 threads: thread (r = tid & 63, part = tid >> 6) sums a quarter of
// the 64 columns of each tile; the diagonal tile is used as tril(T) + strict-tril(T)^T).  The
// row / column tile lists are M's own tiles (CholPlan::mrow / mcol, plan.cu): the factor's fill
// tiles hold zeros in M and are skipped (config 4: 19% of the band's tiles are read).
__global__ void __launch_bounds__(256) k_spmv_sym(const double* __restrict__ Mb, const int* __restrict__ diag_tid,
                                                  const int* __restrict__ rptr, const int2* __restrict__ rdep,
                                                  const int* __restrict__ cptr, const int2* __restrict__ cdep,
                                                  const double* __restrict__ x, double* __restrict__ y) {
    // thread (r, column group p of 16): x segments read straight from global memory (L1-cached,
    // shared by the 64 rows), no barrier per tile; one fixed-order reduction at the end
    __shared__ double part[4][NB];
    const int I = blockIdx.x, tid = threadIdx.x, r = tid & 63, p = tid >> 6;
    double acc = 0.0;
    const int r0 = rptr[I], nr = rptr[I + 1] - r0;
    for (int q = 0; q <= nr; ++q) {
        const int J = q < nr ? rdep[r0 + q].x : I;
        const double* T = Mb + (int64_t)(q < nr ? rdep[r0 + q].y : diag_tid[I]) * ELM_TS;
        const double* xs = x + (int64_t)J * NB;
#pragma unroll 4
        for (int c = p * 16; c < p * 16 + 16; ++c) {
            double v = T[c * LP + r];  // element (r, c)
            if (J == I && c > r) v = T[r * LP + c];  // upper part of the diagonal tile = transpose
            acc += v * __ldg(xs + c);
        }
    }
    // transposed part: y[j] += sum_i T(i, j) x[i] over the column tiles (I', I); warp w owns the
    // columns j in [8w, 8w + 8), lanes the rows i = lane, lane + 32 -- coalesced tile reads, one
    // warp reduction per column at the end
    __shared__ double part2[NB];
    const int lane = tid & 31, w = tid >> 5;
    double tacc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) tacc[u] = 0.0;
    const int c0 = cptr[I], nc = cptr[I + 1] - c0;
    for (int q = 0; q < nc; ++q) {
        const int Ip = cdep[c0 + q].x;
        const double* T = Mb + (int64_t)cdep[c0 + q].y * ELM_TS;
        const double* xs = x + (int64_t)Ip * NB;
        const double x0 = __ldg(xs + lane), x1 = __ldg(xs + lane + 32);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = 8 * w + u;
            tacc[u] += T[lane + j * LP] * x0 + T[lane + 32 + j * LP] * x1;
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        double v = tacc[u];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part2[8 * w + u] = v;
    }
    part[p][r] = acc;
    __syncthreads();
    if (tid < NB)
        y[(int64_t)I * NB + tid] = ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid])) + part2[tid];
}

__global__ void k_cg_gather(const double* __restrict__ g, const int* __restrict__ fbase, int q, int64_t G,
                            double* __restrict__ y, int64_t n) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) y[x] = 0.0;
}
__global__ void k_cg_gather2(const double* __restrict__ g, const int* __restrict__ fbase, int q, int64_t G,
                             double* __restrict__ y) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < G) y[fbase[x / q] + x % q] = g[x];
}
__global__ void k_cg_scatter(const double* __restrict__ y, const int* __restrict__ fbase, int q, int64_t G,
                             double* __restrict__ u, int64_t Gpad) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < G) u[x] = y[fbase[x / q] + x % q];
    else if (x < Gpad) u[x] = 0.0;
}

// partial dot products: part[b] = sum over the b-th 1024-chunk of a . b  (fixed order)
__global__ void __launch_bounds__(256) k_dot_part(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                                  double* __restrict__ part) {
    __shared__ double red[8];
    const int64_t i0 = (int64_t)blockIdx.x * 1024;
    double s = 0.0;
    for (int k = threadIdx.x; k < 1024; k += 256)
        if (i0 + k < n) s += a[i0 + k] * b[i0 + k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        part[blockIdx.x] = t;
    }
}

// sum the partials (one warp, fixed order) into *out
__global__ void k_dot_final(const double* __restrict__ part, int nparts, double* __restrict__ out) {
    double s = 0.0;
    for (int k = threadIdx.x; k < nparts; k += 32) s += part[k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
}

// scalars: sc[0] = r.r, sc[1] = p.q, sc[2] = new r.r
// x += alpha p, r -= alpha q   with alpha = rr / pq
__global__ void k_cg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                        const double* __restrict__ q, const double* __restrict__ sc, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double alpha = sc[1] != 0.0 ? sc[0] / sc[1] : 0.0;
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
}
// p = r + beta p with beta = rr_new / rr;  then rr <- rr_new (one thread after the grid: see host)
__global__ void k_cg_p(double* __restrict__ p, const double* __restrict__ r, const double* __restrict__ sc, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double beta = sc[0] != 0.0 ? sc[2] / sc[0] : 0.0;
    p[i] = r[i] + beta * p[i];
}
__global__ void k_cg_roll(double* sc) { sc[0] = sc[2]; }

}  // namespace

// y = M x for the symmetric matrix in packed tiles (the CG's matrix-vector product), for the
// iterative refinement of the direct interface solve (chol.cu)
static __global__ void k_resid(const double* __restrict__ g, double* __restrict__ r, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) r[i] = g[i] - r[i];
}
static __global__ void k_axpy1(double* __restrict__ x, const double* __restrict__ d, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] += d[i];
}

cudaError_t launch_residual(const elmddm_ctx* c, const double* Mband, const double* x, const double* g, double* r,
                            cudaStream_t st) {
    const CholPlan& pl = c->plan;
    {
        KTimer kt(c, ELMDDM_K_TRSV, st);
        k_spmv_sym<<<pl.nblk, 256, 0, st>>>(Mband, c->d_diag_tid, c->d_mrow_ptr, c->d_mrow, c->d_mcol_ptr, c->d_mcol, x, r);
    }
    k_resid<<<(unsigned)((pl.n + 255) / 256), 256, 0, st>>>(g, r, pl.n);
    return cudaGetLastError();
}

cudaError_t launch_axpy1(double* x, const double* d, int64_t n, cudaStream_t st) {
    k_axpy1<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, d, n);
    return cudaGetLastError();
}

cudaError_t run_interface_cg(const elmddm_ctx* c, const double* Mband, const double* g, double* uG, double* work,
                             double tol, int maxit, int* iters, double* relres, cudaStream_t st) {
    const CholPlan& pl = c->plan;
    const int64_t Gp = pl.n, G = c->sz.G;
    const int nblk = pl.nblk, qd = c->plan_q;
    const int nparts = (int)((Gp + 1023) / 1024);
    double* r = work;
    double* p = r + Gp;
    double* q = p + Gp;
    double* xn = q + Gp;     // solution in the factorisation order
    double* gn = xn + Gp;    // right-hand side in the factorisation order
    double* part = gn + Gp;
    double* sc = part + nparts;  // [4]: rr, pq, rr_new, gg
    cudaError_t e;
    const int nb = (int)((Gp + 255) / 256);
    auto dot = [&](const double* a, const double* b, double* out) -> cudaError_t {
        k_dot_part<<<nparts, 256, 0, st>>>(a, b, Gp, part);
        k_dot_final<<<1, 32, 0, st>>>(part, nparts, out);
        return cudaGetLastError();
    };
    // x = 0, r = p = g (in the factorisation order)
    k_cg_gather<<<nb, 256, 0, st>>>(g, c->d_fbase, qd, G, gn, Gp);
    if (G > 0) k_cg_gather2<<<(unsigned)((G + 255) / 256), 256, 0, st>>>(g, c->d_fbase, qd, G, gn);
    if ((e = cudaMemsetAsync(xn, 0, sizeof(double) * Gp, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(r, gn, sizeof(double) * Gp, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(p, gn, sizeof(double) * Gp, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    if ((e = dot(r, r, sc)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(sc + 3, sc, sizeof(double), cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    double h[4] = {0, 0, 0, 0};
    if ((e = cudaMemcpyAsync(h, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    const double gg = h[3];
    int it = 0;
    double rel = gg > 0.0 ? 1.0 : 0.0;
    const int check = 16;  // convergence is read back every `check` iterations
    while (rel > tol && it < maxit) {
        for (int k = 0; k < check && it < maxit; ++k, ++it) {
            {
                KTimer kt(c, ELMDDM_K_TRSV, st);
                k_spmv_sym<<<nblk, 256, 0, st>>>(Mband, c->d_diag_tid, c->d_mrow_ptr, c->d_mrow, c->d_mcol_ptr, c->d_mcol, p, q);
            }
            if ((e = dot(p, q, sc + 1)) != cudaSuccess) return e;
            k_cg_xr<<<nb, 256, 0, st>>>(xn, r, p, q, sc, Gp);
            if ((e = dot(r, r, sc + 2)) != cudaSuccess) return e;
            k_cg_p<<<nb, 256, 0, st>>>(p, r, sc, Gp);
            k_cg_roll<<<1, 1, 0, st>>>(sc);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        if ((e = cudaMemcpyAsync(h, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
        rel = gg > 0.0 ? sqrt(h[0] / gg) : 0.0;
    }
    k_cg_scatter<<<(unsigned)((c->sz.G_pad + 255) / 256), 256, 0, st>>>(xn, c->d_fbase, qd, G, uG, c->sz.G_pad);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (iters) *iters = it;
    if (relres) *relres = rel;
    return cudaSuccess;
}
