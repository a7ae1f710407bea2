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
#include <cstdio>

namespace {

constexpr int NB = ELM_NB;

__device__ __forceinline__ void dmma_c(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

constexpr int LP = NB + 4;  // padded row stride (== 4 mod 16): conflict-free DMMA fragments

// In-place Cholesky of the 64x64 tile L[i*LP + j] (lower part used), blocked by 8 columns:
//   8x8 diagonal block by warp 0 (lanes = rows, rsqrt, no divisions),
//   panel solve below it (one thread per row, reciprocal diagonal),
//   rank-8 trailing update of the lower 8x8 tiles on the FP64 tensor pipe.
// rd[] receives the reciprocal diagonal.  Returns false on a non-positive pivot.
__device__ bool potrf_tile(double* L, double* rd) {
    __shared__ int bad;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) bad = -1;
    for (int j0 = 0; j0 < NB; j0 += 8) {
        if (warp == 0) {
            const int r = lane & 7, i = j0 + r;
            double row[8];
#pragma unroll
            for (int l = 0; l < 8; ++l) row[l] = L[i * LP + j0 + l];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double d = row[c];
#pragma unroll
                for (int l = 0; l < 8; ++l)
                    if (l < c) d -= row[l] * row[l];
                double dc = __shfl_sync(0xffffffffu, d, c);
                if (lane == 0 && !(dc > 0.0) && bad < 0) bad = j0 + c;
                dc = fmax(dc, 1e-300);
                const double rs = rsqrt(dc);
                double lc[8];
#pragma unroll
                for (int l = 0; l < 8; ++l) lc[l] = __shfl_sync(0xffffffffu, row[l], c);
                if (r > c) {
                    double v = row[c];
#pragma unroll
                    for (int l = 0; l < 8; ++l)
                        if (l < c) v -= row[l] * lc[l];
                    row[c] = v * rs;
                } else if (r == c) {
                    row[c] = dc * rs;
                }
                if (lane == c) rd[j0 + c] = rs;
            }
            if (lane < 8)
#pragma unroll
                for (int l = 0; l < 8; ++l)
                    if (l <= r) L[i * LP + j0 + l] = row[l];
        }
        __syncthreads();
        // panel rows below the diagonal block
        for (int i = j0 + 8 + threadIdx.x; i < NB; i += blockDim.x) {
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = L[i * LP + j0 + c];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double v = x[c];
#pragma unroll
                for (int l = 0; l < 8; ++l)
                    if (l < c) v -= x[l] * L[(j0 + c) * LP + j0 + l];
                x[c] = v * rd[j0 + c];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) L[i * LP + j0 + c] = x[c];
        }
        __syncthreads();
        // trailing update, lower 8x8 tiles (I >= J) of the remaining block, K = 8
        const int b0 = j0 + 8, nt = (NB - b0) / 8;
        const int ntiles = nt * (nt + 1) / 2;
        for (int tt = warp; tt < ntiles; tt += blockDim.x / 32) {
            int J = 0, rem = tt;
            while (rem >= nt - J) {
                rem -= nt - J;
                ++J;
            }
            const int I = J + rem;
            const int ri = b0 + 8 * I + (lane >> 2), cl = b0 + 8 * J + 2 * (lane & 3);
            double c0 = -L[ri * LP + cl], c1 = -L[ri * LP + cl + 1];
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int kk = j0 + ks * 4 + (lane & 3);
                dmma_c(c0, c1, L[(b0 + 8 * I + (lane >> 2)) * LP + kk], L[(b0 + 8 * J + (lane >> 2)) * LP + kk]);
            }
            L[ri * LP + cl] = -c0;
            L[ri * LP + cl + 1] = -c1;
        }
        __syncthreads();
    }
    return bad < 0;
}

constexpr int POTRF_SMEM = (2 * NB * LP + NB) * 8;

// grid 1 + nsub, 256 threads.  Every CTA factors A_kk = L L^T in shared memory; CTA 0 writes
// L_kk, CTA t >= 1 solves X L^T = A_{k+t,k} in place: 8-column blocks, each a DMMA update with
// the already solved columns followed by an 8x8 triangular solve per row.
__global__ void __launch_bounds__(256) k_potrf_trsm(double* __restrict__ Mb, int64_t LD, int k, int n,
                                                    ElmStatus* status) {
    extern __shared__ __align__(16) double psm[];
    double* L = psm;              // [i*LP + j]
    double* Xs = L + NB * LP;     // [i*LP + j]  panel tile, solved in place
    double* rd = Xs + NB * LP;
    (void)n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t k0 = (int64_t)k * NB;
    double* Akk = Mb + k0 + k0 * LD;
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        int i = t % NB, j = t / NB;
        L[i * LP + j] = (i >= j) ? Akk[i + (int64_t)j * LD] : 0.0;
    }
    double* Ap = Mb + (k0 + (int64_t)blockIdx.x * NB) + k0 * LD;
    if (blockIdx.x > 0)
        for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
            int i = t % NB, j = t / NB;
            Xs[i * LP + j] = Ap[i + (int64_t)j * LD];
        }
    __syncthreads();
    const bool ok = potrf_tile(L, rd);
    if (blockIdx.x == 0) {
        if (!ok && threadIdx.x == 0) elm_set_status(status, ELMDDM_ENUMERIC, (int)k0);
        for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
            int i = t % NB, j = t / NB;
            if (i >= j) Akk[i + (int64_t)j * LD] = L[i * LP + j];
        }
        return;
    }
    for (int b = 0; b < NB / 8; ++b) {
        const int c8 = 8 * b;
        if (b > 0 && warp < NB / 8) {
            // Xs[:, c8:c8+8] -= Xs[:, 0:c8] L[c8:c8+8, 0:c8]^T   (warp = 8-row m-tile)
            const int ri = warp * 8 + (lane >> 2), cl = c8 + 2 * (lane & 3);
            double c0 = -Xs[ri * LP + cl], c1 = -Xs[ri * LP + cl + 1];
            for (int ks = 0; ks < 2 * b; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                dmma_c(c0, c1, Xs[(warp * 8 + (lane >> 2)) * LP + kk], L[(c8 + (lane >> 2)) * LP + kk]);
            }
            Xs[ri * LP + cl] = -c0;
            Xs[ri * LP + cl + 1] = -c1;
        }
        __syncthreads();
        if (threadIdx.x < NB) {
            const int i = threadIdx.x;
            double x[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = Xs[i * LP + c8 + c];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                double v = x[c];
#pragma unroll
                for (int l = 0; l < 8; ++l)
                    if (l < c) v -= x[l] * L[(c8 + c) * LP + c8 + l];
                x[c] = v * rd[c8 + c];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) Xs[i * LP + c8 + c] = x[c];
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        int i = t % NB, j = t / NB;
        Ap[i + (int64_t)j * LD] = Xs[i * LP + j];
    }
}

// ------------------------------------------------------------------------------------------
// Band SYRK update of step k: C_ij -= L_i L_j^T for the lower tiles 0 <= j <= i < nsub of the
// window starting at block k+1 (L_i = tile (k+1+i, k)).  The tile list (column-major lower
// triangle) is cut into contiguous chunks, one per CTA: the B tile L_j stays in shared memory
// while j is unchanged, A tiles are double-buffered with cp.async, C tiles are prefetched into
// registers one tile ahead.  grid min(ntiles, 2*SMs), 256 threads, ~104 KB shared memory.
// ------------------------------------------------------------------------------------------
constexpr int SYRK_SMEM = 3 * NB * LP * 8;        // KP = 1
constexpr int SYRK2_SMEM = 6 * NB * LP * 8;       // KP = 2

__device__ __forceinline__ void cpa16(double* dst, const double* src) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// tile (stored column-major in the band, rows r0.., cols c0..) -> dst[row][col] with stride LP?
// We keep A and B as [row][k] (row-major, k = column of the panel) so that both DMMA fragments
// read (row = lane/4, k = lane%4) with stride LP == 4 (mod 16).
__device__ __forceinline__ void load_panel_tile(double* dst, const double* src, int64_t LD) {
    // src: 64 rows x 64 cols column-major (ld LD); dst[r*LP + c].  16 B chunks along rows need a
    // transpose, so copy column segments of 2 rows with two 8 B writes instead: use cp.async on
    // the column-major layout into a [c][r] buffer and read fragments as [k][row] instead.
    for (int ch = threadIdx.x; ch < NB * NB / 2; ch += 256) {
        int c = ch / (NB / 2), r = (ch % (NB / 2)) * 2;
        cpa16(dst + c * LP + r, src + r + (int64_t)c * LD);
    }
}

__device__ __forceinline__ void tile_of(int t, int nsub, int& i, int& j) {
    // column-major lower triangle: column j has nsub - j tiles
    j = 0;
    int rem = t;
    while (rem >= nsub - j) {
        rem -= nsub - j;
        ++j;
    }
    i = j + rem;
}

// KP = 1: C_ij -= L_{i,k} L_{j,k}^T for the window at block k+1 (tiles 0 <= j <= i < nsub).
// KP = 2: two Cholesky steps merged into one rank-128 update of the window at block k+2:
//         C_ij -= L_{i,k} L_{j,k}^T + L_{i,k+1} L_{j,k+1}^T, where tiles of column k beyond the
//         band (relative row > nbw-2) are zero and skipped.
template <int KP>
__global__ void __launch_bounds__(256, KP == 1 ? 2 : 1) k_syrk_band(double* __restrict__ Mb, int64_t LD, int k, int nsub,
                                                                    int ntiles, int nbw) {
    extern __shared__ __align__(16) double ssm[];
    double* Bs = ssm;                   // KP tiles of column j: Bs[p][c*LP + r] = L_{j,k+p}[r][c]
    double* As0 = ssm + KP * NB * LP;   // 2 buffers x KP tiles of row i
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp & 1, wn = warp >> 1;
    const int per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
    if (t0 >= t1) return;
    const int64_t k0 = (int64_t)k * NB, w0 = k0 + KP * NB;  // window origin
    // panel p (column k+p), relative window tile row i -> tile (k+KP+i, k+p); valid iff KP-p+i <= nbw
    auto panel = [&](int p, int i) -> const double* { return Mb + (w0 + (int64_t)i * NB) + (k0 + (int64_t)p * NB) * LD; };
    auto valid = [&](int p, int i) { return KP - p + i <= nbw; };
    int i, j;
    tile_of(t0, nsub, i, j);
    int jb = -1;
#pragma unroll
    for (int p = 0; p < KP; ++p)
        if (valid(p, i)) load_panel_tile(As0 + p * NB * LP, panel(p, i), LD);
    cpa_commit();
    double cn[4][2][2];
    auto load_c = [&](int ti, int tj, double (&cr)[4][2][2]) {
        const double* Ct = Mb + (w0 + (int64_t)ti * NB) + (w0 + (int64_t)tj * NB) * LD;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm * 32 + mt * 8 + (lane >> 2), c = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    cr[mt][nt][e] = Ct[r + (int64_t)c * LD];
                }
    };
    load_c(i, j, cn);
    for (int t = t0; t < t1; ++t) {
        const int ci = i, cj = j, buf = (t - t0) & 1;
        if (cj != jb) {
#pragma unroll
            for (int p = 0; p < KP; ++p)
                if (valid(p, cj)) load_panel_tile(Bs + p * NB * LP, panel(p, cj), LD);
            cpa_commit();
            jb = cj;
        }
        double acc[4][2][2];  // holds -C: the DMMAs add A B^T, the store negates back
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = -cn[mt][nt][0], acc[mt][nt][1] = -cn[mt][nt][1];
        if (t + 1 < t1) {
            if (++i == nsub) i = ++j;  // next tile of the column-major lower triangle
#pragma unroll
            for (int p = 0; p < KP; ++p)
                if (valid(p, i)) load_panel_tile(As0 + ((buf ^ 1) * KP + p) * NB * LP, panel(p, i), LD);
        }
        cpa_commit();
        if (t + 1 < t1) load_c(i, j, cn);
        cpa_wait<1>();
        __syncthreads();
#pragma unroll
        for (int p = 0; p < KP; ++p) {
            if (!valid(p, ci) || !valid(p, cj)) continue;  // tile outside the band: zero contribution
            const double* As = As0 + (buf * KP + p) * NB * LP;
            const double* Bp = Bs + p * NB * LP;
#pragma unroll 4
            for (int ks = 0; ks < NB / 4; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                double af[4], bf[2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = As[kk * LP + wm * 32 + mt * 8 + (lane >> 2)];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) bf[nt] = Bp[kk * LP + wn * 16 + nt * 8 + (lane >> 2)];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt) dmma_c(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
            }
        }
        double* Ct = Mb + (w0 + (int64_t)ci * NB) + (w0 + (int64_t)cj * NB) * LD;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    int r = wm * 32 + mt * 8 + (lane >> 2), c = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                    Ct[r + (int64_t)c * LD] = -acc[mt][nt][e];
                }
        __syncthreads();  // buffers of this tile may be overwritten by the next prefetch
    }
}

// ------------------------------------------------------------------------------------------
// Band triangular solve as ONE cooperative (co-resident) kernel: block-row i is owned by CTA
// i mod gridDim.x; each CTA processes its rows in dependency order, streams the band tiles of the
// row through a 2-stage cp.async ring, waits for the producers of the solved blocks it needs on
// per-block completion flags (acquire/release, monotonically increasing epoch), subtracts the
// GEMV contributions, solves with the diagonal tile and publishes its block.
//   dir 0: L z = rhs  (row i needs z_j, j in [i-nbw, i))
//   dir 1: L^T u = rhs (row i needs u_j, j in (i, i+nbw]; tiles (j, i) used transposed)
// ------------------------------------------------------------------------------------------
constexpr int TP = NB + 1;
constexpr int TRSV_SMEM = (2 * NB * TP + 4 * NB + 3 * NB) * 8;

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void load_tile_async(double* dst, const double* src, int64_t LD) {
    // 64 x 64 column-major tile (ld LD) -> dst[c*TP + r]; 8-byte cp.async (TP is odd)
    for (int t = threadIdx.x; t < NB * NB; t += blockDim.x) {
        const int r = t & 63, c = t >> 6;
        unsigned d = (unsigned)__cvta_generic_to_shared(dst + c * TP + r);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + r + (int64_t)c * LD));
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

__global__ void __launch_bounds__(256) k_band_trsv(const double* __restrict__ Mb, int64_t LD, int nblk, int nbw,
                                                   const double* __restrict__ rhs, double* __restrict__ out, int* flags,
                                                   int epoch, int dir, ElmStatus* status) {
    extern __shared__ __align__(16) double tsm[];
    double* tiles = tsm;                  // [2][64 cols][TP]
    double* part = tiles + 2 * NB * TP;   // [4][64]
    double* acc = part + 4 * NB;          // [64]
    double* xs = acc + NB;                // [64]
    double* rdv = xs + NB;                // [64] reciprocal diagonal
    const int tid = threadIdx.x;
    for (int it = blockIdx.x; it < nblk; it += gridDim.x) {
        const int i = dir == 0 ? it : nblk - 1 - it;
        const int64_t i0 = (int64_t)i * NB;
        // dependency list: forward j = i-nbw .. i-1 (oldest first); backward j = i+nbw .. i+1
        const int jlo = dir == 0 ? max(0, i - nbw) : i + 1;
        const int jhi = dir == 0 ? i - 1 : min(nblk - 1, i + nbw);
        const int nj = jhi - jlo + 1;
        auto tile_of = [&](int q) -> const double* {  // q-th dependency tile, then the diagonal
            if (q == nj) return Mb + i0 + i0 * LD;
            const int j = dir == 0 ? jlo + q : jhi - q;
            return dir == 0 ? Mb + i0 + (int64_t)j * NB * LD        // tile (i, j)
                            : Mb + (int64_t)j * NB + i0 * LD;       // tile (j, i)
        };
        if (tid < NB) acc[tid] = rhs[i0 + tid];
        load_tile_async(tiles, tile_of(0), LD);
        for (int q = 0; q <= nj; ++q) {
            const int st = q & 1;
            if (q < nj) load_tile_async(tiles + (st ^ 1) * NB * TP, tile_of(q + 1), LD);
            else asm volatile("cp.async.commit_group;\n" ::);
            if (q < nj) {
                const int j = dir == 0 ? jlo + q : jhi - q;
                if (tid == 0) {
                    // bounded spin (~1 s): a missing producer reports ELMDDM_ENUMERIC instead of hanging
                    for (long long spin = 0; ld_acquire(flags + j) < epoch; ++spin) {
                        __nanosleep(64);
                        if (spin > (1LL << 24)) {
                            elm_set_status(status, ELMDDM_ENUMERIC, -1 - j);
                            break;
                        }
                    }
                }
                __syncthreads();
                if (tid < NB) xs[tid] = __ldcg(out + (int64_t)j * NB + tid);
            }
            asm volatile("cp.async.wait_group 1;\n" ::);
            __syncthreads();
            const double* T = tiles + st * NB * TP;
            if (q < nj) {
                // forward: acc[r] -= sum_c T[r][c] xs[c];  backward: acc[c] -= sum_r T[r][c] xs[r]
                const int o = tid & 63, p = tid >> 6;
                double s = 0.0;
                if (dir == 0) {
#pragma unroll 4
                    for (int c = p * 16; c < p * 16 + 16; ++c) s += T[c * TP + o] * xs[c];
                } else {
#pragma unroll 4
                    for (int r = p * 16; r < p * 16 + 16; ++r) s += T[o * TP + r] * xs[r];
                }
                part[p * NB + o] = s;
                __syncthreads();
                if (tid < NB) acc[tid] -= part[tid] + part[NB + tid] + part[2 * NB + tid] + part[3 * NB + tid];
            } else {
              if (tid < NB) rdv[tid] = 1.0 / T[tid * TP + tid];
              __syncthreads();
              if (tid < 32) {
                // diagonal solve with the tile (i, i) (lower): warp-level, reciprocal diagonal
                const int lane = tid;
                double z0 = acc[lane], z1 = acc[lane + 32];
                if (dir == 0) {
                    for (int cc = 0; cc < NB; ++cc) {
                        double xc = __shfl_sync(0xffffffffu, cc < 32 ? z0 : z1, cc & 31);
                        xc = xc * rdv[cc];
                        if (lane > cc) z0 -= T[cc * TP + lane] * xc;
                        if (lane + 32 > cc) z1 -= T[cc * TP + lane + 32] * xc;
                        if (lane == (cc & 31)) {
                            if (cc < 32) z0 = xc;
                            else z1 = xc;
                        }
                    }
                } else {
                    for (int cc = NB - 1; cc >= 0; --cc) {
                        double xc = __shfl_sync(0xffffffffu, cc < 32 ? z0 : z1, cc & 31);
                        xc = xc * rdv[cc];
                        if (lane < cc) z0 -= T[lane * TP + cc] * xc;
                        if (lane + 32 < cc) z1 -= T[(lane + 32) * TP + cc] * xc;
                        if (lane == (cc & 31)) {
                            if (cc < 32) z0 = xc;
                            else z1 = xc;
                        }
                    }
                }
                out[i0 + lane] = z0;
                out[i0 + lane + 32] = z1;
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(flags + i, epoch);
              }
            }
            __syncthreads();
        }
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
    static bool attr = false;
    if (!attr) {
        if ((e = cudaFuncSetAttribute(k_potrf_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF_SMEM)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_syrk_band<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SYRK_SMEM)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_syrk_band<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SYRK2_SMEM)) !=
                cudaSuccess)
            return e;
        attr = true;
    }
    if ((e = cudaMemcpyAsync(y, g, sizeof(double) * Gp, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    auto potrf = [&](int k) -> cudaError_t {
        const int nsub = (nblk - 1 - k) < nbw ? (nblk - 1 - k) : nbw;
        KTimer kt(c, ELMDDM_K_POTRF, st);
        k_potrf_trsm<<<1 + nsub, 256, POTRF_SMEM, st>>>(Mband, LD, k, NB, c->d_status);
        return cudaGetLastError();
    };
    auto syrk1 = [&](int k, int ntiles_limit) -> cudaError_t {  // window at k+1, first ntiles tiles
        const int nsub = (nblk - 1 - k) < nbw ? (nblk - 1 - k) : nbw;
        if (nsub <= 0) return cudaSuccess;
        int ntiles = nsub * (nsub + 1) / 2;
        if (ntiles_limit >= 0 && ntiles_limit < ntiles) ntiles = ntiles_limit;
        const int grid = ntiles < 2 * c->nsm ? ntiles : 2 * c->nsm;
        KTimer kt(c, ELMDDM_K_GEMM_CHOL, st);
        k_syrk_band<1><<<grid, 256, SYRK_SMEM, st>>>(Mband, LD, k, nsub, ntiles, nbw);
        return cudaGetLastError();
    };
    int k = 0;
    for (; k + 1 < nblk; k += 2) {
        // step k, then only column k+1 of its update, step k+1, then one rank-128 update of the rest
        const int nsub1 = (nblk - 1 - k) < nbw ? (nblk - 1 - k) : nbw;
        if ((e = potrf(k)) != cudaSuccess) return e;
        if ((e = syrk1(k, nsub1)) != cudaSuccess) return e;  // the first window column = block column k+1
        if ((e = potrf(k + 1)) != cudaSuccess) return e;
        const int nsub2 = (nblk - 2 - k) < nbw ? (nblk - 2 - k) : nbw;
        if (nsub2 > 0) {
            const int ntiles = nsub2 * (nsub2 + 1) / 2;
            const int grid = ntiles < c->nsm ? ntiles : c->nsm;
            KTimer kt(c, ELMDDM_K_GEMM_CHOL, st);
            k_syrk_band<2><<<grid, 256, SYRK2_SMEM, st>>>(Mband, LD, k, nsub2, ntiles, nbw);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    if (k < nblk) {
        if ((e = potrf(k)) != cudaSuccess) return e;
        if ((e = syrk1(k, -1)) != cudaSuccess) return e;
    }
    // triangular solves: one cooperative wavefront kernel per direction
    {
        static int coop_grid = 0;
        if (!coop_grid) {
            if ((e = cudaFuncSetAttribute(k_band_trsv, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSV_SMEM)) !=
                cudaSuccess)
                return e;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_band_trsv, 256, TRSV_SMEM);
            coop_grid = (per_sm > 0 ? 1 : 0) * c->nsm;
            if (coop_grid <= 0) coop_grid = 1;
        }
        int grid = nblk < coop_grid ? nblk : coop_grid;
        int* flags = c->d_flags;
        for (int dir = 0; dir < 2; ++dir) {
            int epoch = ++c->trsv_epoch;
            const double* rhs = dir == 0 ? y : z;
            double* out = dir == 0 ? z : uG;
            int64_t LDv = LD;
            int nblk_v = nblk, nbw_v = nbw;
            ElmStatus* stp = c->d_status;
            void* args[] = {(void*)&Mband, (void*)&LDv, (void*)&nblk_v, (void*)&nbw_v, (void*)&rhs, (void*)&out,
                            (void*)&flags, (void*)&epoch, (void*)&dir, (void*)&stp};
            KTimer kt(c, ELMDDM_K_TRSV, st);
            if ((e = cudaLaunchCooperativeKernel((void*)k_band_trsv, dim3(grid), dim3(256), args, TRSV_SMEM, st)) !=
                cudaSuccess)
                return e;
        }
    }
    return cudaSuccess;
}
