// gemm.cu -- batched fp64 GEMM on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64) for sm_100a.
//
// Used for every dense contraction of the hot path: the compact-WY trailing updates of the
// blocked Householder QR (W = V^T C, Z = T^T W, C -= V Z), the TRSM update and flux product of
// the Schur elimination (W_s = A R11^{-1}, P_s = W_s [R12|y]), the Gram blocks T^T T, the Q-row
// Grams of the interface system and the band-Cholesky SYRK updates.
//
// tcgen05/UMMA has no f64 kind, so on B200 the FP64 tensor path is warp-level DMMA.8x8x4
// (DESIGN.md §5).  Tile 64x64x16, 8 warps (2 x 4), each warp 32x16 = 4x2 DMMA tiles; operands
// staged global -> shared with a 3-stage cp.async pipeline; shared layouts padded so that every
// DMMA fragment load is conflict-free (2 wavefronts per 32 x 8 B).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "tma.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 32, STAGES = 3, NT = 256;
constexpr int PAD_MN = BM + 8;  // stride of [k][m|n] layouts (== 8 mod 16 doubles)
constexpr int PAD_K = BK + 4;   // stride of [m|n][k] layouts (== 4 mod 16 doubles)
constexpr int A_ELEMS = (BM * PAD_K > BK * PAD_MN) ? BM * PAD_K : BK * PAD_MN;
constexpr int B_ELEMS = A_ELEMS;
constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8;

__device__ __forceinline__ void cp_async16(double* dst, const double* src, int src_bytes) {
    unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Load a (rows x cols) tile whose contiguous (first) dimension has extent `nc` elements, from
// src (leading dim ld) into shared dst with row stride `pad` (dst[j*pad + i] = src[i + j*ld]).
// rows_valid / cols_valid clip the tile (zero fill).  Chunks of 2 doubles (16 B).
template <int NC, int NS>  // NC contiguous extent, NS strided extent of the tile
__device__ __forceinline__ void load_tile(double* dst, int pad, const double* src, int64_t ld, int c_valid,
                                          int s_valid, int tid) {
    constexpr int CH = NC / 2;  // chunks per strided index
    constexpr int TOTAL = CH * NS;
#pragma unroll
    for (int it = 0; it < (TOTAL + NT - 1) / NT; ++it) {
        int ch = tid + it * NT;
        if (TOTAL % NT != 0 && ch >= TOTAL) break;
        int j = ch / CH;
        int i = (ch % CH) * 2;
        int bytes = 0;
        if (j < s_valid) bytes = (i + 1 < c_valid) ? 16 : (i < c_valid ? 8 : 0);
        const double* s = bytes ? src + i + (int64_t)j * ld : src;
        cp_async16(dst + j * pad + i, s, bytes);
    }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT, 2) k_gemm(GemmArgs g) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, bz = blockIdx.z;
    if (g.lower_only && m0 + BM <= n0) return;
    const double* A = g.A + (int64_t)bz * g.sA;
    const double* B = g.B + (int64_t)bz * g.sB;
    double* C = g.C + (int64_t)bz * g.sC;

    const int mv = min(BM, g.M - m0), nv = min(BN, g.N - n0);
    const int ktiles = (g.K + BK - 1) / BK;

    auto issue = [&](int kt, int stage) {
        double* As = smem + stage * STAGE_ELEMS;
        double* Bs = As + A_ELEMS;
        const int k0 = kt * BK, kv = min(BK, g.K - k0);
        if (!TA)  // A[i + k lda]: contiguous m, layout As[k][m]
            load_tile<BM, BK>(As, PAD_MN, A + m0 + (int64_t)k0 * g.lda, g.lda, mv, kv, tid);
        else  // A[k + i lda]: contiguous k, layout As[m][k]
            load_tile<BK, BM>(As, PAD_K, A + k0 + (int64_t)m0 * g.lda, g.lda, kv, mv, tid);
        if (!TB)  // B[k + n ldb]: contiguous k, layout Bs[n][k]
            load_tile<BK, BN>(Bs, PAD_K, B + k0 + (int64_t)n0 * g.ldb, g.ldb, kv, nv, tid);
        else  // B[n + k ldb]: contiguous n, layout Bs[k][n]
            load_tile<BN, BK>(Bs, PAD_MN, B + n0 + (int64_t)k0 * g.ldb, g.ldb, nv, kv, tid);
    };

    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) issue(s, s);
        cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            int nk = kt + STAGES - 1;
            if (nk < ktiles) issue(nk, nk % STAGES);
            cp_commit();
        }
        const double* As = smem + (kt % STAGES) * STAGE_ELEMS;
        const double* Bs = As + A_ELEMS;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            const int kk = ks * 4 + (lane & 3);
            double af[4], bf[2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                int i = wm * 32 + mt * 8 + (lane >> 2);
                af[mt] = TA ? As[i * PAD_K + kk] : As[kk * PAD_MN + i];
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                int n = wn * 16 + nt * 8 + (lane >> 2);
                bf[nt] = TB ? Bs[kk * PAD_MN + n] : Bs[n * PAD_K + kk];
            }
            // (8 x 8 sub-tiles wholly outside the valid rows / columns -- the last row or column
            // tile of a batch, e.g. kaug = 4q + 1 -- are skipped: warp-uniform predicates)
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
                    if (wm * 32 + mt * 8 < mv && wn * 16 + nt * 8 < nv)
                        dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
    }
    cp_wait<0>();

    // epilogue: C = alpha acc + beta C
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        int i = wm * 32 + mt * 8 + (lane >> 2);
        if (i >= mv) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int j = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                if (j >= nv) continue;
                double* cp = C + (m0 + i) + (int64_t)(n0 + j) * g.ldc;
                double v = g.alpha * acc[mt][nt][e];
                if (g.beta != 0.0) v += g.beta * *cp;
                *cp = v;
            }
        }
    }
}

// TMA version for C = alpha A^T B + beta C with both operands k-contiguous (A[k + i lda],
// B[k + n ldb]: every GEMM of the path): 64 x 64 output tile, K in chunks of 32 rows staged by
// cp.async.bulk.tensor (two 16 x 64 boxes per operand, 128B swizzle, out-of-range rows / columns
// read as zero) through a 3-stage ring; a warp arrives on the stage's mbarrier when done with it
// and only the issuing thread waits there -- no CTA-wide barrier per chunk.  Same warp tiling
// and DMMA order per output element as k_gemm<1, 0>.
namespace gt {
constexpr int NST = 3;
constexpr int STAGE = 4 * elmtma::BOX;
constexpr int SMEM = NST * STAGE * 8 + 64 + 1024;
}  // namespace gt

__global__ void __launch_bounds__(NT, 2) k_gemm_tn_tma(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB, GemmArgs g) {
    using namespace elmtma;
    using namespace gt;
    extern __shared__ uint8_t raw[];
    double* base = reinterpret_cast<double*>(raw + ((1024u - (su32(raw) & 1023u)) & 1023u));
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + NST * STAGE);  // [NST] full, [NST] empty
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN, bz = blockIdx.z;
    if (g.lower_only && m0 + BM <= n0) return;
    const int mv = min(BM, g.M - m0), nv = min(BN, g.N - n0);
    const int nk = (g.K + 31) / 32;
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&bar[s], 1);
            mbar_init(&bar[NST + s], NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int kc) {  // thread 0
        const int s = kc % NST;
        double* d = base + s * STAGE;
        if (kc >= NST) mbar_wait(&bar[NST + s], ((kc / NST) - 1) & 1);  // every warp done with its last use
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect(&bar[s], 4 * BOX * 8);
        const int k0 = 32 * kc;
        tma_load(d, &tmA, k0, m0, bz, &bar[s]);
        tma_load(d + BOX, &tmA, k0 + 16, m0, bz, &bar[s]);
        tma_load(d + 2 * BOX, &tmB, k0, n0, bz, &bar[s]);
        tma_load(d + 3 * BOX, &tmB, k0 + 16, n0, bz, &bar[s]);
    };
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    if (tid == 0)
        for (int kc = 0; kc < NST - 1 && kc < nk; ++kc) issue(kc);
    for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % NST;
        if (tid == 0 && kc + NST - 1 < nk) issue(kc + NST - 1);
        mbar_wait(&bar[s], (kc / NST) & 1);
        const double* As = base + s * STAGE;
        const double* Bs = As + 2 * BOX;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int kk = ks * 4 + (lane & 3);
            double af[4], bf[2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = As[sw(kk, wm * 32 + mt * 8 + (lane >> 2))];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) bf[nt] = Bs[sw(kk, wn * 16 + nt * 8 + (lane >> 2))];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
                    if (wm * 32 + mt * 8 < mv && wn * 16 + nt * 8 < nv)
                        dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[NST + s]);
    }
    double* C = g.C + (int64_t)bz * g.sC;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int i = wm * 32 + mt * 8 + (lane >> 2);
        if (i >= mv) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = wn * 16 + nt * 8 + 2 * (lane & 3) + e;
                if (j >= nv) continue;
                double* cp = C + (m0 + i) + (int64_t)(n0 + j) * g.ldc;
                double v = g.alpha * acc[mt][nt][e];
                if (g.beta != 0.0) v += g.beta * *cp;
                *cp = v;
            }
        }
    }
}

// C = beta C for an empty contraction (K = 0), column-major, batched; 8 columns per CTA.
__global__ void k_scale_c(int M, int N, double* C, int64_t ldc, int64_t sC, double beta, int lower_only) {
    double* Cb = C + (int64_t)blockIdx.y * sC;
    for (int j = blockIdx.x * 8 + threadIdx.x / 32; j < min(N, (int)blockIdx.x * 8 + 8); j += 8)
        for (int i = threadIdx.x % 32; i < M; i += 32) {
            if (lower_only && i / 64 < j / 64) continue;
            double* cp = Cb + i + (int64_t)j * ldc;
            *cp = beta == 0.0 ? 0.0 : beta * *cp;
        }
}

template <bool TA, bool TB>
cudaError_t launch(const GemmArgs& g, cudaStream_t st, const elmddm_ctx* c, int cls) {
    // (a per-device attribute: set on every launch, a few microseconds of host time)
    cudaError_t e = cudaFuncSetAttribute(k_gemm<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN, g.batch);
    KTimer kt(c, cls, st);
    k_gemm<TA, TB><<<grid, NT, SMEM_BYTES, st>>>(g);
    return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_launch(bool transA, bool transB, const GemmArgs& g, cudaStream_t st, const elmddm_ctx* c,
                        int cls) {
    if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return cudaSuccess;
    if (g.K <= 0) {  // empty contraction: C = beta C (beta = 0 writes zeros, even over NaN)
        if (g.beta == 1.0) return cudaSuccess;
        dim3 grid((g.N + 7) / 8, g.batch);
        k_scale_c<<<grid, 256, 0, st>>>(g.M, g.N, g.C, g.ldc, g.sC, g.beta, g.lower_only);
        return cudaGetLastError();
    }
    if (transA && !transB && c->gemm_tma) {
        CUtensorMap tA, tB;
        if (elm_encode_tmap_s(&tA, g.A, g.K, g.M, g.batch, g.lda, g.sA) &&
            elm_encode_tmap_s(&tB, g.B, g.K, g.N, g.batch, g.ldb, g.sB)) {
            cudaError_t e = cudaFuncSetAttribute(k_gemm_tn_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, gt::SMEM);
            if (e != cudaSuccess) return e;
            dim3 grid((g.M + BM - 1) / BM, (g.N + BN - 1) / BN, g.batch);
            KTimer kt(c, cls, st);
            k_gemm_tn_tma<<<grid, NT, gt::SMEM, st>>>(tA, tB, g);
            return cudaGetLastError();
        }
    }
    if (transA) return transB ? launch<true, true>(g, st, c, cls) : launch<true, false>(g, st, c, cls);
    return transB ? launch<false, true>(g, st, c, cls) : launch<false, false>(g, st, c, cls);
}

// ---- diagnostic: sustained DMMA throughput (register-resident operands, 8 independent chains) ----
namespace {
__global__ void __launch_bounds__(256) k_dmma_probe(int64_t iters, double* out) {
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;  // keep the work alive
}
}  // namespace

extern "C" elmddm_status elmddm_dmma_probe(int device, double ms, double* tflops) {
    if (!tflops || !(ms > 0)) return ELMDDM_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return ELMDDM_ECUDA;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    double* out;
    if (cudaMalloc(&out, 8) != cudaSuccess) return ELMDDM_ECUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = nsm * 4, threads = 256;
    int64_t iters = 4096;
    float t = 0.f;
    for (int pass = 0; pass < 8; ++pass) {
        cudaEventRecord(e0);
        k_dmma_probe<<<blocks, threads>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t, e0, e1);
        if (t >= ms) break;
        iters = (int64_t)(iters * (ms / (t > 0.01f ? t : 0.01f)) * 1.1);
    }
    // one DMMA.8x8x4 = 256 FMA = 512 flop per warp instruction
    double flop = (double)blocks * (threads / 32) * (double)iters * 8.0 * 512.0;
    *tflops = flop / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? ELMDDM_OK : ELMDDM_ECUDA;
}
