// chol.cu -- Cholesky factorisation of the interface Schur matrix (eqn:schur is SPD, P:412;
// reading R12: a direct solve instead of the paper's CG) and the two triangular solves.
//
// Storage (internal.h): the 64 x 64 tiles of the lower factor's tile structure
// (plan.cu: strip/envelope or nested-dissection order, symbolic factorisation on tiles), tile t
// contiguous at t * ELM_TS, element (r, c) at r + c * ELM_TLD (ELM_TLD = 68).  A tile (or its
// first 32 columns) is therefore one contiguous bulk copy that lands in shared memory already in
// the padded, bank-conflict-free layout the DMMA fragments read.
//
// Factorisation: ONE persistent kernel, left-looking over the tiles of L.  Tile (I, J) is
//     C      = M(I, J) - sum_{k in klist(I, J)} L(I, k) L(J, k)^T              (DMMA)
//     L(J,J), Y_J = L(J,J)^{-1} from C           (I == J: unblocked Cholesky + inverse in smem)
//     L(I,J) = C L(J,J)^{-T}                      (I > J: X0 = C Y_J^T and one refinement step
//                                                  X = X0 + (C - X0 L(J,J)^T) Y_J^T, three 64^3 DMMAs)
// where klist(I, J) = {k < J : L(I, k) and L(J, k) structurally nonzero} comes with the plan
// (pairs of tile ids).  The k-sum streams 32-column halves of L(I,k) and L(J,k) through a
// 3-stage TMA bulk-copy / mbarrier pipeline issued by one thread.  Tasks are listed column by
// column (critical tiles I - J <= crit_band first, worked by dedicated CTAs) and dealt
// round-robin to co-resident CTAs; each finished tile publishes a per-tile flag (release /
// acquire) and bumps its column's counter.  A task waits only for tiles of earlier columns or
// for the diagonal of its own column, so the smallest unfinished task can always run (no
// deadlock) and the trailing work of many columns overlaps the critical path.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"

#ifdef ELM_CHOL_PROF
// per-task timeline of the factorisation (profiling builds only): start, end, flag-wait ns,
// data-wait ns, epilogue start, CTA
__device__ unsigned long long g_chol_prof[400000 * 6];
__device__ unsigned long long g_chol_dprof[4096 * 8];  // diagonal tasks: stage timestamps
#endif

namespace {

constexpr int NB = ELM_NB;
constexpr int LP = ELM_TLD;

__device__ __forceinline__ void dmma_c(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// system scope: flags written by (or for) the other GPUs of a multi-rank factorisation
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Spin until *flag >= epoch; after ~10 s report ELMDDM_ENUMERIC (info = -1 - tag) and give up
// instead of hanging the device.
__device__ __forceinline__ void wait_flag(const int* flag, int epoch, ElmStatus* status, int tag, bool sys = false) {
    auto ld = [&]() { return sys ? ld_acquire_sys(flag) : ld_acquire(flag); };
    if (ld() >= epoch) return;
    const uint64_t t0 = globaltimer();
    while (ld() < epoch) {
        __nanosleep(64);
        if (globaltimer() - t0 > 10000000000ull) {
            elm_set_status(status, ELMDDM_ENUMERIC, -1 - tag);
            return;
        }
    }
}

// ---- mbarrier + bulk copy (TMA, non-tensor) -------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
// orders this thread's generic-proxy view (incl. tiles other CTAs published and this thread
// acquired) before its following async-proxy (bulk copy) accesses, in every state space
// (global: tiles written by other CTAs' generic stores, read by the bulk copy; shared::cta: the
// stage this thread's CTA read with generic loads, about to be overwritten by the async proxy.
// The unqualified fence costs a MEMBAR.ALL.GPU, these two a CTA membar.)
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;\nfence.proxy.async.shared::cta;\n" ::: "memory");
}

// ------------------------------------------------------------------------------------------
// the left-looking tile Cholesky
// ------------------------------------------------------------------------------------------
namespace llc {
constexpr int NT = 256;
constexpr int TILE = ELM_TS;                  // doubles per packed 64-wide tile
constexpr int HALF = 32 * LP;                 // doubles per 32-column half tile
constexpr int NSTAGE = 3;                     // stage = (A half, B half) = one tile of smem
constexpr uint32_t HALF_BYTES = HALF * 8;
constexpr int SMEM = NSTAGE * TILE * 8 + 10 * NB * 8 + 16 * 8;  // stages, potrf scratch, mbarriers
}  // namespace llc

// acc[r][n] += sum_kk A[kk*LP + r] B[kk*LP + n], kk < KW; warp tile 32 x 16 (wm = warp & 1, wn = warp >> 1)
template <int KW>
__device__ __forceinline__ void mma_tile(double (&acc)[4][2][2], const double* As, const double* Bs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp & 1, wn = warp >> 1;
#pragma unroll 4
    for (int ks = 0; ks < KW / 4; ++ks) {
        const int kk = ks * 4 + (lane & 3);
        double af[4], bf[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[mt] = As[kk * LP + wm * 32 + mt * 8 + (lane >> 2)];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bf[nt] = Bs[kk * LP + wn * 16 + nt * 8 + (lane >> 2)];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) dmma_c(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
}

// fragment element (mt, nt, e) of this thread -> tile coordinates (r, c)
__device__ __forceinline__ int frag_r(int mt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    return (warp & 1) * 32 + mt * 8 + (lane >> 2);
}
__device__ __forceinline__ int frag_c(int nt, int e) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    return (warp >> 1) * 16 + nt * 8 + 2 * (lane & 3) + e;
}
#define FOR_FRAG                                     \
    _Pragma("unroll") for (int mt = 0; mt < 4; ++mt) \
    _Pragma("unroll") for (int nt = 0; nt < 2; ++nt) \
    _Pragma("unroll") for (int e = 0; e < 2; ++e)

// Cholesky and inverse of one SPD 64 x 64 tile.  Input A[c * LP + r] (lower part valid); output
// L (lower, zeros above) into the same buffer and Y = L^{-1} (lower, zeros above) into Y.
// Blocked by 8 columns: warp 0 factors the 8-wide panel with shuffles (rows c0 + lane and
// c0 + 32 + lane in registers), then all warps apply the rank-8 trailing update on the FP64
// tensor pipe (8 x 8 DMMA tiles, K = 8).  The inverse is blocked the same way: the 8 diagonal
// 8 x 8 blocks are inverted in parallel (one warp each, 1/l_rr from the panel), then block row
// i of Y is Y_ij = -Y_ii sum_{k=j}^{i-1} L_ik Y_kj (DMMA), one barrier per block row.
// xbuf: >= 10 * 64 doubles of scratch ([64] 1/l_rr, pivot flag, [8 warps][64] staging).  Returns the first non-positive pivot (local) or -1.
__device__ int potrf_inv_tile(double* A, double* Y, double* xbuf) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* rsv = xbuf;              // [64] 1 / l_rr
    int* badp = reinterpret_cast<int*>(xbuf + NB);
    if (tid == 0) *badp = -1;
    // zero Y (the off-diagonal upper blocks stay zero)
    for (int x = tid; x < NB * NB; x += llc::NT) Y[(x >> 6) * LP + (x & 63)] = 0.0;
    __syncthreads();
    for (int p = 0; p < 8; ++p) {
        const int c0 = 8 * p;
        if (warp == 0) {
            const int r0 = c0 + lane, r1 = c0 + 32 + lane;
            double x0[8], x1[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                x0[j] = r0 < NB ? A[(c0 + j) * LP + r0] : 0.0;
                x1[j] = r1 < NB ? A[(c0 + j) * LP + r1] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double d = __shfl_sync(0xffffffffu, x0[k], k);
                if (lane == 0 && !(d > 0.0) && *badp < 0) *badp = c0 + k;
                const double rs = rsqrt(d > 0.0 ? d : 1e-300);
                if (lane == 0) rsv[c0 + k] = rs;
                x0[k] = lane >= k ? x0[k] * rs : 0.0;  // column k of L (rows c0+lane >= c0+k)
                x1[k] *= rs;
#pragma unroll
                for (int j = k + 1; j < 8; ++j) {
                    const double lj = __shfl_sync(0xffffffffu, x0[k], j);  // L(c0+j, c0+k)
                    if (lane > k) x0[j] = fma(-x0[k], lj, x0[j]);
                    x1[j] = fma(-x1[k], lj, x1[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (r0 < NB) A[(c0 + j) * LP + r0] = x0[j];
                if (r1 < NB) A[(c0 + j) * LP + r1] = x1[j];
            }
        }
        __syncthreads();
        // rank-8 trailing update of the lower 8 x 8 tiles (I >= J) of rows / columns >= c0 + 8
        const int nt = 7 - p, ntiles = nt * (nt + 1) / 2;
        for (int t = warp; t < ntiles; t += llc::NT / 32) {
            int J = 0, rem = t;
            while (rem >= nt - J) {
                rem -= nt - J;
                ++J;
            }
            const int i0 = c0 + 8 + 8 * (J + rem), j0 = c0 + 8 + 8 * J;
            const int ri = i0 + (lane >> 2), cj = j0 + 2 * (lane & 3);
            double e0 = -A[cj * LP + ri], e1 = -A[(cj + 1) * LP + ri];
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int kk = c0 + ks * 4 + (lane & 3);
                dmma_c(e0, e1, A[kk * LP + i0 + (lane >> 2)], A[kk * LP + j0 + (lane >> 2)]);
            }
            A[cj * LP + ri] = -e0;
            A[(cj + 1) * LP + ri] = -e1;
        }
        __syncthreads();
    }
    // zeros above the diagonal of L
    for (int x = tid; x < NB * NB; x += llc::NT) {
        const int r = x & 63, c = x >> 6;
        if (r < c) A[c * LP + r] = 0.0;
    }
    // diagonal blocks of Y: warp w inverts L_ww (lanes 0..7: one column each)
    if (lane < 8) {
        const int b0 = 8 * warp, c = lane;
        double y[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            double s = r == c ? 1.0 : 0.0;
#pragma unroll
            for (int l = 0; l < 8; ++l)
                if (l < r) s = fma(-A[(b0 + l) * LP + b0 + r], y[l], s);
            y[r] = r >= c ? s * rsv[b0 + r] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) Y[(b0 + c) * LP + b0 + r] = y[r];
    }
    __syncthreads();
    // off-diagonal blocks, block row by block row: warp j < i computes Y_ij
    for (int i = 1; i < 8; ++i) {
        if (warp < i) {
            const int j = warp;
            // S = sum_{k=j}^{i-1} L_ik Y_kj   (8 x 8, K = 8 per term)
            double s0 = 0.0, s1 = 0.0;
            for (int k = j; k < i; ++k) {
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const int kk = ks * 4 + (lane & 3);
                    dmma_c(s0, s1, A[(8 * k + kk) * LP + 8 * i + (lane >> 2)], Y[(8 * j + (lane >> 2)) * LP + 8 * k + kk]);
                }
            }
            // stage S (C fragment: row lane>>2, cols 2(lane&3)+e) as the B operand of Y_ii S
            double* sw = xbuf + 2 * NB + warp * 64;  // per-warp 8 x 8, [col * 8 + row]
            sw[(2 * (lane & 3)) * 8 + (lane >> 2)] = s0;
            sw[(2 * (lane & 3) + 1) * 8 + (lane >> 2)] = s1;
            __syncwarp();
            double y0 = 0.0, y1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                const int kk = ks * 4 + (lane & 3);
                dmma_c(y0, y1, Y[(8 * i + kk) * LP + 8 * i + (lane >> 2)], sw[(lane >> 2) * 8 + kk]);
            }
            const int ri = 8 * i + (lane >> 2), cj = 8 * j + 2 * (lane & 3);
            Y[cj * LP + ri] = -y0;
            Y[(cj + 1) * LP + ri] = -y1;
            __syncwarp();
        }
        __syncthreads();
    }
    return *badp;
}

// X = C L^{-T} for C in As (layout [c * LP + r]), L = L(J,J) in Bs and Y = L(J,J)^{-1} in Ys:
// X0 = C Y^T, then one refinement step X = X0 + (C - X0 L^T) Y^T (three 64^3 DMMA products; the
// inverse alone would lose accuracy on ill-conditioned diagonal blocks).  As is clobbered.
__device__ __forceinline__ void trsm_refined(double (&x)[4][2][2], double* As, const double* Bs, const double* Ys,
                                             bool refine = true) {
    double r[4][2][2];
    FOR_FRAG x[mt][nt][e] = 0.0;
    mma_tile<NB>(x, As, Ys);                                    // X0 = C Y^T
    if (!refine) return;
    FOR_FRAG r[mt][nt][e] = -As[frag_c(nt, e) * LP + frag_r(mt)];  // -C
    __syncthreads();
    FOR_FRAG As[frag_c(nt, e) * LP + frag_r(mt)] = x[mt][nt][e];
    __syncthreads();
    mma_tile<NB>(r, As, Bs);                                    // X0 L^T - C = -R
    __syncthreads();
    FOR_FRAG As[frag_c(nt, e) * LP + frag_r(mt)] = -r[mt][nt][e];
    __syncthreads();
    mma_tile<NB>(x, As, Ys);                                    // X0 + R Y^T
}

struct CholArgs {
    double* Mb;            // tile pool: tile id t at t * ELM_TS (this replica)
    double* Ybuf;          // [nblk] packed tiles: L(J,J)^{-1}
    double* Cbuf;          // [nblk] packed tiles: C(I, klast(I)) before its triangular solve
    int* cready;           // [nblk] Cbuf[I] published (epoch)
    const TaskDesc* tasks; // [0, ncrit) critical band, then the other tiles; each column by column
    int ntasks;
    int ncrit;
    int crit_ctas;         // CTAs [0, crit_ctas) work the critical list, the rest the others
    const int4* klist;     // per-task update lists: (tile (I,k), tile (J,k), k, 0)
    const int* diag_tid;   // [nblk] tile id of (J, J)
    int* flags;            // [ntiles] per-tile completion (epoch)
    int* colcnt;           // [nblk] finished tiles of column J, summed over factorisations
    const int* ntc;        // [nblk] tiles of column J
    int epoch;             // tile flags: 2 epoch when L(I,J) is final, 2 epoch - 1 when a split
                           // task's pre-aggregation is in the tile; cready and colcnt count epochs
    const int* epoch_dev;  // non-null: the epoch is read from here at kernel entry (one rank: a
                           // device counter bumped in-stream by k_launch_prep, so a captured CUDA
                           // graph advances it on every replay); null: `epoch` (multi-rank path)
    ElmStatus* status;
    int* next;             // non-null: tasks dealt dynamically in list order (zeroed counter)
    // multi-rank factorisation (nrep > 1, dynamic dealing through the shared counter `next`):
    // every rank holds a full replica of the tile pool, Ybuf, Cbuf and the flags; a finished tile
    // is written to every replica, then its flag is released in every replica (system scope), so
    // all k-loop reads stay in the rank's own HBM.  CTA b works as replica rep_base + b / ctas_per_rep
    // (one launch per GPU: rep_base = rank, ctas_per_rep = gridDim.x; one-GPU emulation of several
    // ranks: rep_base = 0 and the grid split among the replicas).
    int nrep, rep_base, ctas_per_rep;
    const CholRep* reps;   // [nrep]
    double* Msave;         // non-null (one rank): every task that reads an assembled tile of M
                           // (kinds 0 and 1) also stores it here -- the copy of M the
                           // refinement step's residual needs, without a separate copy pass
    int trsm_refine;       // 1: one refinement step in every tile solve X = C L(J,J)^{-T}
    const unsigned char* tile_m;  // [ntiles] 1: tile of M (saved to Msave), 0: fill (zero in M)
};

__global__ void __launch_bounds__(llc::NT, 2) k_chol_ll(CholArgs a) {
    using namespace llc;
    extern __shared__ __align__(128) double csm[];
    double* St = csm;                                      // NSTAGE x (A half | B half)
    double* rsv = St + NSTAGE * TILE;                      // [10 * 64] potrf scratch
    uint64_t* bar = reinterpret_cast<uint64_t*>(rsv + 10 * NB);  // [NSTAGE] chunk loads, [NSTAGE] epilogue
                                                                  // loads, [NSTAGE] stage released by all warps
    double* As = St;                                       // epilogue: C / X0 / R
    double* Bs = St + TILE;                                // epilogue: L(J,J)
    double* Ys = St + 2 * TILE;                            // epilogue: Y_J
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < 2 * NSTAGE; ++s) mbar_init(&bar[s], 1);
        for (int s = 0; s < NSTAGE; ++s) mbar_init(&bar[2 * NSTAGE + s], NT / 32);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const bool dist = a.nrep > 1;
    const int epoch = a.epoch_dev ? *a.epoch_dev : a.epoch;
    const int fin_ep = 2 * epoch, pre_ep = fin_ep - 1;
    const int my = dist ? a.rep_base + (int)blockIdx.x / a.ctas_per_rep : 0;
    double* const Mb = dist ? a.reps[my].Mb : a.Mb;
    double* const Ybuf = dist ? a.reps[my].Ybuf : a.Ybuf;
    double* const Cbuf = dist ? a.reps[my].Cbuf : a.Cbuf;
    int* const flags = dist ? a.reps[my].flags : a.flags;
    int* const cready = dist ? a.reps[my].cready : a.cready;
    auto tileptr = [&](int t) { return Mb + (int64_t)t * TILE; };
    // copy a finished 64-tile (offset off doubles in each replica's region `which`) from this
    // replica to all the others (16-byte vector loads / stores, all threads), then make the
    // stores visible system-wide; the caller releases the flags afterwards
    auto push = [&](int which, int64_t off) {
        const double2* src = reinterpret_cast<const double2*>((which == 0 ? Mb : (which == 1 ? Ybuf : Cbuf)) + off);
        for (int r = 0; r < a.nrep; ++r) {
            if (r == my) continue;
            double* base = which == 0 ? a.reps[r].Mb : (which == 1 ? a.reps[r].Ybuf : a.reps[r].Cbuf);
            double2* dst2 = reinterpret_cast<double2*>(base + off);
            for (int x = tid; x < TILE / 2; x += NT) dst2[x] = __ldcg(src + x);
        }
    };
    uint32_t gchunk = 0;  // chunk loads issued by this CTA so far (stage = gchunk % NSTAGE)
    uint32_t epi_uses = 0;
#ifdef ELM_CHOL_PROF
    unsigned long long pf_flag = 0, pf_data = 0;
#endif
    // warp 0 (all lanes, q warp-uniform): make sure L(I, k) and L(J, k) of update klist[q] are
    // final.  Lane l checks the two tile flags of update q + l, one ballot gives the number of
    // consecutive ready updates from q (kept in rdy): one L2 round trip per 32 updates instead
    // of two per update on the thread that issues the chunk loads (the loads of the next chunk
    // -- and so every warp -- waited for it)
    int rdy = 0;
    auto ensure_w = [&](int q, int qend, int J) {
        if (q < rdy) return;
#ifdef ELM_CHOL_PROF
        const uint64_t q0 = globaltimer();
#endif
        const int lane = tid & 31;
        uint64_t t0 = 0;
        for (;;) {
            int ok = 1;
            if (q + lane < qend) {
                const int4 e = a.klist[q + lane];
                ok = (dist ? ld_acquire_sys(flags + e.x) : ld_acquire(flags + e.x)) >= fin_ep &&
                     (dist ? ld_acquire_sys(flags + e.y) : ld_acquire(flags + e.y)) >= fin_ep;
            }
            const unsigned nr = ~__ballot_sync(0xffffffffu, ok);
            const int nready = nr ? __ffs(nr) - 1 : 32;
            if (nready > 0) {
                rdy = q + nready;
                break;
            }
            if (!t0) {
                t0 = globaltimer();
            } else if (globaltimer() - t0 > 10000000000ull) {  // as wait_flag: report, give up
                if (lane == 0) elm_set_status(a.status, ELMDDM_ENUMERIC, -1 - a.klist[q].z);
                rdy = qend;
                break;
            }
            __nanosleep(64);
        }
#ifdef ELM_CHOL_PROF
        pf_flag += globaltimer() - q0;
#endif
    };
    // static dealing: CTAs [0, crit_ctas) take the critical list round-robin, the others the
    // rest; dynamic dealing (a.next): every CTA takes the next task of the (list-scheduled) order
    // when it is free.  Both deadlock-free: the lists are topological and a CTA holds one task.
    __shared__ int s_next;
    const bool critw = (int)blockIdx.x < a.crit_ctas;
    const int t_begin = critw ? (int)blockIdx.x : a.ncrit + (int)blockIdx.x - a.crit_ctas;
    const int t_end = a.next ? a.ntasks : (critw ? a.ncrit : a.ntasks);
    const int t_step = critw ? a.crit_ctas : (int)gridDim.x - a.crit_ctas;
    for (int t = t_begin;; t += t_step) {
        if (a.next) {
            if (tid == 0) s_next = dist ? atomicAdd_system(a.next, 1) : atomicAdd(a.next, 1);
            __syncthreads();
            t = s_next;
        }
        if (t >= t_end) break;
        const TaskDesc td = a.tasks[t];
        const int I = td.I, J = td.J;
        // the diagonal task applies its last update column klast itself: it solves for
        // L(J, klast) from the published C(J, klast) (one flag hop less on the critical path)
        const bool pre = td.kind == 1;
        const bool dsub = !pre && I == J && td.klast >= 0;
        const int kb = td.kbeg, ke = dsub ? td.kend - 1 : td.kend;
        const int nch = 2 * (ke - kb);
#ifdef ELM_CHOL_PROF
        const uint64_t pt0 = globaltimer();
        pf_flag = pf_data = 0;
#endif
        const uint32_t g0 = gchunk;
        // chunk c: columns [32h, 32h + 32) of L(I, k) and L(J, k), k = klist[kb + c/2], h = c & 1
        auto issue = [&](int c) {  // thread 0 only
            const int4 ke4 = a.klist[kb + (c >> 1)];
            const int h = c & 1;
            const uint32_t g = g0 + c;
            double* st = St + (g % NSTAGE) * TILE;
            uint64_t* b = &bar[g % NSTAGE];
            // every warp has released the stage's previous chunk (its phase g / NSTAGE - 1)
            if (g >= (uint32_t)NSTAGE) mbar_wait(&bar[2 * NSTAGE + g % NSTAGE], ((g / NSTAGE) - 1) & 1);
            fence_proxy_async();
            mbar_expect(b, 2 * HALF_BYTES);
            bulk_load(st, tileptr(ke4.x) + h * HALF, HALF_BYTES, b);
            bulk_load(st + HALF, tileptr(ke4.y) + h * HALF, HALF_BYTES, b);
        };
        double acc[4][2][2];  // holds -C while the updates are added
        if (td.kind == 2) {   // the tile holds M minus the pre-aggregated updates once flagged
            if (tid == 0) wait_flag(flags + td.tid, pre_ep, a.status, J, dist);
            __syncthreads();
        }
        {
            const double* Ct = tileptr(td.tid);
            FOR_FRAG acc[mt][nt][e] = -__ldcg(Ct + frag_r(mt) + frag_c(nt, e) * LP);
            if (a.Msave && td.kind != 2 && a.tile_m[td.tid]) {  // (fill tiles: never read by the SpMV)
                double* ms = a.Msave + (int64_t)td.tid * TILE;
                FOR_FRAG __stcs(ms + frag_r(mt) + frag_c(nt, e) * LP, -acc[mt][nt][e]);
            }
        }
        rdy = kb;
        if (tid < 32) {
            for (int c = 0; c < NSTAGE - 1 && c < nch; ++c) {
                if ((c & 1) == 0) ensure_w(kb + (c >> 1), ke, J);
                if (tid == 0) issue(c);
            }
            __syncwarp();
        }
        for (int c = 0; c < nch; ++c) {
            if (tid < 32 && c + NSTAGE - 1 < nch) {
                const int cn = c + NSTAGE - 1;
                if ((cn & 1) == 0) ensure_w(kb + (cn >> 1), ke, J);
                if (tid == 0) issue(cn);
                __syncwarp();
            }
            const uint32_t g = g0 + c;
#ifdef ELM_CHOL_PROF
            const uint64_t pw = globaltimer();
#endif
            mbar_wait(&bar[g % NSTAGE], (g / NSTAGE) & 1);
#ifdef ELM_CHOL_PROF
            pf_data += globaltimer() - pw;
#endif
            const double* st = St + (g % NSTAGE) * TILE;
            mma_tile<32>(acc, st, st + HALF);
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&bar[2 * NSTAGE + g % NSTAGE]);  // stage free for its refill
        }
        gchunk = g0 + nch;
        __syncthreads();
#ifdef ELM_CHOL_PROF
        const uint64_t pte = globaltimer();
#endif
        double* dst = tileptr(td.tid);
        if (pre) {
            // partial sum C = M - sum_{k in pre list} L(I,k) L(J,k)^T back into the tile
            FOR_FRAG dst[frag_r(mt) + frag_c(nt, e) * LP] = -acc[mt][nt][e];
            if (dist) {
                __threadfence_block();
                __syncthreads();
                push(0, (int64_t)td.tid * TILE);
            }
        } else if (I == J) {
#ifdef ELM_CHOL_PROF
            uint64_t dts[8] = {globaltimer(), 0, 0, 0, 0, 0, 0, 0};
#define DSTAMP(k) dts[k] = globaltimer()
#else
#define DSTAMP(k)
#endif
            if (dsub) {
                uint64_t* eb = &bar[NSTAGE + (epi_uses % NSTAGE)];
                const uint32_t epar = (epi_uses / NSTAGE) & 1;
                ++epi_uses;
                if (tid == 0) {
                    wait_flag(cready + J, epoch, a.status, J, dist);
                    wait_flag(flags + a.diag_tid[td.klast], fin_ep, a.status, td.klast, dist);
                    fence_proxy_async();
                    mbar_expect(eb, 3 * TILE * 8);
                    bulk_load(As, Cbuf + (int64_t)J * TILE, TILE * 8, eb);
                    bulk_load(Bs, tileptr(a.diag_tid[td.klast]), TILE * 8, eb);
                    bulk_load(Ys, Ybuf + (int64_t)td.klast * TILE, TILE * 8, eb);
                }
                DSTAMP(1);
                mbar_wait(eb, epar);
                DSTAMP(2);
                double x[4][2][2];
                trsm_refined(x, As, Bs, Ys, a.trsm_refine);       // L(J, klast)
                DSTAMP(3);
                __syncthreads();
                FOR_FRAG As[frag_c(nt, e) * LP + frag_r(mt)] = x[mt][nt][e];
                __syncthreads();
                mma_tile<NB>(acc, As, As);                        // -C(J,J) + L(J,klast) L(J,klast)^T
                __syncthreads();
            }
            FOR_FRAG As[frag_c(nt, e) * LP + frag_r(mt)] = -acc[mt][nt][e];
            __syncthreads();
            DSTAMP(4);
            const int bad = potrf_inv_tile(As, Ys, rsv);
            DSTAMP(5);
            if (bad >= 0 && tid == 0) elm_set_status(a.status, ELMDDM_ENUMERIC, J * NB + bad);
            double* yd = Ybuf + (int64_t)J * TILE;
            for (int x = tid; x < TILE / 2; x += NT) {
                reinterpret_cast<double2*>(dst)[x] = reinterpret_cast<const double2*>(As)[x];
                reinterpret_cast<double2*>(yd)[x] = reinterpret_cast<const double2*>(Ys)[x];
            }
            if (dist) {  // L(J,J) and its inverse to the other replicas
                __threadfence_block();
                __syncthreads();
                push(0, (int64_t)td.tid * TILE);
                push(1, (int64_t)J * TILE);
            }
            DSTAMP(6);
            __threadfence();
            DSTAMP(7);
#ifdef ELM_CHOL_PROF
            if (tid == 0 && J < 4096)
                for (int q = 0; q < 8; ++q) g_chol_dprof[8 * J + q] = dts[q];
#endif
#undef DSTAMP
        } else {
            // C -> As[c * LP + r]
            FOR_FRAG As[frag_c(nt, e) * LP + frag_r(mt)] = -acc[mt][nt][e];
            if (td.pub) {  // publish C(I, J = klast(I)) for the diagonal task of row I
                double* cb = Cbuf + (int64_t)I * TILE;
                FOR_FRAG cb[frag_c(nt, e) * LP + frag_r(mt)] = -acc[mt][nt][e];
                if (dist) {
                    __syncthreads();
                    push(2, (int64_t)I * TILE);
                    __threadfence_system();
                    __syncthreads();
                    if (tid == 0)
                        for (int r = 0; r < a.nrep; ++r) st_release_sys(a.reps[r].cready + I, epoch);
                } else {
                    __threadfence();
                    __syncthreads();
                    if (tid == 0) st_release(cready + I, epoch);
                }
            }
            // L(I,J) solves X L_JJ^T = C
            uint64_t* eb = &bar[NSTAGE + (epi_uses % NSTAGE)];
            const uint32_t epar = (epi_uses / NSTAGE) & 1;
            ++epi_uses;
            if (tid == 0) {
#ifdef ELM_CHOL_PROF
                const uint64_t pw = globaltimer();
#endif
                wait_flag(flags + a.diag_tid[J], fin_ep, a.status, J, dist);
#ifdef ELM_CHOL_PROF
                pf_flag += globaltimer() - pw;
#endif
                fence_proxy_async();
                mbar_expect(eb, 2 * TILE * 8);
                bulk_load(Ys, Ybuf + (int64_t)J * TILE, TILE * 8, eb);
                bulk_load(Bs, tileptr(a.diag_tid[J]), TILE * 8, eb);
            }
            __syncthreads();  // C visible to every warp
            mbar_wait(eb, epar);
            double x0[4][2][2];
            trsm_refined(x0, As, Bs, Ys, a.trsm_refine);
            FOR_FRAG dst[frag_r(mt) + frag_c(nt, e) * LP] = x0[mt][nt][e];
            if (dist) {  // L(I,J) to the other replicas
                __threadfence_block();
                __syncthreads();
                push(0, (int64_t)td.tid * TILE);
            }
        }
        const int fval = pre ? pre_ep : fin_ep;
        if (dist) {
            __threadfence_system();
            __syncthreads();
            if (tid == 0)
                for (int r = 0; r < a.nrep; ++r) st_release_sys(a.reps[r].flags + td.tid, fval);
        } else {
            __threadfence();
            __syncthreads();
        }
        if (tid == 0 && !dist) {
            st_release(flags + td.tid, fval);
            if (!pre) asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(a.colcnt + J) : "memory");
#ifdef ELM_CHOL_PROF
            if (t < 400000) {
                unsigned long long* r = g_chol_prof + 6 * (size_t)t;
                r[0] = pt0; r[1] = globaltimer(); r[2] = pf_flag; r[3] = pf_data; r[4] = pte; r[5] = blockIdx.x;
            }
#endif
        }
    }
}
#undef FOR_FRAG

// ------------------------------------------------------------------------------------------
// Triangular solves as ONE cooperative (co-resident) kernel per direction.  Tasks (block rows, or
// chunks of a block row's dependency list: plan.cu build_trsv_tasks) are dealt in list order
// through a counter; a CTA streams the dependency tiles of its task straight from global memory
// into registers (no shared-memory staging, no block barrier per tile), each warp on its own:
// lane k checks the completion flag of dependency q + k (acquire), one ballot tells the warp how
// many of the next 32 dependencies are published, and those tiles are consumed without further
// polling, two at a time for memory-level parallelism.  The products are reduced once per task
// in a fixed order, then the diagonal tile (prefetched into shared memory) is solved by
// warp-level substitution and the block's flag released.
//   dir 0: L z = rhs    tiles (i, j), first[i] <= j < i     thread (row r, column group of 16)
//   dir 1: L^T u = rhs  tiles (j, i), i < j <= last[i]      warp: 8 columns c, lanes: rows r, r + 32
// ------------------------------------------------------------------------------------------
constexpr int TRSV_SMEM = (ELM_TS + 4 * NB + 2 * NB) * 8;

__device__ __forceinline__ void load_tile_async(double* dst, const double* src) {
    for (int t = threadIdx.x; t < ELM_TS / 2; t += blockDim.x) {
        unsigned d = su32(dst + 2 * t);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src + 2 * t));
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

#ifdef ELM_CHOL_PROF
// per task of the last launch of each direction: start, end, flag-wait ns, CTA (tools/trsv_prof.py)
__device__ unsigned long long g_trsv_prof[2][400000][4];
#endif

// The solution blocks are their own completion flags: the output vector is filled with an
// all-ones NaN pattern before the launch (no arithmetic result has it: computed NaNs are the
// canonical 0x7FF8...), a block's 64 values are written once with relaxed stores, and a consumer
// reads them with relaxed loads until none is the pattern (8-byte accesses are single-copy
// atomic).  One L2 round trip per dependency instead of a flag poll plus a data load, and no
// fence + release on the producer's side of the chain.
constexpr long long TRSV_EMPTY = -1LL;
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}

// One dependency tile in registers: forward, thread (r, cg) holds T(r, 16 cg + u), u < 16, and lane
// l holds x_j[16 cg + l % 16] (broadcast by shuffles); backward, lane l of warp w holds
// T(l, 8 w + u), T(l + 32, 8 w + u), u < 8, and x_j[l], x_j[l + 32].  Loaded one tile ahead, so
// the next tile's loads are in flight while this one is checked and consumed.
template <int DIR>
struct TrsvTile {
    double t[16];
    double x0, x1;
};
template <int DIR>
__device__ __forceinline__ void trsv_load(TrsvTile<DIR>& v, const double* __restrict__ Mb, int2 d, const double* out,
                                          int r, int cg, int lane, int w) {
    const double* T = Mb + (int64_t)d.y * ELM_TS;
    const double* xj = out + (int64_t)d.x * NB;
    if (DIR == 0) {  // element (r, c) at r + c LP
#pragma unroll
        for (int u = 0; u < 16; ++u) v.t[u] = __ldg(T + (cg * 16 + u) * LP + r);
        v.x0 = ld_relaxed_f64(xj + cg * 16 + (lane & 15));
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v.t[u] = __ldg(T + (8 * w + u) * LP + lane);
            v.t[u + 8] = __ldg(T + (8 * w + u) * LP + lane + 32);
        }
        v.x0 = ld_relaxed_f64(xj + lane);
        v.x1 = ld_relaxed_f64(xj + lane + 32);
    }
}
// wait until the x_j values of the tile are published (re-reading them), then accumulate:
// s[r] += sum_c T(r, c) x_j[c] (forward) / s[c] += sum_r T(r, c) x_j[r] (backward)
template <int DIR>
__device__ __forceinline__ void trsv_use(TrsvTile<DIR>& v, int2 d, const double* out, int cg, int lane,
                                         double& sacc, double (&tacc)[8], ElmStatus* status, int tag) {
    uint64_t t0 = 0;
    for (;;) {
        const bool ok = __double_as_longlong(v.x0) != TRSV_EMPTY && (DIR == 0 || __double_as_longlong(v.x1) != TRSV_EMPTY);
        if (__all_sync(0xffffffffu, ok)) break;
        if (!t0) {
            t0 = globaltimer();
        } else if (globaltimer() - t0 > 10000000000ull) {  // as wait_flag: report, give up
            if (lane == 0) elm_set_status(status, ELMDDM_ENUMERIC, -1 - tag);
            break;
        }
        __nanosleep(32);
        const double* xj = out + (int64_t)d.x * NB;
        if (DIR == 0) {
            v.x0 = ld_relaxed_f64(xj + cg * 16 + (lane & 15));
        } else {
            v.x0 = ld_relaxed_f64(xj + lane);
            v.x1 = ld_relaxed_f64(xj + lane + 32);
        }
    }
    if (DIR == 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) sacc += v.t[u] * __shfl_sync(0xffffffffu, v.x0, u);
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) tacc[u] += v.t[u] * v.x0 + v.t[u + 8] * v.x1;
    }
}

template <int DIR>
__global__ void __launch_bounds__(256, 2) k_band_trsv(const double* __restrict__ Mb, int ntasks, int nblk,
                                                      const int* __restrict__ diag_tid, const int4* __restrict__ tasks,
                                                      const int* __restrict__ rowslot, const int2* __restrict__ dep,
                                                      const double* __restrict__ rhs, double* out, int* flags,
                                                      int* pflags, double* __restrict__ ppart,
                                                      const int* __restrict__ epoch_dev, ElmStatus* status,
                                                      const double* __restrict__ Yb) {
    const int epoch = *epoch_dev;  // bumped in-stream by k_launch_prep (graph-replay safe)
    extern __shared__ __align__(16) double tsm[];
    double* dtile = tsm;                  // [ELM_TS] the diagonal tile (i, i)
    double* part = dtile + ELM_TS;        // [4][64]
    double* acc = part + 4 * NB;          // [64]
    double* rdv = acc + NB;               // [64] reciprocal diagonal
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int r = tid & 63, cg = tid >> 6;
    __shared__ int s_next;
    for (;;) {
        if (tid == 0) s_next = atomicAdd(flags + nblk, 1);
        __syncthreads();
        const int it = s_next;
        if (it >= ntasks) break;
        const int4 tk = tasks[it];
        const int i = tk.x;
        const bool fin = tk.w < 0;
        const int64_t i0 = (int64_t)i * NB;
        const int d0 = tk.y, nj = tk.z - tk.y;
#ifdef ELM_CHOL_PROF
        unsigned long long pt0 = globaltimer(), pfw = 0;
#endif
        if (fin) {  // the diagonal block's inverse Y = L(i,i)^{-1} (Yb), else the tile L(i,i)
            load_tile_async(dtile, Yb ? Yb + i0 * LP : Mb + (int64_t)diag_tid[i] * ELM_TS);
            if (tid < NB) acc[tid] = rhs[i0 + tid];
        }
        double sacc = 0.0, tacc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tacc[u] = 0.0;
        if (nj > 0) {
            TrsvTile<DIR> ta, tb;
            int2 da = dep[d0], db;
            trsv_load<DIR>(ta, Mb, da, out, r, cg, lane, w);
            for (int q = 0;;) {
                if (q + 1 < nj) {
                    db = dep[d0 + q + 1];
                    trsv_load<DIR>(tb, Mb, db, out, r, cg, lane, w);
                }
                trsv_use<DIR>(ta, da, out, cg, lane, sacc, tacc, status, i);
                if (++q >= nj) break;
                if (q + 1 < nj) {
                    da = dep[d0 + q + 1];
                    trsv_load<DIR>(ta, Mb, da, out, r, cg, lane, w);
                }
                trsv_use<DIR>(tb, db, out, cg, lane, sacc, tacc, status, i);
                if (++q >= nj) break;
            }
        }
        // reduce the partial products in a fixed order
        if (DIR == 0) {
            part[cg * NB + r] = sacc;
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                double v = tacc[u];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) part[8 * w + u] = v;
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::);  // the diagonal tile
        __syncthreads();
        if (!fin) {  // partial task: publish the chunk's 64 sums in slot tk.w
            if (tid < NB) {
                ppart[(int64_t)tk.w * NB + tid] =
                    DIR == 0 ? (part[tid] + part[NB + tid]) + (part[2 * NB + tid] + part[3 * NB + tid]) : part[tid];
                __threadfence();
            }
            __syncthreads();
            if (tid == 0) st_release(pflags + tk.w, epoch);
#ifdef ELM_CHOL_PROF
            if (tid == 0 && it < 400000) {
                unsigned long long* rp = g_trsv_prof[DIR][it];
                rp[0] = pt0; rp[1] = globaltimer(); rp[2] = pfw; rp[3] = blockIdx.x;
            }
#endif
            continue;
        }
        const int nparts = -1 - tk.w;
        const int s0 = rowslot[i];
        if (nparts > 0) {  // the row's partial tasks (earlier in the list) have published their slots
            if (tid == 0)
                for (int c = 0; c < nparts; ++c) wait_flag(pflags + s0 + c, epoch, status, i);
            __syncthreads();
        }
        if (tid < NB) {
            if (nj > 0) {
                const double own = DIR == 0 ? (part[tid] + part[NB + tid]) + (part[2 * NB + tid] + part[3 * NB + tid]) : part[tid];
                double tot = 0.0;  // the chunks' sums in fixed order, the own (last) chunk last
                for (int c = 0; c < nparts; ++c) tot += __ldcg(ppart + (int64_t)(s0 + c) * NB + tid);
                acc[tid] -= nparts == 0 ? own : tot + own;
            }
            if (!Yb) rdv[tid] = 1.0 / dtile[tid * LP + tid];
        }
        __syncthreads();
        if (Yb) {  // x_i = Y acc (forward) / Y^T acc (backward): one 64 x 64 GEMV, no serial chain
            if (DIR == 0) {
                const int r = tid & 63, cg = tid >> 6;
                double p = 0.0;
#pragma unroll
                for (int u = 0; u < 16; ++u) p += dtile[r + (16 * cg + u) * LP] * acc[16 * cg + u];
                part[cg * NB + r] = p;  // (part was read into acc before the barrier above)
                __syncthreads();
                if (tid < NB)
                    st_relaxed_f64(out + i0 + tid, (part[tid] + part[NB + tid]) + (part[2 * NB + tid] + part[3 * NB + tid]));
            } else {
                const int r = tid >> 2, q = tid & 3;
                double p = 0.0;
#pragma unroll
                for (int u = 0; u < 16; ++u) p += dtile[(q + 4 * u) + r * LP] * acc[q + 4 * u];
                p += __shfl_xor_sync(0xffffffffu, p, 1);
                p += __shfl_xor_sync(0xffffffffu, p, 2);
                if (q == 0) st_relaxed_f64(out + i0 + r, p);
            }
        } else if (tid < 32) {
            // diagonal solve with the lower tile (i, i): warp-level substitution
            const double* T = dtile;
            double z0 = acc[lane], z1 = acc[lane + 32];
            if (DIR == 0) {
                for (int cc = 0; cc < NB; ++cc) {
                    double xc = __shfl_sync(0xffffffffu, cc < 32 ? z0 : z1, cc & 31) * rdv[cc];
                    if (lane > cc) z0 -= T[cc * LP + lane] * xc;
                    if (lane + 32 > cc) z1 -= T[cc * LP + lane + 32] * xc;
                    if (lane == (cc & 31)) {
                        if (cc < 32) z0 = xc;
                        else z1 = xc;
                    }
                }
            } else {
                for (int cc = NB - 1; cc >= 0; --cc) {
                    double xc = __shfl_sync(0xffffffffu, cc < 32 ? z0 : z1, cc & 31) * rdv[cc];
                    if (lane < cc) z0 -= T[lane * LP + cc] * xc;
                    if (lane + 32 < cc) z1 -= T[(lane + 32) * LP + cc] * xc;
                    if (lane == (cc & 31)) {
                        if (cc < 32) z0 = xc;
                        else z1 = xc;
                    }
                }
            }
            st_relaxed_f64(out + i0 + lane, z0);  // (the values are the block's completion flag)
            st_relaxed_f64(out + i0 + lane + 32, z1);
#ifdef ELM_CHOL_PROF
            if (lane == 0 && it < 400000) {
                unsigned long long* rp = g_trsv_prof[DIR][it];
                rp[0] = pt0; rp[1] = globaltimer(); rp[2] = pfw; rp[3] = blockIdx.x;
            }
#endif
        }
        __syncthreads();
    }
}

// interface unknowns: strip order (the ABI's g / u_Gamma) <-> factorisation order
__global__ void k_perm_zero(double* __restrict__ y, int64_t n) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < n) y[x] = 0.0;  // padding unknowns keep 0 (unit diagonal)
}
__global__ void k_perm_gather(const double* __restrict__ g, const int* __restrict__ fbase, int q, int64_t G,
                              double* __restrict__ y) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < G) y[fbase[x / q] + x % q] = g[x];
}
__global__ void k_perm_scatter(const double* __restrict__ y, const int* __restrict__ fbase, int q, int64_t G,
                               double* __restrict__ u, int64_t Gpad) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x < G) u[x] = y[fbase[x / q] + x % q];
    else if (x < Gpad) u[x] = 0.0;
}

}  // namespace

#ifdef ELM_CHOL_PROF
extern "C" int elmddm_debug_chol_prof(void* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_chol_prof, sizeof(unsigned long long) * 6 * (size_t)n);
}
extern "C" int elmddm_debug_trsv_tasks(const elmddm_ctx* c, int dir, void* host) {  // int4[sv_ntasks[dir]]
    if (!host) return c->sv_ntasks[dir];
    return (int)cudaMemcpy(host, c->d_sv_tasks[dir], sizeof(int4) * c->sv_ntasks[dir], cudaMemcpyDeviceToHost);
}
extern "C" int elmddm_debug_trsv_prof(void* host, int dir, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_trsv_prof, sizeof(unsigned long long) * 4 * (size_t)n,
                                     sizeof(unsigned long long) * 4 * 400000 * (size_t)dir);
}
extern "C" int elmddm_debug_chol_dprof(void* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_chol_dprof, sizeof(unsigned long long) * 8 * (size_t)n);
}
#endif

namespace {
// multi-rank: wait until every tile of this replica has arrived (the factorisation kernel of
// this rank can end while other ranks still push their last tiles)
// Before a persistent launch on one rank: zero its task counter (if any) and advance its epoch
// counter in-stream, so that the kernel's flag comparisons stay fresh when the whole solve is
// captured once in a CUDA graph and replayed (a host-side epoch would be frozen into the graph).
__global__ void k_launch_prep(int* counter, int* epoch) {
    if (threadIdx.x == 0) {
        if (counter) *counter = 0;
        *epoch += 1;
    }
}

__global__ void k_drain(const int* flags, int ntiles, int epoch, ElmStatus* status) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x)
        wait_flag(flags + t, epoch, status, t, true);
}
// number of differing doubles between two buffers (one-GPU emulation check)
__global__ void k_count_diff(const double* a, const double* b, int64_t n, unsigned long long* cnt) {
    unsigned long long loc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        loc += __double_as_longlong(a[i]) != __double_as_longlong(b[i]);
    if (loc) atomicAdd(cnt, loc);
}
}  // namespace

cudaError_t dist_count_diff(const double* a, const double* b, int64_t n, unsigned long long* d_cnt, cudaStream_t st) {
    k_count_diff<<<592, 256, 0, st>>>(a, b, n, d_cnt);
    return cudaGetLastError();
}

cudaError_t run_cholesky_solve(const elmddm_ctx* c, double* Mband, const double* g, double* uG, double* work,
                               cudaStream_t st) {
    const CholPlan& pl = c->plan;
    const int64_t n = pl.n, G = c->sz.G;
    const int nblk = pl.nblk, q = c->plan_q;  // unknowns per plan face (64 on the dense plan of layout 1)
    double* yv = work;          // right-hand side, then the solution, in the factorisation order
    double* z = yv + n;
    double* Ybuf = z + n;       // [nblk] packed tiles (n is a multiple of 64: 16-byte aligned)
    double* Cbuf = Ybuf + (int64_t)nblk * ELM_TS;
    // iterative refinement (one step): the assembled M and the right-hand side are kept
    double* Mcopy = Cbuf + (int64_t)nblk * ELM_TS;  // [band_elems]
    double* gn = Mcopy + c->sz.band_elems;           // [n]
    double* rr = gn + n;                             // [n]
    cudaError_t e;
    // per-context (per-device) launch configuration, set up on the first call
    int& grid_ll = c->chol_grid;
    int& grid_sv = c->trsv_grid;
    if (!grid_ll) {
        if ((e = cudaFuncSetAttribute(k_chol_ll, cudaFuncAttributeMaxDynamicSharedMemorySize, llc::SMEM)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_band_trsv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSV_SMEM)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(k_band_trsv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSV_SMEM)) !=
                cudaSuccess)
            return e;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_ll, llc::NT, llc::SMEM);
        if (const char* env = getenv("ELMDDM_CHOL_CTAS_PER_SM")) per_sm = std::min(per_sm, atoi(env));
        grid_ll = (per_sm > 0 ? per_sm : 1) * c->nsm;
        // the solves are latency-bound (one dependent chain per tile row): as many co-resident
        // CTAs as fit, at most 3 per SM (cfg3: 2.79 ms at 1, 2.02 ms at 3)
        int sv_per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sv_per, k_band_trsv<1>, 256, TRSV_SMEM);
        {
            int sv0 = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sv0, k_band_trsv<0>, 256, TRSV_SMEM);
            sv_per = std::min(sv_per, sv0);
        }
        sv_per = std::min(sv_per, 3);
        if (const char* env = getenv("ELMDDM_TRSV_CTAS_PER_SM")) sv_per = std::min(sv_per, atoi(env));
        grid_sv = std::max(sv_per, 1) * c->nsm;
    }
    // right-hand side into the factorisation order
    k_perm_zero<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(yv, n);
    if (G > 0) k_perm_gather<<<(unsigned)((G + 255) / 256), 256, 0, st>>>(g, c->d_fbase, q, G, yv);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // factorisation: one cooperative launch over the task list
    const DistState& ds = c->dist;
    const bool dist = ds.nrep > 1;
    const double* Ybuf_solve = Ybuf;  // L(J,J)^{-1} tiles of the replica the solves read
    if (c->iface_refine) {
        // (one rank: the factorisation kernel saves the tiles of M as it reads them)
        if ((dist && (e = cudaMemcpyAsync(Mcopy, Mband, sizeof(double) * c->sz.band_elems, cudaMemcpyDeviceToDevice,
                                          st)) != cudaSuccess) ||
            (e = cudaMemcpyAsync(gn, yv, sizeof(double) * n, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return e;
    }
    if (dist) {
        const int nrep = ds.nrep;
        const int epoch = ++c->dist.epoch;
        int grid = grid_ll, per = grid_ll;
        if (ds.emulate) {
            per = grid_ll / nrep;
            grid = per * nrep;
            if ((e = cudaMemsetAsync(ds.counter + (epoch & 1), 0, sizeof(int), st)) != cudaSuccess) return e;
        } else if (ds.rank == 0) {
            // slot epoch & 1 was zeroed one factorisation ago; zero the next one (no rank can
            // still be using it: every rank finished the previous factorisation before the
            // all-reduce that precedes this one)
            if ((e = cudaMemsetAsync(ds.counter + ((epoch + 1) & 1), 0, sizeof(int), st)) != cudaSuccess) return e;
        }
        const CholRep& mine = ds.reps[ds.emulate ? 0 : ds.rank];
        CholArgs a{mine.Mb, mine.Ybuf, mine.Cbuf, mine.cready, c->d_tasks, (int)pl.tasks.size(), 0, 0, c->d_klist,
                   c->d_diag_tid, mine.flags, c->d_colcnt, c->d_ntc, epoch, nullptr, c->d_status, ds.counter + (epoch & 1),
                   nrep, ds.emulate ? 0 : ds.rank, per, ds.d_reps, nullptr, c->chol_trsm_refine, c->d_tile_m};
        void* args[] = {(void*)&a};
        {
            KTimer kt(c, ELMDDM_K_POTRF, st);
            if ((e = cudaLaunchCooperativeKernel((void*)k_chol_ll, dim3(grid), dim3(llc::NT), args, llc::SMEM, st)) !=
                cudaSuccess)
                return e;
        }
        k_drain<<<(unsigned)c->nsm, 256, 0, st>>>(mine.flags, pl.ntiles, 2 * epoch, c->d_status);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        Mband = mine.Mb;  // the triangular solves read this rank's replica
        Ybuf_solve = mine.Ybuf;
    } else {
        int grid = grid_ll;
        int crit = 32;
        if (const char* env = getenv("ELMDDM_CHOL_CRIT")) crit = atoi(env);
        crit = std::max(1, std::min(crit, grid / 4));  // grid >= 148 on this part: both groups non-empty
        CholArgs a{Mband, Ybuf, Cbuf, c->d_cready, c->d_tasks, (int)pl.tasks.size(), pl.ncrit, crit, c->d_klist,
                   c->d_diag_tid, c->d_cflags, c->d_colcnt, c->d_ntc, 0, c->d_epoch, c->d_status,
                   c->chol_sched ? c->d_chol_next : nullptr, 1, 0, grid, nullptr, c->iface_refine ? Mcopy : nullptr,
                   c->chol_trsm_refine, c->d_tile_m};
        k_launch_prep<<<1, 32, 0, st>>>(c->chol_sched ? c->d_chol_next : nullptr, c->d_epoch);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        void* args[] = {(void*)&a};
        KTimer kt(c, ELMDDM_K_POTRF, st);
        if ((e = cudaLaunchCooperativeKernel((void*)k_chol_ll, dim3(grid), dim3(llc::NT), args, llc::SMEM, st)) !=
            cudaSuccess)
            return e;
    }
    // triangular solves: one cooperative wavefront kernel per direction (b -> z -> x)
    auto solve = [&](double* b, double* x) -> cudaError_t {
        int* flags = c->d_flags;
        for (int dir = 0; dir < 2; ++dir) {
            int* epoch = c->d_epoch + 1;
            const double* rhs = dir == 0 ? b : z;
            double* out = dir == 0 ? z : x;
            int nblk_v = nblk, ntasks = c->sv_ntasks[dir];
            const int grid = ntasks < grid_sv ? ntasks : grid_sv;
            const int* dt = c->d_diag_tid;
            const int4* tl = c->d_sv_tasks[dir];
            const int* rs = c->d_sv_slot[dir];
            const int2* dl = dir == 0 ? c->d_fwd : c->d_bwd;
            int* pf = c->d_pflags;
            double* pp = c->d_ppart;
            ElmStatus* stp = c->d_status;
            const double* yinv = c->trsv_inv ? Ybuf_solve : nullptr;
            void* args[] = {(void*)&Mband, (void*)&ntasks, (void*)&nblk_v, (void*)&dt, (void*)&tl, (void*)&rs,
                            (void*)&dl,    (void*)&rhs,    (void*)&out,    (void*)&flags, (void*)&pf, (void*)&pp,
                            (void*)&epoch, (void*)&stp,  (void*)&yinv};
            k_launch_prep<<<1, 32, 0, st>>>(flags + nblk, epoch);  // the task counter, the epoch
            cudaError_t e1 = cudaGetLastError();
            if (e1 == cudaSuccess) e1 = cudaMemsetAsync(out, 0xFF, sizeof(double) * nblk * NB, st);  // TRSV_EMPTY
            if (e1 != cudaSuccess) return e1;
            KTimer kt(c, ELMDDM_K_TRSV, st);
            cudaError_t e2 = cudaLaunchCooperativeKernel(dir == 0 ? (void*)k_band_trsv<0> : (void*)k_band_trsv<1>, dim3(grid), dim3(256), args, TRSV_SMEM, st);
            if (e2 != cudaSuccess) return e2;
        }
        return cudaSuccess;
    };
    if ((e = solve(yv, yv)) != cudaSuccess) return e;
    // one step of iterative refinement with the assembled M (reading R30): x += M^{-1}(g - M x)
    // through the same factor.  The tile factorisation's explicit diagonal-block inverses leave a
    // forward error a few times that of a dense factorisation on the same M (measured at config
    // 2: 6.5e-10 -> 5.3e-11 vs the exact solution, tools/accuracy_study.py)
    if (c->iface_refine) {
        if ((e = launch_residual(c, Mcopy, yv, gn, rr, st)) != cudaSuccess) return e;
        if ((e = solve(rr, rr)) != cudaSuccess) return e;
        if ((e = launch_axpy1(yv, rr, n, st)) != cudaSuccess) return e;
    }
    // solution back into the strip order of u_Gamma
    const int64_t Gp = c->sz.G_pad;
    k_perm_scatter<<<(unsigned)((Gp + 255) / 256), 256, 0, st>>>(yv, c->d_fbase, q, G, uG, Gp);
    return cudaGetLastError();
}
