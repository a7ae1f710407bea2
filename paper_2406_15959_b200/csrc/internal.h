// internal.h -- private declarations of the elmddm CUDA library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/elmddm.h"

#define ELM_NB 64      // panel width of the blocked QR, tile of the band Cholesky
#define ELM_BB 8       // base block width inside a QR panel
#define ELM_TLD 68     // column stride inside a packed 64 x 64 tile of the Schur matrix (== 4 mod 16)
#define ELM_TS (ELM_NB * ELM_TLD)  // doubles per packed tile

// Implicit E_Gamma: column col of K_aug is never written by elmddm_assemble when
// the 64-column tile of the first trailing update (j0 = 0: tiles start at min(64, M) + 64 t)
// holding it lies entirely inside the E_Gamma block [M, M + ne) (ne = 4q, or 4q + 4 with the
// lattice's corners); that update synthesises the unit columns in shared memory instead of loading
// them.  Returns [begin, end) of those columns.
inline void elm_e_implicit_range(int M, int ne, int* begin, int* end) {
    const int c0 = M < ELM_NB ? M : ELM_NB;
    const int t_first = c0 + ((M - c0 + ELM_NB - 1) / ELM_NB) * ELM_NB;   // first tile start >= M
    int t_end = c0 + ((M + ne - c0) / ELM_NB) * ELM_NB;                  // last tile end <= M + ne
    if (t_end < t_first) t_end = t_first;
    *begin = t_first;
    *end = t_end;
}

// Packed tile storage of the Schur matrix: tile t of the factor's tile structure
// (CholPlan::tile_map) is stored contiguously at t * ELM_TS with element (r, c) at r + c * ELM_TLD,
// so one bulk copy reproduces the conflict-free padded shared-memory layout of the DMMA kernels.

// Device status word: [0] error code (ELMDDM_ENUMERIC), [1] info (column / index).
// ElmStatus.info of ELMDDM_ENUMERIC: >= 0 interface Cholesky row of a non-positive pivot;
// -1 - tag: a dependency wait that exceeded 10 s; <= ELM_INFO_NONFINITE_QR: non-finite R11 of
// subdomain ELM_INFO_NONFINITE_QR - info
constexpr int ELM_INFO_NONFINITE_QR = -(1 << 30);
struct ElmStatus {
    int code;   // first error (ELMDDM_ENUMERIC ...) and its info
    int info;
    int wcode;  // first warning (ELMDDM_WRANK) and its info (global subdomain index)
    int winfo;
};

// One contribution to an interface-matrix face block, see schur.cu.
struct FaceTerm {
    int kind;  // 0: S1 block of Sbuf[s], 1: Ga block of face a
    int src;   // s or a
    int r0;    // row offset inside the source block
    int c0;    // column offset inside the source block
};

// one tile task of the interface Cholesky (plan.cu / chol.cu)
struct TaskDesc {
    int I, J;        // tile of L
    int tid;         // its tile id (offset tid * ELM_TS in the tile pool)
    int kbeg, kend;  // its update list klist[kbeg, kend)
    int klast;       // diagonal tasks: the last update column (applied by the task itself), or -1
    int pub;         // publish C(I, J) for the diagonal task of row I (J == klast(I))
    int kind;        // 0 whole task; 1 pre-aggregation: the updates from columns below J's
                     // dissection node, summed into the tile of M in place (flag 2 epoch - 1);
                     // 2 the rest of a split task (waits for its pre-aggregation first)
};

// ordering and symbolic factorisation of the interface Schur matrix at 64-tile granularity
// One replica of the multi-rank interface factorisation (chol.cu k_chol_ll, nrep > 1).
struct CholRep {
    double* Mb;     // tile pool [ntiles][ELM_TS]
    double* Ybuf;   // [nblk][ELM_TS] L(J,J)^{-1}
    double* Cbuf;   // [nblk][ELM_TS] published C(I, klast(I))
    int* flags;     // [ntiles] tile completion (epoch)
    int* cready;    // [nblk] Cbuf published (epoch)
};
// Multi-rank state: every rank holds a full replica in one cudaMalloc'd region (exported /
// imported with CUDA IPC); one-GPU emulation keeps all replicas in this process.
struct DistState {
    int nrep = 1, rank = 0;
    int epoch = 0;               // factorisation epoch of the shared protocol (agreed: reset at import)
    bool emulate = false;
    std::vector<CholRep> reps;   // host copy of the table
    CholRep* d_reps = nullptr;   // device table [nrep]
    int* counter = nullptr;      // task counter slots [2] in rank 0's region (epoch parity)
    void* region = nullptr;      // this rank's region
    size_t region_bytes = 0;
    std::vector<void*> opened;   // peer regions opened through IPC (closed on destroy)
};

struct CholPlan {
    int ordering = 0;                 // 0 strip (envelope), 1 nested dissection
    int64_t n = 0;                    // unknowns in the factorisation order (multiple of 64)
    int nblk = 0, ntiles = 0, ncrit = 0;
    int64_t nupd = 0;                 // tile updates (work = 2 * 64^3 * nupd)
    std::vector<int> fbase, pad, tile_map, diag_tid, ntc, fwd_ptr, bwd_ptr;
    std::vector<int> blk_depth;       // nested-dissection depth of each tile column (0 = top separator)
    std::vector<int> blk_node0;       // first tile column of the dissection node of each column
    int npre = 0;                     // pre-aggregation tasks (kind 1)
    std::vector<TaskDesc> tasks;      // critical band first, then the rest; each column by column
    std::vector<int4> klist;
    std::vector<int2> fwd, bwd;
    // the tiles of M itself (before fill): row lists (J, tile (I, J)), J < I, and column lists
    // (J, tile (J, I)), J > I, descending -- the packed-tile SpMV of M (refinement residual, CG)
    // reads only these (the fill tiles of the factorisation are zero in M)
    std::vector<int> mrow_ptr, mcol_ptr;
    std::vector<unsigned char> tile_m;  // [ntiles] 1: a tile of M itself, 0: fill
    std::vector<int2> mrow, mcol;
};
int64_t build_chol_plan(int P, int q, int F, const std::vector<std::pair<int, int>>& face_pairs, int ordering,
                        int crit_band, CholPlan& pl, int split_min = 0);
double schedule_chol_tasks(CholPlan& pl, int workers);
// Task list of one triangular-solve direction (dir 0 forward, 1 backward; chol.cu k_band_trsv):
// the dependency list of a block row longer than `chunk` tiles is split into balanced chunks;
// every chunk but the last is a partial task {i, q0, q1, slot} writing its 64 partial sums to a
// slot, placed in the list right after the row its latest dependency waits for; the row's final
// task {i, q0, q1, -1 - nparts} takes the last chunk, the partial slots rowslot[i] ..
// rowslot[i] + nparts - 1 in fixed order, and the diagonal solve.  Returns the slot count.
int build_trsv_tasks(const CholPlan& pl, int dir, int chunk, std::vector<int4>& tasks, std::vector<int>& rowslot);
int chol_split_min();
int panel_cl_stage(int64_t ld, int smem_optin);  // qr.cu: ring stage of the cluster panel, 0 = ld too tall
void export_tasks(const CholPlan& pl, int32_t* tasks);
void interface_face_pairs(int P, std::vector<std::pair<int, int>>& out);
double chol_eval(const CholPlan& pl, const std::vector<int>& order, int workers);

struct elmddm_ctx {
    elmddm_config cfg;
    int device;
    elmddm_sizes_t sz;
    std::string err;
    ElmStatus* d_status = nullptr;
    int nsm = 148;

    // geometry (host)
    int faces = 0;
    std::vector<int> face_sub;   // [faces][2] subdomains (lower/left first)
    std::vector<int> face_edge;  // [faces][2] local edge of the face in each subdomain
    std::vector<int> sub_face;   // [N][4] face of edge e of subdomain s, -1 = Dirichlet
    // flux-face neighbour slots (Q row blocks): nbr[a][7] faces, -1 = empty
    std::vector<int> nbr;
    // device copies
    int* d_sub_face = nullptr;   // [N][4]
    int* d_qsrc = nullptr;       // [faces][8 slots][2 contributors][3] = (s, row edge, col edge) or -1
    int* d_pair_ptr = nullptr;   // CSR over face-block pairs (b, c), b >= c
    int* d_pair_bc = nullptr;    // [npairs][2]
    FaceTerm* d_terms = nullptr; // contributions of each pair
    int* d_gterm_ptr = nullptr;  // CSR over faces b for g terms
    FaceTerm* d_gterms = nullptr;
    int* d_umap = nullptr;       // [N][ne] local interface column -> global unknown or -1 (both layouts)
    int* d_eqsrc = nullptr;      // layout 1: [n_eq][2 contributors][(s, flux row)], ascending s
    int* d_rmap = nullptr;       // layout 1: [G][4][(s, local column)], ascending s, -1 padded
    int* d_tile_I = nullptr;     // layout 1: tile id -> (I, J) of the dense plan
    int* d_tile_J = nullptr;
    int* d_feq = nullptr;        // layout 1: [faces][q + 2] equations of each face block (-1 padded)
    int* d_fpair = nullptr;      // layout 1: [faces][2] the block's two subdomains (ascending)
    int* d_flist = nullptr;      // layout 1: [G][16][(face, column)] copies of every unknown
    int lat_nrow = 0;            // layout 1: rows of a face block (q + 2)
    int plan_q = 0;              // unknowns per plan "face" (q, or 64 for the dense plan of layout 1)
    int64_t ld_q = 0;            // layout 1: leading dimension of the dense Q (n_eq rounded up)
    int npairs = 0, nterms = 0, ngterms = 0;
    int qrow_ld = 0, qrow_cols = 0, ga_ld = 0;  // Q row block: q x (7q+1), ld qrow_ld; Ga: ga_ld^2
    int64_t work_factor = 0, work_iface = 0, work_back = 0;

    // instrumentation (mutable: launch wrappers take a const context)
    mutable int timing = 0;
    int schur_side = 1;  // S_s GEMM on a side stream beside the TRSM (ELMDDM_SCHUR_SIDE=0: in order)
    mutable int64_t launches = 0;
    mutable int64_t cls_count[ELMDDM_NCLASS] = {};
    mutable double cls_ms[ELMDDM_NCLASS] = {};
    mutable std::vector<cudaEvent_t> ev_pool;                 // free events
    mutable std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;

    // internal streams for the subdomain groups of the QR (fork / join with events)
    int qr_groups = 4;
    int use_tma = 1;  // TMA-staged trailing update (ELMDDM_TMA=0 selects the cp.async kernel)
    int wy_hint3 = 1;  // trailing update phase 3: C loads / stores evict-first in L2 (ELMDDM_WY_HINT3)
    int wy_rev3 = 1;  // trailing update phase 3 bottom-up (L2 reuse of phase 1's last chunks; ELMDDM_WY_REV3)
    // k_panel_t on <= 2048 rows with 256 TMEM columns / 112 KB, so that two panel CTAs can share an SM
    // (ELMDDM_PANEL_PAIR=0: 512 / 116 KB, one per SM).  Config 4 local_factor 195.0 -> 193.0 ms
    // (8 groups); with 1 group (panels never beside trailing updates) 216.0 -> 199.1 ms
    int panel_pair = 1;
    // Schur TRSM with the flux-row tiles of a subdomain as one cluster, R11 chunks TMA-multicast
    // (ELMDDM_TRSM_CLUSTER=1; bit-identical, but config 4 TRSM 10.6 -> 12.5 ms: the per-chunk
    // cluster-wide empty handshake makes the slowest CTA gate all four)
    int trsm_cluster = 0;
    // Schur TRSM with 128 flux rows per CTA (ELMDDM_TRSM_WIDE=1; bit-identical, halves the R11
    // traffic, but config 4 TRSM 10.7 -> 11.4 ms: one 512-thread CTA per SM has no second CTA to
    // fill the pipe during its diagonal solves)
    int trsm_wide = 0;
    int gemm_tma = 1;      // batched A^T B GEMMs through the TMA / mbarrier kernel (ELMDDM_GEMM_TMA=0: cp.async)
    int panel_grid = 0;    // cooperative grid panel (automatic for very tall local problems; ELMDDM_PANEL_GRID=1)
    int iface_refine = 1;  // one step of iterative refinement of the interface solve (ELMDDM_IFACE_REFINE)
    int implicit_e = 1;  // E_Gamma tiles never written by the assembly, synthesised by the first
                         // trailing update (elm_e_implicit; needs use_tma; ELMDDM_IMPLICIT_E=0 off)
    int panel_cluster = 0;  // QR panel blocks on 4-CTA clusters (default for S <= 48; ELMDDM_PANEL_CLUSTER)
    int* d_flags = nullptr;          // per 64-block completion flags of the wavefront triangular solves
    int* d_epoch = nullptr;          // [2] device epoch counters: factorisation, triangular solves
                                     // (advanced in-stream by k_launch_prep: graph-replay safe)
    // refinement step in the factorisation's tile solves X = C L(J,J)^{-T} (ELMDDM_CHOL_TRSM_REFINE;
    // default: only when the solution-level refinement step R30 is off -- with it, config 4
    // 84.1 -> 80.2 ms factorisation, error vs exact 1.2e-11 -> 6.1e-11, config 3 3.1e-9 -> 6.3e-10)
    int chol_trsm_refine = -1;
    int trsv_inv = 1;                   // triangular solves: diagonal blocks by their explicit inverse (ELMDDM_TRSV_INV)
    int trsv_chunk = 0;                 // dependency tiles per triangular-solve task, 0 = whole rows
                                        // (ELMDDM_TRSV_CHUNK; 32 / 64 measured slower at config 4)
    int4* d_sv_tasks[2] = {nullptr, nullptr};  // per direction: the task lists of build_trsv_tasks
    int* d_sv_slot[2] = {nullptr, nullptr};    // per direction: first partial slot of each block row
    int sv_ntasks[2] = {0, 0};
    int* d_pflags = nullptr;            // [slots] completion flags of the partial tasks
    double* d_ppart = nullptr;          // [slots][64] partial sums
    // ordering + symbolic factorisation of the Schur matrix (plan.cu) and its device copies
    CholPlan plan;
    int ncrit = 0;                   // the first ncrit tasks are the critical band (I - J <= crit_band)
    int crit_band = 3;               // ELMDDM_CHOL_CRITBAND
    double* d_grf = nullptr;         // problem 6: eqn:grf parameters [ngrf][4] (elmddm_set_coefficient)
    int ngrf = 0;
    double* d_coef = nullptr;        // problem 6: [S][p*p][4] rho, grad rho at the interior points
    mutable DistState dist;          // multi-rank interface factorisation (elmddm_dist_*)
    int panel_prio = 1;              // ELMDDM_PANEL_PRIO: panels on high-priority streams (with k_panel_t)
    int panel8_tmem = 0;             // ELMDDM_PANEL8_TMEM: 8-CTA cluster panel in TMEM (k_panel_c8t)
    int panel_tmem = 1;              // ELMDDM_PANEL_TMEM: TMEM-resident panel block (k_panel_t)
    int panel_merged = 1;            // ELMDDM_PANEL_MERGED: one launch per panel, merged Gram pass (k_panel_p)
    int panel8 = 0;                  // ELMDDM_PANEL8: on-chip 8-CTA cluster panels (qr.cu k_panel_c8)
    int chol_sched = 1;              // ELMDDM_CHOL_SCHED: 1 list-scheduled task order, dynamic dealing
    double chol_sim_us = 0.0;        // simulated makespan of the scheduled order
    int* d_chol_next = nullptr;      // dynamic task counter
    int64_t chol_flops = 0;          // 2 * 64^3 per tile update
    int* d_fbase = nullptr;          // [faces] first unknown of each face in the factorisation order
    int* d_pad = nullptr;            // [npad] padding unknowns (unit diagonal, zero right-hand side)
    int* d_tile_map = nullptr;       // [nblk * nblk] tile id of (I, J), I >= J, or -1
    TaskDesc* d_tasks = nullptr;     // [ntasks]
    int4* d_klist = nullptr;         // [nupd] (tile (I,k), tile (J,k), k, 0)
    int* d_diag_tid = nullptr;       // [nblk]
    int* d_fwd_ptr = nullptr;        // [nblk + 1] CSR of the forward-solve dependencies
    int2* d_fwd = nullptr;           // (j, tile (i, j)), ascending j
    int* d_bwd_ptr = nullptr;        // [nblk + 1] CSR of the backward-solve dependencies
    int2* d_bwd = nullptr;           // (j, tile (j, i)), descending j
    unsigned char* d_tile_m = nullptr;  // [ntiles] CholPlan::tile_m
    int* d_mrow_ptr = nullptr;       // CSR of M's own off-diagonal tiles (CholPlan::mrow / mcol)
    int2* d_mrow = nullptr;
    int* d_mcol_ptr = nullptr;
    int2* d_mcol = nullptr;
    int* d_cflags = nullptr;         // [ntiles] per-tile completion flags of the factorisation
    int* d_colcnt = nullptr;         // [nblk] finished tiles of column J (summed over factorisations)
    int* d_ntc = nullptr;            // [nblk] tiles of column J
    int* d_cready = nullptr;         // [nblk] C(I, klast(I)) published for the diagonal task of row I
    mutable int chol_grid = 0, trsv_grid = 0;  // persistent-kernel grids (chol.cu, first call)
    mutable std::vector<cudaStream_t> gstreams;
    mutable cudaEvent_t ev_fork = nullptr;
    mutable std::vector<cudaEvent_t> ev_join;
    cudaError_t ensure_streams(int n) const {
        cudaError_t e = cudaSuccess;
        if (!ev_fork && (e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        while ((int)gstreams.size() < n) {
            cudaStream_t s;
            cudaEvent_t ev;
            if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
            gstreams.push_back(s);
            ev_join.push_back(ev);
        }
        return e;
    }
    // high-priority panel streams (one per subdomain group) and the panel / trailing-update
    // hand-over events: a pending co-residable panel CTA takes the next free half-SM first
    mutable std::vector<cudaStream_t> pstreams;
    mutable std::vector<cudaEvent_t> ev_panel, ev_wy;
    cudaError_t ensure_panel_streams(int n) const {
        cudaError_t e = cudaSuccess;
        int least = 0, greatest = 0;
        if ((e = cudaDeviceGetStreamPriorityRange(&least, &greatest)) != cudaSuccess) return e;
        while ((int)pstreams.size() < n) {
            cudaStream_t s;
            cudaEvent_t a, b;
            if ((e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, greatest)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) return e;
            pstreams.push_back(s);
            ev_panel.push_back(a);
            ev_wy.push_back(b);
        }
        return e;
    }
};

// RAII probe around one kernel launch: counts it and, when timing is on, brackets it with a
// CUDA event pair on the launch stream.
struct KTimer {
    const elmddm_ctx* c;
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    KTimer(const elmddm_ctx* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
        if (!c) return;
        ++c->launches;
        ++c->cls_count[cls];
        if (c->timing) {
            a = take();
            b = take();
            cudaEventRecord(a, st);
        }
    }
    ~KTimer() {
        if (c && c->timing && a) {
            cudaEventRecord(b, st);
            c->ev_pending.push_back({cls, {a, b}});
        }
    }
    cudaEvent_t take() {
        if (!c->ev_pool.empty()) {
            cudaEvent_t e = c->ev_pool.back();
            c->ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};

// ------------------------------------------------------------------------------------------
// batched DMMA GEMM:  C[b] = alpha * op(A[b]) op(B[b]) + beta * C[b], column-major, fp64
// ------------------------------------------------------------------------------------------
struct GemmArgs {
    int M, N, K;
    const double* A;
    int64_t lda, sA;
    const double* B;
    int64_t ldb, sB;
    double* C;
    int64_t ldc, sC;
    double alpha, beta;
    int batch;
    int lower_only;  // skip 64x64 output tiles strictly above the diagonal
};
// r = g - M x (packed-tile symmetric M, factorisation order; cg.cu) and x += d
cudaError_t run_interface_assemble_lattice(const elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband,
                                           double* g, double* work, cudaStream_t st);
cudaError_t launch_residual(const elmddm_ctx* c, const double* Mband, const double* x, const double* g, double* r,
                            cudaStream_t st);
cudaError_t launch_axpy1(double* x, const double* d, int64_t n, cudaStream_t st);
cudaError_t gemm_launch(bool transA, bool transB, const GemmArgs& g, cudaStream_t st,
                        const elmddm_ctx* c = nullptr, int cls = ELMDDM_K_GEMM_QR);

// kernels in the other translation units
cudaError_t launch_init_hidden(const elmddm_ctx* c, double* W, double* b, double* xi, cudaStream_t st);
cudaError_t launch_assemble(const elmddm_ctx* c, const double* W, const double* b, double* Kaug, double* At,
                            cudaStream_t st);
cudaError_t launch_evaluate(const elmddm_ctx* c, const double* W, const double* b, const double* coef,
                            const double* xy, int64_t n, double* u, cudaStream_t st);
cudaError_t run_local_factor(const elmddm_ctx* c, double* Kaug, double* tau, double* work, cudaStream_t st);
cudaError_t run_schur_accumulate(const elmddm_ctx* c, double* Kaug, double* At, double* Pbuf, double* Sbuf,
                                 double* work, cudaStream_t st);
cudaError_t run_interface_assemble(const elmddm_ctx* c, const double* Pbuf, const double* Sbuf, double* Mband,
                                   double* g, double* work, cudaStream_t st);
cudaError_t dist_count_diff(const double* a, const double* b, int64_t n, unsigned long long* d_cnt, cudaStream_t st);
cudaError_t run_cholesky_solve(const elmddm_ctx* c, double* Mband, const double* g, double* uG, double* work,
                               cudaStream_t st);
cudaError_t run_interface_cg(const elmddm_ctx* c, const double* Mband, const double* g, double* uG, double* work,
                             double tol, int maxit, int* iters, double* relres, cudaStream_t st);
cudaError_t run_back_solve(const elmddm_ctx* c, const double* Kaug, const double* uG, double* coef, double* resid,
                           double* work, cudaStream_t st);

#ifdef __CUDACC__
__device__ __forceinline__ void elm_set_status(ElmStatus* st, int code, int info) {
    if (atomicCAS(&st->code, 0, code) == 0) st->info = info;
}
__device__ __forceinline__ void elm_set_warning(ElmStatus* st, int code, int info) {
    if (atomicCAS(&st->wcode, 0, code) == 0) st->winfo = info;
}
#endif
