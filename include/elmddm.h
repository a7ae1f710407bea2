/*
 * elmddm.h -- C ABI of the B200-native DDM-ELM hot path
 * (arxiv 2406.15959: "nonoverlapping domain decomposition for extreme learning machines").
 *
 * The calls follow Algorithm 1:
 *     Set theta^s randomly                     -> elmddm_init_hidden   (eqn:init)
 *     for s in parallel: construct K,A,B,F     -> elmddm_assemble      (eqn:nonoverlap_discrete)
 *     [factor every local LS]                  -> elmddm_local_factor  (K^+ of P:356 via Householder QR)
 *     [eliminate c into the Schur system]      -> elmddm_schur_accumulate  (eqn:eliminated..eqn:schur)
 *     Solve eqn:schur for u_Gamma              -> elmddm_interface_assemble + elmddm_interface_factor_solve
 *                                                 (= elmddm_interface_solve)
 *     for s in parallel: solve for c^s         -> elmddm_back_solve
 *     [evaluate the solution]                  -> elmddm_evaluate      (error tables, e.g. P:593)
 *
 * Conventions (DESIGN.md §2 has the full statement):
 *  - Geometry: (0,1)^2 split into P x P squares, subdomain s = j*P + i (i along x).  Each subdomain
 *    has p*p interior collocation points and q points on each of its 4 edges (endpoints excluded),
 *    m = p*p + 4q rows ordered [interior (row-major b, a) | left | right | bottom | top].
 *  - Interface unknowns u_Gamma: G = 2P(P-1)q, face-major in strip order, points in increasing
 *    coordinate (elmddm_interface_points exports the coordinates).
 *  - Every array argument is a DEVICE pointer owned by the caller (e.g. a torch tensor), fp64,
 *    column-major, 16-byte aligned; the library never allocates or frees caller memory.  Sizes
 *    and leading dimensions come from elmddm_sizes.  The library owns only its opaque context and
 *    small internal tables (< a few MB).  Work is enqueued on the given stream; calls return
 *    after enqueueing (asynchronous) except where stated.
 *  - A rank owns the contiguous subdomain range [s_begin, s_end); per-subdomain arrays are
 *    indexed by the local index s - s_begin ("S_local" slots) unless stated "global".
 *  - Errors: arguments are validated synchronously before any launch (ELMDDM_EINVAL, nothing
 *    enqueued).  Numerical failures detected on the device (non-positive Cholesky pivot,
 *    non-finite value) set a device status word, reported by elmddm_sync and by the return of
 *    elmddm_interface_solve (which synchronises its stream); elmddm_last_error gives text.  The
 *    per-phase calls, elmddm_interface_factor_solve included, never synchronise, so a whole
 *    solve can be enqueued back to back (and captured in a CUDA graph) with one elmddm_sync at
 *    the end.
 *  - Threading: one context per device per host thread.
 */
#ifndef ELMDDM_H
#define ELMDDM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ELMDDM_OK = 0,
    ELMDDM_EINVAL = 1,   /* bad argument / configuration (nothing was enqueued) */
    ELMDDM_ENUMERIC = 2, /* non-positive pivot or non-finite value detected on the device */
    ELMDDM_ECUDA = 3,    /* CUDA runtime error (text in elmddm_last_error) */
    ELMDDM_ENOMEM = 4,   /* internal table allocation failed */
    ELMDDM_WRANK = 100   /* WARNING, not an error (SPEC factorize_ls: "warns (not errors) when
                            sigma_min/sigma_max < 1e-14"): some subdomain's R11 has
                            min|R11_ii| < 1e-14 max|R11_ii| (which implies sigma_min/sigma_max <
                            1e-14 for K^s); every output is still computed.  Reported once by the
                            next elmddm_sync / elmddm_interface_solve, subdomain in
                            elmddm_last_error.  Expected for the BASELINE configs >= 1: ELM
                            collocation matrices are numerically rank deficient (reading R11). */
} elmddm_status;

typedef struct elmddm_ctx elmddm_ctx;

typedef struct {
    int32_t P;              /* subdomains per axis (N = P*P subdomains of side h = 1/P)        */
    int32_t M;              /* hidden neurons per subdomain, n_N of P:199 (multiple of 8)      */
    int32_t p;              /* interior collocation points per axis per subdomain              */
    int32_t q;              /* collocation points per subdomain edge (even)                    */
    int32_t problem;        /* manufactured solution: 0 sin(pi x)sin(pi y) | 1 e^{x+y}sin(2pi x)cos(2pi y)
                               | 2 sin(4pi x)sin(4pi y) | 3 sin(8pi x)sin(8pi y) | 4 sin(2pi x)e^y
                                | 5 u = 0 | 6 variable coefficient -div(rho grad u) = 1,
                               u = 0 on the boundary, rho = tanh(grf) + 1.1 (eqn:varpoisson,
                               P:694-701; needs elmddm_set_coefficient) | 7 Kirchhoff plate
                               Lap^2 u = q/D, u = Lap u = 0 on the boundary, q = sin(pi x)sin(pi y),
                               E = 1e7, H = 1e-3, nu = 0.3: TWO traces per edge point, so
                               q = 2 x (points per edge), each edge's rows / interface unknowns
                               [u at the q/2 points | Lap u at the same points] (reading R28)  */
    int32_t init_scheme;    /* 0 paper eqn:init l = c sqrt(N*M) | 1 manual l = 1 | 2 He l = sqrt(2/M), b = 0 */
    double init_c;          /* c of eqn:init (1/8 for Poisson)                          */
    double r_over_diam;     /* r = r_over_diam * diam(Omega_s) (1/2)                    */
    uint64_t seed;          /* counter-based RNG key (reading R9)                    */
    int32_t s_begin, s_end; /* subdomains owned by this rank: [s_begin, s_end) of 0..N-1       */
    int32_t interface_mode; /* factorisation order of the Schur matrix: 0 auto (less work) |
                               1, 2 strip order (envelope) | 3 nested dissection             */
    int32_t layout;         /* collocation layout: 0 face points (reading R1: p x p interior + q per
                               edge, endpoints excluded) | 1 the paper's shared lattice (P:436-438,
                               reading R32; p == q == n - 1 for n lattice cells per subdomain side):
                               the 4 subdomain corners are rows too, interior corners are cross
                               points -- interface unknowns shared by 4 subdomains, numbered after
                               the face unknowns -- with one flux row per edge through the corner
                               (the corner remark); interface solved densely (G small)  */
    double tikhonov;        /* lambda (0: off).  lambda > 0 appends M rows lambda e_j^T (right-
                               hand side 0) to every K^s, i.e. each local LS becomes
                               min ||K c - r||^2 + lambda^2 ||c||^2 (reading R29): the near-square,
                               numerically rank-deficient local problems of the paper's Table 2
                               need such damping of K^{s+} (the paper's least-squares solver
                               truncates).  ld = round_up(m + M, 32); r_s includes lambda ||c||.
                               lambda < 0: the fixed rule lambda_s = eps max(m, M) ||K^s||_F per
                               subdomain (reading R33; the collocation rows' Frobenius norm).    */
} elmddm_config;

typedef struct {
    int64_t N;          /* total subdomains P*P                                               */
    int64_t S;          /* local subdomains s_end - s_begin                                   */
    int64_t m;          /* collocation rows of K^s: p*p + 4q (+ M Tikhonov rows below them)   */
    int64_t ld;         /* leading dimension of K_aug (m rounded up to 32; rows m..ld-1 are 0) */
    int64_t ncols;      /* columns of K_aug: M + 4q + 1  ([K | E_Gamma | F])                  */
    int64_t kaug;       /* augmented columns 4q + 1                                            */
    int64_t G;          /* interface unknowns 2P(P-1)q                                         */
    int64_t faces;      /* interface faces 2P(P-1)                                             */
    int64_t kaug_elems; /* doubles of K_aug for the S local subdomains: S*ld*ncols            */
    int64_t at_elems;   /* doubles of At (flux rows, transposed): S*M*4q                      */
    int64_t tau_elems;  /* S*M                                                                 */
    int64_t pbuf_ld, pbuf_elems; /* flux Schur block per subdomain: 4q x kaug, ld pbuf_ld; N slots (global) */
    int64_t sbuf_ld, sbuf_elems; /* Gram block per subdomain: kaug x kaug, ld sbuf_ld; N slots (global) */
    int64_t work_elems;          /* doubles of the caller-provided work buffer (max over calls)  */
    int64_t band_ld, band_nbw, band_elems; /* Schur matrix storage, see elmddm_band_index       */
    int64_t G_pad;                          /* G rounded up to the 64-tile                       */
    int64_t halfband;                       /* exact half-bandwidth of the Schur matrix          */
    int64_t chol_tasks;                     /* 64 x 64 tiles of L (symbolic factorisation)        */
    int64_t chol_flops;                     /* Cholesky work: 2 * 64^3 per tile update            */
    int64_t chol_n;                         /* unknowns in the factorisation order (padded, %64)  */
    int64_t chol_blocks;                    /* chol_n / 64                                        */
    int64_t chol_ordering;                  /* 0 strip (envelope), 1 nested dissection            */
    int64_t e_impl_begin, e_impl_end;       /* implicit E_Gamma columns [begin, end) of K_aug: not
                                               written by elmddm_assemble (see there)             */
    int64_t ne;         /* E_Gamma columns per subdomain: 4q (layout 0) | 4q + 4 (layout 1)      */
    int64_t na;         /* flux rows per subdomain (rows of At): 4q | 4q + 8                     */
    int64_t n_eq;       /* global flux equations (rows of Q): G (layout 0) | faces q + 4 (P-1)^2  */
} elmddm_sizes_t;

/* ---- context ------------------------------------------------------------------------------ */
/* Validates cfg (P>=1, M%8==0, q even <= 256, p>=1, m >= M, 0<=s_begin<s_end<=N, tikhonov finite
 * >= 0, problem 0..7, ld = rows of K^s rounded to 32 <= ~9.6k: up to 3008 rows every QR panel
 * variant, beyond that the 4-CTA cluster panel with a reduced ring), builds the geometry and
 * face tables and uploads them to `device`.  Synchronous.                                     */
elmddm_status elmddm_create(const elmddm_config* cfg, int device, elmddm_ctx** out);
void elmddm_destroy(elmddm_ctx* ctx);
const char* elmddm_last_error(const elmddm_ctx* ctx);
elmddm_status elmddm_sizes(const elmddm_ctx* ctx, elmddm_sizes_t* out);
/* Waits for `stream` (a cudaStream_t), then reads and clears the device status word.          */
elmddm_status elmddm_sync(elmddm_ctx* ctx, void* stream);
/* Host export of the u_Gamma ordering: xy_host[G][2] coordinates of the interface unknowns.   */
elmddm_status elmddm_interface_points(const elmddm_ctx* ctx, double* xy_host);
/* Offset of Schur-matrix element (i, j) (interface unknowns in strip order, either triangle) in
 * the packed tile storage of M / L: the unknowns are renumbered into the factorisation order
 * (strip order, or nested dissection with tile-aligned padding, see chol_ordering); element
 * (a, b), a >= b, of the renumbered lower triangle lives in tile (a/64, b/64), stored
 * contiguously (64 columns of band_ld = 68 doubles) at tile_id * 64 * band_ld.  -1 if the
 * element is outside the structure of L.                                                        */
int64_t elmddm_band_index(const elmddm_ctx* ctx, int64_t i, int64_t j);
/* Host export of the factorisation plan (each pointer may be NULL): newidx[G] = factorisation-
 * order index of every interface unknown; tile_map[chol_blocks^2] = tile id of (I, J), I >= J,
 * or -1; tasks[chol_tasks][4] = (I, J, kind, updates) of every task in the kernel's list order:
 * kind 0 a whole tile task, 1 the pre-aggregation of a split tile task (the updates from columns
 * below J's dissection node, summed into the tile in place), 2 the rest of a split task.      */
elmddm_status elmddm_chol_plan(const elmddm_ctx* ctx, int32_t* newidx, int32_t* tile_map, int32_t* tasks);
/* Host-only planning query (no device, no context): the interface factorisation plan of a P x P
 * grid with q points per face, ordering 0 strip / 1 nested dissection (reading R25), task list
 * scheduled for `workers` CTAs (0: column order).  stats[6] = {n, nblk, ntiles, tile updates,
 * tasks, simulated makespan in ns}; newidx[G], tile_map[nblk*nblk], tasks[ntasks][4] as for
 * elmddm_chol_plan (each may be NULL; size them from a first call with NULL arrays).
 * EINVAL for P outside [2, 1024], q outside [1, 4096], another ordering or stats == NULL.     */
elmddm_status elmddm_plan_query(int32_t P, int32_t q, int32_t ordering, int32_t workers, int64_t* stats,
                                int32_t* newidx, int32_t* tile_map, int32_t* tasks);

/* ---- hot path ----------------------------------------------------------------------------- */
/* eqn:init: W[S][M][2], b[S][M] for the local subdomains; xi[S][M][2] (may be NULL)
 * receives the sampled centres.  w ~ U([-l,l]^2), xi ~ U(closed r-neighbourhood of Omega_s),
 * b = -w.xi, bit-identical to the oracle's counter-based draw (reading R9).                   */
elmddm_status elmddm_init_hidden(elmddm_ctx* ctx, double* W, double* b, double* xi, void* stream);

/* eqn:nonoverlap_discrete, L = -Laplacian:
 *   Kaug[S][ncols][ld]: columns 0..M-1 = K^s (interior rows -|w|^2 sigma''(z) -- problem 6:
 *   -rho |w|^2 sigma''(z) - (grad rho . w) sigma'(z) --, boundary and
 *   interface rows sigma(z)); columns M..M+4q-1 = E_Gamma (unit column at each interface row;
 *   zero column for a Dirichlet edge point; B^s = -E_Gamma); column M+4q = F^s = [f; g; 0];
 *   rows m..ld-1 = 0.  The E_Gamma columns [e_impl_begin, e_impl_end) of elmddm_sizes are
 *   IMPLICIT: not written here (their contents are unspecified until elmddm_local_factor, whose
 *   first trailing update synthesises the unit columns on chip instead of reading them).
 *   At[S][4q][M] = (A^s)^T: flux row e*q+k holds (w_j . n_e) sigma'(z) at edge e point k,
 *   outward axis normals; zero for Dirichlet edges.                                            */
elmddm_status elmddm_assemble(elmddm_ctx* ctx, const double* W, const double* b, double* Kaug, double* At,
                              void* stream);

/* Problem 6 only: the coefficient field of eqn:varpoisson, rho = tanh(grf) + 1.1 with
 * grf(x) = sum_i a_i sin(w_i . x + b_i) of eqn:grf.  params: HOST array [nterms][4] =
 * (a_i, w_ix, w_iy, b_i) (the paper's random draws, supplied by the caller; copied, not kept).
 * Interior rows of K^s become -rho Lap phi - grad rho . grad phi (rho and its analytic gradient at
 * each interior point, evaluated inside elmddm_assemble).  EINVAL for another problem id, nterms
 * outside [1, 65536] or a NULL array; elmddm_assemble of problem 6 without it is EINVAL.       */
elmddm_status elmddm_set_coefficient(elmddm_ctx* ctx, const double* params, int32_t nterms);

/* Batched blocked Householder QR (no pivoting) of every K^s, applied to all ncols columns:
 *   Q^T [K | E_Gamma | F] = [[R11, R12, y], [0, T_E, t_F]]  (in place in Kaug; Householder vectors
 *   below the diagonal of the first M columns, tau[S][M]).  work: >= work_elems doubles.       */
elmddm_status elmddm_local_factor(elmddm_ctx* ctx, double* Kaug, double* tau, double* work, void* stream);

/* Elimination of c^s (eqn:eliminated -> eqn:schur), per local subdomain s:
 *   At <- R11^{-T} At (so At^T = W_s = A^s R11^{-1}, the flux operator A^s K^{s+} restricted to
 *   range(Q_1));  Pbuf[s] = W_s [R12 | y]  (4q x kaug: flux of c^s(u) = q_s + P_s u_s);
 *   Sbuf[s] = [T_E | t_F]^T [T_E | t_F]   (kaug x kaug Gram, symmetric: only its lower triangle
 *             i >= j is guaranteed; 64 x 64 tiles strictly above the diagonal are not written).
 * Pbuf and Sbuf are GLOBAL (N slots); only slots [s_begin, s_end) are written, so a sum over
 * ranks of zero-filled buffers is their exact union (the NCCL reduce of DESIGN.md §6).        */
elmddm_status elmddm_schur_accumulate(elmddm_ctx* ctx, double* Kaug, double* At, double* Pbuf, double* Sbuf,
                                      double* work, void* stream);

/* Rank-0 interface system (eqn:schur) from the global Pbuf/Sbuf:
 *   M = sum_s scatter(T_E^T T_E) + Q^T Q,  g = -sum_s scatter(T_E^T t_F) - Q^T q,
 *   Q = sum_s scatter(P_s), q = sum_s scatter(q_s)   (reading R13; fixed summation order).
 * Writes Mband (band_elems doubles, lower band, see elmddm_band_index; padding diagonal = 1)
 * and g[G_pad].  work: >= work_elems doubles.                                                 */
elmddm_status elmddm_interface_assemble(elmddm_ctx* ctx, const double* Pbuf, const double* Sbuf, double* Mband,
                                        double* g, double* work, void* stream);
/* Cholesky M = L L^T in place over the tile structure of the factorisation order (64 x 64
 * tiles of L, nested dissection by default -- see elmddm_chol_plan; one persistent left-looking
 * kernel over a list-scheduled task order) and u = M^{-1} g into uG[G_pad] (strip order).  On
 * return the tiles of Mband hold L (diagonal tiles: L(J,J), lower triangular).  g is not
 * modified.  Asynchronous: a non-positive pivot (or a dependency wait exceeding 10 s) sets the
 * device status word, reported as ELMDDM_ENUMERIC by the next elmddm_sync.                                                             */
elmddm_status elmddm_interface_factor_solve(elmddm_ctx* ctx, double* Mband, const double* g, double* uG,
                                            double* work, void* stream);
/* The paper's interface solver: unpreconditioned conjugate gradients on
 * eqn:schur, M u = g with M from elmddm_interface_assemble (not modified), x0 = 0, stopping at
 * ||g - M u|| <= tol ||g|| (recurrence residual; the paper uses tol = 1e-9) or after maxit
 * iterations.  Deterministic (fixed-order reductions).  work: >= work_elems doubles.  Synchronous (reads the residual back every 16 iterations).  *iters and *relres (may
 * be NULL) receive the iteration count and final relative residual; ELMDDM_ENUMERIC if the
 * tolerance was not reached.                                                                   */
elmddm_status elmddm_interface_cg(elmddm_ctx* ctx, const double* Mband, const double* g, double* uG, double* work,
                                  double tol, int32_t maxit, int32_t* iters, double* relres, void* stream);
/* ---- multi-rank interface factorisation ------------------------------
 * Every rank keeps a full replica of the factor's tile pool (plus L(J,J)^{-1}, the published
 * C(J, klast) and the completion flags) in one library-owned device region.  All ranks run the
 * persistent factorisation kernel on the SAME list-scheduled task list, taking tasks through one
 * shared counter (in rank 0's region); a finished tile is written to every replica over NVLink
 * peer memory and its flag released in every replica (system scope), so every k-loop reads its
 * own HBM.  Afterwards every rank holds the whole L and solves for u_Gamma itself (no broadcast).
 * Protocol: every rank elmddm_dist_export -> all-gather the 64-byte handles -> every rank
 * elmddm_dist_import(rank, world, handles[world][64]); then per solve: all-reduce Pbuf / Sbuf,
 * elmddm_interface_assemble into elmddm_dist_pool's buffer, elmddm_interface_factor_solve with
 * that buffer (every rank, the same number of times).  CUDA IPC (cudaIpcGetMemHandle /
 * cudaIpcOpenMemHandle): one process per GPU, peer access over NVLink.  EINVAL on bad
 * arguments / order; ECUDA if IPC fails (the caller then keeps the rank-0 path).
 * elmddm_dist_import with world == 1 (handles may be NULL) returns to the single-rank path.    */
elmddm_status elmddm_dist_export(elmddm_ctx* ctx, void* handle /*[64] bytes out*/);
elmddm_status elmddm_dist_import(elmddm_ctx* ctx, int32_t rank, int32_t world, const void* handles);
elmddm_status elmddm_dist_pool(const elmddm_ctx* ctx, double** pool);
/* IPC sanity check after elmddm_dist_import (all ranks, with a host barrier between the phases):
 * phase 0 stores a word into every peer's region (system-scope release) and adds to a counter in
 * rank 0's region (system-scope atomic); phase 1 sets *ok = 1 iff every peer's word arrived (and,
 * on rank 0, the counter is consistent).  Synchronous.                                         */
elmddm_status elmddm_dist_handshake(elmddm_ctx* ctx, int32_t phase, int32_t* ok);
/* One-GPU emulation of nrep (2..8) ranks for testing: ONE cooperative launch whose CTAs are split
 * into nrep groups, each working as one rank on its own replica (separate allocations), with the
 * multi-rank publication protocol.  Factors a copy of the assembled Mband (not modified), solves
 * into uG from replica 0, and returns in *ndiff the number of doubles in which the other
 * replicas' factors differ from replica 0's (0 expected: every tile is computed once and
 * copied).                                                                                     */
elmddm_status elmddm_debug_dist_emulate(elmddm_ctx* ctx, int32_t nrep, const double* Mband, const double* g,
                                        double* uG, double* work, int64_t* ndiff, void* stream);
/* = interface_assemble + interface_factor_solve + elmddm_sync(stream): returns ELMDDM_ENUMERIC
 * on a non-positive pivot, else the pending ELMDDM_WRANK warning if any. */
elmddm_status elmddm_interface_solve(elmddm_ctx* ctx, const double* Pbuf, const double* Sbuf, double* Mband,
                                     double* g, double* uG, double* work, void* stream);

/* Local back-solve (Alg. 1) with the global uG[G]:
 *   u_s = uG at s's interface points (0 on Dirichlet edges);
 *   coef[S][M] = R11^{-1} (y + R12 u_s);  resid[S] = || t_F + T_E u_s ||_2.                     */
elmddm_status elmddm_back_solve(elmddm_ctx* ctx, const double* Kaug, const double* uG, double* coef,
                                double* resid, double* work, void* stream);

/* u(x) = sum_j c_j^s tanh(w_j^s . x + b_j^s) with s = owner of x (column min(floor(xP), P-1),
 * same for y; reading R15) for points xy[n][2] owned by this rank; other u[i] are left as is. */
elmddm_status elmddm_evaluate(elmddm_ctx* ctx, const double* W, const double* b, const double* coef,
                              const double* xy, int64_t n, double* u, void* stream);

/* ---- instrumentation (measurement only; no effect on results) ------------------------------ */
/* kernel classes timed by elmddm_timing */
enum {
    ELMDDM_K_INIT = 0,       /* init_hidden                                   */
    ELMDDM_K_ASSEMBLE = 1,   /* assembly of K_aug and At                      */
    ELMDDM_K_PANEL = 2,      /* QR panel base blocks                          */
    ELMDDM_K_GEMM_QR = 3,    /* QR compact-WY trailing-update GEMMs (DMMA)    */
    ELMDDM_K_TRSM = 4,       /* R11^{-T} At diagonal-block solves             */
    ELMDDM_K_GEMM_SCHUR = 5, /* TRSM updates, flux product, Gram (DMMA)       */
    ELMDDM_K_IFACE = 6,      /* Q-row gather, M / g assembly (+ Q^T Q GEMM)   */
    ELMDDM_K_POTRF = 7,      /* interface Cholesky: persistent left-looking tile kernel (DMMA) */
    ELMDDM_K_GEMM_CHOL = 8,  /* (reserved; no kernel of this class since the persistent factorisation) */
    ELMDDM_K_TRSV = 9,       /* interface forward / backward substitution     */
    ELMDDM_K_BACK = 10,      /* local back-solve                              */
    ELMDDM_K_EVAL = 11,      /* evaluation                                    */
    ELMDDM_NCLASS = 12
};
typedef struct {
    int64_t launches;              /* kernels launched by this context since the last reset    */
    int64_t count[ELMDDM_NCLASS];  /* launches per class                                        */
    double ms[ELMDDM_NCLASS];      /* summed device time per class (CUDA events on the launch
                                      stream; only while timing is enabled)                     */
} elmddm_timing_t;
/* enable != 0: record a CUDA event pair around every kernel launch (adds ~2 us per launch). */
elmddm_status elmddm_set_timing(elmddm_ctx* ctx, int enable);
/* Synchronises the device, fills *out (may be NULL) and, if reset != 0, clears the counters. */
elmddm_status elmddm_timing(elmddm_ctx* ctx, elmddm_timing_t* out, int reset);
/* Diagnostic: sustained FP64 tensor (DMMA.8x8x4) throughput of `device`, measured with a
 * register-resident mma.sync loop on every SM for about `ms` milliseconds.  Synchronous.        */
elmddm_status elmddm_dmma_probe(int device, double ms, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* ELMDDM_H */
