/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle of the DDM-ELM method
 * (arxiv 2406.15959, "nonoverlapping domain decomposition for extreme learning machines").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2406_15959_b200/) never links, imports or executes anything under oracle/.
 * This file shares no code, header, table or constant generator with the CUDA path.
 *
 * Citation convention: "P:<line>" = /root/reference/PAPER.md line; equations by LaTeX label.
 * Readings of ambiguous passages are those of SURVEY.md §8(c) and are listed in DESIGN.md §3.
 *
 * What it computes (per DESIGN.md §3 and SURVEY.md §8(c)):
 *   1. geometry and collocation points              P:204-225, reading R1/R14
 *   2. hidden layer by the paper's initialisation   eqn:init P:535-546, reading R6-R9
 *   3. K^s, A^s, B^s = [0;0;-I], F^s                eqn:nonoverlap_discrete P:231-280
 *   4. unblocked Householder QR of K^s, no pivoting  (realises K^+ of P:356, reading R11)
 *   5. the literal pieces of eqn:schur P:407-410, with KK^+ = Q_1 Q_1^T and the flux operator
 *        A^s K^{s+} = (A^s R^{-1}) Q_1^T formed once:  B^T(I-KK^+)B, B^T(I-KK^+)F,
 *        AK^+B = sum_s (A^s K^{s+}) B^s,  AK^+F = sum_s (A^s K^{s+}) F^s
 *   6. M = B^T(I-KK^+)B + (AK^+B)^T(AK^+B),  g = B^T(I-KK^+)F + (AK^+B)^T(AK^+F)
 *   7. plain Cholesky (Crout, rows in parallel), forward/back substitution: dense, or on the
 *      band of the strip order (reading R14) for the large interfaces (configs 3-4)
 *   8. c^s = K^{s+}(F^s - B^s u_Gamma) (Alg. 1), r_s = ||(Q^T(F+E u_s))_{M:m}||
 *   9. u(x) = owner subdomain's network (reading R15)
 *
 * Parity pins: tests/test_oracle_*.py.  Functions without a pin say so.
 * Build: gcc -O2 -fPIC -shared -ffp-contract=off -pthread oracle.c -lm -o liboracle.so
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
    int32_t P, M, p, q;     /* P x P subdomains; M neurons each; p x p interior pts; q pts per edge */
    int32_t problem;        /* manufactured solution id, see orc_problem */
    int32_t init_scheme;    /* 0 paper eqn:init, 1 manual l=1, 2 He l=sqrt(2/M), b=0 */
    double init_c;          /* c in l = c sqrt(n), P:544 (1/8 for Poisson) */
    double r_over_diam;     /* r = r_over_diam * diam(Omega_s), P:546 (1/2) */
    uint64_t seed;
    double tikhonov;        /* lambda >= 0: M extra rows lambda * e_j^T of K^s (reading R29);
                               < 0: the fixed rule lambda_s = eps max(m, M) ||K^s||_F (R33)      */
    int32_t layout;         /* 0: face points (reading R1); 1: the paper's shared lattice with
                               cross points (reading R32), p == q        */
} orc_cfg;

static const double PI = 3.14159265358979323846;

/* ------------------------------------------------------------------------------------------ */
/* timing + tiny thread pool                                                                  */
/* ------------------------------------------------------------------------------------------ */
static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

typedef void (*work_fn)(void *ctx, int item, int tid);
typedef struct {
    work_fn fn;
    void *ctx;
    int n_items;
    int next;
    pthread_mutex_t mu;
} pool_job;
typedef struct {
    pool_job *job;
    int tid;
} pool_arg;

static void *pool_main(void *a_) {
    pool_arg *a = (pool_arg *)a_;
    for (;;) {
        pthread_mutex_lock(&a->job->mu);
        int it = a->job->next++;
        pthread_mutex_unlock(&a->job->mu);
        if (it >= a->job->n_items) break;
        a->job->fn(a->job->ctx, it, a->tid);
    }
    return NULL;
}

static void run_parallel(int n_items, int nthreads, work_fn fn, void *ctx) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_items) nthreads = n_items > 0 ? n_items : 1;
    pool_job job;
    job.fn = fn;
    job.ctx = ctx;
    job.n_items = n_items;
    job.next = 0;
    pthread_mutex_init(&job.mu, NULL);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    pool_arg *args = (pool_arg *)malloc(sizeof(pool_arg) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        args[t].job = &job;
        args[t].tid = t;
        if (t > 0) pthread_create(&th[t], NULL, pool_main, &args[t]);
    }
    pool_main(&args[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&job.mu);
    free(th);
    free(args);
}

/* ------------------------------------------------------------------------------------------ */
/* manufactured problems (P:587 for problem 4)                            */
/* u_exact and f = -Lap u_exact, written out by hand; pinned by FD in tests                   */
/* ------------------------------------------------------------------------------------------ */
void orc_problem(int problem, double x, double y, double *u, double *f) {
    double uu = 0.0, ff = 0.0;
    switch (problem) {
    case 0: /* sin(pi x) sin(pi y) */
        uu = sin(PI * x) * sin(PI * y);
        ff = 2.0 * PI * PI * uu;
        break;
    case 1: { /* e^{x+y} sin(2 pi x) cos(2 pi y) */
        double E = exp(x + y), S = sin(2.0 * PI * x), C = cos(2.0 * PI * y);
        double cx = cos(2.0 * PI * x), sy = sin(2.0 * PI * y);
        uu = E * S * C;
        ff = -E * (2.0 * (1.0 - 4.0 * PI * PI) * S * C + 4.0 * PI * cx * C - 4.0 * PI * S * sy);
        break;
    }
    case 2: /* sin(4 pi x) sin(4 pi y) */
        uu = sin(4.0 * PI * x) * sin(4.0 * PI * y);
        ff = 32.0 * PI * PI * uu;
        break;
    case 3: /* sin(8 pi x) sin(8 pi y) */
        uu = sin(8.0 * PI * x) * sin(8.0 * PI * y);
        ff = 128.0 * PI * PI * uu;
        break;
    case 4: /* the paper's Table 2 solution sin(2 pi x) e^y */
        uu = sin(2.0 * PI * x) * exp(y);
        ff = (4.0 * PI * PI - 1.0) * uu;
        break;
    case 6: /* variable coefficient, eqn:varpoisson: f = 1, g = 0, no closed form */
        uu = 0.0;
        ff = 1.0;
        break;
    case 7: /* plate bending: Lap^2 u = q/D, q = sin(pi x) sin(pi y), D = E H^3 / (12 (1 - nu^2)),
               E = 1e7, H = 1e-3, nu = 0.3; u = sin(pi x) sin(pi y) / (4 pi^4 D) */
    {
        double D = 1e7 * 1e-9 / (12.0 * (1.0 - 0.3 * 0.3));
        double sq = sin(PI * x) * sin(PI * y);
        uu = sq / (4.0 * PI * PI * PI * PI * D);
        ff = sq / D;
        break;
    }
    default: /* 5: homogeneous problem u = 0 */
        uu = 0.0;
        ff = 0.0;
        break;
    }
    *u = uu;
    *f = ff;
}

/* ------------------------------------------------------------------------------------------ */
/* geometry (readings R1 point layout, R14 strip order)                            */
/* ------------------------------------------------------------------------------------------ */
/* edges: 0 left (x = x0), 1 right (x = x0+h), 2 bottom (y = y0), 3 top (y = y0+h)           */
/* layout 1 adds the 4 subdomain corners as rows [BL, BR, TL, TR] after the edge rows */
static int orc_ncorner(const orc_cfg *c) { return c->layout == 1 ? 4 : 0; }
static int orc_m(const orc_cfg *c) { return c->p * c->p + 4 * c->q + orc_ncorner(c); }
/* flux rows of A^s: one per edge point, and (layout 1) two per corner -- "a row to A^s for each
 * edge to which x belongs" (the corner remark): [edge e point k at e*q + k | corner cc
 * at 4q + 2cc + d, d = 0 the normal of the corner's vertical edge, d = 1 of its horizontal edge] */
static int orc_na(const orc_cfg *c) { return 4 * c->q + 2 * orc_ncorner(c); }
/* rows of K^s: the m collocation rows, then (reading R29, Tikhonov damping of the local LS)
 * M rows lambda e_j^T with right-hand side 0, so that min ||K c - r||^2 + lambda^2 ||c||^2      */
static int orc_mk(const orc_cfg *c) { return orc_m(c) + (c->tikhonov != 0.0 ? c->M : 0); }

/* Face id of edge e of subdomain (i,j), or -1 if the edge lies on dOmega (Dirichlet).
 * Strip order: strip j holds V(0..P-2, j) then H(0..P-1, j) (j < P-1).                        */
static int face_of(const orc_cfg *c, int i, int j, int e) {
    int P = c->P;
    int strip = 2 * P - 1;
    switch (e) {
    case 0: return i > 0 ? j * strip + (i - 1) : -1;
    case 1: return i < P - 1 ? j * strip + i : -1;
    case 2: return j > 0 ? (j - 1) * strip + (P - 1) + i : -1;
    default: return j < P - 1 ? j * strip + (P - 1) + i : -1;
    }
}

/* row points of subdomain s in K^s order [interior (b-major, a fastest) | L | R | B | T].
 * Every coordinate is one correctly-rounded division of integers, so a point shared by two
 * subdomains is bit-identical in both.  edge[r] = -1 interior else 0..3; gidx[r] = global
 * interface unknown (face*q + k) or -1.                                                      */
/* Plate bending (problem 7; reading R28): two traces per edge point (u and Lap u), so
 * an edge holds q = 2 npts rows / interface unknowns: [u at points 0..npts-1 | Lap u at points
 * 0..npts-1], npts = q / 2 collocation points per edge. */
static int orc_npts(const orc_cfg *c) { return c->problem == 7 ? c->q / 2 : c->q; }

void orc_rows(const orc_cfg *c, int s, double *xy, int32_t *edge, int32_t *gidx) {
    int P = c->P, p = c->p, q = c->q, np = orc_npts(c);
    int i = s % P, j = s / P;
    int r = 0;
    for (int t = orc_m(c); t < orc_mk(c); ++t) { /* Tikhonov rows: no point, edge -2 */
        xy[2 * t] = xy[2 * t + 1] = 0.0;
        edge[t] = -2;
        gidx[t] = -1;
    }
    for (int b = 0; b < p; ++b)
        for (int a = 0; a < p; ++a, ++r) {
            xy[2 * r] = (double)(i * (p + 1) + a + 1) / (double)(P * (p + 1));
            xy[2 * r + 1] = (double)(j * (p + 1) + b + 1) / (double)(P * (p + 1));
            edge[r] = -1;
            gidx[r] = -1;
        }
    for (int e = 0; e < 4; ++e) {
        int f = face_of(c, i, j, e);
        for (int k = 0; k < q; ++k, ++r) {
            int kp = k % np;
            double t_y = (double)(j * (np + 1) + kp + 1) / (double)(P * (np + 1));
            double t_x = (double)(i * (np + 1) + kp + 1) / (double)(P * (np + 1));
            switch (e) {
            case 0: xy[2 * r] = (double)i / (double)P; xy[2 * r + 1] = t_y; break;
            case 1: xy[2 * r] = (double)(i + 1) / (double)P; xy[2 * r + 1] = t_y; break;
            case 2: xy[2 * r] = t_x; xy[2 * r + 1] = (double)j / (double)P; break;
            default: xy[2 * r] = t_x; xy[2 * r + 1] = (double)(j + 1) / (double)P; break;
            }
            edge[r] = e;
            gidx[r] = f >= 0 ? f * q + k : -1;
        }
    }
    /* layout 1: the corners; an interior one is a cross point, an interface unknown shared by
     * four subdomains, numbered after the face unknowns (row-major over the (P-1)^2 crossings) */
    for (int cc = 0; cc < orc_ncorner(c); ++cc, ++r) {
        int ci = cc & 1, cj = cc >> 1, X = i + ci, Y = j + cj;
        xy[2 * r] = (double)X / (double)P;
        xy[2 * r + 1] = (double)Y / (double)P;
        edge[r] = 4 + cc;
        gidx[r] = (X > 0 && X < P && Y > 0 && Y < P) ? 2 * P * (P - 1) * q + (Y - 1) * (P - 1) + (X - 1) : -1;
    }
}

/* Global flux equation of flux row ar (0 .. orc_na - 1) of subdomain s, or -1 (Dirichlet edge or
 * a corner on dOmega).  Edge points: the face unknown's index f*q + k (one equation per face
 * point, the two subdomains' rows summed: A = [A^1 ... A^N]).  Layout 1, corner cc of
 * s at the cross point X (index x): one equation per face incident to X, numbered after the face
 * equations at Gf + 4x + t, t = 0 the vertical face below X, 1 above, 2 the horizontal face left
 * of X, 3 right -- each summing the rows of the two subdomains that share that face.           */
int orc_flux_eq(const orc_cfg *c, int s, int ar) {
    int P = c->P, q = c->q, i = s % P, j = s / P;
    if (ar < 4 * q) {
        int f = face_of(c, i, j, ar / q);
        return f >= 0 ? f * q + ar % q : -1;
    }
    int cc = (ar - 4 * q) / 2, d = (ar - 4 * q) % 2, ci = cc & 1, cj = cc >> 1, X = i + ci, Y = j + cj;
    if (!(X > 0 && X < P && Y > 0 && Y < P)) return -1;
    int x = (Y - 1) * (P - 1) + (X - 1);
    int t = d == 0 ? (cj == 1 ? 0 : 1) : (ci == 1 ? 2 : 3);
    return 2 * P * (P - 1) * q + 4 * x + t;
}

/* out[0]=m  out[1]=G (interface unknowns)  out[2]=faces  out[3]=N  out[4]=flux equations
 * out[5]=flux rows per subdomain */
void orc_geometry(const orc_cfg *c, int64_t *out) {
    int64_t P = c->P, X = c->layout == 1 ? (P - 1) * (P - 1) : 0;
    out[0] = orc_mk(c);
    out[2] = 2 * P * (P - 1);
    out[1] = out[2] * c->q + X;
    out[3] = P * P;
    out[4] = out[2] * c->q + 4 * X;
    out[5] = orc_na(c);
}

/* ------------------------------------------------------------------------------------------ */
/* counter-based RNG (reading R9) and the paper's initialisation eqn:init         */
/* ------------------------------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* uniform double in [0,1) keyed by (seed, subdomain, neuron, draw number) */
static double uniform01(uint64_t seed, int s, int j, int d) {
    uint64_t ctr = ((uint64_t)(uint32_t)s << 40) ^ ((uint64_t)(uint32_t)j << 16) ^ (uint64_t)(uint32_t)d;
    uint64_t x = mix64(ctr + mix64(seed + 0x9E3779B97F4A7C15ULL));
    return (double)(x >> 11) * 0x1.0p-53;
}

#define ORC_MAX_COLLAR_TRIES 1000

/* W[s][j][2], b[s][j], xi[s][j][2] (may be NULL), tries[s][j] (may be NULL)
 *   w ~ U([-l,l]^2), l = c sqrt(n), n = N*M                       (eqn:init, reading R6)
 *   xi ~ U(closed r-neighbourhood of Omega_s), r = diam/2, by rejection from the box  (R7)
 *   b = -w . xi                                                    (eqn:init)              */
void orc_init_hidden(const orc_cfg *c, double *W, double *b, double *xi, int32_t *tries) {
    int P = c->P, M = c->M, N = P * P;
    double h = 1.0 / (double)P;
    double l;
    if (c->init_scheme == 0) l = c->init_c * sqrt((double)N * (double)M);
    else if (c->init_scheme == 1) l = 1.0;
    else l = sqrt(2.0 / (double)M);
    double r = c->r_over_diam * (sqrt(2.0) * h);
    double r2 = r * r;
    double span = h + 2.0 * r;
    for (int s = 0; s < N; ++s) {
        int i = s % P, j = s / P;
        double x0 = (double)i / (double)P, y0 = (double)j / (double)P;
        double x1 = (double)(i + 1) / (double)P, y1 = (double)(j + 1) / (double)P;
        double lox = x0 - r, loy = y0 - r;
        for (int n = 0; n < M; ++n) {
            double wx = (2.0 * uniform01(c->seed, s, n, 0) - 1.0) * l;
            double wy = (2.0 * uniform01(c->seed, s, n, 1) - 1.0) * l;
            double ex = 0.5 * (x0 + x1), ey = 0.5 * (y0 + y1);
            int t = 0;
            if (c->init_scheme != 2) {
                for (t = 0; t < ORC_MAX_COLLAR_TRIES; ++t) {
                    double px = lox + uniform01(c->seed, s, n, 2 + 2 * t) * span;
                    double py = loy + uniform01(c->seed, s, n, 3 + 2 * t) * span;
                    double dx = fmax(fmax(x0 - px, px - x1), 0.0);
                    double dy = fmax(fmax(y0 - py, py - y1), 0.0);
                    if (dx * dx + dy * dy <= r2) {
                        ex = px;
                        ey = py;
                        break;
                    }
                }
            }
            size_t k = (size_t)s * M + n;
            W[2 * k] = wx;
            W[2 * k + 1] = wy;
            b[k] = c->init_scheme == 2 ? 0.0 : -(wx * ex + wy * ey);
            if (xi) {
                xi[2 * k] = ex;
                xi[2 * k + 1] = ey;
            }
            if (tries) tries[k] = t + 1;
        }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* variable coefficient (problem 6), eqn:varpoisson with eqn:grf:      */
/*   grf(x) = sum_i a_i sin(w_i . x + b_i)  (the 256 draws a_i, w_i, b_i are an input: params  */
/*   [i][4] = (a_i, w_ix, w_iy, b_i), from the seeded generator module, reading R26),          */
/*   rho = tanh(grf) + 1.1, grad rho = (1 - tanh^2 grf) grad grf (analytic).        */
/* ------------------------------------------------------------------------------------------ */
static double *g_grf = NULL;
static int g_grf_n = 0;

void orc_set_grf(const double *params, int nterms) {
    free(g_grf);
    g_grf = NULL;
    g_grf_n = 0;
    if (nterms > 0) {
        g_grf = (double *)malloc(sizeof(double) * 4 * (size_t)nterms);
        memcpy(g_grf, params, sizeof(double) * 4 * (size_t)nterms);
        g_grf_n = nterms;
    }
}

/* rho and its gradient at (x, y) */
void orc_rho(double x, double y, double *rho, double *rx, double *ry) {
    double g = 0.0, gx = 0.0, gy = 0.0;
    for (int i = 0; i < g_grf_n; ++i) {
        const double *t = g_grf + 4 * (size_t)i;
        double arg = t[1] * x + t[2] * y + t[3];
        g += t[0] * sin(arg);
        double c = t[0] * cos(arg);
        gx += c * t[1];
        gy += c * t[2];
    }
    double th = tanh(g);
    *rho = th + 1.1;
    *rx = (1.0 - th * th) * gx;
    *ry = (1.0 - th * th) * gy;
}

/* ------------------------------------------------------------------------------------------ */
/* assembly: eqn:nonoverlap_discrete, Poisson L = -Lap (reading R4)               */
/*   K^s rows: interior  -|w|^2 sigma''(z);  boundary/interface  sigma(z)                      */
/*   problem 6 interior: -div(rho grad phi) = -rho |w|^2 sigma'' - (grad rho . w) sigma'         */
/*   A^s rows (interface points): (w . n_s) sigma'(z), outward axis normals (reading R5)      */
/*   F^s = [f(x_i); g(x_b); 0], g = u_exact on dOmega (reading R3)                            */
/*   sigma = tanh, sigma' = 1 - sigma^2, sigma'' = -2 sigma sigma'                             */
/* ------------------------------------------------------------------------------------------ */
/* K: m x M column-major (ld m).  F: m.  A: na x M column-major (ld na = orc_na), row e*q+k =
 * flux row of edge e point k, rows 4q + 2cc + d of corner cc (layout 1; see orc_na); zero rows
 * where there is no interface.                                                                 */
void orc_assemble(const orc_cfg *c, int s, const double *W, const double *b, double *K, double *F,
                  double *A) {
    int M = c->M, q = c->q, m = orc_m(c), mk = orc_mk(c), na = orc_na(c), pp = c->p * c->p;
    double *xy = (double *)malloc(sizeof(double) * 2 * (size_t)mk);
    int32_t *edge = (int32_t *)malloc(sizeof(int32_t) * (size_t)mk);
    int32_t *gidx = (int32_t *)malloc(sizeof(int32_t) * (size_t)mk);
    orc_rows(c, s, xy, edge, gidx);
    static const double nx[4] = {-1.0, 1.0, 0.0, 0.0};
    static const double ny[4] = {0.0, 0.0, -1.0, 1.0};
    if (A)
        for (size_t t = 0; t < (size_t)na * M; ++t) A[t] = 0.0;
    const double *Ws = W + (size_t)2 * s * M;
    const double *bs = b + (size_t)s * M;
    const int np = orc_npts(c);
    const int plate = c->problem == 7;
    /* kind of an edge row: 0 the u trace, 1 the Lap u trace (plate only) */
#define ROW_KIND(r) (plate ? ((r) - (m - 4 * q)) % q / np : 0)
    for (int r = 0; r < m; ++r) {
        double u, f;
        orc_problem(c->problem, xy[2 * r], xy[2 * r + 1], &u, &f);
        if (edge[r] < 0) F[r] = f;
        else if (gidx[r] >= 0) F[r] = 0.0;
        else F[r] = ROW_KIND(r) == 0 ? u : -2.0 * PI * PI * u; /* plate: Lap u = -2 pi^2 u */
    }
    for (int n = 0; n < M; ++n) {
        double wx = Ws[2 * n], wy = Ws[2 * n + 1], bb = bs[n];
        double w2 = wx * wx + wy * wy;
        for (int r = 0; r < m; ++r) {
            double z = wx * xy[2 * r] + wy * xy[2 * r + 1] + bb;
            double t = tanh(z);
            double d1 = 1.0 - t * t;
            double d2 = -2.0 * t * d1;
            double val;
            if (plate) {
                /* s3 = sigma''' = -2 sigma'^2 - 2 sigma sigma'', s4 = sigma'''' = -6 sigma' sigma'' - 2 sigma s3 */
                double d3 = -2.0 * d1 * d1 - 2.0 * t * d2;
                double d4 = -6.0 * d1 * d2 - 2.0 * t * d3;
                if (edge[r] < 0) val = w2 * w2 * d4;                 /* Lap^2 phi = |w|^4 sigma'''' */
                else val = ROW_KIND(r) == 0 ? t : w2 * d2;           /* phi, Lap phi = |w|^2 sigma'' */
                K[(size_t)n * mk + r] = val;
                if (edge[r] >= 0 && A) {
                    int e = edge[r];
                    int ar = r - (m - 4 * q);
                    double wn = wx * nx[e] + wy * ny[e];
                    A[(size_t)n * na + ar] =
                        gidx[r] >= 0 ? (ROW_KIND(r) == 0 ? wn * d1 : w2 * wn * d3) : 0.0; /* d/dn phi, d/dn Lap phi */
                }
                continue;
            }
            if (edge[r] < 0) {
                if (c->problem == 6) {
                    double rho, rx, ry;
                    orc_rho(xy[2 * r], xy[2 * r + 1], &rho, &rx, &ry);
                    val = -rho * w2 * d2 - (rx * wx + ry * wy) * d1;
                } else {
                    val = -w2 * d2;
                }
            } else {
                val = t;
            }
            K[(size_t)n * mk + r] = val;
            if (edge[r] >= 0 && edge[r] < 4 && A) {
                int e = edge[r];
                int ar = r - pp; /* = e*q + k */
                A[(size_t)n * na + ar] = gidx[r] >= 0 ? (wx * nx[e] + wy * ny[e]) * d1 : 0.0;
            } else if (edge[r] >= 4 && A && gidx[r] >= 0) {
                /* corner remark: one flux row per edge through the corner, with that
                 * edge's outward normal: d = 0 the vertical edge (left or right), d = 1 the
                 * horizontal edge (bottom or top) */
                int cc = edge[r] - 4, ci = cc & 1, cj = cc >> 1;
                A[(size_t)n * na + 4 * q + 2 * cc] = (ci ? wx : -wx) * d1;
                A[(size_t)n * na + 4 * q + 2 * cc + 1] = (cj ? wy : -wy) * d1;
            }
        }
    }
    if (mk > m) { /* reading R29: damping rows lambda e_j^T, right-hand side 0 */
        double lam = c->tikhonov;
        if (lam < 0.0) { /* reading R33: lambda_s = eps max(m, M) ||K^s||_F over the collocation rows */
            double f2 = 0.0;
            for (int n = 0; n < M; ++n)
                for (int r = 0; r < m; ++r) f2 += K[(size_t)n * mk + r] * K[(size_t)n * mk + r];
            lam = sqrt(f2) * (0x1.0p-52 * (double)(m > M ? m : M));
        }
        for (int r = m; r < mk; ++r) {
            F[r] = 0.0;
            for (int n = 0; n < M; ++n) K[(size_t)n * mk + r] = (r - m == n) ? lam : 0.0;
        }
    }
    free(xy);
    free(edge);
    free(gidx);
#undef ROW_KIND
}

/* ------------------------------------------------------------------------------------------ */
/* unblocked Householder QR, no pivoting (reading R11/R20)                                    */
/*   column j: x = A[j:m, j], alpha = -sign(x0) ||x|| (sign(0)=+1), v = (x - alpha e1)/(x0-alpha),
 *   tau = (alpha - x0)/alpha; ||x|| = 0 -> tau = 0.  A <- (I - tau v v^T) A.                  */
/* ------------------------------------------------------------------------------------------ */
void orc_qr(int m, int n, double *A, int lda, double *tau) {
    int kmax = m < n ? m : n;
    for (int j = 0; j < kmax; ++j) {
        double *x = A + (size_t)j * lda;
        double s2 = 0.0;
        for (int i = j; i < m; ++i) s2 += x[i] * x[i];
        double nrm = sqrt(s2);
        if (nrm == 0.0) {
            tau[j] = 0.0;
            continue;
        }
        double x0 = x[j];
        double alpha = x0 >= 0.0 ? -nrm : nrm;
        double scale = 1.0 / (x0 - alpha);
        for (int i = j + 1; i < m; ++i) x[i] *= scale;
        tau[j] = (alpha - x0) / alpha;
        x[j] = alpha; /* R_jj; v_j = 1 implicit */
        for (int l = j + 1; l < n; ++l) {
            double *y = A + (size_t)l * lda;
            double dot = y[j];
            for (int i = j + 1; i < m; ++i) dot += x[i] * y[i];
            dot *= tau[j];
            y[j] -= dot;
            for (int i = j + 1; i < m; ++i) y[i] -= dot * x[i];
        }
    }
}

/* vec <- Q^T vec  (Q = H_0 H_1 ... H_{k-1}) */
void orc_apply_qt(int m, int k, const double *A, int lda, const double *tau, double *vec) {
    for (int j = 0; j < k; ++j) {
        const double *x = A + (size_t)j * lda;
        double dot = vec[j];
        for (int i = j + 1; i < m; ++i) dot += x[i] * vec[i];
        dot *= tau[j];
        vec[j] -= dot;
        for (int i = j + 1; i < m; ++i) vec[i] -= dot * x[i];
    }
}

/* vec <- Q vec */
void orc_apply_q(int m, int k, const double *A, int lda, const double *tau, double *vec) {
    for (int j = k - 1; j >= 0; --j) {
        const double *x = A + (size_t)j * lda;
        double dot = vec[j];
        for (int i = j + 1; i < m; ++i) dot += x[i] * vec[i];
        dot *= tau[j];
        vec[j] -= dot;
        for (int i = j + 1; i < m; ++i) vec[i] -= dot * x[i];
    }
}

/* solve R z = y (R upper n x n in the QR'd A), in place */
static void back_subst(int n, const double *A, int lda, double *z) {
    for (int i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (int l = i + 1; l < n; ++l) s -= A[(size_t)l * lda + i] * z[l];
        z[i] = s / A[(size_t)i * lda + i];
    }
}

/* ------------------------------------------------------------------------------------------ */
/* per-subdomain literal pieces of eqn:schur                                       */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int m, M, mg, ma;     /* rows, neurons, interface points m_Gamma^s, flux rows */
    double *K;            /* factored K^s (m x M) */
    double *tau;          /* M */
    double *F;            /* m */
    int32_t *irow;        /* [mg] row of K^s for interface point k */
    int32_t *ig;          /* [mg] global index of interface point k */
    int32_t *aeq;         /* [ma] global flux equation of flux row k (orc_flux_eq) */
    double *Aflux;        /* [ma x M] row-major: the flux rows (layout 0: one per interface point) */
    double *S1;           /* B^T (I - K K^+) B: mg x mg */
    double *g1;           /* B^T (I - K K^+) F: mg */
    double *PB;           /* A K^+ B: ma x mg row-major (rows = flux rows) */
    double *pF;           /* A K^+ F: ma */
} orc_local;

static void local_free(orc_local *L) {
    free(L->K); free(L->tau); free(L->F); free(L->irow); free(L->ig); free(L->aeq); free(L->Aflux);
    free(L->S1); free(L->g1); free(L->PB); free(L->pF);
    memset(L, 0, sizeof(*L));
}

/* Steps 2-5 of the oracle for one subdomain. */
static void local_build(const orc_cfg *c, int s, const double *W, const double *b, orc_local *L) {
    int M = c->M, m = orc_mk(c), na = orc_na(c); /* rows of K^s, flux rows of A^s */
    L->m = m;
    L->M = M;
    double *xy = (double *)malloc(sizeof(double) * 2 * (size_t)m);
    int32_t *edge = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int32_t *gidx = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    orc_rows(c, s, xy, edge, gidx);
    int mg = 0;
    for (int r = 0; r < m; ++r) mg += gidx[r] >= 0;
    L->mg = mg;
    L->K = (double *)malloc(sizeof(double) * (size_t)m * M);
    L->tau = (double *)malloc(sizeof(double) * (size_t)M);
    L->F = (double *)malloc(sizeof(double) * (size_t)m);
    L->irow = (int32_t *)malloc(sizeof(int32_t) * (size_t)(mg + 1));
    L->ig = (int32_t *)malloc(sizeof(int32_t) * (size_t)(mg + 1));
    double *A4 = (double *)calloc((size_t)na * M, sizeof(double));
    orc_assemble(c, s, W, b, L->K, L->F, A4);
    int k = 0;
    for (int r = 0; r < m; ++r)
        if (gidx[r] >= 0) {
            L->irow[k] = r;
            L->ig[k] = gidx[r];
            ++k;
        }
    int ma = 0;
    for (int ar = 0; ar < na; ++ar) ma += orc_flux_eq(c, s, ar) >= 0;
    L->ma = ma;
    L->aeq = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ma + 1));
    L->Aflux = (double *)malloc(sizeof(double) * (size_t)(ma + 1) * M);
    k = 0;
    for (int ar = 0; ar < na; ++ar) {
        int eq = orc_flux_eq(c, s, ar);
        if (eq < 0) continue;
        L->aeq[k] = eq;
        for (int n = 0; n < M; ++n) L->Aflux[(size_t)k * M + n] = A4[(size_t)n * na + ar];
        ++k;
    }
    free(A4);
    free(xy);
    free(edge);
    free(gidx);

    /* Householder QR of K^s */
    orc_qr(m, M, L->K, m, L->tau);

    /* rows of Q_1 at the interface rows: t_k = Q_1^T e_{row_k} (first M entries of Q^T e_row) */
    double *t = (double *)malloc(sizeof(double) * (size_t)(mg + 1) * M);
    double *vec = (double *)malloc(sizeof(double) * (size_t)m);
    for (k = 0; k < mg; ++k) {
        memset(vec, 0, sizeof(double) * (size_t)m);
        vec[L->irow[k]] = 1.0;
        orc_apply_qt(m, M, L->K, m, L->tau, vec);
        memcpy(t + (size_t)k * M, vec, sizeof(double) * (size_t)M);
    }
    double *yF = (double *)malloc(sizeof(double) * (size_t)m); /* Q^T F; Q_1^T F = yF[0:M] */
    memcpy(yF, L->F, sizeof(double) * (size_t)m);
    orc_apply_qt(m, M, L->K, m, L->tau, yF);

    /* B^T (I - K K^+) B = E^T (I - Q_1 Q_1^T) E  and  B^T (I - K K^+) F = (Q_1 Q_1^T F)_Gamma - F_Gamma */
    L->S1 = (double *)malloc(sizeof(double) * (size_t)(mg + 1) * (mg + 1));
    L->g1 = (double *)malloc(sizeof(double) * (size_t)(mg + 1));
    for (k = 0; k < mg; ++k) {
        for (int l = 0; l < mg; ++l) {
            double d = 0.0;
            for (int n = 0; n < M; ++n) d += t[(size_t)k * M + n] * t[(size_t)l * M + n];
            L->S1[(size_t)k * mg + l] = (k == l ? 1.0 : 0.0) - d;
        }
        double d = 0.0;
        for (int n = 0; n < M; ++n) d += t[(size_t)k * M + n] * yF[n];
        /* -e_k^T (F - Q1 Q1^T F) = d - F_k, and F_k = 0 on interface rows */
        L->g1[k] = d - L->F[L->irow[k]];
    }

    /* The flux operator A^s K^{s+} = (A^s R^{-1}) Q_1^T is formed ONCE (forward substitution
     * R^T w_a = a for every flux row a), then applied to B^s and to F^s:
     *     A K^+ B = -(A R^{-1}) (Q_1^T E),   A K^+ F = (A R^{-1}) (Q_1^T F).
     * This is the association (A K^+) B of eqn:schur.  Forming K^+ B column by column
     * first (i.e. A (K^+ B)) is NOT used: when K^s is numerically rank-deficient each column
     * carries its own resolution of the near-null space and the flux term loses all accuracy
     * (reading R23: u_Gamma error 1.4e-2 vs 1.6e-11 at config 1).                  */
    double *wr = (double *)malloc(sizeof(double) * (size_t)M);
    L->PB = (double *)malloc(sizeof(double) * (size_t)(ma + 1) * (mg + 1));
    L->pF = (double *)malloc(sizeof(double) * (size_t)(ma + 1));
    for (k = 0; k < ma; ++k) {
        const double *a = L->Aflux + (size_t)k * M;
        for (int i = 0; i < M; ++i) { /* R^T w = a, R^T lower triangular */
            double sacc = a[i];
            for (int l = 0; l < i; ++l) sacc -= L->K[(size_t)i * m + l] * wr[l];
            wr[i] = sacc / L->K[(size_t)i * m + i];
        }
        for (int l = 0; l < mg; ++l) {
            double d = 0.0;
            const double *tl = t + (size_t)l * M;
            for (int n = 0; n < M; ++n) d += wr[n] * tl[n];
            L->PB[(size_t)k * mg + l] = -d;
        }
        double d = 0.0;
        for (int n = 0; n < M; ++n) d += wr[n] * yF[n];
        L->pF[k] = d;
    }
    free(wr);
    free(t);
    free(vec);
    free(yF);
}

/* back-solve with a given global u_Gamma (Alg. 1):
 *   c = K^+ (F - B u_s) = R^{-1} (Q^T (F + E u_s))_{0:M},   r = ||(Q^T (F + E u_s))_{M:m}||   */
static void local_back(const orc_local *L, const double *uG, double *coef, double *resid) {
    int M = L->M, m = L->m, mg = L->mg;
    double *vec = (double *)malloc(sizeof(double) * (size_t)m);
    memcpy(vec, L->F, sizeof(double) * (size_t)m);
    for (int k = 0; k < mg; ++k) vec[L->irow[k]] += uG[L->ig[k]];
    orc_apply_qt(m, M, L->K, m, L->tau, vec);
    double s2 = 0.0;
    for (int i = M; i < m; ++i) s2 += vec[i] * vec[i];
    *resid = sqrt(s2);
    memcpy(coef, vec, sizeof(double) * (size_t)M);
    back_subst(M, L->K, m, coef);
    free(vec);
}

/* ------------------------------------------------------------------------------------------ */
/* evaluation (reading R15): owner column min(floor(x P), P-1) by integer rule on the grid;    */
/* for general points we use the same rule on floor(x*P).                                      */
/* ------------------------------------------------------------------------------------------ */
static int owner_of(int P, double x, double y) {
    int i = (int)floor(x * (double)P), j = (int)floor(y * (double)P);
    if (i > P - 1) i = P - 1;
    if (j > P - 1) j = P - 1;
    if (i < 0) i = 0;
    if (j < 0) j = 0;
    return j * P + i;
}

void orc_evaluate(const orc_cfg *c, const double *W, const double *b, const double *coef,
                  const double *xy, int64_t n, double *u) {
    int M = c->M;
    for (int64_t t = 0; t < n; ++t) {
        int s = owner_of(c->P, xy[2 * t], xy[2 * t + 1]);
        const double *Ws = W + (size_t)2 * s * M;
        const double *bs = b + (size_t)s * M;
        const double *cs = coef + (size_t)s * M;
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += cs[j] * tanh(Ws[2 * j] * xy[2 * t] + Ws[2 * j + 1] * xy[2 * t + 1] + bs[j]);
        u[t] = acc;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* plain Cholesky (Crout, row-major lower; rows of each column in parallel) + substitution    */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    double *L;   /* G x G row-major, lower part overwritten by the factor */
    int64_t G;
    int j;
    int nthreads;
    int bad;
} chol_ctx;

static void chol_rows(void *ctx_, int item, int tid) {
    (void)tid;
    chol_ctx *C = (chol_ctx *)ctx_;
    int64_t G = C->G;
    int j = C->j;
    const double *Lj = C->L + (size_t)j * G;
    for (int64_t i = j + 1 + item; i < G; i += C->nthreads) {
        double *Li = C->L + (size_t)i * G;
        double s = Li[j];
        for (int k = 0; k < j; ++k) s -= Li[k] * Lj[k];
        Li[j] = s / Lj[j];
    }
}

/* returns 0 on success, 1 + column of the first non-positive pivot otherwise */
int orc_cholesky(double *L, int64_t G, int nthreads) {
    chol_ctx C;
    C.L = L;
    C.G = G;
    C.nthreads = nthreads < 1 ? 1 : nthreads;
    for (int64_t j = 0; j < G; ++j) {
        double *Lj = L + (size_t)j * G;
        double s = Lj[j];
        for (int64_t k = 0; k < j; ++k) s -= Lj[k] * Lj[k];
        if (!(s > 0.0)) return (int)(1 + j);
        Lj[j] = sqrt(s);
        C.j = (int)j;
        if (G - j - 1 > 256 && C.nthreads > 1) run_parallel(C.nthreads, C.nthreads, chol_rows, &C);
        else {
            int nt = C.nthreads;
            C.nthreads = 1;
            chol_rows(&C, 0, 0);
            C.nthreads = nt;
        }
    }
    return 0;
}

void orc_chol_solve(const double *L, int64_t G, double *x) {
    for (int64_t i = 0; i < G; ++i) {
        double s = x[i];
        const double *Li = L + (size_t)i * G;
        for (int64_t k = 0; k < i; ++k) s -= Li[k] * x[k];
        x[i] = s / Li[i];
    }
    for (int64_t i = G - 1; i >= 0; --i) {
        double s = x[i];
        for (int64_t k = i + 1; k < G; ++k) s -= L[(size_t)k * G + i] * x[k];
        x[i] = s / L[(size_t)i * G + i];
    }
}

/* ------------------------------------------------------------------------------------------ */
/* plain BANDED Cholesky in strip order (reading R14)                     */
/* ------------------------------------------------------------------------------------------ */
/* In strip order the interface matrix M of eqn:schur is banded: S1 couples the faces
 * of one subdomain, (AK^+B)^T(AK^+B) the faces of the two subdomains beside one flux face, and
 * both lie within (4P-1)q - 1 unknowns of each other (reading R14).  Storage: the lower band,
 * row-major, row i holding columns i-bw .. i at B[i*(bw+1) + (k - i + bw)] (entries left of
 * column 0 are unused zeros).  The factorisation is the same Crout recurrence as orc_cholesky,
 *     L_jj = sqrt(M_jj - sum_k L_jk^2),   L_ij = (M_ij - sum_k L_ik L_jk) / L_jj   (i > j),
 * with the sums running over the band only (k >= i - bw): outside the band M and L are exactly
 * zero, so the terms dropped are exact zeros.  Rows of a column are computed in parallel; every
 * thread forms L_jj itself from finished data (one barrier per column).                       */
typedef struct {
    double *B;
    int64_t G, bw;
    int nthreads;
    int bad;              /* 1 + first non-positive pivot column */
    pthread_barrier_t bar;
} bchol_ctx;

typedef struct {
    bchol_ctx *C;
    int tid;
} bchol_arg;

static void *bchol_main(void *a_) {
    bchol_arg *a = (bchol_arg *)a_;
    bchol_ctx *C = a->C;
    const int64_t G = C->G, bw = C->bw, w = bw + 1;
    double *B = C->B;
    for (int64_t j = 0; j < G; ++j) {
        double *Lj = B + (size_t)j * w;              /* Lj[k - j + bw] = L_jk */
        int64_t lo = j - bw > 0 ? j - bw : 0;
        double s = Lj[bw];
        for (int64_t k = lo; k < j; ++k) s -= Lj[k - j + bw] * Lj[k - j + bw];
        if (!(s > 0.0)) {                            /* every thread sees the same pivot */
            if (a->tid == 0) C->bad = (int)(1 + j);
            return NULL;
        }
        double d = sqrt(s);
        int64_t iend = j + bw < G - 1 ? j + bw : G - 1;
        for (int64_t i = j + 1 + a->tid; i <= iend; i += C->nthreads) {
            double *Li = B + (size_t)i * w;          /* Li[k - i + bw] = L_ik */
            int64_t klo = i - bw > 0 ? i - bw : 0;
            double t = Li[j - i + bw];
            for (int64_t k = klo; k < j; ++k) t -= Li[k - i + bw] * Lj[k - j + bw];
            Li[j - i + bw] = t / d;
        }
        pthread_barrier_wait(&C->bar);               /* column j done; every thread has read M_jj */
        if (a->tid == 0) Lj[bw] = d;                 /* column j+1 never reads L_jj */
    }
    return NULL;
}

/* returns 0 on success, 1 + column of the first non-positive pivot otherwise */
int orc_band_cholesky(double *B, int64_t G, int64_t bw, int nthreads) {
    bchol_ctx C;
    C.B = B;
    C.G = G;
    C.bw = bw;
    C.nthreads = nthreads < 1 ? 1 : nthreads;
    C.bad = 0;
    pthread_barrier_init(&C.bar, NULL, (unsigned)C.nthreads);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)C.nthreads);
    bchol_arg *args = (bchol_arg *)malloc(sizeof(bchol_arg) * (size_t)C.nthreads);
    for (int t = 0; t < C.nthreads; ++t) {
        args[t].C = &C;
        args[t].tid = t;
        if (t > 0) pthread_create(&th[t], NULL, bchol_main, &args[t]);
    }
    bchol_main(&args[0]);
    for (int t = 1; t < C.nthreads; ++t) pthread_join(th[t], NULL);
    pthread_barrier_destroy(&C.bar);
    free(th);
    free(args);
    return C.bad;
}

/* L y = g, then L^T x = y, on the band factor (in place on x) */
void orc_band_chol_solve(const double *B, int64_t G, int64_t bw, double *x) {
    const int64_t w = bw + 1;
    for (int64_t i = 0; i < G; ++i) {
        const double *Li = B + (size_t)i * w;
        int64_t lo = i - bw > 0 ? i - bw : 0;
        double s = x[i];
        for (int64_t k = lo; k < i; ++k) s -= Li[k - i + bw] * x[k];
        x[i] = s / Li[bw];
    }
    for (int64_t i = G - 1; i >= 0; --i) {
        int64_t hi = i + bw < G - 1 ? i + bw : G - 1;
        double s = x[i];
        for (int64_t k = i + 1; k <= hi; ++k) s -= B[(size_t)k * w + (i - k + bw)] * x[k];
        x[i] = s / B[(size_t)i * w + bw];
    }
}

/* ------------------------------------------------------------------------------------------ */
/* the whole method (Algorithm 1)                                                   */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    const orc_cfg *c;
    const double *W, *b;
    orc_local *L;
    const double *uG;
    double *coef, *resid;
} solve_ctx;

static void job_local(void *ctx_, int s, int tid) {
    (void)tid;
    solve_ctx *X = (solve_ctx *)ctx_;
    local_build(X->c, s, X->W, X->b, &X->L[s]);
}
static void job_back(void *ctx_, int s, int tid) {
    (void)tid;
    solve_ctx *X = (solve_ctx *)ctx_;
    local_back(&X->L[s], X->uG, X->coef + (size_t)s * X->c->M, &X->resid[s]);
}

/* Steps 5-7 on the band (reading R14 strip order, half-bandwidth bw = (4P-1)q - 1): the same
 * sums as the dense route below, element by element in the same order (S1 blocks in ascending s,
 * then the rows a of AK^+B in ascending a), stored as the lower band.  Row a of AK^+B is
 * sum_s (A^s K^{s+}) B^s restricted to flux row a: the PB rows of the two subdomains beside the
 * face of a, added in ascending s into a zeroed window a-bw .. a+bw.  Returns 0, 2 on a
 * non-positive pivot, 3 if an entry falls outside the band (a geometry error).                 */
typedef struct {
    const orc_local *L;
    int N;
    int64_t G, bw;
    const int32_t *own_s, *own_k;   /* [G][2] contributors (s ascending; -1 = none) */
    int32_t *qnz;                   /* [G][qcap] column indices of row a of AK^+B */
    double *qval;                   /* [G][qcap] values */
    int32_t *qn;                    /* [G] count */
    int qcap;
    int bad;
} qrow_ctx;

static void job_qrow(void *ctx_, int a, int tid) {
    (void)tid;
    qrow_ctx *Q = (qrow_ctx *)ctx_;
    int64_t bw = Q->bw, G = Q->G;
    double *win = (double *)calloc((size_t)(2 * bw + 1), sizeof(double));
    int64_t lo = G, hi = -1;
    for (int t = 0; t < 2; ++t) {
        int s = Q->own_s[2 * a + t];
        if (s < 0) continue;
        const orc_local *Ls = &Q->L[s];
        int k = Q->own_k[2 * a + t];
        for (int l = 0; l < Ls->mg; ++l) {
            int64_t gl = Ls->ig[l];
            if (gl < a - bw || gl > a + bw) { Q->bad = 1; continue; }
            win[gl - a + bw] += Ls->PB[(size_t)k * Ls->mg + l];
            if (gl < lo) lo = gl;
            if (gl > hi) hi = gl;
        }
    }
    int n = 0;
    for (int64_t gl = lo; gl <= hi; ++gl) {
        double v = win[gl - a + bw];
        if (v != 0.0) {
            if (n >= Q->qcap) { Q->bad = 1; break; }
            Q->qnz[(size_t)a * Q->qcap + n] = (int32_t)gl;
            Q->qval[(size_t)a * Q->qcap + n] = v;
            ++n;
        }
    }
    Q->qn[a] = n;
    free(win);
}

typedef struct {
    const qrow_ctx *Q;
    double *Mb, *g;
    const double *qg;
    int nthreads;
} qtq_ctx;

/* thread t owns the band rows kx with kx % nthreads == t and adds every row a's terms to them in
 * ascending a -- the dense route's order for each element */
static void job_qtq(void *ctx_, int t, int tid) {
    (void)tid;
    qtq_ctx *X = (qtq_ctx *)ctx_;
    const qrow_ctx *Q = X->Q;
    int64_t bw = Q->bw, w = bw + 1;
    for (int64_t a = 0; a < Q->G; ++a) {
        const int32_t *nz = Q->qnz + (size_t)a * Q->qcap;
        const double *v = Q->qval + (size_t)a * Q->qcap;
        int n = Q->qn[a];
        for (int x = 0; x < n; ++x) {
            int64_t kx = nz[x];
            if (kx % X->nthreads != t) continue;
            double rx = v[x];
            X->g[kx] += rx * X->qg[a];
            double *Mk = X->Mb + (size_t)kx * w;
            for (int y = 0; y < n; ++y) {
                int64_t ky = nz[y];
                if (ky <= kx) Mk[ky - kx + bw] += rx * v[y];
            }
        }
    }
}

static int iface_band(const orc_cfg *c, const orc_local *L, int N, int64_t G, int nthreads, double *uG,
                      double *tas, double *tsol) {
    double t0 = now_s();
    int64_t bw = (int64_t)(4 * c->P - 1) * c->q - 1;
    if (bw > G - 1) bw = G - 1;
    int64_t w = bw + 1;
    double *Mb = (double *)calloc((size_t)G * (size_t)w, sizeof(double));
    double *g = (double *)calloc((size_t)G, sizeof(double));
    double *qg = (double *)calloc((size_t)G, sizeof(double));
    int32_t *own_s = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)G);
    int32_t *own_k = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)G);
    int bad = 0;
    if (!Mb || !g || !qg || !own_s || !own_k) return 4;
    for (int64_t a = 0; a < 2 * G; ++a) own_s[a] = own_k[a] = -1;
    for (int s = 0; s < N; ++s) {
        const orc_local *Ls = &L[s];
        for (int k = 0; k < Ls->ma; ++k) {  /* layout 0 (the only one on this route): equation = unknown */
            int64_t ek = Ls->aeq[k];
            qg[ek] += Ls->pF[k];
            int slot = own_s[2 * ek] < 0 ? 0 : 1;
            own_s[2 * ek + slot] = s;
            own_k[2 * ek + slot] = k;
        }
        for (int k = 0; k < Ls->mg; ++k) {
            int64_t gk = Ls->ig[k];
            g[gk] += Ls->g1[k];
            double *Mk = Mb + (size_t)gk * w;
            for (int l = 0; l < Ls->mg; ++l) {
                int64_t gl = Ls->ig[l];
                if (gl > gk) continue;
                if (gk - gl > bw) { bad = 1; continue; }
                Mk[gl - gk + bw] += Ls->S1[(size_t)k * Ls->mg + l];
            }
        }
    }
    qrow_ctx Q;
    Q.L = L;
    Q.N = N;
    Q.G = G;
    Q.bw = bw;
    Q.own_s = own_s;
    Q.own_k = own_k;
    Q.qcap = 8 * c->q;
    Q.qnz = (int32_t *)malloc(sizeof(int32_t) * (size_t)G * Q.qcap);
    Q.qval = (double *)malloc(sizeof(double) * (size_t)G * Q.qcap);
    Q.qn = (int32_t *)calloc((size_t)G, sizeof(int32_t));
    Q.bad = 0;
    if (!Q.qnz || !Q.qval || !Q.qn) return 4;
    run_parallel((int)G, nthreads, job_qrow, &Q);
    qtq_ctx X = {&Q, Mb, g, qg, nthreads < 1 ? 1 : nthreads};
    run_parallel(X.nthreads, X.nthreads, job_qtq, &X);
    free(Q.qnz);
    free(Q.qval);
    free(Q.qn);
    free(own_s);
    free(own_k);
    free(qg);
    double t1 = now_s();
    int rc = 0;
    if (bad || Q.bad) rc = 3;
    else if (orc_band_cholesky(Mb, G, bw, nthreads) != 0) rc = 2;
    else {
        memcpy(uG, g, sizeof(double) * (size_t)G);
        orc_band_chol_solve(Mb, G, bw, uG);
    }
    free(Mb);
    free(g);
    *tas = t1 - t0;
    *tsol = now_s() - t1;
    return rc;
}

/* times[0] local (assemble+QR+Schur pieces), [1] interface assembly, [2] Cholesky+solve,
 * [3] back-solve, [4] evaluate.  Mout (G x G row-major, full symmetric) and gout optional
 * (dense route only).  band: 0 auto (band if G > 20000), 1 dense, 2 band.
 * Returns 0 ok, 2 if Cholesky hit a non-positive pivot, 1 if G too large for dense storage,
 * 3 band geometry error, 4 out of memory.                                                     */
int orc_solve(const orc_cfg *c, const double *W, const double *b, int nthreads, double *uG,
              double *coef, double *resid, const double *xy_eval, int64_t n_eval, double *u_eval,
              double *Mout, double *gout, double *times, int band) {
    int64_t geo[6];
    orc_geometry(c, geo);
    int64_t G = geo[1];
    int N = (int)geo[3];
    if (band == 0) band = G > 20000 ? 2 : 1;
    if (band == 1 && G > 20000) return 1;
    if (band == 2 && c->layout != 0) return 3; /* cross points are outside the strip-order band */
    double t0 = now_s();
    orc_local *L = (orc_local *)calloc((size_t)N, sizeof(orc_local));
    solve_ctx X = {c, W, b, L, uG, coef, resid};
    run_parallel(N, nthreads, job_local, &X);
    double t1 = now_s();
    if (band == 2) {
        double tas = 0.0, tsol = 0.0;
        int rc = G > 0 ? iface_band(c, L, N, G, nthreads, uG, &tas, &tsol) : 0;
        double t3 = now_s();
        if (rc == 0) run_parallel(N, nthreads, job_back, &X);
        double t4 = now_s();
        if (rc == 0 && xy_eval && n_eval > 0) orc_evaluate(c, W, b, coef, xy_eval, n_eval, u_eval);
        double t5 = now_s();
        if (times) {
            times[0] = t1 - t0;
            times[1] = tas;
            times[2] = tsol;
            times[3] = t4 - t3;
            times[4] = t5 - t4;
        }
        for (int s = 0; s < N; ++s) local_free(&L[s]);
        free(L);
        return rc;
    }

    /* global pieces: sum in ascending s (step 5-6 of SURVEY §8(c)) */
    const int64_t NE = geo[4]; /* flux equations: rows of A K^+ B (= G in layout 0) */
    double *Mm = (double *)calloc((size_t)(G > 0 ? G : 1) * (G > 0 ? G : 1), sizeof(double));
    double *g = (double *)calloc((size_t)(G > 0 ? G : 1), sizeof(double));
    double *Qg = (double *)calloc((size_t)(NE > 0 ? NE : 1) * (G > 0 ? G : 1), sizeof(double)); /* A K^+ B */
    double *qg = (double *)calloc((size_t)(NE > 0 ? NE : 1), sizeof(double));                   /* A K^+ F */
    for (int s = 0; s < N; ++s) {
        orc_local *Ls = &L[s];
        for (int k = 0; k < Ls->mg; ++k) {
            int gk = Ls->ig[k];
            g[gk] += Ls->g1[k];
            for (int l = 0; l < Ls->mg; ++l) {
                int gl = Ls->ig[l];
                Mm[(size_t)gk * G + gl] += Ls->S1[(size_t)k * Ls->mg + l];
            }
        }
        for (int k = 0; k < Ls->ma; ++k) {
            int ek = Ls->aeq[k];
            qg[ek] += Ls->pF[k];
            for (int l = 0; l < Ls->mg; ++l) {
                int gl = Ls->ig[l];
                Qg[(size_t)ek * G + gl] += Ls->PB[(size_t)k * Ls->mg + l];
            }
        }
    }
    /* (AK^+B)^T (AK^+B) and (AK^+B)^T (AK^+F), row by row of AK^+B over its nonzeros */
    int32_t *nz = (int32_t *)malloc(sizeof(int32_t) * (size_t)(G > 0 ? G : 1));
    for (int64_t a = 0; a < NE; ++a) {
        const double *row = Qg + (size_t)a * G;
        int nnz = 0;
        for (int64_t k = 0; k < G; ++k)
            if (row[k] != 0.0) nz[nnz++] = (int32_t)k;
        for (int x = 0; x < nnz; ++x) {
            int kx = nz[x];
            double rx = row[kx];
            g[kx] += rx * qg[a];
            double *Mk = Mm + (size_t)kx * G;
            for (int y = 0; y < nnz; ++y) Mk[nz[y]] += rx * row[nz[y]];
        }
    }
    free(nz);
    if (Mout) memcpy(Mout, Mm, sizeof(double) * (size_t)G * G);
    if (gout) memcpy(gout, g, sizeof(double) * (size_t)G);
    double t2 = now_s();
    int rc = 0;
    if (G > 0) {
        if (orc_cholesky(Mm, G, nthreads) != 0) rc = 2;
        else {
            memcpy(uG, g, sizeof(double) * (size_t)G);
            orc_chol_solve(Mm, G, uG);
        }
    }
    double t3 = now_s();
    run_parallel(N, nthreads, job_back, &X);
    double t4 = now_s();
    if (xy_eval && n_eval > 0) orc_evaluate(c, W, b, coef, xy_eval, n_eval, u_eval);
    double t5 = now_s();
    if (times) {
        times[0] = t1 - t0;
        times[1] = t2 - t1;
        times[2] = t3 - t2;
        times[3] = t4 - t3;
        times[4] = t5 - t4;
    }
    for (int s = 0; s < N; ++s) local_free(&L[s]);
    free(L);
    free(Mm);
    free(g);
    free(Qg);
    free(qg);
    return rc;
}

/* Per-subdomain pieces for sampled checks at sizes where the full oracle is too slow.
 * Outputs (nullable): S1 (mg x mg row-major), g1 (mg), PB (ma x mg), pF (ma), ig (mg), aeq (ma),
 * *ma_out, and -- given a global u_Gamma -- coef (M) and resid.  Returns mg.                    */
int orc_local_pieces(const orc_cfg *c, int s, const double *W, const double *b, const double *uG,
                     double *S1, double *g1, double *PB, double *pF, int32_t *ig, double *coef,
                     double *resid, int32_t *aeq, int32_t *ma_out) {
    orc_local L;
    memset(&L, 0, sizeof(L));
    local_build(c, s, W, b, &L);
    int mg = L.mg, ma = L.ma;
    if (S1) memcpy(S1, L.S1, sizeof(double) * (size_t)mg * mg);
    if (g1) memcpy(g1, L.g1, sizeof(double) * (size_t)mg);
    if (PB) memcpy(PB, L.PB, sizeof(double) * (size_t)ma * mg);
    if (pF) memcpy(pF, L.pF, sizeof(double) * (size_t)ma);
    if (ig) memcpy(ig, L.ig, sizeof(int32_t) * (size_t)mg);
    if (aeq) memcpy(aeq, L.aeq, sizeof(int32_t) * (size_t)ma);
    if (ma_out) *ma_out = ma;
    if (uG && coef && resid) local_back(&L, uG, coef, resid);
    local_free(&L);
    return mg;
}

/* CPU baseline leg: the local phase (assemble + QR + Schur pieces + back-solve against
 * u_Gamma = uG or 0) for the n subdomains in s_list, threaded over subdomains.  Returns the
 * wall seconds.                                                                               */
typedef struct {
    const orc_cfg *c;
    const double *W, *b, *uG;
    const int32_t *s_list;
    double *sink;
} sample_ctx;

static void job_sample(void *ctx_, int item, int tid) {
    (void)tid;
    sample_ctx *X = (sample_ctx *)ctx_;
    orc_local L;
    memset(&L, 0, sizeof(L));
    int s = X->s_list[item];
    local_build(X->c, s, X->W, X->b, &L);
    double *coef = (double *)malloc(sizeof(double) * (size_t)L.M);
    double r = 0.0;
    if (X->uG) local_back(&L, X->uG, coef, &r);
    X->sink[item] = r + coef[0] * 0.0;
    free(coef);
    local_free(&L);
}

double orc_sample_local(const orc_cfg *c, const double *W, const double *b, const double *uG,
                        const int32_t *s_list, int n, int nthreads, double *sink) {
    double t0 = now_s();
    sample_ctx X = {c, W, b, uG, s_list, sink};
    run_parallel(n, nthreads, job_sample, &X);
    return now_s() - t0;
}
