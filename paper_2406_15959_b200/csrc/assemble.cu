// assemble.cu -- hidden-layer initialisation (eqn:init), collocation assembly
// (eqn:nonoverlap_discrete) and solution evaluation, for sm_100a.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "internal.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

// ---- counter-based RNG (reading R9) ---------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// uniform double in [0,1) keyed by (seed, subdomain, neuron, draw number)
__device__ __forceinline__ double uniform01(uint64_t key, int s, int j, int d) {
    uint64_t ctr = ((uint64_t)(uint32_t)s << 40) ^ ((uint64_t)(uint32_t)j << 16) ^ (uint64_t)(uint32_t)d;
    uint64_t x = mix64(ctr + key);
    return __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
}

constexpr int kMaxCollarTries = 1000;

// eqn:init.  Every floating-point step is an explicitly rounded IEEE op so that the
// draw is bit-identical to any other implementation of the same recipe (no FMA contraction).
__global__ void k_init_hidden(elmddm_config cfg, double* __restrict__ W, double* __restrict__ b,
                              double* __restrict__ xi) {
    const int P = cfg.P, M = cfg.M, N = P * P;
    const int S = cfg.s_end - cfg.s_begin;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)S * M) return;
    const int sl = (int)(t / M), n = (int)(t % M);
    const int s = cfg.s_begin + sl;
    const int i = s % P, j = s / P;
    const uint64_t key = mix64(cfg.seed + 0x9E3779B97F4A7C15ULL);
    const double h = 1.0 / (double)P;
    double l;
    if (cfg.init_scheme == 0) l = __dmul_rn(cfg.init_c, sqrt(__dmul_rn((double)N, (double)M)));
    else if (cfg.init_scheme == 1) l = 1.0;
    else l = sqrt(2.0 / (double)M);
    const double r = __dmul_rn(cfg.r_over_diam, __dmul_rn(sqrt(2.0), h));
    const double r2 = __dmul_rn(r, r);
    const double span = __dadd_rn(h, __dmul_rn(2.0, r));
    const double x0 = (double)i / (double)P, y0 = (double)j / (double)P;
    const double x1 = (double)(i + 1) / (double)P, y1 = (double)(j + 1) / (double)P;
    const double lox = __dsub_rn(x0, r), loy = __dsub_rn(y0, r);
    const double wx = __dmul_rn(__dsub_rn(__dmul_rn(2.0, uniform01(key, s, n, 0)), 1.0), l);
    const double wy = __dmul_rn(__dsub_rn(__dmul_rn(2.0, uniform01(key, s, n, 1)), 1.0), l);
    double ex = __dmul_rn(0.5, __dadd_rn(x0, x1)), ey = __dmul_rn(0.5, __dadd_rn(y0, y1));
    if (cfg.init_scheme != 2) {
        for (int tr = 0; tr < kMaxCollarTries; ++tr) {
            double px = __dadd_rn(lox, __dmul_rn(uniform01(key, s, n, 2 + 2 * tr), span));
            double py = __dadd_rn(loy, __dmul_rn(uniform01(key, s, n, 3 + 2 * tr), span));
            double dx = fmax(fmax(__dsub_rn(x0, px), __dsub_rn(px, x1)), 0.0);
            double dy = fmax(fmax(__dsub_rn(y0, py), __dsub_rn(py, y1)), 0.0);
            if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r2) {
                ex = px;
                ey = py;
                break;
            }
        }
    }
    W[2 * t] = wx;
    W[2 * t + 1] = wy;
    b[t] = cfg.init_scheme == 2 ? 0.0 : -__dadd_rn(__dmul_rn(wx, ex), __dmul_rn(wy, ey));
    if (xi) {
        xi[2 * t] = ex;
        xi[2 * t + 1] = ey;
    }
}

// ---- manufactured problems -----------------------------------------------------
__device__ void problem_uf(int pid, double x, double y, double& u, double& f) {
    switch (pid) {
        case 0: {
            double s = sin(kPi * x) * sin(kPi * y);
            u = s;
            f = 2.0 * kPi * kPi * s;
        } break;
        case 1: {
            double E = exp(x + y);
            double sx, cx, sy, cy;
            sincos(2.0 * kPi * x, &sx, &cx);
            sincos(2.0 * kPi * y, &sy, &cy);
            u = E * sx * cy;
            f = -E * (2.0 * (1.0 - 4.0 * kPi * kPi) * sx * cy + 4.0 * kPi * (cx * cy - sx * sy));
        } break;
        case 2: {
            double s = sin(4.0 * kPi * x) * sin(4.0 * kPi * y);
            u = s;
            f = 32.0 * kPi * kPi * s;
        } break;
        case 3: {
            double s = sin(8.0 * kPi * x) * sin(8.0 * kPi * y);
            u = s;
            f = 128.0 * kPi * kPi * s;
        } break;
        case 4: {
            double s = sin(2.0 * kPi * x) * exp(y);
            u = s;
            f = (4.0 * kPi * kPi - 1.0) * s;
        } break;
        case 6:  // variable coefficient, eqn:varpoisson: f = 1, g = 0
            u = 0.0;
            f = 1.0;
            break;
        case 7: {  // plate bending: Lap^2 u = q/D, u = sin(pi x)sin(pi y)/(4 pi^4 D)
            const double D = 1e7 * 1e-9 / (12.0 * (1.0 - 0.3 * 0.3));
            const double sq = sin(kPi * x) * sin(kPi * y);
            u = sq / (4.0 * kPi * kPi * kPi * kPi * D);
            f = sq / D;
        } break;
        default:
            u = 0.0;
            f = 0.0;
    }
}

// Collocation point of row r of subdomain (i, j); kind = -1 interior, 0..3 edge, -2 padding.
// Each coordinate is one correctly rounded division of integers (shared face points are
// bit-identical in both neighbours).
__device__ __forceinline__ void row_point(const elmddm_config& c, int i, int j, int r, double& x, double& y,
                                          int& kind, int& k) {
    const int P = c.P, p = c.p, q = c.q, pp = p * p;
    if (r < pp) {
        int a = r % p, bb = r / p;
        double den = (double)(P * (p + 1));
        x = (double)(i * (p + 1) + a + 1) / den;
        y = (double)(j * (p + 1) + bb + 1) / den;
        kind = -1;
        k = 0;
        return;
    }
    r -= pp;
    if (r >= 4 * q && c.layout == 1 && r < 4 * q + 4) {  // lattice corner cc = (ci, cj): kind 4 + cc
        const int cc = r - 4 * q;
        x = (double)(i + (cc & 1)) / (double)P;
        y = (double)(j + (cc >> 1)) / (double)P;
        kind = 4 + cc;
        k = 0;
        return;
    }
    if (r >= 4 * q) {
        kind = -2;
        x = y = 0.0;
        k = 0;
        return;
    }
    int e = r / q;
    k = r % q;
    kind = e;
    // plate (problem 7, reading R28): q = 2 npts rows per edge, [u traces | Lap u traces]
    const int np = c.problem == 7 ? q / 2 : q, kp = k % np;
    double den = (double)(P * (np + 1));
    double ty = (double)(j * (np + 1) + kp + 1) / den;
    double tx = (double)(i * (np + 1) + kp + 1) / den;
    switch (e) {
        case 0: x = (double)i / (double)P; y = ty; break;
        case 1: x = (double)(i + 1) / (double)P; y = ty; break;
        case 2: x = tx; y = (double)j / (double)P; break;
        default: x = tx; y = (double)(j + 1) / (double)P; break;
    }
}

// edge e < 4 of subdomain (i, j) is an interface face; e = 4 + cc: the lattice corner cc is a
// cross point (inside the domain)
__device__ __forceinline__ bool edge_is_interface(int P, int i, int j, int e) {
    switch (e) {
        case 0: return i > 0;
        case 1: return i < P - 1;
        case 2: return j > 0;
        case 3: return j < P - 1;
        default: {
            const int X = i + ((e - 4) & 1), Y = j + ((e - 4) >> 1);
            return X > 0 && X < P && Y > 0 && Y < P;
        }
    }
}

// Problem 6 coefficient at the interior collocation points, eqn:varpoisson with
// eqn:grf: grf = sum_i a_i sin(w_i . x + b_i), rho = tanh(grf) + 1.1,
// grad rho = (1 - tanh^2 grf) grad grf (analytic).  coef[S][p*p][4] =
// (rho, d rho/dx, d rho/dy, 0); params[i] = (a_i, w_ix, w_iy, b_i) in global memory.
// Separable on the p x p interior lattice of a subdomain: e^{i(w.x + b)} = [e^{i(w_x x_a + b)}]
// [e^{i w_y y_b}], the two factors tabulated per term over the p lattice coordinates (one CTA per
// subdomain, terms in chunks of CT), so each point costs one complex product per term instead
// of a sincos.
constexpr int CT = 32;
__global__ void __launch_bounds__(512) k_coef(elmddm_config cfg, const double4* __restrict__ params, int nterms,
                                              double4* __restrict__ coef) {
    extern __shared__ double ctab[];  // [CT][p][4]: (cos, sin) of the x factor, (cos, sin) of the y factor
    const int p = cfg.p, pp = p * p, P = cfg.P;
    const int sl = blockIdx.x, s = cfg.s_begin + sl;
    const int i = s % P, j = s / P;
    const double den = (double)(P * (p + 1));
    constexpr int NPT = 8;  // points per thread (p*p <= 512 * 8 is checked by the launcher)
    double g[NPT], gx[NPT], gy[NPT];
#pragma unroll
    for (int u = 0; u < NPT; ++u) g[u] = gx[u] = gy[u] = 0.0;
    for (int k0 = 0; k0 < nterms; k0 += CT) {
        const int nk = min(CT, nterms - k0);
        __syncthreads();
        for (int t = threadIdx.x; t < nk * p; t += blockDim.x) {
            const int k = t / p, a = t % p;
            const double4 pr = params[k0 + k];
            const double xa = (double)(i * (p + 1) + a + 1) / den, yb = (double)(j * (p + 1) + a + 1) / den;
            double sx, cx, sy, cy;
            sincos(pr.y * xa + pr.w, &sx, &cx);
            sincos(pr.z * yb, &sy, &cy);
            double* e = ctab + (size_t)t * 4;
            e[0] = cx; e[1] = sx; e[2] = cy; e[3] = sy;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < NPT; ++u) {
            const int r = threadIdx.x + u * blockDim.x;
            if (r >= pp) break;
            const int a = r % p, bb = r / p;
            for (int k = 0; k < nk; ++k) {
                const double4 pr = params[k0 + k];
                const double* ex = ctab + ((size_t)k * p + a) * 4;
                const double* ey = ctab + ((size_t)k * p + bb) * 4;
                const double sn = fma(ex[1], ey[2], ex[0] * ey[3]);   // sin(A + B)
                const double cs = fma(ex[0], ey[2], -ex[1] * ey[3]);  // cos(A + B)
                g[u] = fma(pr.x, sn, g[u]);
                const double c = pr.x * cs;
                gx[u] = fma(c, pr.y, gx[u]);
                gy[u] = fma(c, pr.z, gy[u]);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < NPT; ++u) {
        const int r = threadIdx.x + u * blockDim.x;
        if (r >= pp) break;
        const double th = tanh(g[u]), d = 1.0 - th * th;
        coef[(int64_t)sl * pp + r] = make_double4(th + 1.1, d * gx[u], d * gy[u], 0.0);
    }
}

constexpr int AS_COLS = 8;   // columns per CTA in the K_aug kernel: must divide 8 (M % 8 == 0 is
                             // validated), so no CTA straddles the neuron / augmented boundary
constexpr int AS_NT = 256;

// 1/x for x in [1, 1e30]: MUFU.RCP64H seed + two Newton steps (full double precision)
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// Kaug[s][col][row]: grid (ceil(ncols / AS_COLS), S).
// Neuron columns use the separable form of SURVEY §8(a): with the subdomain centre c and
// b~ = b + w.c,  E = e^{2z} = [e^{2 w_x (x - c_x) + 2 b~}] [e^{2 w_y (y - c_y)}], the two factors
// tabulated per neuron over the p+q+2 distinct x (resp. y) coordinates of the subdomain's rows;
// then d = 1/(1+E), sigma = 1 - 2d, sigma' = 4 E d^2, -|w|^2 sigma'' = 2|w|^2 sigma sigma'.
// |z| <= |w|_1 (h/2 + r) stays O(10) for the paper's initialisation, so E never overflows.
// OP: 0 Poisson, 1 variable coefficient (problem 6), 2 plate bending (problem 7)
template <int OP>
__global__ void __launch_bounds__(AS_NT) k_assemble(elmddm_config cfg, int64_t ld, int64_t ncols,
                                                    const double* __restrict__ W, const double* __restrict__ b,
                                                    double* __restrict__ Kaug, double* __restrict__ At,
                                                    const double4* __restrict__ coef, int e_impl_begin,
                                                    int e_impl_end) {
    const int M = cfg.M, q = cfg.q, P = cfg.P, p = cfg.p, pp = p * p;
    const int nc = cfg.layout == 1 ? 4 : 0;  // lattice corners (rows after the edge rows)
    const int m = pp + 4 * q + nc, na = 4 * q + 2 * nc;
    const int sl = blockIdx.y, s = cfg.s_begin + sl;
    const int i = s % P, j = s / P;
    int c0 = blockIdx.x * AS_COLS;
    if (c0 >= e_impl_begin) c0 += e_impl_end - e_impl_begin;  // the grid skips the implicit columns
    double* Ks = Kaug + (int64_t)sl * ld * ncols;
    if (c0 < M) {
        extern __shared__ double tab[];      // [AS_COLS][2][ntab]
        __shared__ double w2s[AS_COLS], wxs[AS_COLS], wys[AS_COLS], bts[AS_COLS];
        const int ntab = p + q + 2;
        // distinct coordinates: [interior (p) | x0 | x0+h | edge positions (q)], same for y
        const double cx = (double)(2 * i + 1) / (double)(2 * P), cy = (double)(2 * j + 1) / (double)(2 * P);
        if (threadIdx.x < AS_COLS) {
            const int col = min(c0 + (int)threadIdx.x, M - 1);
            const double wx = W[((int64_t)sl * M + col) * 2], wy = W[((int64_t)sl * M + col) * 2 + 1];
            w2s[threadIdx.x] = 2.0 * (wx * wx + wy * wy);
            wxs[threadIdx.x] = wx;
            wys[threadIdx.x] = wy;
            bts[threadIdx.x] = b[(int64_t)sl * M + col] + wx * cx + wy * cy;  // b~ = b + w . c
        }
        __syncthreads();
        // one coordinate per thread (one correctly rounded division, shared by the 8 neurons),
        // then e^{2 w_x (x - c_x) + 2 b~} (axis 0) or e^{2 w_y (y - c_y)} (axis 1) for each neuron
        for (int t = threadIdx.x; t < 2 * ntab; t += AS_NT) {
            const int axis = t >= ntab, k = t - axis * ntab;
            const int ij = axis == 0 ? i : j;
            double coord;
            if (k < p) coord = (double)(ij * (p + 1) + k + 1) / (double)(P * (p + 1));
            else if (k == p) coord = (double)ij / (double)P;
            else if (k == p + 1) coord = (double)(ij + 1) / (double)P;
            else {
                const int np = OP == 2 ? q / 2 : q;  // plate: edge rows k and k + np share a point
                coord = (double)(ij * (np + 1) + (k - p - 2) % np + 1) / (double)(P * (np + 1));
            }
            const double dc = coord - (axis == 0 ? cx : cy);
#pragma unroll 2
            for (int cc = 0; cc < AS_COLS; ++cc)
                tab[cc * 2 * ntab + t] = exp(axis == 0 ? 2.0 * (wxs[cc] * dc + bts[cc]) : 2.0 * wys[cc] * dc);
        }
        __syncthreads();
        const int ncc = min(AS_COLS, M - c0);
        // flux rows (A^s)^T for the same neurons: At[s][e*q + k][c0 .. c0+8), sigma' = 4 E d^2 at the
        // edge point from the same tables, times w . n_e (outward axis normal); one flux row per
        // thread, four 16-byte stores of neuron pairs.  Dirichlet edges are zero.
        {
            double* Arow = At + (int64_t)sl * na * M;
            for (int row = threadIdx.x; row < na; row += AS_NT) {
                int e, k, xi, yi;
                bool nx, iface;
                double sgn;
                if (row < 4 * q) {
                    e = row / q;
                    k = row - e * q;
                    iface = edge_is_interface(P, i, j, e);
                    xi = e == 0 ? p : (e == 1 ? p + 1 : p + 2 + k);
                    yi = e == 2 ? p : (e == 3 ? p + 1 : p + 2 + k);
                    nx = e < 2;                       // normal along x (e 0, 1) or y (e 2, 3)
                    sgn = (e & 1) ? 1.0 : -1.0;       // outward: left / bottom negative
                } else {  // lattice corner cc, d = 0: its vertical edge's normal, d = 1: horizontal
                    const int cc = (row - 4 * q) >> 1, d = (row - 4 * q) & 1, ci = cc & 1, cj = cc >> 1;
                    e = 4 + cc;
                    k = 0;
                    iface = edge_is_interface(P, i, j, e);
                    xi = p + ci;
                    yi = p + cj;
                    nx = d == 0;
                    sgn = (d == 0 ? ci : cj) ? 1.0 : -1.0;
                }
                double* dst = Arow + (int64_t)row * M + c0;
#pragma unroll 1
                for (int pr = 0; pr < AS_COLS; pr += 2) {
                    double v[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int cc = pr + h;
                        v[h] = 0.0;
                        if (iface && cc < ncc) {
                            const double* tx = tab + cc * 2 * ntab;
                            const double E = tx[xi] * tx[ntab + yi];
                            const double d = fast_rcp(1.0 + E);
                            const double wn = sgn * (nx ? wxs[cc] : wys[cc]);
                            const double s1 = 4.0 * E * d * d;
                            if (OP == 2 && k >= q / 2) {  // plate: d/dn Lap phi = |w|^2 (w.n) sigma'''
                                const double sg = fma(-2.0, d, 1.0), s2 = -2.0 * sg * s1;
                                v[h] = 0.5 * w2s[cc] * wn * (-2.0 * s1 * s1 - 2.0 * sg * s2);
                            } else {
                                v[h] = wn * s1;
                            }
                        }
                    }
                    if (pr + 1 < ncc)
                        *reinterpret_cast<double2*>(dst + pr) = make_double2(v[0], v[1]);
                    else if (pr < ncc)
                        dst[pr] = v[0];
                }
            }
        }
        // interior rows, Poisson (OP 0) with p even: a row pair (r, r+1) shares the lattice row b and
        // starts at an even a, so both x-factors come from ONE 16-byte table load (conflict-free),
        // the y-factor is a broadcast, and the row kind needs no per-element selection.  Only
        // the FP64 arithmetic of the separable form remains per element.
        int r2_begin = 0;
        if (OP == 0 && (p & 1) == 0 && ncc == AS_COLS) {
            double w2r[AS_COLS];
#pragma unroll
            for (int cc = 0; cc < AS_COLS; ++cc) w2r[cc] = w2s[cc];
            const int npair = pp / 2;
            for (int r2 = threadIdx.x; r2 < npair; r2 += AS_NT) {
                const int r = 2 * r2, a = r % p, bb = r / p;
                double* dst = Ks + (int64_t)c0 * ld + r;
#pragma unroll
                for (int cc = 0; cc < AS_COLS; ++cc) {
                    const double* tx = tab + cc * 2 * ntab;
                    const double2 ex = *reinterpret_cast<const double2*>(tx + a);
                    const double ey = tx[ntab + bb];
                    const double E0 = ex.x * ey, E1 = ex.y * ey;
                    const double d0 = fast_rcp(1.0 + E0), d1 = fast_rcp(1.0 + E1);
                    // -Lap phi = 2|w|^2 sigma sigma', sigma = 1 - 2d, sigma' = 4 E d^2
                    const double v0 = w2r[cc] * fma(-2.0, d0, 1.0) * (4.0 * E0 * d0 * d0);
                    const double v1 = w2r[cc] * fma(-2.0, d1, 1.0) * (4.0 * E1 * d1 * d1);
                    *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
                    dst += ld;
                }
            }
            r2_begin = npair;
        }
        // two consecutive rows per thread -> 16-byte stores
        for (int r2 = r2_begin + threadIdx.x; r2 < ld / 2; r2 += AS_NT) {
            int xi[2], yi[2], kind[2];
            double4 rc[2] = {make_double4(1.0, 0.0, 0.0, 0.0), make_double4(1.0, 0.0, 0.0, 0.0)};
            bool lapt[2] = {false, false};  // plate: a Lap u trace row
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 2 * r2 + e;
                if (r < pp) {
                    xi[e] = r % p;
                    yi[e] = r / p;
                    kind[e] = 0;
                    if (OP == 1) rc[e] = coef[(int64_t)sl * pp + r];
                } else if (r < pp + 4 * q) {
                    const int t = r - pp, ed = t / q, k = t % q;
                    kind[e] = 1;
                    lapt[e] = OP == 2 && k >= q / 2;
                    xi[e] = ed == 0 ? p : (ed == 1 ? p + 1 : p + 2 + k);
                    yi[e] = ed == 2 ? p : (ed == 3 ? p + 1 : p + 2 + k);
                } else if (r < m) {  // lattice corner: a value row at (x0 or x0+h, y0 or y0+h)
                    const int cc = r - pp - 4 * q;
                    kind[e] = 1;
                    xi[e] = p + (cc & 1);
                    yi[e] = p + (cc >> 1);
                } else {
                    kind[e] = 2;  // padding, or (reading R29) the damping row lambda e_{r-m}^T
                    xi[e] = yi[e] = 0;
                }
            }
#pragma unroll
            for (int cc = 0; cc < AS_COLS; ++cc) {
                if (cc >= ncc) break;
                const double* tx = tab + cc * 2 * ntab;
                const double* ty = tx + ntab;
                double v[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double E = tx[xi[e]] * ty[yi[e]];
                    const double d = fast_rcp(1.0 + E);
                    const double sg = fma(-2.0, d, 1.0);
                    const double s1 = 4.0 * E * d * d;
                    if (OP == 2) {
                        // plate: interior Lap^2 phi = |w|^4 sigma'''', traces phi and Lap phi = |w|^2 sigma''
                        const double w2 = 0.5 * w2s[cc];
                        const double s2 = -2.0 * sg * s1, s3 = -2.0 * s1 * s1 - 2.0 * sg * s2;
                        const double s4 = -6.0 * s1 * s2 - 2.0 * sg * s3;
                        v[e] = kind[e] == 0 ? w2 * w2 * s4 : (kind[e] == 1 ? (lapt[e] ? w2 * s2 : sg) : 0.0);
                    } else {
                        // interior: -Lap phi, or -rho Lap phi - grad rho . grad phi (problem 6)
                        const double lap = OP == 1 ? rc[e].x * (w2s[cc] * sg) - (rc[e].y * wxs[cc] + rc[e].z * wys[cc])
                                                   : w2s[cc] * sg;
                        v[e] = kind[e] == 0 ? lap * s1 : (kind[e] == 1 ? sg : 0.0);
                    }
                    // (tikhonov < 0, reading R33: the per-subdomain lambda is written by k_damping)
                    if (kind[e] == 2) v[e] = (2 * r2 + e - m == c0 + cc && cfg.tikhonov > 0.0) ? cfg.tikhonov : 0.0;
                }
                *reinterpret_cast<double2*>(Ks + (int64_t)(c0 + cc) * ld + 2 * r2) = make_double2(v[0], v[1]);
            }
        }
        return;
    }
    // augmented columns: E_Gamma (unit interface columns) and F = [f; g; 0]
    for (int cc = 0; cc < AS_COLS; ++cc) {
        const int col = c0 + cc;
        if (col >= ncols) break;
        if (col >= e_impl_begin && col < e_impl_end) continue;  // implicit: synthesised by the QR
        if (col < M + 4 * q + nc) {  // ld is even: 16-byte stores of row pairs
            const int t = col - M;
            const int one = edge_is_interface(P, i, j, t < 4 * q ? t / q : 4 + (t - 4 * q)) ? pp + t : -1;
            double2* dst = reinterpret_cast<double2*>(Ks + (int64_t)col * ld);
            for (int r2 = threadIdx.x; r2 < ld / 2; r2 += AS_NT)
                dst[r2] = make_double2(2 * r2 == one ? 1.0 : 0.0, 2 * r2 + 1 == one ? 1.0 : 0.0);
        } else {
            for (int r = threadIdx.x; r < ld; r += AS_NT) {
                double v = 0.0;
                if (r < m) {
                    double x, y, u, f;
                    int kind, k;
                    row_point(cfg, i, j, r, x, y, kind, k);
                    if (kind == -1) {
                        problem_uf(cfg.problem, x, y, u, f);
                        v = f;
                    } else if (!edge_is_interface(P, i, j, kind)) {
                        problem_uf(cfg.problem, x, y, u, f);
                        // plate: the Lap u trace rows carry Lap u = -2 pi^2 u of the exact solution
                        v = (cfg.problem == 7 && k >= q / 2) ? -2.0 * kPi * kPi * u : u;
                    }
                }
                Ks[(int64_t)col * ld + r] = v;
            }
        }
    }
}

// Reading R33 (tikhonov < 0): lambda_s = eps max(m, M) ||K^s||_F over the m collocation rows, written
// on the diagonal of the damping rows m .. m+M-1 (k_assemble left them zero).  grid S, 512 threads;
// fixed-order reduction.
__global__ void __launch_bounds__(512) k_damping(double* __restrict__ Kaug, int64_t ld, int64_t ncols, int m,
                                                 int M) {
    __shared__ double red[16];
    double* Ks = Kaug + (int64_t)blockIdx.x * ld * ncols;
    double ss = 0.0;
    for (int n = 0; n < M; ++n)
        for (int r = threadIdx.x; r < m; r += 512) {
            const double v = Ks[(int64_t)n * ld + r];
            ss = fma(v, v, ss);
        }
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 16; ++w) t += red[w];
        red[0] = sqrt(t) * (0x1.0p-52 * (double)(m > M ? m : M));
    }
    __syncthreads();
    const double lam = red[0];
    for (int n = threadIdx.x; n < M; n += 512) Ks[(int64_t)n * ld + m + n] = lam;
}

// one warp per point: lane l sums neurons l, l + 32, ...; fixed-order butterfly reduction
__global__ void k_evaluate(elmddm_config cfg, const double* __restrict__ W, const double* __restrict__ b,
                           const double* __restrict__ coef, const double* __restrict__ xy, int64_t n,
                           double* __restrict__ u) {
    const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= n) return;
    const int P = cfg.P, M = cfg.M;
    double x = xy[2 * t], y = xy[2 * t + 1];
    int i = (int)floor(x * (double)P), j = (int)floor(y * (double)P);
    i = min(max(i, 0), P - 1);
    j = min(max(j, 0), P - 1);
    int s = j * P + i;
    if (s < cfg.s_begin || s >= cfg.s_end) return;
    int sl = s - cfg.s_begin;
    const double* Ws = W + (int64_t)sl * M * 2;
    const double* bs = b + (int64_t)sl * M;
    const double* cs = coef + (int64_t)sl * M;
    double acc = 0.0;
    for (int k = lane; k < M; k += 32) acc += cs[k] * tanh(Ws[2 * k] * x + Ws[2 * k + 1] * y + bs[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) u[t] = acc;
}

}  // namespace

cudaError_t launch_init_hidden(const elmddm_ctx* c, double* W, double* b, double* xi, cudaStream_t st) {
    int64_t n = c->sz.S * c->cfg.M;
    int nt = 128;
    KTimer kt(c, ELMDDM_K_INIT, st);
    k_init_hidden<<<(unsigned)((n + nt - 1) / nt), nt, 0, st>>>(c->cfg, W, b, xi);
    return cudaGetLastError();
}

cudaError_t launch_assemble(const elmddm_ctx* c, const double* W, const double* b, double* Kaug, double* At,
                            cudaStream_t st) {
    // (the implicit E_Gamma columns [e_impl_begin, e_impl_end) are multiples of AS_COLS apart)
    dim3 g1((unsigned)((c->sz.ncols - (c->sz.e_impl_end - c->sz.e_impl_begin) + AS_COLS - 1) / AS_COLS),
            (unsigned)c->sz.S);
    const size_t tab_bytes = sizeof(double) * AS_COLS * 2 * (c->cfg.p + c->cfg.q + 2);
    if (tab_bytes > 48 * 1024) {  // (the lattice's 1 x 1: 512 coordinates per axis)
        cudaError_t e = cudaFuncSetAttribute(c->cfg.problem == 7 ? k_assemble<2> : (c->cfg.problem == 6 ? k_assemble<1>
                                                                                                 : k_assemble<0>),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab_bytes);
        if (e != cudaSuccess) return e;
    }
    { KTimer kt(c, ELMDDM_K_ASSEMBLE, st);
    const double4* coef = nullptr;
    if (c->cfg.problem == 6) {
        const int pp = c->cfg.p * c->cfg.p;
        const int nt = std::min(512, std::max(32, (pp + 7) / 8 + 31) / 32 * 32);
        // (a per-device attribute: set on every call)
        cudaError_t e = cudaFuncSetAttribute(k_coef, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        if (e != cudaSuccess) return e;
        k_coef<<<(unsigned)c->sz.S, nt, sizeof(double) * 4 * CT * c->cfg.p, st>>>(
            c->cfg, reinterpret_cast<const double4*>(c->d_grf), c->ngrf, reinterpret_cast<double4*>(c->d_coef));
        coef = reinterpret_cast<const double4*>(c->d_coef);
    }
    if (coef)
        k_assemble<1><<<g1, AS_NT, tab_bytes, st>>>(c->cfg, c->sz.ld, c->sz.ncols, W, b, Kaug, At, coef,
                                  (int)c->sz.e_impl_begin, (int)c->sz.e_impl_end);
    else if (c->cfg.problem == 7)
        k_assemble<2><<<g1, AS_NT, tab_bytes, st>>>(c->cfg, c->sz.ld, c->sz.ncols, W, b, Kaug, At, nullptr,
                                  (int)c->sz.e_impl_begin, (int)c->sz.e_impl_end);
    else
        k_assemble<0><<<g1, AS_NT, tab_bytes, st>>>(c->cfg, c->sz.ld, c->sz.ncols, W, b, Kaug, At, nullptr,
                                  (int)c->sz.e_impl_begin, (int)c->sz.e_impl_end);
    if (c->cfg.tikhonov < 0.0)
        k_damping<<<(unsigned)c->sz.S, 512, 0, st>>>(Kaug, c->sz.ld, c->sz.ncols,
                                                    (int)(c->cfg.p * c->cfg.p + 4 * c->cfg.q + (c->cfg.layout == 1 ? 4 : 0)),
                                                    c->cfg.M); }
    return cudaGetLastError();
}

cudaError_t launch_evaluate(const elmddm_ctx* c, const double* W, const double* b, const double* coef,
                            const double* xy, int64_t n, double* u, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int nt = 256;  // 8 points per CTA, one warp each
    KTimer kt(c, ELMDDM_K_EVAL, st);
    k_evaluate<<<(unsigned)((n * 32 + nt - 1) / nt), nt, 0, st>>>(c->cfg, W, b, coef, xy, n, u);
    return cudaGetLastError();
}
