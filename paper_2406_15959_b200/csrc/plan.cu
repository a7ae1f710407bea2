// plan.cu -- host-side ordering and symbolic factorisation of the interface Schur matrix
// (eqn:schur) at 64-tile granularity, for the persistent left-looking Cholesky of
// chol.cu.  Two face orderings:
//   * strip order (reading R14): the envelope ordering of the original build;
//   * nested dissection: recursive bisection of the P x P subdomain grid;
//     a separator is every face touching the middle subdomain column (row) -- two faces thick,
//     because Q^T Q couples faces within any pair of adjacent subdomains -- and every tree node
//     starts on a tile boundary (padding unknowns with unit diagonal), so subtrees never share a
//     tile and fill stays inside the elimination tree.
// The symbolic factorisation (elimination tree on tiles) gives the tile structure of L, the
// column-ordered task list with per-task lists of update tiles k (rows I and J both nonzero in
// column k), the triangular-solve dependency lists, and the work 2 * 64^3 per tile update; the
// auto mode keeps the ordering with less work.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <functional>
#include <map>
#include <tuple>
#include <utility>
#include <vector>

#include "internal.h"

namespace {

struct FaceGeo {
    int vertical, i, j;  // V(i,j) between subdomains (i,j)-(i+1,j); H(i,j) between (i,j)-(i,j+1)
};

FaceGeo face_geo(int P, int f) {
    const int strip = 2 * P - 1, j = f / strip, t = f % strip;
    if (t < P - 1) return {1, t, j};
    return {0, t - (P - 1), j};
}

// nested-dissection node list (faces of each node, in elimination order)
void nd_nodes(int P, std::vector<std::vector<int>>& nodes) {
    const int F = 2 * P * (P - 1);
    std::vector<int> all(F);
    for (int f = 0; f < F; ++f) all[f] = f;
    auto key = [&](int f) {
        FaceGeo g = face_geo(P, f);
        return std::make_tuple(g.j, g.i, g.vertical);
    };
    auto by_pos = [&](std::vector<int>& v) { std::sort(v.begin(), v.end(), [&](int a, int b) { return key(a) < key(b); }); };
    std::function<void(std::vector<int>&, int, int, int, int)> rec = [&](std::vector<int>& fs, int i0, int i1, int j0,
                                                                          int j1) {
        if (fs.empty()) return;
        const int w = i1 - i0 + 1, h = j1 - j0 + 1;
        if ((w <= 1 && h <= 1) || fs.size() <= 2) {
            by_pos(fs);
            nodes.push_back(fs);
            return;
        }
        std::vector<int> sep, L, R;
        if (w >= h) {
            const int cm = (i0 + i1) / 2;
            for (int f : fs) {
                FaceGeo g = face_geo(P, f);
                const int lo = g.i, hi = g.vertical ? g.i + 1 : g.i;  // subdomain columns touched
                (hi < cm ? L : (lo > cm ? R : sep)).push_back(f);
            }
            rec(L, i0, cm - 1, j0, j1);
            rec(R, cm + 1, i1, j0, j1);
        } else {
            const int cm = (j0 + j1) / 2;
            for (int f : fs) {
                FaceGeo g = face_geo(P, f);
                const int lo = g.j, hi = g.vertical ? g.j : g.j + 1;  // subdomain rows touched
                (hi < cm ? L : (lo > cm ? R : sep)).push_back(f);
            }
            rec(L, i0, i1, j0, cm - 1);
            rec(R, i0, i1, cm + 1, j1);
        }
        by_pos(sep);
        nodes.push_back(sep);
    };
    rec(all, 0, P - 1, 0, P - 1);
}

}  // namespace

// Build the plan for `ordering` (0 strip, 1 nested dissection).  face_pairs: (b, c), b >= c,
// structurally nonzero q x q face blocks of M.  Returns the work (tile updates).
int64_t build_chol_plan(int P, int q, int F, const std::vector<std::pair<int, int>>& face_pairs, int ordering,
                        int crit_band, CholPlan& pl) {
    const int T = ELM_NB;
    pl.ordering = ordering;
    // 1. face bases in the new order (+ padding to tile boundaries between ND nodes)
    std::vector<std::vector<int>> nodes;
    if (ordering == 1 && F > 0) {
        nd_nodes(P, nodes);
    } else {
        nodes.emplace_back(F);
        for (int f = 0; f < F; ++f) nodes[0][f] = f;
    }
    pl.fbase.assign(std::max(F, 1), 0);
    int64_t off = 0;
    std::vector<char> used;
    for (auto& nd : nodes) {
        for (int f : nd) {
            pl.fbase[f] = (int)off;
            off += q;
        }
        if (ordering == 1) off = (off + T - 1) / T * T;
    }
    pl.n = std::max<int64_t>((off + T - 1) / T * T, T);
    pl.nblk = (int)(pl.n / T);
    used.assign(pl.n, 0);
    for (int f = 0; f < F; ++f)
        for (int k = 0; k < q; ++k) used[pl.fbase[f] + k] = 1;
    pl.pad.clear();
    for (int64_t x = 0; x < pl.n; ++x)
        if (!used[x]) pl.pad.push_back((int)x);
    // 2. tile adjacency of M (lower)
    const int nb = pl.nblk;
    std::vector<std::vector<int>> cols(nb);
    for (int J = 0; J < nb; ++J) cols[J].push_back(J);
    auto tiles_of = [&](int f, int& t0, int& t1) {
        t0 = pl.fbase[f] / T;
        t1 = (pl.fbase[f] + q - 1) / T;
    };
    for (auto& bc : face_pairs) {
        int a0, a1, b0, b1;
        tiles_of(bc.first, a0, a1);
        tiles_of(bc.second, b0, b1);
        for (int I = a0; I <= a1; ++I)
            for (int J = b0; J <= b1; ++J) cols[std::min(I, J)].push_back(std::max(I, J));
    }
    // 3. symbolic factorisation (children merge into their elimination-tree parent)
    for (int J = 0; J < nb; ++J) {
        auto& c = cols[J];
        std::sort(c.begin(), c.end());
        c.erase(std::unique(c.begin(), c.end()), c.end());
        if (c.size() > 1) {
            auto& p = cols[c[1]];
            p.insert(p.end(), c.begin() + 1, c.end());
        }
    }
    // 4. tile ids (column by column), row structures
    pl.tile_map.assign((size_t)nb * nb, -1);
    std::vector<std::vector<int>> rows(nb);
    int tid = 0;
    for (int J = 0; J < nb; ++J)
        for (int I : cols[J]) {
            pl.tile_map[(size_t)I * nb + J] = tid++;
            rows[I].push_back(J);  // ascending J
        }
    pl.ntiles = tid;
    pl.diag_tid.assign(nb, 0);
    for (int J = 0; J < nb; ++J) pl.diag_tid[J] = pl.tile_map[(size_t)J * nb + J];
    // 5. tasks and k-lists
    std::vector<int> klast(nb, -1);
    for (int I = 0; I < nb; ++I)
        if (rows[I].size() > 1) klast[I] = rows[I][rows[I].size() - 2];
    std::vector<TaskDesc> crit, reg;
    pl.klist.clear();
    pl.ntc.assign(nb, 0);
    int64_t nupd = 0;
    for (int J = 0; J < nb; ++J) {
        for (int I : cols[J]) {
            TaskDesc td{};
            td.I = I;
            td.J = J;
            td.tid = pl.tile_map[(size_t)I * nb + J];
            td.kbeg = (int)pl.klist.size();
            // k < J with L(I,k) and L(J,k) nonzero: merge of rows[I] and rows[J]
            const auto& rI = rows[I];
            const auto& rJ = rows[J];
            size_t a = 0, b = 0;
            while (a < rI.size() && b < rJ.size()) {
                const int ka = rI[a], kb = rJ[b];
                if (ka >= J || kb >= J) break;
                if (ka == kb) {
                    pl.klist.push_back({pl.tile_map[(size_t)I * nb + ka], pl.tile_map[(size_t)J * nb + ka], ka, 0});
                    ++a;
                    ++b;
                } else if (ka < kb) {
                    ++a;
                } else {
                    ++b;
                }
            }
            td.kend = (int)pl.klist.size();
            nupd += td.kend - td.kbeg;
            td.klast = (I == J && td.kend > td.kbeg) ? pl.klist[td.kend - 1].z : -1;
            td.pub = (I > J && klast[I] == J) ? 1 : 0;  // C(I, J) feeds the diagonal task of row I
            ++pl.ntc[J];
            (I - J <= crit_band ? crit : reg).push_back(td);
        }
    }
    pl.ncrit = (int)crit.size();
    pl.tasks = crit;
    pl.tasks.insert(pl.tasks.end(), reg.begin(), reg.end());
    // 6. triangular-solve dependency lists: row i (tiles (i, j), j < i, ascending) and column i
    //    (tiles (j, i), j > i, descending)
    pl.fwd_ptr.assign(nb + 1, 0);
    pl.bwd_ptr.assign(nb + 1, 0);
    pl.fwd.clear();
    pl.bwd.clear();
    for (int i = 0; i < nb; ++i) {
        for (int j : rows[i])
            if (j < i) pl.fwd.push_back({j, pl.tile_map[(size_t)i * nb + j]});
        pl.fwd_ptr[i + 1] = (int)pl.fwd.size();
        for (auto it = cols[i].rbegin(); it != cols[i].rend(); ++it)
            if (*it > i) pl.bwd.push_back({*it, pl.tile_map[(size_t)(*it) * nb + i]});
        pl.bwd_ptr[i + 1] = (int)pl.bwd.size();
    }
    pl.nupd = nupd;
    return nupd;
}
