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
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <queue>
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

// nested-dissection node list (faces of each node, in elimination order) and each node's depth
// in the dissection tree (0 = the top separator)
void nd_nodes(int P, std::vector<std::vector<int>>& nodes, std::vector<int>& depth) {
    const int F = 2 * P * (P - 1);
    std::vector<int> all(F);
    for (int f = 0; f < F; ++f) all[f] = f;
    auto key = [&](int f) {
        FaceGeo g = face_geo(P, f);
        return std::make_tuple(g.j, g.i, g.vertical);
    };
    auto by_pos = [&](std::vector<int>& v) { std::sort(v.begin(), v.end(), [&](int a, int b) { return key(a) < key(b); }); };
    std::function<void(std::vector<int>&, int, int, int, int, int)> rec = [&](std::vector<int>& fs, int i0, int i1,
                                                                               int j0, int j1, int dep) {
        if (fs.empty()) return;
        const int w = i1 - i0 + 1, h = j1 - j0 + 1;
        if ((w <= 1 && h <= 1) || fs.size() <= 2) {
            by_pos(fs);
            nodes.push_back(fs);
            depth.push_back(dep);
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
            rec(L, i0, cm - 1, j0, j1, dep + 1);
            rec(R, cm + 1, i1, j0, j1, dep + 1);
        } else {
            const int cm = (j0 + j1) / 2;
            for (int f : fs) {
                FaceGeo g = face_geo(P, f);
                const int lo = g.j, hi = g.vertical ? g.j : g.j + 1;  // subdomain rows touched
                (hi < cm ? L : (lo > cm ? R : sep)).push_back(f);
            }
            rec(L, i0, i1, j0, cm - 1, dep + 1);
            rec(R, i0, i1, cm + 1, j1, dep + 1);
        }
        by_pos(sep);
        nodes.push_back(sep);
        depth.push_back(dep);
    };
    rec(all, 0, P - 1, 0, P - 1, 0);
}

}  // namespace

// Structurally nonzero q x q face blocks (b, c), b >= c, of the interface matrix M = sum_s
// scatter(T_E^T T_E) + Q^T Q (eqn:schur): faces of one subdomain (the S1 term), and the faces of
// the two subdomains adjacent to a flux face (the Q^T Q term).  Strip face numbering (R14).
void interface_face_pairs(int P, std::vector<std::pair<int, int>>& out) {
    out.clear();
    if (P < 2) return;
    const int N = P * P, F = 2 * P * (P - 1), strip = 2 * P - 1;
    auto fid = [&](int i, int j, int e) {
        if (e == 0) return i > 0 ? j * strip + (i - 1) : -1;
        if (e == 1) return i < P - 1 ? j * strip + i : -1;
        if (e == 2) return j > 0 ? (j - 1) * strip + (P - 1) + i : -1;
        return j < P - 1 ? j * strip + (P - 1) + i : -1;
    };
    std::vector<int> sub_of(2 * F, -1);
    for (int s = 0; s < N; ++s)
        for (int e = 0; e < 4; ++e) {
            const int f = fid(s % P, s / P, e);
            if (f >= 0) sub_of[2 * f + ((e == 1 || e == 3) ? 0 : 1)] = s;
        }
    std::vector<std::pair<int, int>> v;
    for (int a = 0; a < F; ++a) {
        int nb[9], n = 0;
        nb[n++] = a;
        for (int k = 0; k < 2; ++k) {
            const int s = sub_of[2 * a + k];
            for (int e = 0; e < 4; ++e) {
                const int f = fid(s % P, s / P, e);
                if (f >= 0 && f != a) nb[n++] = f;
            }
        }
        for (int x = 0; x < n; ++x)
            for (int y = 0; y < n; ++y)
                if (nb[x] >= nb[y]) v.push_back({nb[x], nb[y]});
    }
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    out.swap(v);
}

// Build the plan for `ordering` (0 strip, 1 nested dissection).  face_pairs: (b, c), b >= c,
// structurally nonzero q x q face blocks of M.  Returns the work (tile updates).
int64_t build_chol_plan(int P, int q, int F, const std::vector<std::pair<int, int>>& face_pairs, int ordering,
                        int crit_band, CholPlan& pl, int split_min) {
    const int T = ELM_NB;
    pl.ordering = ordering;
    // 1. face bases in the new order (+ padding to tile boundaries between ND nodes)
    std::vector<std::vector<int>> nodes;
    std::vector<int> ndepth;
    if (ordering == 1 && F > 0) {
        nd_nodes(P, nodes, ndepth);
    } else {
        nodes.emplace_back(F);
        for (int f = 0; f < F; ++f) nodes[0][f] = f;
        ndepth.push_back(0);
    }
    pl.fbase.assign(std::max(F, 1), 0);
    int64_t off = 0;
    std::vector<char> used;
    std::vector<int64_t> node_end;
    for (auto& nd : nodes) {
        for (int f : nd) {
            pl.fbase[f] = (int)off;
            off += q;
        }
        if (ordering == 1) off = (off + T - 1) / T * T;
        node_end.push_back(off);
    }
    pl.n = std::max<int64_t>((off + T - 1) / T * T, T);
    pl.nblk = (int)(pl.n / T);
    // dissection depth of every tile column (strip order: all 0)
    pl.blk_depth.assign(pl.nblk, 0);
    pl.blk_node0.assign(pl.nblk, 0);
    for (int J = 0, nd = 0; J < pl.nblk; ++J) {
        while (nd + 1 < (int)node_end.size() && (int64_t)J * T >= node_end[nd]) ++nd;
        pl.blk_depth[J] = ndepth[nd];
        pl.blk_node0[J] = nd > 0 ? (int)(node_end[nd - 1] / T) : 0;
    }
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
    std::vector<std::vector<int>> mcols(nb);  // M's own tile structure (lower), kept for the SpMV lists
    for (int J = 0; J < nb; ++J) {
        mcols[J] = cols[J];
        std::sort(mcols[J].begin(), mcols[J].end());
        mcols[J].erase(std::unique(mcols[J].begin(), mcols[J].end()), mcols[J].end());
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
    {
        std::vector<std::vector<int2>> mr(nb), mc(nb);
        for (int J = 0; J < nb; ++J)
            for (int I : mcols[J])
                if (I > J) {
                    const int t = pl.tile_map[(size_t)I * nb + J];
                    mr[I].push_back({J, t});
                    mc[J].push_back({I, t});
                }
        pl.tile_m.assign(tid, 0);
        for (int J = 0; J < nb; ++J)
            for (int I : mcols[J]) pl.tile_m[pl.tile_map[(size_t)I * nb + J]] = 1;
        for (int J = 0; J < nb; ++J) pl.tile_m[pl.tile_map[(size_t)J * nb + J]] = 1;  // (padding diagonals)
        pl.mrow_ptr.assign(nb + 1, 0);
        pl.mcol_ptr.assign(nb + 1, 0);
        pl.mrow.clear();
        pl.mcol.clear();
        for (int I = 0; I < nb; ++I) {
            std::sort(mr[I].begin(), mr[I].end(), [](const int2& x, const int2& y) { return x.x < y.x; });
            std::sort(mc[I].begin(), mc[I].end(), [](const int2& x, const int2& y) { return x.x > y.x; });
            pl.mrow.insert(pl.mrow.end(), mr[I].begin(), mr[I].end());
            pl.mcol.insert(pl.mcol.end(), mc[I].begin(), mc[I].end());
            pl.mrow_ptr[I + 1] = (int)pl.mrow.size();
            pl.mcol_ptr[I + 1] = (int)pl.mcol.size();
        }
    }
    pl.diag_tid.assign(nb, 0);
    for (int J = 0; J < nb; ++J) pl.diag_tid[J] = pl.tile_map[(size_t)J * nb + J];
    // 5. tasks and k-lists
    std::vector<int> klast(nb, -1);
    for (int I = 0; I < nb; ++I)
        if (rows[I].size() > 1) klast[I] = rows[I][rows[I].size() - 2];
    std::vector<TaskDesc> crit, reg;
    pl.klist.clear();
    pl.npre = 0;
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
            td.kind = 0;
            ++pl.ntc[J];
            auto& lst = I - J <= crit_band ? crit : reg;
            // split: the updates from columns below J's dissection node are final long before
            // the node itself is factored; summed by a task of their own (in place into the tile
            // of M), they no longer hold a CTA that waits for the node's columns
            if (split_min > 0) {
                int npre = 0;
                while (td.kbeg + npre < td.kend && pl.klist[td.kbeg + npre].z < pl.blk_node0[J]) ++npre;
                if (I == J && td.kend > td.kbeg) npre = std::min(npre, td.kend - td.kbeg - 1);  // klast stays
                if (npre >= split_min) {
                    TaskDesc pre = td;
                    pre.kend = td.kbeg + npre;
                    pre.klast = -1;
                    pre.pub = 0;
                    pre.kind = 1;
                    lst.push_back(pre);
                    td.kbeg += npre;
                    td.kind = 2;
                    ++pl.npre;
                }
            }
            lst.push_back(td);
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

int build_trsv_tasks(const CholPlan& pl, int dir, int chunk, std::vector<int4>& tasks, std::vector<int>& rowslot) {
    const int nb = pl.nblk;
    const std::vector<int>& ptr = dir == 0 ? pl.fwd_ptr : pl.bwd_ptr;
    const std::vector<int2>& dep = dir == 0 ? pl.fwd : pl.bwd;
    if (chunk < 1) chunk = 1 << 30;
    // 1. tasks in solve order: a row's partial chunks, then its final task
    std::vector<int4> lst;
    rowslot.assign(nb, 0);
    int nslots = 0;
    for (int t = 0; t < nb; ++t) {
        const int i = dir == 0 ? t : nb - 1 - t;
        const int d0 = ptr[i], nj = ptr[i + 1] - d0;
        const int nch = nj <= chunk ? 1 : (nj + chunk - 1) / chunk;
        rowslot[i] = nslots;
        for (int c = 0; c + 1 < nch; ++c)
            lst.push_back(int4{i, d0 + (int)((int64_t)nj * c / nch), d0 + (int)((int64_t)nj * (c + 1) / nch), nslots++});
        lst.push_back(int4{i, d0 + (int)((int64_t)nj * (nch - 1) / nch), d0 + nj, -nch});  // -1 - nparts
    }
    // 2. list order = earliest-start order of a latency model of the kernel (unbounded CTAs): a task
    //    consumes its tiles in order, each no earlier than TL/2 after its block's solution is
    //    published, TT per tile; a final task adds the partial sums and the diagonal solve.  The
    //    key of a task, the model time its last input is published, is strictly larger than the
    //    key of every task it waits for, so the sorted list stays topological (deadlock freedom of
    //    the in-order dealing).  The row order alone leaves the backward solve's CTAs blocked on
    //    the top separators' chain while ready rows wait further down the list.
    const double TT = 1.0, TL = 3.0, TD = 1.5;
    std::vector<double> fin_row(nb, 0.0), fin_task(lst.size(), 0.0), key(lst.size(), 0.0);
    for (size_t k = 0; k < lst.size(); ++k) {
        const int4 tk = lst[k];
        double t = 0.0, last_in = 0.0;
        for (int q = tk.y; q < tk.z; ++q) {
            const double rdy = fin_row[dep[q].x];
            last_in = std::max(last_in, rdy);
            t = std::max(t, rdy + TL / 2) + TT;
        }
        if (tk.w < 0) {
            const int np = -1 - tk.w;
            for (int c = 0; c < np; ++c) {
                const double rdy = fin_task[k - np + c];  // the row's partial tasks precede it
                last_in = std::max(last_in, rdy);
                t = std::max(t, rdy + TL / 2);
            }
            t += TL / 2 + TD;
            fin_row[tk.x] = t;
        } else {
            t += TL / 2;
        }
        fin_task[k] = t;
        key[k] = last_in;
    }
    std::vector<int> ord(lst.size());
    for (size_t k = 0; k < ord.size(); ++k) ord[k] = (int)k;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return key[x] < key[y]; });
    tasks.clear();
    for (int k : ord) tasks.push_back(lst[k]);
    return nslots;
}

// Task order of the persistent factorisation kernel.  The kernel deals tasks to whichever CTA is
// free, in list order (dynamic counter); a CTA streams the k-list of its task, waiting for each
// update's tiles only when it reaches them, then waits for the diagonal tile and finishes.  So the
// list must be topological (deadlock freedom), and a good list starts early what can run early.
// Column order wastes the tree parallelism of a nested-dissection order: all CTAs wait inside one
// subtree while the independent subtrees sit further down the list.
//
// Model (tools/chol_prof.py medians): one tile update UPD us, epilogue EPI_OFF (refined triangular
// solve) or EPI_DIAG (Cholesky + inverse of the diagonal tile).  chol_eval() replays a list on
// `workers` CTAs with exactly the kernel's dealing and waiting rules; schedule_chol_tasks() ranks
// the tasks by their finish time with unlimited CTAs (as-soon-as-possible streaming schedule),
// and keeps that order if the replay beats the column order.
namespace {
// model constants (us); ELMDDM_CHOL_MODEL="upd,epi_off,epi_diag,epi_pre" overrides them
double UPD = 3.5, EPI_OFF = 10.0, EPI_DIAG = 45.0, EPI_PRE = 3.0;
void model_from_env() {
    if (const char* env = getenv("ELMDDM_CHOL_MODEL")) {
        double v[4] = {UPD, EPI_OFF, EPI_DIAG, EPI_PRE};
        if (sscanf(env, "%lf,%lf,%lf,%lf", &v[0], &v[1], &v[2], &v[3]) >= 1) {
            UPD = v[0];
            EPI_OFF = v[1];
            EPI_DIAG = v[2];
            EPI_PRE = v[3];
        }
    }
}

// task index of every tile's final task (tix) and of its pre-aggregation task (ptix, -1: none)
void task_index(const CholPlan& pl, std::vector<int>& tix, std::vector<int>& ptix) {
    tix.assign(pl.ntiles, -1);
    ptix.assign(pl.ntiles, -1);
    for (int t = 0; t < (int)pl.tasks.size(); ++t) (pl.tasks[t].kind == 1 ? ptix : tix)[pl.tasks[t].tid] = t;
}

// finish time of task t started at time s, given the finish times of the tasks before it
double task_finish(const CholPlan& pl, const std::vector<int>& tix, const std::vector<int>& ptix,
                   const std::vector<double>& fin, int t, double s) {
    const TaskDesc& td = pl.tasks[t];
    double x = td.kind == 2 ? std::max(s, fin[ptix[td.tid]]) : s;
    const bool dsub = td.kind != 1 && td.I == td.J && td.klast >= 0;
    const int ke = dsub ? td.kend - 1 : td.kend;
    for (int e = td.kbeg; e < ke; ++e) {
        const int4 k4 = pl.klist[e];
        x = std::max(x, std::max(fin[tix[k4.x]], fin[tix[k4.y]])) + UPD;
    }
    if (td.kind == 1) return x + EPI_PRE;
    if (td.I > td.J) return std::max(x, fin[tix[pl.diag_tid[td.J]]]) + EPI_OFF;
    if (dsub) {  // L(J, klast) from the published C(J, klast): needs that tile's k-sum and L(klast, klast)
        const int4 k4 = pl.klist[td.kend - 1];
        x = std::max(x, std::max(fin[tix[k4.x]] - EPI_OFF, fin[tix[pl.diag_tid[td.klast]]])) + EPI_OFF + UPD;
    }
    return x + EPI_DIAG;
}
}  // namespace

// replay `order` (a permutation of pl.tasks, topological) with dynamic dealing on `workers` CTAs
double chol_eval(const CholPlan& pl, const std::vector<int>& order, int workers) {
    const int nt = (int)pl.tasks.size();
    std::vector<int> tix, ptix;
    task_index(pl, tix, ptix);
    std::vector<double> fin(nt, 1e300);
    std::priority_queue<double, std::vector<double>, std::greater<double>> freeat;
    for (int w = 0; w < workers; ++w) freeat.push(0.0);
    double span = 0.0;
    for (int t : order) {
        const double s = freeat.top();
        freeat.pop();
        fin[t] = task_finish(pl, tix, ptix, fin, t, s);
        freeat.push(fin[t]);
        span = std::max(span, fin[t]);
    }
    return span;
}

double schedule_chol_tasks(CholPlan& pl, int workers) {
    const int nt = (int)pl.tasks.size();
    if (nt == 0 || workers < 1) return 0.0;
    model_from_env();
    std::vector<int> tix, ptix;
    task_index(pl, tix, ptix);
    // column order (a topological order: off-diagonal tiles of column J after (J, J), a tile's
    // pre-aggregation before the rest of it)
    std::vector<int> col(nt);
    for (int t = 0; t < nt; ++t) col[t] = t;
    std::stable_sort(col.begin(), col.end(), [&](int x, int y) {
        const TaskDesc &a = pl.tasks[x], &b = pl.tasks[y];
        if (a.J != b.J) return a.J < b.J;
        return (a.I == a.J) > (b.I == b.J);
    });
    // dependency graph: the tiles of the k-list, the diagonal tile of column J (off-diagonal
    // tiles) or of column klast (diagonal tiles), the tile's own pre-aggregation
    auto for_deps = [&](int t, auto&& f) {
        const TaskDesc& td = pl.tasks[t];
        for (int e = td.kbeg; e < td.kend; ++e) {
            const int4 k4 = pl.klist[e];
            f(tix[k4.x]);
            if (k4.y != k4.x) f(tix[k4.y]);
        }
        if (td.kind == 1) return;
        if (td.kind == 2) f(ptix[td.tid]);
        if (td.I > td.J) f(tix[pl.diag_tid[td.J]]);
        else if (td.klast >= 0) f(tix[pl.diag_tid[td.klast]]);
    };
    std::vector<int> ndep(nt, 0), sptr(nt + 1, 0);
    for (int t = 0; t < nt; ++t) for_deps(t, [&](int d) { ++ndep[t]; ++sptr[d + 1]; });
    for (int t = 0; t < nt; ++t) sptr[t + 1] += sptr[t];
    std::vector<int> succ(sptr[nt]), fill(sptr.begin(), sptr.end() - 1);
    for (int t = 0; t < nt; ++t) for_deps(t, [&](int d) { succ[fill[d]++] = t; });
    std::vector<double> cost(nt), blev(nt, 0.0);
    for (int t = 0; t < nt; ++t) {
        const TaskDesc& td = pl.tasks[t];
        cost[t] = UPD * (td.kend - td.kbeg) + (td.kind == 1 ? EPI_PRE : (td.I == td.J ? EPI_DIAG : EPI_OFF));
    }
    for (int i = nt - 1; i >= 0; --i) {  // bottom levels, reverse topological order
        const int t = col[i];
        double m = 0.0;
        for (int j = sptr[t]; j < sptr[t + 1]; ++j) m = std::max(m, blev[succ[j]]);
        blev[t] = cost[t] + m;
    }
    // greedy list construction with the kernel's dealing rule: the earliest-free CTA takes the
    // next task.  Candidates are the tasks whose dependencies are all dealt (their finish times
    // known); a candidate is "ready" at r = its stall-free start (finish with an early start minus
    // its own cost).  Pick the ready task with the longest path to the end, else the one that
    // gets ready first.
    // (ELMDDM_CHOL_LOCALITY = bucket width in us, experiment: bottom levels within one bucket
    // rank equal and the tie goes to the lower column J, then row I, so that tasks sharing the
    // tiles L(J, k) are dealt together and read them while they are in L2)
    double loc_w = 0.0;
    if (const char* env = getenv("ELMDDM_CHOL_LOCALITY")) loc_w = std::max(0.0, atof(env));
    using KV = std::pair<double, int>;
    std::priority_queue<KV, std::vector<KV>, std::greater<KV>> pending;  // (r, task)
    auto rkey = [&](int t) {
        if (loc_w <= 0.0) return blev[t];
        const TaskDesc& td = pl.tasks[t];
        return std::floor(blev[t] / loc_w) * 1e9 - (double)td.J * 1e5 - (double)td.I;
    };
    std::priority_queue<KV> ready;                                        // (bottom level, task)
    std::priority_queue<double, std::vector<double>, std::greater<double>> freeat;
    for (int w = 0; w < workers; ++w) freeat.push(0.0);
    std::vector<double> fin(nt, 1e300);
    std::vector<int> left(ndep), ord;
    ord.reserve(nt);
    for (int t = 0; t < nt; ++t)
        if (left[t] == 0) pending.push({0.0, t});
    double span = 0.0;
    while ((int)ord.size() < nt) {
        const double s = freeat.top();
        freeat.pop();
        while (!pending.empty() && pending.top().first <= s) {
            ready.push({rkey(pending.top().second), pending.top().second});
            pending.pop();
        }
        int t;
        if (!ready.empty()) {
            t = ready.top().second;
            ready.pop();
        } else {
            t = pending.top().second;
            pending.pop();
        }
        fin[t] = task_finish(pl, tix, ptix, fin, t, s);
        span = std::max(span, fin[t]);
        freeat.push(fin[t]);
        ord.push_back(t);
        for (int j = sptr[t]; j < sptr[t + 1]; ++j) {
            const int u = succ[j];
            if (--left[u] == 0) pending.push({std::max(0.0, task_finish(pl, tix, ptix, fin, u, 0.0) - cost[u]), u});
        }
    }
    const double t_col = chol_eval(pl, col, workers);
    const std::vector<int>& best = span <= t_col ? ord : col;
    std::vector<TaskDesc> nl(nt);
    for (int t = 0; t < nt; ++t) nl[t] = pl.tasks[best[t]];
    pl.tasks.swap(nl);
    pl.ncrit = 0;
    return std::min(span, t_col);
}

// minimum pre-aggregation length of a split task (ELMDDM_CHOL_SPLIT; 0 = no split).  Measured
// (chol kernel, configs 3 / 4): no split 17.64 / 93.15 ms, 4: 17.60 / 91.62, 16: 17.34 / 91.07.
int chol_split_min() {
    int v = 16;
    if (const char* env = getenv("ELMDDM_CHOL_SPLIT")) v = std::max(0, atoi(env));
    return v;
}

// tasks[ntasks][4] = (I, J, kind, updates) in list order
void export_tasks(const CholPlan& pl, int32_t* tasks) {
    for (size_t t = 0; t < pl.tasks.size(); ++t) {
        const TaskDesc& td = pl.tasks[t];
        tasks[4 * t] = td.I;
        tasks[4 * t + 1] = td.J;
        tasks[4 * t + 2] = td.kind;
        tasks[4 * t + 3] = td.kend - td.kbeg;
    }
}
