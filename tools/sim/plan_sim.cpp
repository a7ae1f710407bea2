// Host-only study of the interface-Cholesky plan (paper_2406_15959_b200/csrc/plan.cu): builds the
// face coupling pattern of the Schur matrix for a P x P subdomain grid (the same pairs as
// elmddm.cu build_tables), the strip / nested-dissection plans, and the list-scheduling simulation.
// build: g++ -O2 -std=c++17 -I/usr/local/cuda/include -x c++ tools/sim/plan_sim.cpp -o /tmp/plan_sim
// usage: /tmp/plan_sim P q [workers]
#include "../../paper_2406_15959_b200/csrc/plan.cu"

#include <cstdio>
#include <cstdlib>
#include <set>

static int face_id(int P, int i, int j, int e) {
    const int strip = 2 * P - 1;
    if (e == 0) return i > 0 ? j * strip + (i - 1) : -1;
    if (e == 1) return i < P - 1 ? j * strip + i : -1;
    if (e == 2) return j > 0 ? (j - 1) * strip + (P - 1) + i : -1;
    return j < P - 1 ? j * strip + (P - 1) + i : -1;
}

int main(int argc, char** argv) {
    const int P = argc > 1 ? atoi(argv[1]) : 16, q = argc > 2 ? atoi(argv[2]) : 80;
    const int workers = argc > 3 ? atoi(argv[3]) : 296;
    const int N = P * P, F = 2 * P * (P - 1);
    std::vector<int> sub_face(N * 4), face_sub(F * 2, -1);
    for (int s = 0; s < N; ++s)
        for (int e = 0; e < 4; ++e) {
            const int f = face_id(P, s % P, s / P, e);
            sub_face[s * 4 + e] = f;
            if (f >= 0) face_sub[f * 2 + ((e == 1 || e == 3) ? 0 : 1)] = s;
        }
    std::set<std::pair<int, int>> pairs;
    for (int a = 0; a < F; ++a) {
        std::vector<int> nb{a};
        for (int k = 0; k < 2; ++k)
            for (int e = 0; e < 4; ++e) {
                const int f = sub_face[face_sub[a * 2 + k] * 4 + e];
                if (f >= 0 && f != a) nb.push_back(f);
            }
        for (int b : nb)
            for (int c : nb)
                if (b >= c) pairs.insert({b, c});
    }
    std::vector<std::pair<int, int>> fp(pairs.begin(), pairs.end());
    for (int ord = 0; ord < 2; ++ord) {
        CholPlan pl;
        build_chol_plan(P, q, F, fp, ord, 3, pl);
        int maxk = 0;
        for (auto& t : pl.tasks) maxk = std::max(maxk, t.kend - t.kbeg);
        std::vector<int> id(pl.tasks.size());
        for (size_t t = 0; t < id.size(); ++t) id[t] = (int)t;
        std::stable_sort(id.begin(), id.end(), [&](int x, int y) {
            const TaskDesc &a = pl.tasks[x], &b = pl.tasks[y];
            if (a.J != b.J) return a.J < b.J;
            return (a.I == a.J) > (b.I == b.J);
        });
        printf("  column order, dynamic dealing: %.2f ms\n", chol_eval(pl, id, workers) * 1e-3);
        const double ms = schedule_chol_tasks(pl, workers) * 1e-3;
        printf("P=%d q=%d %s: n=%lld nblk=%d tiles=%d tasks=%zu nupd=%lld (%.3g flop) max klist %d, simulated %.2f ms on %d workers\n",
               P, q, ord ? "ND" : "strip", (long long)pl.n, pl.nblk, pl.ntiles, pl.tasks.size(), (long long)pl.nupd,
               2.0 * 64 * 64 * 64 * pl.nupd, maxk, ms, workers);
        std::vector<int> id2(pl.tasks.size());
        for (size_t t = 0; t < id2.size(); ++t) id2[t] = (int)t;
        double work = 0;
        for (auto& t : pl.tasks) work += 3.5 * (t.kend - t.kbeg) + (t.I == t.J ? 45.0 : 10.0);
        printf("  critical path (unlimited CTAs) %.2f ms, work / workers %.2f ms\n", chol_eval(pl, id2, 1 << 20) * 1e-3,
               work / workers * 1e-3);
        if (ord == 1) {
            std::vector<double> upd(16, 0.0), cols(16, 0.0);
            for (auto& t : pl.tasks) upd[std::min(15, pl.blk_depth[t.J])] += t.kend - t.kbeg;
            for (int J = 0; J < pl.nblk; ++J) cols[std::min(15, pl.blk_depth[J])] += 1;
            printf("  updates by dissection depth of the column:");
            for (int d = 0; d < 12; ++d) printf(" d%d %.1f%% (%g cols)", d, 100.0 * upd[d] / pl.nupd, cols[d]);
            printf("\n");
        }
    }
    return 0;
}
