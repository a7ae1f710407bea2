"""Host logic of the interface-factorisation plan (plan.cu via the host-only elmddm_plan_query;
no GPU): nested-dissection renumbering, tile structure vs an independent scalar symbolic
factorisation, task-list order (the persistent kernel's deadlock-freedom condition) and work
counts.  DESIGN.md §5.5, reading R25."""
import itertools

import numpy as np
import pytest

import paper_2406_15959_b200 as E


def face_pattern(P):
    """Face pairs of M = sum_s T_E^T T_E + Q^T Q (eqn:schur), from the geometry alone: faces of
    one subdomain, and faces of the two subdomains adjacent to a flux face."""
    strip = 2 * P - 1
    F = 2 * P * (P - 1)

    def fid(i, j, e):
        if e == 0:
            return j * strip + i - 1 if i > 0 else -1
        if e == 1:
            return j * strip + i if i < P - 1 else -1
        if e == 2:
            return (j - 1) * strip + P - 1 + i if j > 0 else -1
        return j * strip + P - 1 + i if j < P - 1 else -1

    faces_of = [[f for f in (fid(s % P, s // P, e) for e in range(4)) if f >= 0] for s in range(P * P)]
    subs_of = [[] for _ in range(F)]
    for s, fs in enumerate(faces_of):
        for f in fs:
            subs_of[f].append(s)
    pairs = set()
    for a in range(F):
        nb = {x for s in subs_of[a] for x in faces_of[s]}
        pairs |= {(max(x, y), min(x, y)) for x in nb for y in nb}
    return F, pairs


def scalar_fill(P, q, newidx, n):
    """Lower pattern of the Cholesky factor of M in the plan's order (boolean elimination)."""
    F, pairs = face_pattern(P)
    A = np.zeros((n, n), dtype=bool)
    for b, c in pairs:
        ib = newidx[b * q:(b + 1) * q]
        ic = newidx[c * q:(c + 1) * q]
        A[np.ix_(ib, ic)] = True
        A[np.ix_(ic, ib)] = True
    A |= np.eye(n, dtype=bool)
    L = np.tril(A)
    for k in range(n):
        rows = np.nonzero(L[k + 1:, k])[0] + k + 1
        if len(rows) > 1:
            L[np.ix_(rows, rows)] |= np.tril(np.ones((len(rows), len(rows)), dtype=bool))
    return L


CASES = [(2, 3), (3, 5), (4, 4), (5, 3), (4, 24), (3, 70)]


@pytest.mark.parametrize("P,q", CASES)
@pytest.mark.parametrize("ordering", [0, 1])
def test_plan_tiles_cover_scalar_fill(P, q, ordering):
    pl = E.plan_query(P, q, ordering)
    n, nb = pl["n"], pl["nblk"]
    newidx, tmap = pl["newidx"], pl["tile_map"]
    G = 2 * P * (P - 1) * q
    assert n % 64 == 0 and n >= G and nb * 64 == n
    assert len(np.unique(newidx)) == G and newidx.min() >= 0 and newidx.max() < n
    L = scalar_fill(P, q, newidx, n)
    need = L.reshape(nb, 64, nb, 64).any(axis=(1, 3))
    have = tmap >= 0
    assert np.all(have[need]), "a nonzero of L falls outside the plan's tiles"
    assert np.all(np.diag(have)) and not np.any(np.triu(have, 1))
    ids = tmap[have]
    assert sorted(ids.tolist()) == list(range(pl["ntiles"]))


@pytest.mark.parametrize("split,locality", [("0", "0"), ("4", "0"), ("1", "0"), ("4", "500"), ("0", "5000")])
@pytest.mark.parametrize("P,q", [(3, 5), (4, 24), (6, 10), (8, 60)])
def test_plan_task_list_is_topological_and_counts_updates(P, q, split, locality, monkeypatch):
    """The list-scheduled order (dynamic dealing): every task comes after the tiles its k-list
    and its epilogue wait for -- the condition under which the persistent kernel's smallest
    unfinished task can always run -- and the update count is the number of (I, J, k) with
    L(I,k), L(J,k) present, k < J.  Split tasks (ELMDDM_CHOL_SPLIT): the pre-aggregation of
    (I, J) takes the first updates of the k-list (columns below J's dissection node, never the
    diagonal task's last one), waits only for their tiles and comes before the rest of (I, J)."""
    monkeypatch.setenv("ELMDDM_CHOL_SPLIT", split)
    monkeypatch.setenv("ELMDDM_CHOL_LOCALITY", locality)  # (the opt-in locality tie-break keeps it topological)
    pl = E.plan_query(P, q, 1, 296)
    have = pl["tile_map"] >= 0
    fin, pre = {}, {}
    for t, (I, J, kind, nk) in enumerate(pl["tasks"]):
        (pre if kind == 1 else fin)[(int(I), int(J))] = (t, int(kind), int(nk))
    assert len(fin) == pl["ntiles"] and len(fin) + len(pre) == pl["ntasks"]
    if split == "0":
        assert not pre
    elif P >= 4:
        assert pre
    nupd = 0
    for (I, J), (t, kind, nk) in fin.items():
        ks = np.nonzero(have[I, :J] & have[J, :J])[0]
        nupd += len(ks)
        npre = 0
        if kind == 2:
            tp, _, npre = pre[(I, J)]
            assert tp < t and npre >= int(split) and npre + nk == len(ks)
            for k in ks[:npre]:
                assert fin[(I, int(k))][0] < tp and fin[(J, int(k))][0] < tp
        else:
            assert kind == 0 and nk == len(ks) and (I, J) not in pre
        for k in ks[npre:]:
            assert fin[(I, int(k))][0] < t and fin[(J, int(k))][0] < t
        if I > J:
            assert fin[(J, J)][0] < t
        elif len(ks):
            assert npre < len(ks)
            assert fin[(int(ks[-1]), int(ks[-1]))][0] < t
    assert nupd == pl["nupd"]


@pytest.mark.parametrize("P,q", [(4, 24), (6, 10)])
def test_static_lists_are_column_ordered(P, q):
    """Without scheduling (static dealing: the critical band I - J <= 3, then the rest, each
    worked round-robin by its own CTAs) each list is column-ordered with a column's diagonal
    task first -- every dependency of a task lies in an earlier column or is its own column's
    diagonal, the progress argument of the static mode."""
    pl = E.plan_query(P, q, 1, 0)
    tasks = [(int(I), int(J)) for I, J, _, _ in pl["tasks"]]
    crit = [t for t in tasks if t[0] - t[1] <= 3]
    rest = [t for t in tasks if t[0] - t[1] > 3]
    assert tasks == crit + rest
    for lst in (crit, rest):
        keys = [(J, 0 if I == J else 1) for I, J in lst]
        assert keys == sorted(keys)


def test_nested_dissection_reduces_work():
    """At the BASELINE sizes the nested-dissection order needs fewer tile updates than the strip
    (envelope) order (config 3: 8.6e5 vs 1.33e6; config 4: 4.8e6 vs 1.17e7)."""
    for P, q in [(8, 60), (16, 80), (32, 64)]:
        nd = E.plan_query(P, q, 1, arrays=False)
        st = E.plan_query(P, q, 0, arrays=False)
        assert nd["nupd"] < st["nupd"]
    nd3 = E.plan_query(16, 80, 1, arrays=False)
    assert nd3["nupd"] == 861078 and nd3["ntiles"] == 30915


def test_plan_query_rejects_bad_arguments():
    for args in [(1, 4, 1, 0), (4, 0, 1, 0), (4, 4, 2, 0)]:
        with pytest.raises(E.ElmddmError):
            E.plan_query(*args, arrays=False)
