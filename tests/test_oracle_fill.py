"""Pins for oracle O-10..O-12 (Eq. 1 split, feature fill, adjacency fill / Algorithm 1)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests._util import GOLDEN, random_csc

SPEC = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


# ----------------------------------------------------------------------------- Eq. (1)
def test_allocate_spec_example():
    for ex in SPEC["allocate"]:
        assert oracle.allocate(ex["C"], ex["t_sample"], ex["t_feature"]) == (ex["c_adj"], ex["c_feat"])


def test_allocate_eq1_properties():
    """Eq. (1): sum == C exactly, scale invariance of the times, monotone in
    the sample share, Fraction floor agrees, 0/0 -> half, explicit ratio honoured."""
    rng = np.random.default_rng(0)
    for _ in range(1000):
        C = int(rng.integers(0, 2**62))
        n = int(rng.integers(1, 9))
        ts = rng.integers(0, 10**9, n).astype(np.uint64)
        tf = rng.integers(0, 10**9, n).astype(np.uint64)
        a, f = oracle.allocate(C, ts, tf)
        assert a + f == C
        S, F = int(ts.sum()), int(tf.sum())
        if S + F:
            assert Fraction(a) <= Fraction(C * S, S + F) < a + 1
            assert oracle.allocate(C, ts * 3, tf * 3) == (a, f)
    assert oracle.allocate(1001, [0], [0]) == (500, 501)
    assert oracle.allocate(1000, [5], [5], ratio=(1, 4)) == (250, 750)
    assert oracle.allocate(1000, [1], [9]) < oracle.allocate(1000, [2], [8])


# ----------------------------------------------------------------------------- feature fill
def test_feat_fill_spec_examples():
    for ex in SPEC["feat_fill"]:
        slot, adm = oracle.feat_fill(ex["visits"], ex["cap"])
        assert adm.tolist() == ex["admitted"]
        assert [slot[v] for v in ex["admitted"]] == list(range(len(ex["admitted"])))


def test_feat_fill_equals_full_sort():
    """O-11 == first cap entries of numpy.lexsort by (visits desc, id asc), slots by id."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        N = int(rng.integers(1, 300))
        visits = rng.integers(0, 6, N).astype(np.int32)
        cap = int(rng.integers(0, N + 3))
        slot, adm = oracle.feat_fill(visits, cap)
        order = np.lexsort((np.arange(N), -visits.astype(np.int64)))
        want = np.sort(order[: min(cap, N)])
        assert adm.tolist() == want.tolist()
        exp = np.full(N, -1)
        exp[want] = np.arange(len(want))
        assert slot.tolist() == exp.tolist()


def test_feat_fill_matches_paper_rule_when_above_average_fits():
    """nodes with visits > average go in first (no sort), then below-average nodes
    backfill.  When the above-average set fits, the admitted set must contain it and
    every other admitted node must have visits <= average."""
    rng = np.random.default_rng(2)
    for _ in range(200):
        N = int(rng.integers(2, 400))
        visits = rng.poisson(1.5, N).astype(np.int32)
        avg = visits.mean()
        above = np.nonzero(visits > avg)[0]
        cap = int(rng.integers(len(above), N + 1))
        _, adm = oracle.feat_fill(visits, cap)
        assert set(above.tolist()) <= set(adm.tolist())
        assert len(adm) == cap
        rest = np.setdiff1d(adm, above)
        assert np.all(visits[rest] <= avg)


# ----------------------------------------------------------------------------- Algorithm 1
def test_adj_fill_fig6_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "fig6_adj_fill.json")))
    R, cl, co, ac = oracle.adj_fill(g["indptr"], g["indices"], g["counts"], g["c_adj_bytes"])
    ex = g["expected"]
    assert R.tolist() == ex["indices_R"]
    assert cl.tolist() == ex["cached_len"]
    assert ac.tolist() == ex["acache"]
    pf = g["paper_facts"]
    cnt = np.array(g["counts"])
    assert cnt[0:3].sum() == pf["node0_total"] and cnt[3:5].sum() == pf["node1_total"]
    assert R[0:3].tolist() == pf["node0_reordered"] and cl[2] == pf["node2_cached_len"]
    # hit rule: node 2, 1-based n <= cached_len -> hit; 0-based r < cached_len
    assert [r < cl[2] for r in range(2)] == [True, False]


def _brute_adj_fill(indptr, indices, counts, c_adj):
    """Full-sort reference via numpy.lexsort (S:317 'brute-force prefix oracle')."""
    N = len(indptr) - 1
    E = len(indices)
    R = indices.copy()
    tot = np.zeros(N, np.int64)
    for v in range(N):
        a, b = indptr[v], indptr[v + 1]
        c = counts[a:b].astype(np.int64)
        perm = np.lexsort((np.arange(b - a), -c))  # stable: count desc, position asc
        R[a:b] = indices[a:b][perm]
        tot[v] = c.sum()
    deg = np.diff(indptr)
    cap = c_adj // 4
    if E <= cap:
        return R, deg.astype(np.int32)
    order = np.lexsort((np.arange(N), -tot))
    cum = np.cumsum(deg[order])
    prev = np.concatenate([[0], cum[:-1]])
    take = np.clip(cap - prev, 0, deg[order])
    cl = np.zeros(N, np.int32)
    cl[order] = take
    return R, cl


def test_adj_fill_equals_bruteforce_prefix():
    rng = np.random.default_rng(3)
    for trial in range(200):
        N = int(rng.integers(1, 40))
        indptr, indices = random_csc(rng, N, 7)
        E = len(indices)
        counts = rng.integers(0, 4, E).astype(np.int32)
        c_adj = int(rng.integers(0, 4 * E + 12))
        R, cl, co, ac = oracle.adj_fill(indptr, indices, counts, c_adj)
        R2, cl2 = _brute_adj_fill(indptr, indices, counts, c_adj)
        assert R.tolist() == R2.tolist()
        assert cl.tolist() == cl2.tolist()
        assert len(ac) == min(E, c_adj // 4) == int(cl.sum())
        for v in range(N):
            assert ac[co[v]:co[v] + cl[v]].tolist() == R[indptr[v]:indptr[v] + cl[v]].tolist()


def test_adj_fill_invariants_and_monotonicity():
    """counts non-increasing within each reordered run; totals non-increasing
    along the walk; every node's run is a permutation of its original run; larger budget
    never caches fewer elements of any node; whole-fit caches everything."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        N = int(rng.integers(1, 30))
        indptr, indices = random_csc(rng, N, 6)
        E = len(indices)
        counts = rng.integers(0, 5, E).astype(np.int32)
        prev = None
        for c_adj in sorted(rng.integers(0, 4 * E + 8, 5).tolist()):
            R, cl, co, ac = oracle.adj_fill(indptr, indices, counts, c_adj)
            for v in range(N):
                a, b = indptr[v], indptr[v + 1]
                assert sorted(R[a:b].tolist()) == sorted(indices[a:b].tolist())
            if prev is not None:
                assert np.all(cl >= prev)
            prev = cl
        R, cl, co, ac = oracle.adj_fill(indptr, indices, counts, 4 * E)
        assert cl.tolist() == np.diff(indptr).tolist()


def test_table1_redundancy_arithmetic():
    """Table I: Load/Test == Loaded / Test nodes to 3 decimals."""
    t = SPEC["table1"]
    for bs, fan, loaded, ratio in t["rows"]:
        assert round(loaded / t["test_nodes"], 3) == pytest.approx(ratio, abs=1e-3)


# ----------------------------------------------------------------------------- F4 knapsack
def test_knapsack_spec_example():
    """one feature row (count 100, 4 bytes) vs one adjacency element (count 1, 4 bytes),
    budget 4 -> the feature row is admitted."""
    indptr = np.array([0, 1], np.int64)
    slot, cl, used = oracle.knapsack_fill(indptr, [100], [1], 4, 4, 1.0, 1.0)
    assert slot.tolist() == [0] and cl.tolist() == [0] and used == 4


def test_knapsack_properties():
    """Budget respected; full budget admits everything; every non-admitted item that would fit
    the leftover has density no higher than the lowest admitted item of its kind (greedy);
    each node's admitted elements are its top-count elements (the level-2 prefix, so the
    prefix hit rule holds); monotone in the budget."""
    rng = np.random.default_rng(7)
    for _ in range(150):
        N = int(rng.integers(1, 30))
        indptr, _ = random_csc(rng, N, 6)
        E = int(indptr[-1])
        visits = rng.integers(0, 6, N).astype(np.int32)
        counts = rng.integers(0, 5, E).astype(np.int32)
        R = int(rng.choice([16, 64, 400]))
        cf, ca = float(rng.uniform(0.1, 5)), float(rng.uniform(0.1, 5))
        total = N * R + 4 * E
        Cb = int(rng.integers(0, total + 20))
        slot, cl, used = oracle.knapsack_fill(indptr, visits, counts, Cb, R, cf, ca)
        adm = slot >= 0
        assert used <= Cb and used == int(adm.sum()) * R + 4 * int(cl.sum())
        assert slot[adm].tolist() == list(range(int(adm.sum())))
        left = Cb - used
        if (~adm).any() and left >= R:
            raise AssertionError("a feature row still fits but was not admitted")
        for v in range(N):
            run = counts[indptr[v]:indptr[v + 1]]
            order = np.lexsort((np.arange(len(run)), -run.astype(np.int64)))
            top = run[order][: cl[v]]
            rest = run[order][cl[v]:]
            if len(top) and len(rest):
                assert top.min() >= rest.max()  # prefix of the level-2 order
        full_slot, full_cl, _ = oracle.knapsack_fill(indptr, visits, counts, total, R, cf, ca)
        assert (full_slot >= 0).all() and full_cl.tolist() == np.diff(indptr).tolist()
        s2, c2, _ = oracle.knapsack_fill(indptr, visits, counts, Cb + 4 * E + R * N, R, cf, ca)
        assert ((s2 >= 0) | ~adm).all() and (c2 >= cl).all()


KNAP = json.load(open(os.path.join(GOLDEN, "knapsack_cases.json")))


@pytest.mark.parametrize("case", KNAP["cases"], ids=[c["name"] for c in KNAP["cases"]])
def test_knapsack_hand_worked_cases(case):
    """O-14 against hand-worked instances (tests/golden/knapsack_cases.json):
    unequal cost factors, cross-kind and within-kind ties, skip-and-continue."""
    slot, cl, used = oracle.knapsack_fill(np.array(case["indptr"], np.int64), case["visits"], case["counts"],
                                          case["C"], case["row_bytes"], case["cost_feat"], case["cost_adj"])
    n = len(case["indptr"]) - 1
    assert slot[:n].tolist() == case["slot_of"]
    assert cl[:n].tolist() == case["cached_len"]
    assert used == case["used"]


def _exhaustive_greedy(indptr, visits, counts, C, R, cf, ca):
    """SPEC S:503's independent check: every item with its EXACT density (Fraction), all items
    sorted by (density desc, kind: feature first, id asc), each admitted iff it fits what is left."""
    cf, ca = Fraction(cf), Fraction(ca)
    items = [(-Fraction(int(visits[v])) * cf / R, 0, v, R) for v in range(len(visits))]
    items += [(-Fraction(int(counts[e])) * ca / 4, 1, e, 4) for e in range(len(counts))]
    left, feat, elem = C, set(), set()
    for _, kind, i, size in sorted(items):
        if size <= left:
            left -= size
            (feat if kind == 0 else elem).add(i)
    slot, s = [], 0
    for v in range(len(visits)):
        slot.append(s if v in feat else -1)
        s += v in feat
    cl = [sum(1 for e in range(indptr[v], indptr[v + 1]) if e in elem) for v in range(len(visits))]
    return slot, cl, C - left


def test_knapsack_matches_exhaustive_greedy_small_instances():
    """O-14 == the independent exact-arithmetic greedy on 400 random instances of <= 20 items,
    with UNEQUAL, dyadic cost factors (exact in fp64) and small counts, so cross-kind and
    within-kind density ties occur often ("20-item random instance -> admitted set
    matches an independent exhaustive greedy oracle")."""
    rng = np.random.default_rng(2503)
    ties = 0
    for _ in range(400):
        N = int(rng.integers(1, 8))
        E_target = int(rng.integers(0, 21 - N))
        degs = rng.multinomial(E_target, np.ones(N) / N) if E_target else np.zeros(N, np.int64)
        indptr = np.r_[0, np.cumsum(degs)].astype(np.int64)
        E = int(indptr[-1])
        visits = rng.integers(0, 5, N).astype(np.int32)
        counts = rng.integers(0, 5, E).astype(np.int32)
        R = int(rng.choice([4, 8, 16, 64]))
        cf = float(rng.integers(1, 17)) / 8.0
        ca = float(rng.integers(1, 17)) / 8.0
        while ca == cf:
            ca = float(rng.integers(1, 17)) / 8.0
        C = int(rng.integers(0, N * R + 4 * E + 8))
        want = _exhaustive_greedy(indptr, visits, counts, C, R, cf, ca)
        slot, cl, used = oracle.knapsack_fill(indptr, visits, counts, C, R, cf, ca)
        assert (slot[:N].tolist(), cl[:N].tolist(), used) == want
        df = {Fraction(int(x)) * Fraction(cf) / R for x in visits}
        da = {Fraction(int(x)) * Fraction(ca) / 4 for x in counts}
        ties += bool(df & da)
    assert ties > 40  # the instances do exercise the cross-kind tie-break
