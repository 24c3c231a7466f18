"""Pins for oracle O-5..O-9 (batch sampling, gather, presample counts, counters)."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from tests._util import random_csc


def _check_batch_invariants(indptr, indices, seeds, fanouts, b):
    """Invariants every correct batch satisfies (BJ north_star oracle bullet list):
    F_h prefix-nested and unique, seeds first, every sample a true neighbour with
    min(deg, f) distinct ranks, block CSR well formed, |F_L| <= min(N, B*prod(1+f))."""
    N, L = len(indptr) - 1, len(fanouts)
    F, n = b.F, b.sizes
    assert len(set(F.tolist())) == len(F)
    assert F[: len(seeds)].tolist() == list(seeds)
    assert n[0] == len(seeds) and np.all(np.diff(n) >= 0) and n[L] == len(F)
    assert n[L] <= min(N, len(seeds) * np.prod([1 + f for f in fanouts]))
    total = 0
    for h in range(L):
        f = fanouts[L - 1 - h]
        bp, bs = b.bptr[h], b.bsrc[h]
        assert len(bp) == n[h] + 1 and bp[0] == 0 and np.all(np.diff(bp) >= 0)
        assert np.all(bs < n[h + 1]) and np.all(bs >= 0)
        for d in range(n[h]):
            v = F[d]
            deg = indptr[v + 1] - indptr[v]
            k = bp[d + 1] - bp[d]
            assert k == min(deg, f)
            nb = F[bs[bp[d]:bp[d + 1]]]
            # sampled multiset is a sub-multiset of v's in-neighbour multiset
            full = indices[indptr[v]:indptr[v + 1]]
            vals, cnt = np.unique(nb, return_counts=True)
            fv, fc = np.unique(full, return_counts=True)
            fmap = dict(zip(fv.tolist(), fc.tolist()))
            for x, c in zip(vals.tolist(), cnt.tolist()):
                assert fmap.get(x, 0) >= c
            total += k
    assert int(b.counters[0] + b.counters[1]) == total


def test_invariants_on_rmat(tiny_graph):
    indptr, indices = tiny_graph
    batches = synth.inference_batches(indptr, 64)
    for fan in [(2, 2, 2), (15, 10, 5), (8, 4, 2), (3,)]:
        for bi in range(3):
            b = oracle.sample_batch(indptr, indices, batches[bi], fan, seed=4)
            _check_batch_invariants(indptr, indices, batches[bi], fan, b)


def test_full_fanout_equals_khop_closure_and_induced_blocks():
    """Special case f >= max deg: no randomness.  F_L must equal the L-hop in-neighbour
    closure of the seeds (scipy.sparse reachability) and every block must list the full
    in-adjacency in CSC order."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        N = int(rng.integers(5, 60))
        indptr, indices = random_csc(rng, N, 6)
        A = sp.csc_matrix((np.ones(len(indices)), indices, indptr), shape=(N, N))  # A[u, v]=1: u -> v
        seeds = rng.choice(N, size=int(rng.integers(1, min(N, 8) + 1)), replace=False).astype(np.int32)
        L = int(rng.integers(1, 4))
        fan = [6] * L
        b = oracle.sample_batch(indptr, indices, seeds, fan, seed=int(trial))
        x = np.zeros(N, bool)
        x[seeds] = True
        for h in range(L):
            assert set(b.F[: b.sizes[h]].tolist()) == set(np.nonzero(x)[0].tolist())
            x = x | ((A @ x.astype(float)) > 0)
        assert set(b.F.tolist()) == set(np.nonzero(x)[0].tolist())
        for h in range(L):
            for d in range(b.sizes[h]):
                v = b.F[d]
                got = b.F[b.bsrc[h][b.bptr[h][d]:b.bptr[h][d + 1]]]
                assert got.tolist() == indices[indptr[v]:indptr[v + 1]].tolist()


def test_first_occurrence_relabel_order():
    """C6: new nodes get ids in order of first appearance (dst-major, rank-ascending).
    Hand-built graph: 0 <- {2, 1}, 1 <- {3, 0}; seeds [0, 1], full fan-out, 1 hop.
    Visit order: (d=0: 2, 1), (d=1: 3, 0) -> F = [0, 1, 2, 3]."""
    indptr = np.array([0, 2, 4, 4, 4], np.int64)
    indices = np.array([2, 1, 3, 0], np.int32)
    b = oracle.sample_batch(indptr, indices, [0, 1], [5], seed=1)
    assert b.F.tolist() == [0, 1, 2, 3]
    assert b.bptr[0].tolist() == [0, 2, 4]
    assert b.bsrc[0].tolist() == [2, 1, 3, 0]


def test_fanout_dgl_order_and_reframpling_semantics():
    """C2/C3: hop h uses fanouts[L-1-h]; seeds are re-sampled at every hop.
    Star centred at 0 with 10 leaves, each leaf has in-edge from 0: seeds [0],
    fanouts (4, 1): hop 0 samples 1 neighbour of 0, hop 1 samples up to 4 of 0."""
    N = 11
    cols = [list(range(1, 11))] + [[0] for _ in range(10)]
    indptr = np.zeros(N + 1, np.int64)
    indptr[1:] = np.cumsum([len(c) for c in cols])
    indices = np.array(sum(cols, []), np.int32)
    b = oracle.sample_batch(indptr, indices, [0], [4, 1], seed=3)
    assert b.bptr[0].tolist() == [0, 1]           # hop 0: fan-out 1 (last entry)
    assert b.bptr[1][1] - b.bptr[1][0] == 4       # hop 1: seed 0 re-sampled with fan-out 4
    assert b.sizes[0] == 1 and b.sizes[1] == 2 and 5 <= b.sizes[2] <= 6  # 4 leaves drawn, one may be in F_1


def test_seed_errors():
    indptr = np.array([0, 1, 2], np.int64)
    indices = np.array([1, 0], np.int32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_batch(indptr, indices, [0, 0], [2], seed=1)
    assert e.value.code == oracle.EDUP
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_batch(indptr, indices, [2], [2], seed=1)
    assert e.value.code == oracle.ESEED


def test_zero_degree_seed_and_empty_batch():
    """C22 / S:136: a degree-0 seed gets no samples but is still in F and gathered."""
    indptr = np.array([0, 0, 1], np.int64)
    indices = np.array([0], np.int32)
    b = oracle.sample_batch(indptr, indices, [0], [2, 2], seed=1)
    assert b.F.tolist() == [0] and b.bptr[0].tolist() == [0, 0]
    b = oracle.sample_batch(indptr, indices, [], [2], seed=1)
    assert len(b.F) == 0 and b.sizes.tolist() == [0, 0]


def test_determinism_and_batch_composition_invariance(tiny_graph):
    """C4: the key excludes the batch index, so a node's samples at a hop depend only on
    (seed, pass, hop, node): the same node sampled in two different batches at hop 0
    gets the same neighbour multiset."""
    indptr, indices = tiny_graph
    b1 = oracle.sample_batch(indptr, indices, [5, 6, 7], [4], seed=4)
    b2 = oracle.sample_batch(indptr, indices, [7, 100], [4], seed=4)
    n1 = b1.F[b1.bsrc[0][b1.bptr[0][2]:b1.bptr[0][3]]]
    n2 = b2.F[b2.bsrc[0][b2.bptr[0][0]:b2.bptr[0][1]]]
    assert n1.tolist() == n2.tolist()


def test_gather_closed_form_features(tiny_graph):
    """O-7: X[i][d] == feat_fn(F[i], d) (closed form) and hit+miss == |F_L|."""
    indptr, indices = tiny_graph
    N = len(indptr) - 1
    feats = synth.features(N, 13).numpy()
    b = oracle.sample_gather(indptr, indices, feats, synth.inference_batches(indptr, 32)[0], (3, 3), seed=4)
    ref = synth.feat_fn(b.F[:, None], np.arange(13)[None, :])
    assert np.array_equal(b.X, ref)
    assert int(b.counters[2] + b.counters[3]) == len(b.F) and b.counters[2] == 0


def test_counters_budget_extremes(tiny_graph):
    """O-9: hits+misses == accesses; cached_len = 0 -> all misses; cached_len = deg and all
    slots valid -> all hits."""
    indptr, indices = tiny_graph
    N = len(indptr) - 1
    feats = synth.features(N, 4).numpy()
    seeds = synth.inference_batches(indptr, 50)[1]
    deg = np.diff(indptr).astype(np.int32)
    b0 = oracle.sample_gather(indptr, indices, feats, seeds, (5, 5), 4, np.zeros(N, np.int32),
                              np.full(N, -1, np.int32))
    b1 = oracle.sample_gather(indptr, indices, feats, seeds, (5, 5), 4, deg, np.arange(N, dtype=np.int32))
    assert b0.counters[0] == 0 and b0.counters[2] == 0
    assert b1.counters[1] == 0 and b1.counters[3] == 0
    assert b0.counters[1] == b1.counters[0] and b0.counters[3] == b1.counters[2] == len(b1.F)
    assert b0.F.tolist() == b1.F.tolist()  # caches never change what is sampled


def test_presample_star_example():
    """star, centre degree 5, fan-out [5], seed {centre}, one batch -> each centre
    element counted once; centre and each leaf visited once."""
    N = 6
    indptr = np.array([0, 5, 5, 5, 5, 5, 5], np.int64)
    indices = np.array([1, 2, 3, 4, 5], np.int32)
    nv, ec = oracle.presample(indptr, indices, [0], 1, [5], seed=3)
    assert ec.tolist() == [1, 1, 1, 1, 1]
    assert nv.tolist() == [1, 1, 1, 1, 1, 1]


def test_presample_ledger_identities(tiny_graph):
    """sum(edge_counts) == total samples, sum(node_visits) == sum |F_L|, and the
    counts equal a per-batch replay through sample_batch(pass=1)."""
    indptr, indices = tiny_graph
    seeds = synth.presample_seeds(indptr, 4, 40)
    fan = (4, 3)
    nv, ec = oracle.presample(indptr, indices, seeds, 40, fan, seed=3)
    samples, fl = 0, 0
    nv2 = np.zeros_like(nv)
    for b0 in range(0, len(seeds), 40):
        b = oracle.sample_batch(indptr, indices, seeds[b0:b0 + 40], fan, seed=3, pss=1)
        samples += sum(int(b.bptr[h][-1]) for h in range(2))
        fl += len(b.F)
        nv2[b.F] += 1
    assert int(ec.sum()) == samples and int(nv.sum()) == fl
    assert np.array_equal(nv, nv2)
    assert np.all(ec <= 4 * 2)  # at most once per hop per batch


def test_mean_aggregate_equals_sparse_normalised_product(tiny_graph):
    """O-13 against scipy.sparse: H = diag(1/k) . A_block . X, with A_block the sampled block
    (bptr, bsrc) as a 0/1 matrix with multiplicity; zero-degree dst rows give 0."""
    indptr, indices = tiny_graph
    N = len(indptr) - 1
    feats = synth.features(N, 11).numpy()
    seeds = np.concatenate([np.nonzero(np.diff(indptr) == 0)[0][:3], synth.inference_batches(indptr, 40)[0]])
    b = oracle.sample_gather(indptr, indices, feats, seeds.astype(np.int32), (4, 3), seed=4)
    L = 2
    bp, bs = b.bptr[L - 1], b.bsrc[L - 1]
    n_dst = len(bp) - 1
    H = oracle.mean_aggregate(bp, bs, b.X)
    A = sp.csr_matrix((np.ones(len(bs)), bs, bp.astype(np.int64)), shape=(n_dst, len(b.F)))
    k = np.diff(bp).astype(np.float64)
    ref = sp.diags(np.where(k > 0, 1.0 / np.maximum(k, 1), 0.0)) @ (A @ b.X.astype(np.float64))
    assert np.allclose(H, ref, rtol=1e-12, atol=1e-12)
    assert np.all(H[k == 0] == 0) and np.any(k == 0)
    # identical source rows -> the mean is that row
    Xc = np.tile(b.X[:1], (len(b.F), 1))
    Hc = oracle.mean_aggregate(bp, bs, Xc)
    assert np.allclose(Hc[k > 0], np.tile(b.X[:1].astype(np.float64), (int((k > 0).sum()), 1)), rtol=0, atol=0)
    # sum aggregator (Table III "sum"): A_block . X
    Hs = oracle.mean_aggregate(bp, bs, b.X, op="sum")
    assert np.allclose(Hs, A @ b.X.astype(np.float64), rtol=1e-12, atol=1e-12)
