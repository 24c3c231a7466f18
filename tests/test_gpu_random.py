"""Randomised GPU parity: many small random configurations (graph shape, hubs, fan-outs 1..32,
1..4 hops, ragged batch sizes, budgets and explicit splits, presample sizes), each compared bit
for bit against the oracle — presample counts, fill (cache state), and several batches."""
import numpy as np
import pytest

import oracle
import synth
from tests._util import random_csc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2503_01281_b200 as dci  # noqa: E402

DEV = torch.device("cuda", 0)


def _graph(rng, kind):
    if kind == "rmat":
        N = int(rng.integers(50, 4000))
        E = 2 * int(rng.integers(N // 2, 12 * N))
        ip, ix = synth.rmat_csc(N, E, seed=int(rng.integers(1, 1 << 30)))
        return ip.numpy(), ix.numpy()
    if kind == "hub":  # a few very high in-degree nodes (Floyd path with deg >> f)
        N = int(rng.integers(100, 2000))
        deg = rng.integers(0, 6, N)
        deg[rng.choice(N, 3, replace=False)] = rng.integers(500, 3000, 3)
        ip = np.zeros(N + 1, np.int64)
        ip[1:] = np.cumsum(deg)
        ix = rng.integers(0, N, int(ip[-1])).astype(np.int32)
        return ip, ix
    N = int(rng.integers(5, 300))
    return random_csc(rng, N, int(rng.integers(1, 40)))


@pytest.mark.parametrize("trial", range(24))
def test_random_configuration(trial):
    rng = np.random.default_rng(1000 + trial)
    ip, ix = _graph(rng, ["rmat", "hub", "uniform"][trial % 3])
    N, E = len(ip) - 1, len(ix)
    D = int(rng.choice([1, 3, 4, 8, 33, 100]))
    ft = synth.features(N, D).numpy()
    L = int(rng.integers(1, 5))
    fan = tuple(int(x) for x in rng.integers(1, 33, L))
    B = int(rng.integers(1, min(N, 300) + 1))
    ctx = dci.load_graph(ip, ix, ft)
    # presample (random number of batches, ragged last batch)
    el = synth.eligible_nodes(ip)
    if len(el) == 0:
        pytest.skip("graph without edges")
    npre = int(rng.integers(1, min(len(el), 4 * B) + 1))
    pre = rng.permutation(el)[:npre].astype(np.int32)
    pb = int(rng.integers(1, B + 1))
    nv = torch.zeros(N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(max(E, 1), dtype=torch.int32, device=DEV)
    ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(DEV), pb, fan, 77, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, pb, fan, 77)
    assert np.array_equal(nv.cpu().numpy(), nv_o)
    assert np.array_equal(ec.cpu().numpy()[:E], ec_o)
    # random budget and split
    C = int(rng.integers(0, 2 * synth.data_bytes(N, E, D) + 64)) + 1
    r = int(rng.integers(0, 101))
    c_adj, c_feat = dci.allocate(ctx, C, ts, tf, ratio=(r, 100))
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    st = dci.cache_state(ctx)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, adm = oracle.feat_fill(nv_o, c_feat // (4 * ((D + 3) // 4 * 4)))
    assert np.array_equal(st["indices_cur"], R)
    assert np.array_equal(st["cached_len"], cl)
    assert np.array_equal(st["slot_of"], slot_o)
    for v in np.nonzero(cl)[0]:
        a = st["cache_off"][v]
        assert np.array_equal(st["acache"][a:a + cl[v]], ac[co[v]:co[v] + cl[v]])
    if len(adm):
        assert np.array_equal(st["fcache"][:, :D], ft[adm])
    ws = dci.workspace_create(ctx, B, fan)
    seed = int(rng.integers(0, 1 << 62))
    for _ in range(3):
        b = int(rng.integers(0, B + 1))
        seeds = rng.choice(N, size=min(b, N), replace=False).astype(np.int32)
        out = dci.BatchOut(ctx, len(seeds), fan)
        dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, seed, out)
        g = out.result()
        o = oracle.sample_gather(ip, R, ft, seeds, fan, seed, cl, slot_o)
        assert g["status"] == 0
        assert np.array_equal(g["F"], o.F)
        assert np.array_equal(g["sizes"], o.sizes)
        for h in range(L):
            assert np.array_equal(g["bptr"][h], o.bptr[h])
            assert np.array_equal(g["bsrc"][h], o.bsrc[h])
        assert np.array_equal(g["counters"], o.counters)
        assert np.array_equal(g["X"], o.X)


@pytest.mark.parametrize("trial", range(16))
def test_knapsack_fill_parity(trial):
    """NEXT F4: the GPU knapsack (histogram-level walk + scans) equals the oracle's full-sort
    greedy (O-14) for random budgets / cost ratios, and batches sampled on it match."""
    rng = np.random.default_rng(5000 + trial)
    ip, ix = _graph(rng, ["rmat", "hub", "uniform"][trial % 3])
    N, E = len(ip) - 1, len(ix)
    D = int(rng.choice([4, 30, 64]))
    ft = synth.features(N, D).numpy()
    fan = tuple(int(x) for x in rng.integers(1, 16, int(rng.integers(1, 4))))
    ctx = dci.load_graph(ip, ix, ft)
    el = synth.eligible_nodes(ip)
    if len(el) == 0:
        pytest.skip("graph without edges")
    B = int(rng.integers(1, min(len(el), 200) + 1))
    pre = rng.permutation(el)[: 3 * B].astype(np.int32)
    nv = torch.zeros(N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(max(E, 1), dtype=torch.int32, device=DEV)
    dci.presample(ctx, torch.from_numpy(pre).to(DEV), B, fan, 5, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, fan, 5)
    R = 4 * ((D + 3) // 4 * 4)
    Cb = int(rng.integers(0, N * R + 4 * E + 64))
    cf, ca = float(rng.choice([0.5, 1.0, 7.3, 40.0])), float(rng.choice([0.2, 1.0, 3.0]))
    dci.fill_knapsack(ctx, nv, ec, Cb, cf, ca)
    slot_o, cl_o, used = oracle.knapsack_fill(ip, nv_o, ec_o, Cb, R, cf, ca)
    st = dci.cache_state(ctx)
    R_idx, _, _, _ = oracle.adj_fill(ip, ix, ec_o, 0)  # level-2 order (the knapsack keeps it)
    assert np.array_equal(st["indices_cur"], R_idx)
    assert np.array_equal(st["slot_of"], slot_o)
    assert np.array_equal(st["cached_len"], cl_o)
    assert st["info"]["adj_elems"] * 4 + st["info"]["feat_rows"] * R == used
    for v in np.nonzero(cl_o)[0]:
        a = st["cache_off"][v]
        assert np.array_equal(st["acache"][a:a + cl_o[v]], R_idx[ip[v]:ip[v] + cl_o[v]])
    ws = dci.workspace_create(ctx, B, fan)
    seeds = rng.choice(N, size=min(B, N), replace=False).astype(np.int32)
    out = dci.BatchOut(ctx, len(seeds), fan)
    dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, 17, out)
    g = out.result()
    o = oracle.sample_gather(ip, R_idx, ft, seeds, fan, 17, cl_o, slot_o)
    assert np.array_equal(g["F"], o.F) and np.array_equal(g["counters"], o.counters)
    assert np.array_equal(g["X"], o.X)
    # the same caches through a group call
    grp = [rng.choice(N, size=min(B, N), replace=False).astype(np.int32) for _ in range(4)]
    wss = [dci.workspace_create(ctx, B, fan) for _ in grp]
    outs = [dci.BatchOut(ctx, B, fan) for _ in grp]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(x).to(DEV) for x in grp], fan, 17, outs)
    for x, og in zip(grp, outs):
        g = og.result()
        o = oracle.sample_gather(ip, R_idx, ft, x, fan, 17, cl_o, slot_o)
        assert np.array_equal(g["F"], o.F) and np.array_equal(g["counters"], o.counters)
        assert np.array_equal(g["X"], o.X)


@pytest.mark.parametrize("trial", range(40))
def test_random_group_configuration(trial):
    """dci_sample_gather_many on random graphs / fan-outs (1..40: frontier-order and node-sweep
    sampling, G < 4 and G >= 4 lane groups, the wide kernel above 32) / group sizes 1..32 /
    budgets: every batch bit-exact against the oracle; groups issued twice on two streams."""
    rng = np.random.default_rng(9000 + trial)
    ip, ix = _graph(rng, ["rmat", "hub", "uniform"][trial % 3])
    N, E = len(ip) - 1, len(ix)
    D = int(rng.choice([1, 4, 13, 64, 100]))
    ft = synth.features(N, D).numpy()
    L = int(rng.integers(1, 4))
    fan = tuple(int(x) for x in rng.integers(1, 41 if trial % 5 == 0 else 17, L))
    B = int(rng.integers(1, min(N, 128) + 1))
    ctx = dci.load_graph(ip, ix, ft)
    el = synth.eligible_nodes(ip)
    if len(el) == 0:
        pytest.skip("graph without edges")
    pre = rng.permutation(el)[: min(len(el), 2 * B)].astype(np.int32)
    nv = torch.zeros(N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(max(E, 1), dtype=torch.int32, device=DEV)
    dci.presample(ctx, torch.from_numpy(pre).to(DEV), B, fan, 3, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, fan, 3)
    C = int(rng.integers(0, 2 * synth.data_bytes(N, E, D) + 64)) + 1
    r = int(rng.integers(0, 101))
    c_adj, c_feat = oracle.allocate(C, ratio=(r, 100))
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    R, cl, _, _ = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, _ = oracle.feat_fill(nv_o, c_feat // (4 * ((D + 3) // 4 * 4)))
    n = int(rng.integers(1, 33))
    streams = [torch.cuda.Stream(device=DEV) for _ in range(2)]
    wss = [[dci.workspace_create(ctx, B, fan) for _ in range(n)] for _ in range(2)]
    seed = int(rng.integers(0, 1 << 62))
    expect = []
    keep = []
    for k in range(4):  # groups 0..3 on alternating streams, workspaces reused
        group = []
        for _ in range(n):
            b = int(rng.integers(0, B + 1))
            group.append(rng.choice(N, size=min(b, N), replace=False).astype(np.int32))
        outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
        sd = [torch.from_numpy(g).to(DEV) for g in group]
        keep.append(sd)
        dci.sample_gather_many(ctx, wss[k % 2], sd, fan, seed, outs, stream=streams[k % 2])
        expect += list(zip(group, outs))
    torch.cuda.synchronize()
    for seeds, og in expect:
        g = og.result()
        o = oracle.sample_gather(ip, R, ft, seeds, fan, seed, cl, slot_o)
        assert g["status"] == 0
        assert np.array_equal(g["F"], o.F)
        assert np.array_equal(g["sizes"], o.sizes)
        for h in range(L):
            assert np.array_equal(g["bptr"][h], o.bptr[h])
            assert np.array_equal(g["bsrc"][h], o.bsrc[h])
        assert np.array_equal(g["counters"], o.counters)
        assert np.array_equal(g["X"], o.X)
