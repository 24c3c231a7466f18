"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element, on the
same seeded inputs.  Bit-exact for every output (integers and copied fp32 rows)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2503_01281_b200 as dci  # noqa: E402

DEV = torch.device("cuda", 0)


def _graph(N, E, seed, D):
    ip, ix = synth.rmat_csc(N, E, seed=seed)
    return ip.numpy(), ix.numpy(), synth.features(N, D).numpy()


def _assert_batch_equal(g, o, L, with_x=True):
    assert g["status"] == 0
    assert np.array_equal(g["sizes"], o.sizes), (g["sizes"], o.sizes)
    assert np.array_equal(g["F"], o.F)
    for h in range(L):
        assert np.array_equal(g["bptr"][h], o.bptr[h]), h
        assert np.array_equal(g["bsrc"][h], o.bsrc[h]), h
    assert np.array_equal(g["counters"], o.counters), (g["counters"], o.counters)
    if with_x:
        assert np.array_equal(g["X"], o.X)


def _run(ctx, ws, seeds, fan, seed, **kw):
    out = dci.BatchOut(ctx, len(seeds), fan, **kw)
    dci.sample_gather(ctx, ws, torch.from_numpy(np.ascontiguousarray(seeds, np.int32)).to(DEV), fan, seed, out)
    return out.result()


@pytest.fixture(scope="module")
def small():
    ip, ix, ft = _graph(5000, 60000, 21, 13)
    ctx = dci.load_graph(ip, ix, ft)
    return ip, ix, ft, ctx


@pytest.mark.parametrize("fan", [(2, 2, 2), (15, 10, 5), (8, 4, 2), (1,), (32, 3), (5, 17, 9, 2)])
def test_nocache_sampling_parity(small, fan):
    """Before fill: original CSC, no cache (all misses), pass 0."""
    ip, ix, ft, ctx = small
    B = 100
    ws = dci.workspace_create(ctx, B, fan)
    for bi, seeds in enumerate(synth.inference_batches(ip, B)[:3]):
        g = _run(ctx, ws, seeds, fan, 4 + bi)
        o = oracle.sample_gather(ip, ix, ft, seeds, fan, 4 + bi)
        _assert_batch_equal(g, o, len(fan))


def test_ragged_empty_and_degree0(small):
    ip, ix, ft, ctx = small
    fan = (3, 3)
    ws = dci.workspace_create(ctx, 300, fan)
    zero = np.nonzero(np.diff(ip) == 0)[0].astype(np.int32)
    for seeds in [synth.inference_batches(ip, 300)[-1], np.zeros(0, np.int32),
                  np.concatenate([zero[:5], synth.inference_batches(ip, 7)[2]]).astype(np.int32)]:
        g = _run(ctx, ws, seeds, fan, 9)
        o = oracle.sample_gather(ip, ix, ft, seeds, fan, 9)
        _assert_batch_equal(g, o, 2)


def test_seed_errors_reported_in_status(small):
    ip, ix, ft, ctx = small
    fan = (2, 2)
    ws = dci.workspace_create(ctx, 8, fan)
    g = _run(ctx, ws, np.array([1, 2, 1], np.int32), fan, 1)
    assert g["status"] == dci.EDUP
    g = _run(ctx, ws, np.array([1, 5000], np.int32), fan, 1)
    assert g["status"] == dci.ESEED
    # the workspace stays clean: a valid batch afterwards still matches
    seeds = synth.inference_batches(ip, 8)[0]
    g = _run(ctx, ws, seeds, fan, 3)
    _assert_batch_equal(g, oracle.sample_gather(ip, ix, ft, seeds, fan, 3), 2)


def test_x_layouts(small):
    """ldx = D (unaligned rows, scalar copy path) and X = None (sampling only)."""
    ip, ix, ft, ctx = small
    fan = (4, 4)
    ws = dci.workspace_create(ctx, 50, fan)
    seeds = synth.inference_batches(ip, 50)[1]
    o = oracle.sample_gather(ip, ix, ft, seeds, fan, 5)
    g = _run(ctx, ws, seeds, fan, 5, ldx=13)
    _assert_batch_equal(g, o, 2)
    g = _run(ctx, ws, seeds, fan, 5, with_x=False)
    _assert_batch_equal(g, o, 2, with_x=False)


def test_presample_counts_and_times(small):
    ip, ix, ft, ctx0 = small
    ctx = dci.load_graph(ip, ix, ft)
    fan = (5, 3, 2)
    pre = synth.presample_seeds(ip, 5, 90)
    nv = torch.zeros(ctx.N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(ctx.E, dtype=torch.int32, device=DEV)
    ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(DEV), 90, fan, 3, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, 90, fan, 3)
    assert np.array_equal(nv.cpu().numpy(), nv_o)
    assert np.array_equal(ec.cpu().numpy(), ec_o)
    assert len(ts) == 5 and np.all(ts > 0) and np.all(tf > 0)
    # accumulate: a second call doubles the counts
    dci.presample(ctx, torch.from_numpy(pre).to(DEV), 90, fan, 3, nv, ec)
    assert np.array_equal(nv.cpu().numpy(), 2 * nv_o)


@pytest.mark.parametrize("r", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_m1_fill_and_cached_parity(r):
    """Config M1 (BASELINE configs[0]) at explicit split ratios: every fill branch (SURVEY
    A.6) — no adjacency cache, partial node-major prefix, whole fit, top-k tie cut."""
    cfg = synth.CONFIGS["M1"]
    ip, ix, ft = _graph(cfg.N, cfg.E, synth.GRAPH_SEED, cfg.D)
    ctx = dci.load_graph(ip, ix, ft)
    fan, B = cfg.fanouts, cfg.batch
    pre = synth.presample_seeds(ip, 8, B)
    nv = torch.zeros(ctx.N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(ctx.E, dtype=torch.int32, device=DEV)
    ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(DEV), B, fan, synth.PRESAMPLE_SEED, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, fan, synth.PRESAMPLE_SEED)
    assert np.array_equal(nv.cpu().numpy(), nv_o) and np.array_equal(ec.cpu().numpy(), ec_o)
    Cb = synth.parse_budget(cfg.budget, synth.data_bytes(cfg.N, cfg.E, cfg.D))
    num, den = int(round(r * 100)), 100
    c_adj, c_feat = dci.allocate(ctx, Cb, ts, tf, ratio=(num, den))
    assert (c_adj, c_feat) == oracle.allocate(Cb, ts, tf, ratio=(num, den))
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    st = dci.cache_state(ctx)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    pitch = cfg.pitch_floats()
    slot_o, adm = oracle.feat_fill(nv_o, c_feat // (4 * pitch))
    assert np.array_equal(st["indices_cur"], R)
    assert np.array_equal(st["cached_len"], cl)
    assert np.array_equal(st["slot_of"], slot_o)
    # cache contents: per-node prefixes (layout in id order on the GPU) and feature rows
    for v in np.nonzero(cl)[0]:
        a = st["cache_off"][v]
        assert np.array_equal(st["acache"][a:a + cl[v]], ac[co[v]:co[v] + cl[v]])
    assert st["info"]["adj_elems"] == int(cl.sum())
    assert np.array_equal(st["fcache"][:, : cfg.D], ft[adm])
    ws = dci.workspace_create(ctx, B, fan)
    for seeds in synth.inference_batches(ip, B)[:6]:
        g = _run(ctx, ws, seeds, fan, synth.SAMPLE_SEED)
        o = oracle.sample_gather(ip, R, ft, seeds, fan, synth.SAMPLE_SEED, cl, slot_o)
        _assert_batch_equal(g, o, 3)


def test_concurrent_workspaces_on_streams(small):
    """Several batches in flight on distinct streams/workspaces give the serial results."""
    ip, ix, ft, ctx = small
    fan = (10, 5)
    B = 128
    batches = synth.inference_batches(ip, B)[:6]
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(3)]
    streams = [torch.cuda.Stream() for _ in range(3)]
    outs = []
    for i, seeds in enumerate(batches):
        out = dci.BatchOut(ctx, len(seeds), fan)
        sd = torch.from_numpy(seeds).to(DEV)
        torch.cuda.synchronize()
        dci.sample_gather(ctx, wss[i % 3], sd, fan, 11, out, stream=streams[i % 3])
        outs.append(out)
    torch.cuda.synchronize()
    for seeds, out in zip(batches, outs):
        _assert_batch_equal(out.result(), oracle.sample_gather(ip, ix, ft, seeds, fan, 11), 2)


def test_host_seed_variant(small):
    ip, ix, ft, ctx = small
    fan = (6, 3)
    B = 64
    ws = dci.workspace_create(ctx, B, fan)
    seeds = synth.inference_batches(ip, B)[3]
    out = dci.BatchOut(ctx, B, fan)
    sh = torch.from_numpy(seeds).pin_memory()
    sizes = torch.zeros(3, dtype=torch.int64).pin_memory()
    cnt = torch.zeros(4, dtype=torch.int64).pin_memory()
    stt = torch.zeros(1, dtype=torch.int32).pin_memory()
    dci.sample_gather_host(ctx, ws, sh, fan, 2, out, sizes, cnt, stt)
    torch.cuda.synchronize()
    o = oracle.sample_gather(ip, ix, ft, seeds, fan, 2)
    _assert_batch_equal(out.result(), o, 2)
    assert sizes.numpy().tolist() == o.sizes.tolist()
    assert cnt.numpy().astype(np.uint64).tolist() == o.counters.tolist() and stt.item() == 0


def _agg_tol(bp, X, H_ref):
    """|g - r| <= 1e-5 |r| + k_d * 2^-23 * max|x| (fp32 sequential sum of k_d terms, then one
    division)."""
    k = np.diff(bp).astype(np.float64)[:, None]
    return 1e-5 * np.abs(H_ref) + k * 2.0 ** -23 * float(np.abs(X).max() if X.size else 0.0)


@pytest.mark.parametrize("D,ldx", [(13, None), (13, 13), (64, None), (602, None)])
def test_mean_aggregate_parity(D, ldx):
    """NEXT F2: GraphSAGE mean over the input-layer block vs the fp64 oracle (O-13)."""
    ip, ix, ft = _graph(6000, 70000, 31, D)
    ctx = dci.load_graph(ip, ix, ft)
    fan = (10, 5)
    ws = dci.workspace_create(ctx, 80, fan)
    seeds = np.concatenate([np.nonzero(np.diff(ip) == 0)[0][:4], synth.inference_batches(ip, 76)[0]]).astype(np.int32)
    out = dci.BatchOut(ctx, len(seeds), fan, ldx=ldx)
    dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, 5, out)
    H = dci.mean_aggregate(ctx, out)
    Hs = dci.mean_aggregate(ctx, out, op="sum")
    g = out.result()
    o = oracle.sample_gather(ip, ix, ft, seeds, fan, 5)
    _assert_batch_equal(g, o, 2)
    L = 2
    Hr = oracle.mean_aggregate(o.bptr[L - 1], o.bsrc[L - 1], o.X)
    Hg = H[: len(o.bptr[L - 1]) - 1, :D].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Hg - Hr) <= _agg_tol(o.bptr[L - 1], o.X, Hr))
    assert np.all(Hg[np.diff(o.bptr[L - 1]) == 0] == 0)
    Hr_s = oracle.mean_aggregate(o.bptr[L - 1], o.bsrc[L - 1], o.X, op="sum")
    Hg_s = Hs[: len(o.bptr[L - 1]) - 1, :D].cpu().numpy().astype(np.float64)
    k = np.diff(o.bptr[L - 1]).astype(np.float64)[:, None]
    assert np.all(np.abs(Hg_s - Hr_s) <= 1e-5 * np.abs(Hr_s) + k * k * 2.0 ** -24 * float(np.abs(o.X).max()))


def test_abi_error_paths(small):
    """DCI_ESTATE / DCI_ECAP / DCI_EINVAL are returned (and raised by the binding) without
    corrupting the context: a valid batch afterwards still matches the oracle."""
    ip, ix, ft, ctx0 = small
    ctx = dci.load_graph(ip, ix, ft)
    fan = (4, 4)
    ws = dci.workspace_create(ctx, 64, fan)
    seeds = synth.inference_batches(ip, 64)[0]
    sd = torch.from_numpy(seeds).to(DEV)
    # output smaller than dci_output_bounds -> ECAP
    small_out = dci.BatchOut(ctx, 8, fan)
    with pytest.raises(dci.DciError) as e:
        dci.sample_gather(ctx, ws, sd, fan, 1, small_out)
    assert e.value.code in (dci.ECAP, dci.EINVAL)
    # fan-out above the workspace's maximum / above 32 / wrong L
    out = dci.BatchOut(ctx, 64, fan)
    with pytest.raises(dci.DciError) as e:
        dci.sample_gather(ctx, ws, sd, (5, 4), 1, out)
    assert e.value.code == dci.EINVAL
    with pytest.raises(dci.DciError) as e:
        dci.workspace_create(ctx, 64, (1025,))
    assert e.value.code == dci.EINVAL
    with pytest.raises(dci.DciError) as e:
        dci.sample_gather(ctx, ws, sd, (4,), 1, out)
    assert e.value.code == dci.EINVAL
    # workspace of another context
    other = dci.load_graph(ip, ix, ft)
    with pytest.raises(dci.DciError) as e:
        dci.sample_gather(other, ws, sd, fan, 1, out)
    assert e.value.code == dci.EINVAL
    # presample after fill -> ESTATE
    nv = torch.zeros(ctx.N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(ctx.E, dtype=torch.int32, device=DEV)
    dci.fill(ctx, nv, ec, 0, 0)
    with pytest.raises(dci.DciError) as e:
        dci.presample(ctx, sd, 64, fan, 3, nv, ec)
    assert e.value.code == dci.ESTATE
    # partition arguments
    with pytest.raises(dci.DciError) as e:
        dci.fill_partitioned(ctx, nv, ec, 0, 0, 17, 0)
    assert e.value.code == dci.EINVAL
    # still consistent (fill with C = 0: reordered CSC, no caches)
    R, cl, co, ac = oracle.adj_fill(ip, ix, np.zeros(len(ix), np.int32), 0)
    g = _run(ctx, ws, seeds, fan, 2)
    _assert_batch_equal(g, oracle.sample_gather(ip, R, ft, seeds, fan, 2, cl, np.full(len(ip) - 1, -1, np.int32)), 2)


@pytest.mark.parametrize("fan", [(40,), (100, 7), (33, 64), (1024,), (2, 300)])
def test_wide_fanout_parity(fan):
    """Fan-outs 33..1024 (shared-memory Floyd + bitonic sort) on a graph with hubs of degree
    far above and nodes far below the fan-out; presample counts and a filled cache too."""
    rng = np.random.default_rng(len(fan) * 1000 + fan[-1])
    N = 3000
    deg = rng.integers(0, 20, N)
    deg[rng.choice(N, 40, replace=False)] = rng.integers(1100, 5000, 40)
    ip = np.zeros(N + 1, np.int64)
    ip[1:] = np.cumsum(deg)
    ix = rng.integers(0, N, int(ip[-1])).astype(np.int32)
    ft = synth.features(N, 12).numpy()
    ctx = dci.load_graph(ip, ix, ft)
    B = 48
    pre = rng.permutation(np.nonzero(deg)[0])[:3 * B].astype(np.int32)
    nv = torch.zeros(N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(len(ix), dtype=torch.int32, device=DEV)
    dci.presample(ctx, torch.from_numpy(pre).to(DEV), B, fan, 3, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, fan, 3)
    assert np.array_equal(nv.cpu().numpy(), nv_o) and np.array_equal(ec.cpu().numpy(), ec_o)
    c_adj, c_feat = 4 * len(ix) // 3, 64 * 4 * 300
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, _ = oracle.feat_fill(nv_o, c_feat // (4 * 12))
    ws = dci.workspace_create(ctx, B, fan)
    hubs = np.nonzero(deg > 1000)[0].astype(np.int32)
    for seeds in [hubs[:B], rng.choice(N, B, replace=False).astype(np.int32)]:
        g = _run(ctx, ws, seeds, fan, 21)
        o = oracle.sample_gather(ip, R, ft, seeds, fan, 21, cl, slot_o)
        _assert_batch_equal(g, o, len(fan))


def test_dropped_seed_tensors_on_several_streams(small):
    """Seeds uploaded per call and dropped right away while batches run on other streams: the
    binding records the stream on the tensor, so torch's allocator cannot recycle the memory
    under an unfinished batch (this raced before)."""
    ip, ix, ft, ctx = small
    fan = (10, 5)
    B = 128
    batches = synth.inference_batches(ip, B)[:12]
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(12)]
    for i, seeds in enumerate(batches):
        dci.sample_gather(ctx, wss[i % 4], torch.from_numpy(seeds).to(DEV), fan, 13, outs[i], stream=streams[i % 4])
    torch.cuda.synchronize()
    for seeds, out in zip(batches, outs):
        _assert_batch_equal(out.result(), oracle.sample_gather(ip, ix, ft, seeds, fan, 13), 2)


@pytest.mark.parametrize("case", ["L8", "N1_E0", "selfloops", "wide_rows", "wide_rows_odd"])
def test_edge_shapes(case):
    """Shapes at the ABI's limits: 8 hops, a 1-node graph without edges, self-loops only, and
    rows far wider than one warp pass (D = 1500 / 4099) through gather and aggregation."""
    rng = np.random.default_rng(3)
    if case == "L8":
        ip, ix, ft = _graph(3000, 20000, 5, 6)
        fan, seeds = (2, 2, 2, 2, 2, 2, 2, 2), synth.inference_batches(ip, 5)[0]
    elif case == "N1_E0":
        ip, ix, ft = np.array([0, 0], np.int64), np.zeros(0, np.int32), synth.features(1, 3).numpy()
        fan, seeds = (4, 4), np.array([0], np.int32)
    elif case == "selfloops":
        N = 50
        ip = np.arange(N + 1, dtype=np.int64) * 2
        ix = np.repeat(np.arange(N, dtype=np.int32), 2)
        ft, fan, seeds = synth.features(N, 7).numpy(), (3, 1), np.array([4, 9, 0], np.int32)
    else:
        D = 1500 if case == "wide_rows" else 4099
        ip, ix, ft = _graph(2000, 16000, 8, D)
        fan, seeds = (6, 3), synth.inference_batches(ip, 40)[0]
    ctx = dci.load_graph(ip, ix, ft)
    ws = dci.workspace_create(ctx, max(len(seeds), 1), fan)
    out = dci.BatchOut(ctx, len(seeds), fan)
    dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, 3, out)
    H = dci.mean_aggregate(ctx, out)
    g = out.result()
    o = oracle.sample_gather(ip, ix, ft, seeds, fan, 3)
    _assert_batch_equal(g, o, len(fan))
    L = len(fan)
    Hr = oracle.mean_aggregate(o.bptr[L - 1], o.bsrc[L - 1], o.X)
    Hg = H[: len(o.bptr[L - 1]) - 1, : ft.shape[1]].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Hg - Hr) <= _agg_tol(o.bptr[L - 1], o.X, Hr))
    # and with a fill (C = everything) on the same context
    nv = torch.zeros(len(ip) - 1, dtype=torch.int32, device=DEV)
    ec = torch.zeros(max(len(ix), 1), dtype=torch.int32, device=DEV)
    dci.presample(ctx, torch.from_numpy(seeds).to(DEV), max(len(seeds), 1), fan, 1, nv, ec)
    big = 4 * len(ix) + 4 * ((ft.shape[1] + 3) // 4 * 4) * (len(ip) - 1) + 64
    dci.fill(ctx, nv, ec, big // 2, big)
    nv_o, ec_o = oracle.presample(ip, ix, seeds, max(len(seeds), 1), fan, 1)
    R, cl, _, _ = oracle.adj_fill(ip, ix, ec_o, big // 2)
    slot_o, _ = oracle.feat_fill(nv_o, big // (4 * ((ft.shape[1] + 3) // 4 * 4)))
    out2 = dci.BatchOut(ctx, len(seeds), fan)
    dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, 3, out2)
    _assert_batch_equal(out2.result(), oracle.sample_gather(ip, R, ft, seeds, fan, 3, cl, slot_o), L)
