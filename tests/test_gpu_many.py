"""GPU parity of dci_sample_gather_many (groups of batches sampled concurrently, one TMA bulk-copy
gather launch per group) against the oracle, batch by batch, bit-exact."""
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


def _assert_batch_equal(g, o, L):
    assert g["status"] == 0
    assert np.array_equal(g["sizes"], o.sizes), (g["sizes"], o.sizes)
    assert np.array_equal(g["F"], o.F)
    for h in range(L):
        assert np.array_equal(g["bptr"][h], o.bptr[h]), h
        assert np.array_equal(g["bsrc"][h], o.bsrc[h]), h
    assert np.array_equal(g["counters"], o.counters), (g["counters"], o.counters)
    assert np.array_equal(g["X"], o.X)


def _filled(N, E, D, fan, B, ratio, budget_frac, gseed=3):
    """Graph + presample + fill at an explicit split, so both caches have hits AND misses."""
    ip, ix = synth.rmat_csc(N, E, seed=gseed)
    ip, ix = ip.numpy(), ix.numpy()
    ft = synth.features(N, D).numpy()
    ctx = dci.load_graph(ip, ix, ft)
    pre = synth.presample_seeds(ip, 4, B)
    nv = torch.zeros(N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(E, dtype=torch.int32, device=DEV)
    ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(DEV), B, fan, synth.PRESAMPLE_SEED, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, fan, synth.PRESAMPLE_SEED)
    Cb = int(budget_frac * synth.data_bytes(N, E, D))
    c_adj, c_feat = oracle.allocate(Cb, ratio=ratio)
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    R, cl, _, _ = oracle.adj_fill(ip, ix, ec_o, c_adj)
    pitch = (D + 3) // 4 * 4
    slot, _ = oracle.feat_fill(nv_o, c_feat // (4 * pitch))
    return ip, R, ft, ctx, cl, slot


@pytest.fixture(scope="module", params=[13, 100, 602])
def filled(request):
    D = request.param
    fan, B = (8, 4, 2), 128
    return (*_filled(6000, 80000, D, fan, B, (1, 2), 0.3), fan, B)


@pytest.mark.parametrize("n", [1, 2, 5, 16])
def test_many_parity(filled, n):
    ip, R, ft, ctx, cl, slot, fan, B = filled
    batches = synth.inference_batches(ip, B)
    group = [batches[i % len(batches)] for i in range(n)]
    if n >= 5:  # ragged: a short batch and an empty one inside the group
        group[1] = group[1][:17]
        group[3] = np.zeros(0, np.int32)
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(n)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
    seeds = [torch.from_numpy(np.ascontiguousarray(s, np.int32)).to(DEV) for s in group]
    dci.sample_gather_many(ctx, wss, seeds, fan, synth.SAMPLE_SEED, outs)
    hits = 0
    for s, o_gpu in zip(group, outs):
        g = o_gpu.result()
        o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(g, o, len(fan))
        hits += int(g["counters"][2])
    if n >= 5:
        assert 0 < hits  # both feature paths (HBM hit rows, host miss rows) are exercised


def test_group_call_repeated_bit_exact(filled):
    """dci.GroupCall (workspaces, outputs and fan-outs marshalled once) gives every batch the
    oracle's outputs, call after call with new seeds on a side stream, and checks its seeds."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    batches = synth.inference_batches(ip, B)
    n = 6
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(n)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
    gc = dci.GroupCall(ctx, wss, fan, outs)
    st = torch.cuda.Stream()
    for rep in range(3):
        group = [batches[(rep * n + i) % len(batches)] for i in range(n)]
        seeds = [torch.from_numpy(np.ascontiguousarray(s, np.int32)).to(DEV) for s in group]
        gc(seeds, synth.SAMPLE_SEED, stream=st)
        st.synchronize()
        for s, o_gpu in zip(group, outs):
            _assert_batch_equal(o_gpu.result(), oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot),
                                len(fan))
    # the host-seed form: pinned seeds in, results in one copy
    group = [batches[(7 + i) % len(batches)] for i in range(n)]
    hs = [torch.from_numpy(np.ascontiguousarray(s, np.int32)).pin_memory() for s in group]
    res = dci.result_buffer(n)
    gc.host(hs, synth.SAMPLE_SEED, res, stream=st)
    st.synchronize()
    parsed = dci.parse_results(res, len(fan))
    for s, o_gpu, r in zip(group, outs, parsed):
        o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(o_gpu.result(), o, len(fan))
        assert r["status"] == 0 and np.array_equal(r["sizes"], o.sizes)
    with pytest.raises(TypeError):
        gc([torch.zeros(4, dtype=torch.int64, device=DEV)] * n, synth.SAMPLE_SEED)
    with pytest.raises(ValueError):
        gc(seeds[:2], synth.SAMPLE_SEED)


@pytest.fixture(scope="module", params=[(32, 0.3), (602, 0.3), (100, 2.0)])
def dense(request):
    """A small graph where one batch touches most nodes, so groups take the node-sweep path
    (sum of |F_L| >= N): rows read once per group, written to every batch that holds them."""
    D, frac = request.param
    fan, B = (5, 4, 3), 64
    return (*_filled(1500, 40000, D, fan, B, (1, 3), frac, gseed=5), fan, B)


@pytest.mark.parametrize("n", [2, 3, 8, 9, 17, 32])
def test_many_sweep_parity(dense, n):
    ip, R, ft, ctx, cl, slot, fan, B = dense
    batches = synth.inference_batches(ip, B)
    group = [batches[i % len(batches)] for i in range(n)]
    group[-1] = group[-1][: B // 2]  # ragged
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(n)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
    for rep in range(2):  # the second group reuses the workspaces (new epochs in the tables)
        seeds = [torch.from_numpy(np.ascontiguousarray(s, np.int32)).to(DEV) for s in group]
        dci.sample_gather_many(ctx, wss, seeds, fan, synth.SAMPLE_SEED + rep, outs)
        total = 0
        for s, og in zip(group, outs):
            g = og.result()
            o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED + rep, cl, slot)
            _assert_batch_equal(g, o, len(fan))
            total += len(o.F)
        assert total >= ctx.N  # the sweep condition holds


def test_many_groups_pipelined_on_two_streams(filled):
    """Groups issued back to back on two streams, workspaces reused: every batch still exact."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    batches = synth.inference_batches(ip, B)[:12]
    G = 3
    wss = [[dci.workspace_create(ctx, B, fan) for _ in range(G)] for _ in range(2)]
    streams = [torch.cuda.Stream(device=DEV) for _ in range(2)]
    results = []
    for k in range(4):  # groups 0..3, group k on stream k % 2, reusing that stream's workspaces
        grp = batches[k * G:(k + 1) * G]
        outs = [dci.BatchOut(ctx, B, fan) for _ in range(G)]
        seeds = [torch.from_numpy(s).to(DEV) for s in grp]
        dci.sample_gather_many(ctx, wss[k % 2], seeds, fan, synth.SAMPLE_SEED, outs, stream=streams[k % 2])
        results += list(zip(grp, outs))
    torch.cuda.synchronize()
    for s, og in results:
        o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))


def test_many_unaligned_x_falls_back(filled):
    """ldx % 4 != 0 cannot take bulk stores: the group runs batch by batch, same results."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    D = ctx.D
    batches = synth.inference_batches(ip, B)[:3]
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(3)]
    ldx = D + 1 if (D + 1) % 4 else D + 2
    outs = [dci.BatchOut(ctx, B, fan, ldx=ldx) for _ in range(3)]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(s).to(DEV) for s in batches], fan, synth.SAMPLE_SEED, outs)
    for s, og in zip(batches, outs):
        o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))


def test_many_padded_ldx(filled):
    """X rows with a stride > pitch (multiple of 4): per-row bulk stores instead of one per chunk."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    pitch = (ctx.D + 3) // 4 * 4
    batches = synth.inference_batches(ip, B)[:2]
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(2)]
    outs = [dci.BatchOut(ctx, B, fan, ldx=pitch + 8) for _ in range(2)]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(s).to(DEV) for s in batches], fan, synth.SAMPLE_SEED, outs)
    for s, og in zip(batches, outs):
        o = oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))


def test_many_errors_and_status(filled):
    ip, R, ft, ctx, cl, slot, fan, B = filled
    ws = [dci.workspace_create(ctx, B, fan) for _ in range(2)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(2)]
    s = [torch.from_numpy(b).to(DEV) for b in synth.inference_batches(ip, B)[:2]]
    with pytest.raises(dci.DciError) as e:
        dci.sample_gather_many(ctx, [ws[0], ws[0]], s, fan, 1, outs)
    assert e.value.code == dci.EINVAL
    with pytest.raises(dci.DciError):
        dci.sample_gather_many(ctx, [], [], fan, 1, [])
    # a bad seed id in one batch is reported in that batch's status; the other batch is exact
    bad = torch.tensor([1, ctx.N + 5], dtype=torch.int32, device=DEV)
    dci.sample_gather_many(ctx, ws, [bad, s[1]], fan, synth.SAMPLE_SEED, outs)
    assert outs[0].result()["status"] == dci.ESEED
    o = oracle.sample_gather(ip, R, ft, synth.inference_batches(ip, B)[1], fan, synth.SAMPLE_SEED, cl, slot)
    _assert_batch_equal(outs[1].result(), o, len(fan))
    # the workspaces are clean afterwards
    dci.sample_gather_many(ctx, ws, s, fan, synth.SAMPLE_SEED, outs)
    for b, og in zip(synth.inference_batches(ip, B)[:2], outs):
        o = oracle.sample_gather(ip, R, ft, b, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))


def test_many_stats_and_profiling(filled):
    ip, R, ft, ctx, cl, slot, fan, B = filled
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(4)]
    for w in wss:
        w.set_profiling(True)
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(4)]
    batches = synth.inference_batches(ip, B)[:4]
    for _ in range(3):
        dci.sample_gather_many(ctx, wss, [torch.from_numpy(b).to(DEV) for b in batches], fan, 4, outs)
    sts = [w.stats(reset=True) for w in wss]
    assert all(st["batches"] == 3 for st in sts)
    # the group samples with one graph and gathers with one launch, both timed once and booked
    # (times, bytes, rows read) on the group's first workspace
    assert sts[0]["timed_batches"] == 3 * len(wss) and sts[0]["sample_ms"] > 0
    assert all(st["timed_batches"] == 0 for st in sts[1:])
    # (a split group gather, DCI_SPLIT_GATHER=1, is two launches)
    assert sts[0]["gather_launches"] in (3, 6) and sts[0]["gather_ms"] > 0
    assert all(st["gather_launches"] == 0 and st["gather_bytes"] == 0 for st in sts[1:])
    rows = sum(int(o.result()["sizes"][-1]) for o in outs)
    assert sum(st["frontier_rows"] for st in sts) == 3 * rows
    D, N, n = ctx.D, ctx.N, len(wss)
    read = sts[0]["rows_read"]
    kinds = sts[0]["gather_kinds"]
    nl = sts[0]["gather_launches"]
    assert sum(kinds) == nl and all(sum(st["gather_kinds"]) == 0 for st in sts[1:])
    if kinds[0] == 0:  # node sweep (register or bulk copies): each row read once per group (launch)
        assert n >= 2 and sts[0]["table_bytes"] == 8 * N  # sweeps need the dense position table
        assert read <= (nl // 3) * 3 * rows
        assert sts[0]["gather_bytes"] == nl * N * (8 * n + 4) + read * 4 * D + 3 * rows * 4 * D
    else:
        assert read == 3 * rows
        assert sts[0]["gather_bytes"] == 3 * rows * (8 * D + 4)


@pytest.mark.parametrize("ldx_pad", [0, 1])
def test_many_host_results_in_one_copy(filled, ldx_pad):
    """dci_sample_gather_many_host: host seeds in, all results back in one copy (or, on the
    batch-by-batch fallback for unaligned X, per-batch copies into the same records)."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    batches = synth.inference_batches(ip, B)[:4]
    batches[2] = batches[2][:5]
    wss = [dci.workspace_create(ctx, B, fan) for _ in batches]
    ldx = None if not ldx_pad else (ctx.D + 1 if (ctx.D + 1) % 4 else ctx.D + 2)
    outs = [dci.BatchOut(ctx, B, fan, ldx=ldx) for _ in batches]
    res = dci.result_buffer(len(batches))
    st = torch.cuda.Stream()
    dci.sample_gather_many_host(ctx, wss, [torch.from_numpy(b).pin_memory() for b in batches], fan,
                                synth.SAMPLE_SEED, outs, res, stream=st)
    st.synchronize()
    for b, og, r in zip(batches, outs, dci.parse_results(res, len(fan))):
        o = oracle.sample_gather(ip, R, ft, b, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))
        assert np.array_equal(r["sizes"], o.sizes) and np.array_equal(r["counters"], o.counters)
        assert r["status"] == 0


def test_sweep_group_with_seed_errors(dense):
    """A node-sweep group in which one batch has a bad seed and another a repeated seed: those
    batches report DCI_ESEED / DCI_EDUP, every other batch stays bit-exact, and the workspaces
    are clean for the next group (the sweep is skipped when a batch has a seed error)."""
    ip, R, ft, ctx, cl, slot, fan, B = dense
    batches = synth.inference_batches(ip, B)
    n = 6
    group = [batches[i % len(batches)].copy() for i in range(n)]
    group[1][3] = ctx.N + 7          # out of range
    group[4][5] = group[4][2]        # repeated
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(n)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(n)]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(g).to(DEV) for g in group], fan, synth.SAMPLE_SEED, outs)
    res = [o.result() for o in outs]
    assert res[1]["status"] == dci.ESEED and res[4]["status"] == dci.EDUP
    for i in (0, 2, 3, 5):
        o = oracle.sample_gather(ip, R, ft, group[i], fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(res[i], o, len(fan))
    good = [batches[(i + 7) % len(batches)] for i in range(n)]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(g).to(DEV) for g in good], fan, synth.SAMPLE_SEED, outs)
    for g_, og in zip(good, outs):
        o = oracle.sample_gather(ip, R, ft, g_, fan, synth.SAMPLE_SEED, cl, slot)
        _assert_batch_equal(og.result(), o, len(fan))


def test_group_shapes_alternate(filled):
    """A first workspace caches two group graphs: alternating group sizes (and a third shape that
    evicts one) on the same workspaces keeps every batch exact."""
    ip, R, ft, ctx, cl, slot, fan, B = filled
    batches = synth.inference_batches(ip, B)
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(5)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(5)]
    k = 0
    for n in [5, 3, 5, 3, 2, 5, 2, 3]:
        group = [batches[(k + j) % len(batches)] for j in range(n)]
        k += n
        dci.sample_gather_many(ctx, wss[:n], [torch.from_numpy(g).to(DEV) for g in group], fan, synth.SAMPLE_SEED,
                               outs[:n])
        for g_, og in zip(group, outs[:n]):
            o = oracle.sample_gather(ip, R, ft, g_, fan, synth.SAMPLE_SEED, cl, slot)
            _assert_batch_equal(og.result(), o, len(fan))
