"""GPU parity at BASELINE.json's full sizes (M2 Reddit-shaped, M3 products-shaped) in the
bench's launch configuration (several workspaces / streams in flight, CUDA graphs), plus the
workspace statistics and the graph re-capture logic."""
import os
import subprocess
import sys

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
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _same(g, o, L):
    return (g["status"] == 0 and np.array_equal(g["F"], o.F) and np.array_equal(g["counters"], o.counters)
            and all(np.array_equal(g["bptr"][h], o.bptr[h]) and np.array_equal(g["bsrc"][h], o.bsrc[h])
                    for h in range(L)) and np.array_equal(g["X"], o.X))


def _setup(cfg, ratio=None):
    ip, ix = synth.rmat_csc(cfg.N, cfg.E, device=DEV)
    ip, ix = ip.cpu().numpy(), ix.cpu().numpy()
    ft = synth.features(cfg.N, cfg.D, device=DEV).cpu().numpy()
    ctx = dci.load_graph(ip, ix, ft)
    pre = synth.presample_seeds(ip, 8, cfg.batch)
    nv = torch.zeros(cfg.N, dtype=torch.int32, device=DEV)
    ec = torch.zeros(cfg.E, dtype=torch.int32, device=DEV)
    ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(DEV), cfg.batch, cfg.fanouts, synth.PRESAMPLE_SEED, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, cfg.batch, cfg.fanouts, synth.PRESAMPLE_SEED)
    assert np.array_equal(nv.cpu().numpy(), nv_o) and np.array_equal(ec.cpu().numpy(), ec_o)
    return ip, ix, ft, ctx, nv, ec, nv_o, ec_o, ts, tf


def _check_fill_and_batches(cfg, ip, ix, ft, ctx, nv, ec, nv_o, ec_o, c_adj, c_feat, nbatches=3, inflight=3,
                            group=0):
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    st = dci.cache_state(ctx)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, adm = oracle.feat_fill(nv_o, c_feat // (4 * cfg.pitch_floats()))
    assert np.array_equal(st["indices_cur"], R)
    assert np.array_equal(st["cached_len"], cl)
    assert np.array_equal(st["slot_of"], slot_o)
    # sampled cache-content checks (every cached node would be slow at this size)
    rng = np.random.default_rng(0)
    cached = np.nonzero(cl)[0]
    for v in rng.choice(cached, size=min(2000, len(cached)), replace=False) if len(cached) else []:
        a = st["cache_off"][v]
        assert np.array_equal(st["acache"][a:a + cl[v]], R[ip[v]:ip[v] + cl[v]])
    for j in rng.choice(len(adm), size=min(2000, len(adm)), replace=False) if len(adm) else []:
        assert np.array_equal(st["fcache"][j, : cfg.D], ft[adm[j]])
    del st
    fan, B = cfg.fanouts, cfg.batch
    wss = [dci.workspace_create(ctx, B, fan) for _ in range(inflight)]
    streams = [torch.cuda.Stream() for _ in range(inflight)]
    outs = [dci.BatchOut(ctx, B, fan) for _ in range(inflight)]
    batches = synth.inference_batches(ip, B)[:nbatches]
    seeds_dev = [torch.from_numpy(b).to(DEV) for b in batches]  # alive while batches are in flight
    results = []
    for i, seeds in enumerate(batches):
        w = i % inflight
        if i >= inflight:
            results.append(outs[w].result())
        dci.sample_gather(ctx, wss[w], seeds_dev[i], fan, synth.SAMPLE_SEED, outs[w], stream=streams[w])
    torch.cuda.synchronize()
    for i in range(max(0, len(batches) - inflight), len(batches)):
        results.append(outs[i % inflight].result())
    for seeds, g in zip(batches, results):
        o = oracle.sample_gather(ip, R, ft, seeds, fan, synth.SAMPLE_SEED, cl, slot_o)
        assert _same(g, o, len(fan))
    if group:
        # the bench's default call on HBM-resident data: groups of `group` batches, 2 groups in
        # flight on 2 streams, one TMA gather launch per group (node sweep when sum |F_L| >= N)
        batches = synth.inference_batches(ip, B)[nbatches:nbatches + 2 * group]
        gw = [[dci.workspace_create(ctx, B, fan) for _ in range(group)] for _ in range(2)]
        go = [[dci.BatchOut(ctx, B, fan) for _ in range(group)] for _ in range(2)]
        gs = [torch.cuda.Stream() for _ in range(2)]
        sd = [torch.from_numpy(b).to(DEV) for b in batches]
        for k in range(2):
            dci.sample_gather_many(ctx, gw[k], sd[k * group:(k + 1) * group], fan, synth.SAMPLE_SEED, go[k],
                                   stream=gs[k])
        torch.cuda.synchronize()
        for i, seeds in enumerate(batches):
            o = oracle.sample_gather(ip, R, ft, seeds, fan, synth.SAMPLE_SEED, cl, slot_o)
            assert _same(go[i // group][i % group].result(), o, len(fan)), i


def test_m2_reddit_fullsize_auto_budget():
    """configs[1]: 232,965 nodes, 114.6 M edges, D 602, 15,10,5, B 1024, auto budget."""
    cfg = synth.CONFIGS["M2"]
    ip, ix, ft, ctx, nv, ec, nv_o, ec_o, ts, tf = _setup(cfg)
    c_adj, c_feat = dci.allocate(ctx, 0, ts, tf)
    assert c_adj + c_feat > 0
    _check_fill_and_batches(cfg, ip, ix, ft, ctx, nv, ec, nv_o, ec_o, c_adj, c_feat, nbatches=4, group=6)


@pytest.mark.parametrize("r", [None, 0.0, 0.5])
def test_m3_products_fullsize_quarter_budget(r):
    """configs[2]/[4]: 2.45 M nodes, 61.9 M edges, D 100, 8,4,2, budget 25 % of data; Eq. 1
    split (r=None) and explicit splits of the M5 sweep."""
    cfg = synth.CONFIGS["M3"]
    ip, ix, ft, ctx, nv, ec, nv_o, ec_o, ts, tf = _setup(cfg)
    C = synth.parse_budget(cfg.budget, synth.data_bytes(cfg.N, cfg.E, cfg.D))
    ratio = None if r is None else (int(r * 100), 100)
    c_adj, c_feat = dci.allocate(ctx, C, ts, tf, ratio=ratio)
    assert (c_adj, c_feat) == oracle.allocate(C, ts, tf, ratio=ratio)
    _check_fill_and_batches(cfg, ip, ix, ft, ctx, nv, ec, nv_o, ec_o, c_adj, c_feat, nbatches=4,
                            group=3 if r == 0.5 else 0)


def test_workspace_stats_and_graph_recapture():
    """Running totals match the per-batch outputs; a workspace reused with a different output
    struct / fan-out / profiling flag re-captures its CUDA graph and stays bit-exact."""
    ip, ix = synth.rmat_csc(4000, 40000, seed=3)
    ip, ix = ip.numpy(), ix.numpy()
    ft = synth.features(4000, 8).numpy()
    ctx = dci.load_graph(ip, ix, ft)
    ws = dci.workspace_create(ctx, 64, (8, 8))
    ws.stats(reset=True)
    tot_rows, tot_cnt, nb = 0, np.zeros(4, np.uint64), 0
    for i, (fan, prof) in enumerate([((4, 4), False), ((4, 4), False), ((8, 2), True), ((4, 4), True),
                                     ((8, 8), False), ((8, 8), False)]):
        ws.set_profiling(prof)
        out = dci.BatchOut(ctx, 64, fan)
        seeds = synth.inference_batches(ip, 64)[i]
        dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(DEV), fan, 7, out)
        g = out.result()
        o = oracle.sample_gather(ip, ix, ft, seeds, fan, 7)
        assert _same(g, o, 2)
        tot_rows += len(o.F)
        tot_cnt += o.counters
        nb += 1
    st = ws.stats(reset=True)
    assert st["batches"] == nb and st["seeds"] == 64 * nb and st["frontier_rows"] == tot_rows
    assert st["counters"] == tot_cnt.tolist()
    assert st["timed_batches"] == 2 and st["gather_ms"] > 0 and st["sample_ms"] > 0
    assert ws.stats()["batches"] == 0


@pytest.mark.parametrize("env", [{"DCI_GATHER": "tma"}, {"DCI_SWEEP": "0"}, {"DCI_GATHER_SERIAL": "0"},
                                 {"DCI_TMA_WARPS": "2", "DCI_TMA_CHUNK": "2048"}, {"DCI_PHASED": "1"},
                                 {"DCI_SAMPLE_SWEEP": "0"}, {"DCI_PRECHECK": "1"}, {"DCI_SAMPLE_BPS": "1"},
                                 {"DCI_TMA_SMS": "37"}, {"DCI_PHASED": "2"}, {"DCI_PHASED": "2", "DCI_GRAPH": "0"},
                                 {"DCI_TABLE": "hash"}, {"DCI_TABLE": "hash", "DCI_GRAPH": "0"},
                                 {"DCI_SWEEP_KIND": "tma"}, {"DCI_SWEEP_KIND": "tma", "DCI_SWEEP_WARPS": "2"},
                                 {"DCI_SWEEP_BPS": "1", "DCI_SWEEP_SMS": "20"}, {"DCI_SPLIT_GATHER": "0"},
                                 {"DCI_SPLIT_GATHER": "1", "DCI_GRAPH": "0"}, {"DCI_SPLIT_GATHER": "1", "DCI_PHASED": "2"},
                                 {"DCI_SPLIT_GATHER": "1", "DCI_SWEEP_KIND": "ldg"}, {"DCI_NMASK_SWEEP": "0"},
                                 {"DCI_ELEM_POLICY": "0", "DCI_DIR_POLICY": "0"},
                                 {"DCI_ELEM_POLICY": "2", "DCI_DIR_POLICY": "2"}])
def test_gather_variants_subprocess(env):
    """Process-wide switches (read once per process): the TMA gather for single-batch
    calls, row mode for groups, group gathers on the caller's stream, a small TMA ring, phased
    (not overlapped) groups, frontier-order sampling only, the tag pre-read before atomicMax, one
    sampling block per SM, a gather grid on a quarter of the SMs, the split schedule (graphs and
    direct launches), hashed position tables, the bulk-copy node sweep, a small sweep grid, and the
    split group gather (off; without graphs; with the split schedule; register-copy sweeps), and the
    scan's per-candidate tag reads instead of the node-major new-candidate masks."""
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT,
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "smoke ok" in r.stdout


def test_no_graph_path_subprocess():
    """The direct-launch path (DCI_GRAPH=0) passes the same smoke check."""
    env = dict(os.environ, DCI_GRAPH="0")
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "smoke ok" in r.stdout


def test_m2_fullsize_bench_launch_configuration():
    """configs[1] in exactly the launch configuration bench.py times: groups of 20 batches, two
    groups in flight on two streams, X rows padded to whole 128-byte lines (ldx 608), auto budget;
    EVERY batch of both groups bit-exact against the oracle (the bench's parity_check samples 3)."""
    from concurrent.futures import ThreadPoolExecutor
    cfg = synth.CONFIGS["M2"]
    ip, ix, ft, ctx, nv, ec, nv_o, ec_o, ts, tf = _setup(cfg)
    c_adj, c_feat = dci.allocate(ctx, 0, ts, tf)
    fan, B, G = cfg.fanouts, cfg.batch, 20
    ldx = -(-cfg.D // 32) * 32
    gw = [[dci.workspace_create(ctx, B, fan) for _ in range(G)] for _ in range(2)]
    go = [[dci.BatchOut(ctx, B, fan, ldx=ldx) for _ in range(G)] for _ in range(2)]
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    R, cl, _, _ = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, _ = oracle.feat_fill(nv_o, c_feat // (4 * cfg.pitch_floats()))
    batches = synth.inference_batches(ip, B)[: 2 * G]
    sd = [torch.from_numpy(b).to(DEV) for b in batches]
    gs = [torch.cuda.Stream() for _ in range(2)]
    for rep in range(2):  # the second round reuses the workspaces (epochs, cached graphs)
        for k in range(2):
            dci.sample_gather_many(ctx, gw[k], sd[k * G:(k + 1) * G], fan, synth.SAMPLE_SEED, go[k], stream=gs[k])
    torch.cuda.synchronize()
    assert go[0][0].ldx == ldx
    got = [go[i // G][i % G].result() for i in range(2 * G)]

    def check(i):
        o = oracle.sample_gather(ip, R, ft, batches[i], fan, synth.SAMPLE_SEED, cl, slot_o)
        return _same(got[i], o, len(fan))

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        ok = list(ex.map(check, range(2 * G)))
    assert all(ok), [i for i, v in enumerate(ok) if not v]
