"""DCI_ADOPT_HOST (dci.h, dci_load_graph): the caller's host buffers registered in place instead of
copied -- the mechanism that lets the ranks of one node share ONE host-resident graph
(papers100M-shaped data stays in host memory).  Parity: every output bit-exact
against the oracle, single process and two processes adopting one node-shared shm segment
(parallel.SharedGraph) on one GPU, with a budget that leaves both caches with misses so the UVA
paths read the adopted memory."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2503_01281_b200 as dci  # noqa: E402

N, E, D, FAN, B = 5000, 60000, 13, (5, 3, 2), 96  # D = 13: pitch 16 != D (padded adopted rows)


def _graph():
    ip, ix = synth.rmat_csc(N, E, seed=17)
    return ip.numpy(), ix.numpy(), synth.features(N, D).numpy()


def _padded(ft):
    pitch = (D + 3) // 4 * 4
    out = np.zeros((N, pitch), np.float32)
    out[:, :D] = ft
    return out


def _run_and_check(ctx, ip, ix, ft, dev):
    """presample -> fill at a budget with misses on both sides -> single calls and a group, each
    bit-exact against the oracle; the adopted buffers are unchanged afterwards."""
    pre = synth.presample_seeds(ip, 4, B)
    nv = torch.zeros(N, dtype=torch.int32, device=dev)
    ec = torch.zeros(E, dtype=torch.int32, device=dev)
    dci.presample(ctx, torch.from_numpy(pre).to(dev), B, FAN, synth.PRESAMPLE_SEED, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, FAN, synth.PRESAMPLE_SEED)
    pitch = (D + 3) // 4 * 4
    c_adj, c_feat = 4 * E // 3, 4 * pitch * (N // 4)
    dci.fill(ctx, nv, ec, c_adj, c_feat)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot, _ = oracle.feat_fill(nv_o, c_feat // (4 * pitch))
    batches = synth.inference_batches(ip, B)
    ws = dci.workspace_create(ctx, B, FAN)
    ok = True
    for s in batches[:3]:
        out = dci.BatchOut(ctx, B, FAN)
        dci.sample_gather(ctx, ws, torch.from_numpy(s).to(dev), FAN, synth.SAMPLE_SEED, out)
        g, o = out.result(), oracle.sample_gather(ip, R, ft, s, FAN, synth.SAMPLE_SEED, cl, slot)
        ok &= g["status"] == 0 and np.array_equal(g["F"], o.F) and np.array_equal(g["X"], o.X)
        ok &= np.array_equal(g["counters"], o.counters) and all(
            np.array_equal(g["bsrc"][h], o.bsrc[h]) for h in range(len(FAN)))
        ok &= g["counters"][1] > 0 and g["counters"][3] > 0  # both miss paths read adopted memory
    grp = batches[3:9]
    wss = [dci.workspace_create(ctx, B, FAN) for _ in grp]
    outs = [dci.BatchOut(ctx, B, FAN) for _ in grp]
    dci.sample_gather_many(ctx, wss, [torch.from_numpy(s).to(dev) for s in grp], FAN, synth.SAMPLE_SEED, outs)
    for s, og in zip(grp, outs):
        g, o = og.result(), oracle.sample_gather(ip, R, ft, s, FAN, synth.SAMPLE_SEED, cl, slot)
        ok &= np.array_equal(g["F"], o.F) and np.array_equal(g["X"], o.X) and np.array_equal(g["counters"], o.counters)
    return bool(ok)


def test_adopt_single_process_bit_exact_and_untouched():
    dev = torch.device("cuda", 0)
    ip, ix, ft = _graph()
    ix_adopt, ft_adopt = ix.copy(), _padded(ft)
    ctx = dci.load_graph(ip, ix_adopt, ft_adopt, adopt=True, D=D)
    assert _run_and_check(ctx, ip, ix, ft, dev)
    # the library never writes adopted memory (the level-2 reorder lives in its own buffer)
    assert np.array_equal(ix_adopt, ix) and np.array_equal(ft_adopt[:, :D], ft) and not ft_adopt[:, D:].any()
    ctx.close()


def test_adopt_rejects_unpadded_features():
    ip, ix, ft = _graph()
    with pytest.raises(ValueError):
        dci.load_graph(ip, ix, ft, adopt=True)  # [N, 13] is not [N, pitch 16]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shared_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        from paper_2503_01281_b200 import parallel
        parallel.init("gloo")
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        sg = parallel.SharedGraph(N, E, D, _graph, tag=f"adopt{port}")
        ctx = sg.load(0)
        ip, ix, ft = _graph()
        ok = _run_and_check(ctx, ip, ix, ft, dev)
        parallel.barrier()
        q.put((rank, ok, sg.names[2]))
        ctx.close()
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), ""))
        raise


def test_two_processes_adopt_one_shared_graph():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert [r[:2] for r in res] == [(0, True), (1, True)], res
    assert res[0][2] == res[1][2]
