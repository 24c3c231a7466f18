"""NEXT F1 — partitioned feature cache: bit-exact parity with the oracle's feature fill at the
combined capacity (world x per-partition rows), for partitions emulated on one device and for
a real 2-process run on one GPU that exchanges CUDA IPC handles (the multi-GPU mechanism
without the NVLink hop)."""
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

N, E, D, FAN, B = 6000, 80000, 24, (6, 4, 3), 128


def _inputs():
    ip, ix = synth.rmat_csc(N, E, seed=41)
    return ip.numpy(), ix.numpy(), synth.features(N, D).numpy()


def _check(g, o):
    assert g["status"] == 0 and np.array_equal(g["F"], o.F)
    assert np.array_equal(g["counters"], o.counters)
    assert np.array_equal(g["X"], o.X)
    for h in range(len(FAN)):
        assert np.array_equal(g["bsrc"][h], o.bsrc[h])


def _check_batches(ctx, ip, R, ft, cl, slot_o, dev, nb=4):
    ws = dci.workspace_create(ctx, B, FAN)
    batches = synth.inference_batches(ip, B)
    for seeds in batches[:nb]:
        out = dci.BatchOut(ctx, B, FAN)
        dci.sample_gather(ctx, ws, torch.from_numpy(seeds).to(dev), FAN, 9, out)
        _check(out.result(), oracle.sample_gather(ip, R, ft, seeds, FAN, 9, cl, slot_o))
    # groups (one TMA gather launch reading local and peer partitions): 3 batches (row mode) and
    # 8 batches (node sweep: together they hold more rows than N)
    for n in (3, 8):
        grp = [batches[i % len(batches)] for i in range(n)]
        wss = [dci.workspace_create(ctx, B, FAN) for _ in grp]
        outs = [dci.BatchOut(ctx, B, FAN) for _ in grp]
        dci.sample_gather_many(ctx, wss, [torch.from_numpy(s).to(dev) for s in grp], FAN, 9, outs)
        for s, og in zip(grp, outs):
            _check(og.result(), oracle.sample_gather(ip, R, ft, s, FAN, 9, cl, slot_o))


@pytest.mark.parametrize("world", [2, 3, 5])
def test_emulated_partitions(world):
    dev = torch.device("cuda", 0)
    ip, ix, ft = _inputs()
    ctx = dci.load_graph(ip, ix, ft)
    pre = synth.presample_seeds(ip, 6, B)
    nv = torch.zeros(N, dtype=torch.int32, device=dev)
    ec = torch.zeros(E, dtype=torch.int32, device=dev)
    dci.presample(ctx, torch.from_numpy(pre).to(dev), B, FAN, 3, nv, ec)
    nv_o, ec_o = oracle.presample(ip, ix, pre, B, FAN, 3)
    pitch = (D + 3) // 4 * 4
    cap_part = 300
    c_feat, c_adj = cap_part * 4 * pitch, 90_000
    dci.fill_partitioned(ctx, nv, ec, c_adj, c_feat, world, -1)
    st = dci.cache_state(ctx)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
    slot_o, adm = oracle.feat_fill(nv_o, world * cap_part)
    assert np.array_equal(st["slot_of"], slot_o)
    assert st["info"]["feat_partitions"] == world and st["info"]["feat_rows_total"] == len(adm)
    # partition p holds global slots p, p + world, ... in order
    rows = [adm[p::world] for p in range(world)]
    assert np.array_equal(st["fcache"][:, :D], ft[np.concatenate(rows)])
    _check_batches(ctx, ip, R, ft, cl, slot_o, dev)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        import paper_2503_01281_b200 as dci_w
        from paper_2503_01281_b200 import parallel
        parallel.init("gloo")
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(0)
        ip, ix, ft = _inputs()
        ctx = dci_w.load_graph(ip, ix, ft)
        pre = synth.presample_seeds(ip, 6, B)
        batches = [pre[i * B:(i + 1) * B] for i in range(6)]
        nv = torch.zeros(N, dtype=torch.int32, device=dev)
        ec = torch.zeros(E, dtype=torch.int32, device=dev)
        ts, tf = [], []
        for b in parallel.shard(batches, rank, world):
            a, c = dci_w.presample(ctx, torch.from_numpy(b).to(dev), B, FAN, 3, nv, ec)
            ts += a.tolist()
            tf += c.tolist()
        parallel.allreduce_presample(nv, ec, ts, tf)
        pitch = (D + 3) // 4 * 4
        cap_part, c_adj = 300, 90_000
        dci_w.fill_partitioned(ctx, nv, ec, c_adj, cap_part * 4 * pitch, world, rank)
        torch.cuda.synchronize()
        parallel.barrier()
        parallel.exchange_feature_partitions(ctx)
        parallel.barrier()
        nv_o, ec_o = oracle.presample(ip, ix, pre, B, FAN, 3)
        R, cl, co, ac = oracle.adj_fill(ip, ix, ec_o, c_adj)
        slot_o, adm = oracle.feat_fill(nv_o, world * cap_part)
        info = dci_w.cache_info(ctx)
        st = dci_w.cache_state(ctx)
        ok = bool(np.array_equal(st["slot_of"], slot_o)) and info["feat_rows"] == len(adm[rank::world])
        ok &= bool(np.array_equal(st["fcache"][:, :D], ft[adm[rank::world]]))
        _check_batches(ctx, ip, R, ft, cl, slot_o, dev)
        parallel.barrier()
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))
        raise


def test_two_process_ipc_partitions_on_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, True), (1, True)], res
