"""Multi-process host logic on CPU (gloo, world size 2): batch sharding, the presample-count
allreduce (C1) and max/sum over ranks.  The per-rank counting is done by the oracle here (the
CUDA path does it on GPUs); what is tested is that sharding + allreduce reproduce the
single-process presample exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_01281_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        import oracle
        import synth
        r, w, _ = parallel.init("gloo")
        assert (r, w) == (rank, world)
        ip, ix = synth.rmat_csc(1500, 16000, seed=5)
        ip, ix = ip.numpy(), ix.numpy()
        B, fan = 40, (4, 3)
        pre = synth.presample_seeds(ip, 6, B)
        batches = [pre[i * B:(i + 1) * B] for i in range(6)]
        mine = parallel.shard(batches, rank, world)
        nv = np.zeros(len(ip) - 1, np.int32)
        ec = np.zeros(len(ix), np.int32)
        ts, tf = [], []
        for b in mine:
            oracle.presample(ip, ix, b, B, fan, 3, nv, ec)
            ts.append(1000 + rank)
            tf.append(3000 + rank)
        nv_t, ec_t = torch.from_numpy(nv), torch.from_numpy(ec)
        S, F = parallel.allreduce_presample(nv_t, ec_t, ts, tf)
        mx = parallel.max_over_ranks(float(rank + 1))
        sm = parallel.sum_over_ranks([1.0, rank])
        ok = True
        if rank == 0:
            nv1, ec1 = oracle.presample(ip, ix, pre, B, fan, 3)
            ok = bool(np.array_equal(nv_t.numpy(), nv1) and np.array_equal(ec_t.numpy(), ec1))
        q.put((rank, ok, S, F, mx, sm.tolist(), len(mine)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
        raise


def test_sharded_presample_allreduce_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    res = sorted(res)
    for r in res:
        assert len(r) == 7, r
    (_, ok0, S0, F0, mx0, sm0, n0), (_, ok1, S1, F1, mx1, sm1, n1) = res
    assert ok0
    assert n0 == 3 and n1 == 3
    assert S0 == S1 == 3 * 1000 + 3 * 1001 and F0 == F1 == 3 * 3000 + 3 * 3001
    assert mx0 == mx1 == 2.0
    assert sm0 == sm1 == [2.0, 1.0]


def test_shard_round_robin():
    items = list(range(10))
    assert parallel.shard(items, 0, 3) == [0, 3, 6, 9]
    assert parallel.shard(items, 2, 3) == [2, 5, 8]
    assert sorted(sum((parallel.shard(items, r, 4) for r in range(4)), [])) == items


def test_cap_split_to_data():
    """Reading B4: the excess of one side of the split over its data goes to the other; the
    total is unchanged; feature need is per partition."""
    assert parallel.cap_split_to_data(100, 900, 1000, 400) == (600, 400)
    assert parallel.cap_split_to_data(900, 100, 300, 5000) == (300, 700)
    assert parallel.cap_split_to_data(10, 20, 1000, 1000) == (10, 20)  # nothing to move
    a, f = parallel.cap_split_to_data(1_159_508_631, 14_671_851_609, 4 * 1_615_685_872, 512 * 111_059_956, 8)
    assert a == 4 * 1_615_685_872 and a + f == 1_159_508_631 + 14_671_851_609 and f * 8 >= 512 * 111_059_956


def _shm_worker(rank, world, port, q, tag):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        import synth
        parallel.init("gloo")
        N, E, D = 1200, 9000, 13
        calls = []

        def gen():
            calls.append(rank)
            ip, ix = synth.rmat_csc(N, E, seed=9)
            return ip, ix, synth.features(N, D)

        g = parallel.SharedGraph(N, E, D, gen, tag=tag)
        ip, ix = synth.rmat_csc(N, E, seed=9)
        ft = synth.features(N, D).numpy()
        ok = (np.array_equal(g.indptr, ip.numpy()) and np.array_equal(g.indices[:E], ix.numpy())
              and np.array_equal(g.feats[:, :D], ft) and not g.feats[:, D:].any())
        q.put((rank, bool(ok), calls, g.feats.shape, g.names[2]))
        dist.barrier()
        g.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
        raise


def test_shared_graph_generated_once_per_node():
    """parallel.SharedGraph (DCI_ADOPT_HOST's host side): local rank 0 alone generates the graph
    into shm segments; rank 1 maps the same bytes; features are pitch-padded with zeros."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"test{port}"
    procs = [ctx.Process(target=_shm_worker, args=(r, 2, port, q, tag)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5, r
    (_, ok0, calls0, shape0, name0), (_, ok1, calls1, shape1, name1) = res
    assert ok0 and ok1
    assert calls0 == [0] and calls1 == []  # generated once, by local rank 0
    assert shape0 == shape1 == (1200, 16) and name0 == name1
    assert not os.path.exists("/dev/shm/" + name0)  # unlinked once both ranks mapped it
