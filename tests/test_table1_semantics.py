"""Statistical pin of the sampling semantics against PAPER.md Table I: the number
of loaded nodes per test seed (Load/Test) on ogbn-products.  Our products-shaped synthetic
graph (SURVEY A.2 calibration) must reproduce the batch-1024 column within 5 %
under readings C2 (every frontier node re-sampled per hop) and C3 (DGL fan-out order); the
reverse order or tree-only sampling miss it by 15-25 %."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from tests._util import GOLDEN

TABLE1 = {(int(b), f): r for b, f, _, r in json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["table1"]["rows"]}


@pytest.fixture(scope="module")
def products_cpu():
    ip, ix = synth.rmat_csc(2_449_029, 61_859_140)
    return ip.numpy(), ix.numpy()


def test_oracle_reproduces_table1_batch1024(products_cpu):
    ip, ix = products_cpu
    batches = synth.inference_batches(ip, 1024)
    for fan in [(8, 4, 2), (2, 2, 2)]:
        got = np.mean([len(oracle.sample_batch(ip, ix, batches[i], fan, synth.SAMPLE_SEED).F) / 1024
                       for i in range(6)])
        want = TABLE1[(1024, ",".join(map(str, fan)))]
        assert abs(got - want) / want < 0.05, (fan, got, want)
    # the reverse fan-out order (not DGL's) is far off: C3 is what the paper ran
    rev = np.mean([len(oracle.sample_batch(ip, ix, batches[i], (2, 4, 8), synth.SAMPLE_SEED).F) / 1024
                   for i in range(3)])
    assert abs(rev - TABLE1[(1024, "8,4,2")]) / TABLE1[(1024, "8,4,2")] > 0.1


@pytest.mark.gpu
def test_gpu_table1_all_cells():
    """All nine Table I cells through the CUDA path (bit-exact to the oracle elsewhere):
    within 5 % at batch 1024, 25 % at 256 / 4096 (the synthetic graph's
    batch-size dependence differs from the real graph's by up to ~18 %)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2503_01281_b200 as dci
    dev = torch.device("cuda", 0)
    ip, ix = synth.rmat_csc(2_449_029, 61_859_140, device=dev)
    ip, ix = ip.cpu().numpy(), ix.cpu().numpy()
    ctx = dci.load_graph(ip, ix, np.zeros((len(ip) - 1, 4), np.float32))
    res = {}
    for (B, fs), want in TABLE1.items():
        fan = tuple(int(x) for x in fs.split(","))
        ws = dci.workspace_create(ctx, B, fan)
        out = dci.BatchOut(ctx, B, fan, with_x=False)
        batches = synth.inference_batches(ip, B)
        nb = max(4, 16384 // B)
        tot = 0
        for i in range(nb):
            dci.sample_gather(ctx, ws, torch.from_numpy(batches[i]).to(dev), fan, synth.SAMPLE_SEED, out)
            tot += int(out.sizes[len(fan)].item())
        got = tot / (nb * B)
        res[(B, fs)] = (got, want)
        tol = 0.05 if B == 1024 else 0.25
        assert abs(got - want) / want < tol, (B, fs, got, want)
    print(res)
