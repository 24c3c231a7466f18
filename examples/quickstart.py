"""Quick start: DCI mini-batch preparation on one B200, end to end through the Python binding.

  python examples/quickstart.py            (needs a GPU; builds nothing: run __graft_entry__.build() first)

Steps: load the graph into pinned host memory (S0), pre-sample a few batches to
count node / edge hotness (S1), split the HBM budget with Eq. 1 (S2), fill both caches (S3, S4),
then prepare inference batches (S5-S8) in groups with dci_sample_gather_many and aggregate the
input layer with the GraphSAGE mean (NEXT F2).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_01281_b200 as dci  # noqa: E402
import synth  # noqa: E402  (seeded synthetic graphs and features)


def main():
    dev = torch.device("cuda", 0)
    N, E, D, fan, B = 50_000, 2_000_000, 128, (10, 5), 512
    indptr, indices = synth.rmat_csc(N, E, seed=1)
    feats = synth.features(N, D)
    ctx = dci.load_graph(indptr.numpy(), indices.numpy(), feats.numpy(), device=0)  # S0

    # S1: pre-sample 8 batches (pass 1), accumulating hotness histograms on the device
    pre = synth.presample_seeds(indptr.numpy(), 8, B)
    node_visits = torch.zeros(N, dtype=torch.int32, device=dev)
    edge_counts = torch.zeros(E, dtype=torch.int32, device=dev)
    t_sample, t_feature = dci.presample(ctx, torch.from_numpy(pre).to(dev), B, fan, 3, node_visits, edge_counts)

    # S2 + S3/S4: a 64 MB budget split by Eq. 1, then both cache fills
    c_adj, c_feat = dci.allocate(ctx, 64 << 20, t_sample, t_feature)
    dci.fill(ctx, node_visits, edge_counts, c_adj, c_feat)
    info = dci.cache_info(ctx)
    print(f"C_adj={c_adj} C_feat={c_feat}: {info['adj_elems']} adjacency elements, {info['feat_rows']} feature rows")

    # S5-S8: groups of 8 batches, two groups in flight on two streams
    G = 8
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    wss = [[dci.workspace_create(ctx, B, fan) for _ in range(G)] for _ in range(2)]
    outs = [[dci.BatchOut(ctx, B, fan) for _ in range(G)] for _ in range(2)]
    batches = synth.inference_batches(indptr.numpy(), B)
    for k in range(4):
        seeds = [torch.from_numpy(batches[(k * G + j) % len(batches)]).to(dev) for j in range(G)]
        dci.sample_gather_many(ctx, wss[k % 2], seeds, fan, 4, outs[k % 2], stream=streams[k % 2])
    torch.cuda.synchronize()

    r = outs[1][0].result()  # one batch of the last group: frontier, block CSRs, features, counters
    print(f"|F_h| = {r['sizes'].tolist()}, X {r['X'].shape}, counters {r['counters'].tolist()}")
    H = dci.mean_aggregate(ctx, outs[1][0])  # GraphSAGE mean over the input layer's block
    n_dst = int(r["sizes"][len(fan) - 1])  # rows of H that hold results: |F_{L-1}|
    H = H[:n_dst, :D]
    print(f"mean-aggregated input layer: {tuple(H.shape)}, finite={bool(torch.isfinite(H).all())}")
    st = wss[0][0].stats()
    print(f"workspace totals: {st['batches']} batches, {st['frontier_rows']} feature rows")
    ctx.close()


if __name__ == "__main__":
    main()
