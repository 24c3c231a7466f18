"""Diagnostic: one config, print per-batch counters and stage times (not part of the product)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01281_b200 as dci  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "M2"]
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
ip, ix = synth.rmat_csc(cfg.N, cfg.E, device=dev)
ip, ix = ip.cpu().numpy(), ix.cpu().numpy()
ft = synth.features(cfg.N, cfg.D, device=dev).cpu().numpy()
ctx = dci.load_graph(ip, ix, ft)
B, fan = cfg.batch, cfg.fanouts
pre = synth.presample_seeds(ip, 8, B)
nv = torch.zeros(cfg.N, dtype=torch.int32, device=dev)
ec = torch.zeros(cfg.E, dtype=torch.int32, device=dev)
ts, tf = dci.presample(ctx, torch.from_numpy(pre).to(dev), B, fan, 3, nv, ec)
print("presample t_s", ts.tolist(), "t_f", tf.tolist())
C = synth.parse_budget(cfg.budget, synth.data_bytes(cfg.N, cfg.E, cfg.D))
ca, cf = dci.allocate(ctx, C, ts, tf)
dci.fill(ctx, nv, ec, ca, cf)
print("info", dci.cache_info(ctx))
st = dci.cache_state(ctx)
print("slot>=0:", int((st["slot_of"] >= 0).sum()), "cached_len sum", int(st["cached_len"].sum()))
ws = dci.workspace_create(ctx, B, fan)
ws.set_profiling(True)
out = dci.BatchOut(ctx, B, fan)
for b in synth.inference_batches(ip, B)[:nb]:
    sd = torch.from_numpy(b).to(dev)
    torch.cuda.synchronize()
    t0 = time.time()
    dci.sample_gather(ctx, ws, sd, fan, 4, out)
    torch.cuda.synchronize()
    r = out.result()
    print("batch", r["sizes"].tolist(), "counters", r["counters"].tolist(), "stage_ms", ws.stage_ms(),
          "wall_ms", (time.time() - t0) * 1e3)
