"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no sampling, counting, allocation or
fill).  It only produces the inputs the paper's workloads are shaped like
(DESIGN.md §5 "input recipe"):

* ``rmat_csc`` — symmetrised R-MAT graph, (a,b,c,d) = (0.45, 0.22, 0.22, 0.11), E/2
  undirected pairs with both directions stored (exactly E directed edges), endpoints >= N
  rejected and redrawn, Graph500-style random relabelling, self-loops and multi-edges
  kept, CSC neighbours sorted by (dst, src).  Shapes follow PAPER.md Table II
  via BASELINE.json's configs.
* ``feat_fn`` / ``features`` — closed-form fp32 features, uniform in [-1, 1), exactly
  representable, so X can be checked at any size without a second host copy.
* ``inference_batches`` / ``presample_seeds`` — seed lists (eligible = in-degree > 0).

Everything is deterministic for a given (seed, device).  torch is used as a fast array
library here (CPU for the test suite, CUDA for full-size bench graphs); both sides of any
comparison always consume the *same* arrays.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

GRAPH_SEED, PERM_SEED, PRESAMPLE_SEED, SAMPLE_SEED = 1, 2, 3, 4
RMAT_ABC = (0.45, 0.22, 0.22)


@dataclass
class Config:
    """One BASELINE.json workload (M1..M5)."""
    name: str
    N: int
    E: int
    D: int
    fanouts: tuple
    batch: int
    budget: str  # "bytes:<n>" | "frac:<x>" | "auto"
    ratios: tuple = field(default_factory=tuple)  # explicit C_adj/C split points for parity/sweeps

    def pitch_floats(self) -> int:
        return (self.D + 3) // 4 * 4


CONFIGS = {
    # configs[0]: synthetic R-MAT 10K nodes, avg deg 10, 32-dim, 2,2,2, batch 256, 1 MB
    "M1": Config("M1-rmat10k", 10_000, 100_000, 32, (2, 2, 2), 256, "bytes:1048576", (0.0, 0.25, 0.5, 0.75)),
    # configs[1]: Reddit-shaped 233K nodes, 115M edges, 602-dim, 15,10,5, batch 1024
    "M2": Config("M2-reddit", 232_965, 114_615_892, 602, (15, 10, 5), 1024, "auto"),
    # configs[2]: products-shaped 2.4M nodes, 62M edges, 100-dim, 8,4,2, budget 25 % of data
    "M3": Config("M3-products", 2_449_029, 61_859_140, 100, (8, 4, 2), 1024, "frac:0.25"),
    # configs[3]: papers100M-shaped (host-resident, 8-GPU sharded seeds)
    "M4": Config("M4-papers100M", 111_059_956, 1_615_685_872, 128, (15, 10, 5), 1024, "frac:0.25"),
    # configs[3] at 1/10 scale: same average in-degree 14.5, host-resident parity case
    "M4s": Config("M4s-papers100M-tenth", 11_105_996, 161_568_588, 128, (15, 10, 5), 1024, "frac:0.25"),
    # configs[4]: split sweep on products-shaped, r = C_adj/C in 0..1
    "M5": Config("M5-products-sweep", 2_449_029, 61_859_140, 100, (8, 4, 2), 1024, "frac:0.25",
                 tuple(i / 10 for i in range(11))),
}


def rmat_csc(N: int, E: int, seed: int = GRAPH_SEED, device="cpu", abc=RMAT_ABC):
    """Symmetrised R-MAT CSC.  Returns (indptr int64 [N+1], indices int32 [E]) on ``device``.

    E must be even (E/2 undirected pairs stored in both directions)."""
    if E % 2:
        raise ValueError("E must be even (symmetrised R-MAT)")
    if N < 1:
        raise ValueError("N >= 1")
    a, b, c = abc
    scale = max(1, math.ceil(math.log2(N)))
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    need = E // 2
    srcs, dsts, have = [], [], 0
    while have < need:
        m = int((need - have) * 1.15) + 1024
        s = torch.zeros(m, dtype=torch.int64, device=device)
        d = torch.zeros(m, dtype=torch.int64, device=device)
        for _ in range(scale):
            r = torch.rand(m, generator=g, device=device)
            sbit = r >= (a + b)                              # quadrants c, d
            dbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)  # quadrants b, d
            s = s * 2 + sbit.to(torch.int64)
            d = d * 2 + dbit.to(torch.int64)
        keep = (s < N) & (d < N)
        s, d = s[keep], d[keep]
        take = min(need - have, s.numel())
        srcs.append(s[:take])
        dsts.append(d[:take])
        have += take
    s = torch.cat(srcs)
    d = torch.cat(dsts)
    del srcs, dsts
    perm = torch.randperm(N, generator=g, device=device)
    s, d = perm[s], perm[d]
    src = torch.cat([s, d])
    dst = torch.cat([d, s])
    del s, d
    key = dst * N + src
    del src, dst
    key, _ = torch.sort(key)
    dst = key // N
    indices = (key - dst * N).to(torch.int32)
    del key
    counts = torch.bincount(dst, minlength=N)
    indptr = torch.zeros(N + 1, dtype=torch.int64, device=device)
    indptr[1:] = torch.cumsum(counts, 0)
    return indptr, indices


def _mix32(h):
    """murmur3 fmix32 on int64 tensors/arrays holding uint32 values."""
    M = 0xFFFFFFFF
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & M
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & M
    h = h ^ (h >> 16)
    return h


def feat_fn(v, d):
    """Closed-form feature value (numpy): float(mix32(v*0x9E3779B1 ^ d*0x85EBCA6B) >> 8) * 2^-23 - 1."""
    v = np.asarray(v, np.int64)
    d = np.asarray(d, np.int64)
    M = 0xFFFFFFFF
    h = ((v * 0x9E3779B1) & M) ^ ((d * 0x85EBCA6B) & M)
    h = _mix32(h)
    return ((h >> 8).astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)


def features(N: int, D: int, device="cpu", row_block: int = 1 << 16):
    """Dense [N, D] fp32 feature matrix of feat_fn (torch, on ``device``)."""
    out = torch.empty((N, D), dtype=torch.float32, device=device)
    M = 0xFFFFFFFF
    dcol = (torch.arange(D, device=device, dtype=torch.int64) * 0x85EBCA6B) & M
    for r0 in range(0, N, row_block):
        r1 = min(N, r0 + row_block)
        v = (torch.arange(r0, r1, device=device, dtype=torch.int64) * 0x9E3779B1) & M
        h = _mix32(v[:, None] ^ dcol[None, :])
        out[r0:r1] = ((h >> 8).to(torch.float64) * 2.0 ** -23 - 1.0).to(torch.float32)
    return out


def eligible_nodes(indptr):
    """Nodes with in-degree > 0 (seed candidates)."""
    ip = indptr.cpu().numpy() if isinstance(indptr, torch.Tensor) else np.asarray(indptr)
    return np.nonzero(np.diff(ip) > 0)[0].astype(np.int32)


def _perm(n: int, seed: int) -> np.ndarray:
    return np.random.Generator(np.random.Philox(seed)).permutation(n)


def inference_batches(indptr, batch: int, seed: int = PERM_SEED):
    """Eligible nodes, shuffled (Philox stream ``seed``), cut into contiguous batches."""
    el = eligible_nodes(indptr)
    el = el[_perm(len(el), seed)]
    return [el[i:i + batch] for i in range(0, len(el), batch)]


def presample_seeds(indptr, n_batches: int, batch: int, seed: int = PRESAMPLE_SEED):
    """n_batches*batch distinct eligible nodes drawn independently of the inference order (C9)."""
    el = eligible_nodes(indptr)
    el = el[_perm(len(el), seed)]
    return el[: n_batches * batch].copy()


def parse_budget(spec: str, data_bytes: int) -> int:
    """Budget grammar: 'bytes:<n>' | 'frac:<x>' (of feature+index bytes) | 'auto' (-> 0)."""
    if spec == "auto":
        return 0
    kind, val = spec.split(":")
    if kind == "bytes":
        return int(val)
    if kind == "frac":
        return int(float(val) * data_bytes)
    raise ValueError(spec)


def data_bytes(N: int, E: int, D: int) -> int:
    """Bytes the caches can hold: pitch-padded feature rows + 4-byte neighbour ids (C18)."""
    return N * ((D + 3) // 4 * 4) * 4 + 4 * E
