"""DCI oracle — ctypes wrapper around ``oracle/liboracle.so`` (``dci_oracle.c``, plain C11).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
``paper_2503_01281_b200`` never imports it, and this package never imports the product.

Each wrapper names the oracle definition it calls (SURVEY.md §8(c) O-k, restated in
DESIGN.md §3) and the paper passage (P:n = /root/reference/PAPER.md line n).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dci_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, EINVAL, ESEED, EDUP, ECAP = 0, -1, -2, -3, -4

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -O2, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _LIB_PATH, _SRC])
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.oracle_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.oracle_philox4x32_10.restype = None
        L.oracle_draw.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.oracle_draw.restype = C.c_uint64
        L.oracle_bounded.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_bounded.restype = C.c_uint64
        L.oracle_floyd_from_draws.argtypes = [C.c_int64, C.c_int32, _u64p, _i64p]
        L.oracle_floyd_from_draws.restype = None
        L.oracle_select.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int32, C.c_int64, C.c_int32, _i64p]
        L.oracle_select.restype = C.c_int32
        pp = C.POINTER(C.c_void_p)
        L.oracle_sample_batch.argtypes = [C.c_int64, _i64p, _i32p, C.c_void_p, _i32p, C.c_int32, _i32p,
                                          C.c_int32, C.c_uint64, C.c_uint32, _i32p, C.c_int64, _i64p, pp, pp,
                                          _i64p, _u64p, C.c_void_p]
        L.oracle_sample_batch.restype = C.c_int32
        L.oracle_gather.argtypes = [_i32p, C.c_int64, _f32p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, _u64p]
        L.oracle_gather.restype = C.c_int32
        L.oracle_presample.argtypes = [C.c_int64, _i64p, _i32p, _i32p, C.c_int64, C.c_int32, _i32p, C.c_int32,
                                       C.c_uint64, _i32p, _i32p]
        L.oracle_presample.restype = C.c_int32
        L.oracle_allocate.argtypes = [C.c_uint64, _u64p, _u64p, C.c_int32, C.c_int64, C.c_int64,
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_allocate.restype = C.c_int32
        L.oracle_feat_fill.argtypes = [C.c_int64, _i32p, C.c_int64, _i32p, C.c_void_p]
        L.oracle_feat_fill.restype = C.c_int64
        L.oracle_adj_fill.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _i32p, C.c_uint64, _i32p, _i32p, _i64p,
                                      _i32p]
        L.oracle_adj_fill.restype = C.c_int64
        _f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.oracle_block_aggregate.argtypes = [_i32p, _i32p, C.c_int64, _f32p, C.c_int64, C.c_int32, C.c_int32,
                                             _f64p]
        L.oracle_block_aggregate.restype = None
        L.oracle_knapsack_fill.argtypes = [C.c_int64, C.c_int64, _i64p, _i32p, _i32p, C.c_uint64, C.c_int64,
                                           C.c_double, C.c_double, _i32p, _i32p]
        L.oracle_knapsack_fill.restype = C.c_uint64
        L.oracle_sample_gather.argtypes = [C.c_int64, _i64p, _i32p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                           _i32p, C.c_int32, _i32p, C.c_int32, C.c_uint64, _i32p, C.c_int64, _i64p,
                                           pp, pp, _i64p, C.c_void_p, C.c_int64, _u64p]
        L.oracle_sample_gather.restype = C.c_int32
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


def _ptr(a):
    return None if a is None else a.ctypes.data


# ----------------------------------------------------------------------------- O-1..O-4
def philox4x32_10(ctr, key):
    """O-1 Philox4x32-10 block function (Random123)."""
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
    return out


def draw(seed: int, pss: int, hop: int, v: int, i: int) -> int:
    """O-2 u(seed, pass, hop, v, i)."""
    return int(lib().oracle_draw(seed, pss, hop, v, i))


def bounded(u: int, m: int) -> int:
    """O-3 floor(u*m / 2^64)."""
    return int(lib().oracle_bounded(u, m))


def floyd_from_draws(deg: int, t) -> np.ndarray:
    """O-4 Floyd's selection from given bounded draws (draw order, unsorted)."""
    t = np.ascontiguousarray(t, np.uint64)
    out = np.zeros(max(len(t), 1), np.int64)
    lib().oracle_floyd_from_draws(deg, len(t), t, out)
    return out[: len(t)]


def select(seed: int, pss: int, hop: int, v: int, deg: int, f: int) -> np.ndarray:
    """O-4 sorted ranks sampled for node v at this hop (k = min(deg, f))."""
    out = np.zeros(max(min(deg, f), 1), np.int64)
    k = lib().oracle_select(seed, pss, hop, v, deg, f, out)
    return out[:k]


# ----------------------------------------------------------------------------- O-6
def frontier_caps(N: int, B: int, fanouts, L: int):
    """Worst-case |F_h| = min(N, B * prod_{j<h}(1 + f_j)), hop h using fanouts[L-1-h]."""
    caps = [B]
    for h in range(L):
        caps.append(min(N, caps[-1] * (1 + int(fanouts[L - 1 - h]))))
    return caps


class Batch:
    """One sampled mini-batch: F (global ids of F_L, prefix-nested), sizes[L+1],
    per-hop block CSR (bptr[h], bsrc[h]) over dst = F_h, counters, optional X."""

    def __init__(self, F, sizes, bptr, bsrc, counters, X=None):
        self.F, self.sizes, self.bptr, self.bsrc, self.counters, self.X = F, sizes, bptr, bsrc, counters, X


def _alloc_batch(N, B, fanouts, L):
    caps = frontier_caps(N, B, fanouts, L)
    F = np.zeros(max(caps[L], 1), np.int32)
    sizes = np.zeros(L + 1, np.int64)
    bptr = [np.zeros(caps[h] + 1, np.int32) for h in range(L)]
    bcaps = np.array([caps[h] * int(fanouts[L - 1 - h]) for h in range(L)], np.int64)
    bsrc = [np.zeros(max(int(bcaps[h]), 1), np.int32) for h in range(L)]
    bp = (C.c_void_p * L)(*[a.ctypes.data for a in bptr])
    bs = (C.c_void_p * L)(*[a.ctypes.data for a in bsrc])
    return caps, F, sizes, bptr, bsrc, bcaps, bp, bs


def _finish(F, sizes, bptr, bsrc, L):
    n = sizes.copy()
    F = F[: n[L]].copy()
    bptr = [bptr[h][: n[h] + 1].copy() for h in range(L)]
    bsrc = [bsrc[h][: bptr[h][-1]].copy() for h in range(L)]
    return F, n, bptr, bsrc


def sample_batch(indptr, indices_cur, seeds, fanouts, seed: int, pss: int = 0, cached_len=None,
                 edge_counts=None) -> Batch:
    """O-5/O-6 one batch of L-hop sampling."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices_cur = np.ascontiguousarray(indices_cur, np.int32)
    seeds = np.ascontiguousarray(seeds, np.int32)
    fanouts = np.ascontiguousarray(fanouts, np.int32)
    N, L, B = len(indptr) - 1, len(fanouts), len(seeds)
    caps, F, sizes, bptr, bsrc, bcaps, bp, bs = _alloc_batch(N, B, fanouts, L)
    hm = np.zeros(2, np.uint64)
    if cached_len is not None:
        cached_len = np.ascontiguousarray(cached_len, np.int32)
    rc = lib().oracle_sample_batch(N, indptr, indices_cur, _ptr(cached_len), seeds, B, fanouts, L, seed, pss, F,
                                   len(F), sizes, bp, bs, bcaps, hm, _ptr(edge_counts))
    if rc != OK:
        raise OracleError(rc, "sample_batch")
    F, n, bptr, bsrc = _finish(F, sizes, bptr, bsrc, L)
    return Batch(F, n, bptr, bsrc, np.array([hm[0], hm[1], 0, 0], np.uint64))


def gather(F, feats, slot_of=None, with_x=True):
    """O-7 X[i] = feats[F[i]]; returns (X, [feat_hit, feat_miss])."""
    F = np.ascontiguousarray(F, np.int32)
    feats = np.ascontiguousarray(feats, np.float32)
    D = feats.shape[1]
    X = np.zeros((len(F), D), np.float32) if with_x else None
    hm = np.zeros(2, np.uint64)
    if slot_of is not None:
        slot_of = np.ascontiguousarray(slot_of, np.int32)
    lib().oracle_gather(F, len(F), feats, D, _ptr(slot_of), _ptr(X), D, hm)
    return X, hm


def sample_gather(indptr, indices_cur, feats, seeds, fanouts, seed: int, cached_len=None, slot_of=None,
                  with_x=True) -> Batch:
    """One inference step (O-6 pass 0 + O-7).  Counters = [adj_hit, adj_miss, feat_hit, feat_miss]."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices_cur = np.ascontiguousarray(indices_cur, np.int32)
    feats = np.ascontiguousarray(feats, np.float32)
    seeds = np.ascontiguousarray(seeds, np.int32)
    fanouts = np.ascontiguousarray(fanouts, np.int32)
    N, L, B = len(indptr) - 1, len(fanouts), len(seeds)
    D = feats.shape[1]
    caps, F, sizes, bptr, bsrc, bcaps, bp, bs = _alloc_batch(N, B, fanouts, L)
    X = np.zeros((caps[L], D), np.float32) if with_x else None
    cnt = np.zeros(4, np.uint64)
    if cached_len is not None:
        cached_len = np.ascontiguousarray(cached_len, np.int32)
    if slot_of is not None:
        slot_of = np.ascontiguousarray(slot_of, np.int32)
    rc = lib().oracle_sample_gather(N, indptr, indices_cur, _ptr(cached_len), _ptr(slot_of), feats.ctypes.data, D,
                                    seeds, B, fanouts, L, seed, F, len(F), sizes, bp, bs, bcaps, _ptr(X), D, cnt)
    if rc != OK:
        raise OracleError(rc, "sample_gather")
    F, n, bptr, bsrc = _finish(F, sizes, bptr, bsrc, L)
    if X is not None:
        X = X[: n[L]]
    return Batch(F, n, bptr, bsrc, cnt, X)


# ----------------------------------------------------------------------------- O-8..O-12
def presample(indptr, indices, seeds, batch: int, fanouts, seed: int, node_visits=None, edge_counts=None):
    """O-8 presample counts (pass 1, original CSC, no cache).  Accumulates in place."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    seeds = np.ascontiguousarray(seeds, np.int32)
    fanouts = np.ascontiguousarray(fanouts, np.int32)
    N, E = len(indptr) - 1, len(indices)
    if node_visits is None:
        node_visits = np.zeros(N, np.int32)
    if edge_counts is None:
        edge_counts = np.zeros(E, np.int32)
    rc = lib().oracle_presample(N, indptr, indices, seeds, len(seeds), batch, fanouts, len(fanouts), seed,
                                node_visits, edge_counts)
    if rc != OK:
        raise OracleError(rc, "presample")
    return node_visits, edge_counts


def allocate(C_bytes: int, t_sample=(), t_feature=(), ratio=None):
    """O-10 Eq. (1) split; ratio=(num, den) overrides the measured times."""
    ts = np.ascontiguousarray(t_sample, np.uint64).reshape(-1)
    tf = np.ascontiguousarray(t_feature, np.uint64).reshape(-1)
    if len(ts) == 0:
        ts = np.zeros(1, np.uint64)
        tf = np.zeros(1, np.uint64)
        n = 0
    else:
        n = len(ts)
    num, den = (0, 0) if ratio is None else ratio
    a, f = C.c_uint64(0), C.c_uint64(0)
    rc = lib().oracle_allocate(C_bytes, ts, tf, n, num, den, C.byref(a), C.byref(f))
    if rc != OK:
        raise OracleError(rc, "allocate")
    return int(a.value), int(f.value)


def feat_fill(node_visits, cap_rows: int):
    """O-11 top-cap by (visits desc, id asc); slots in ascending id.  Returns (slot_of, admitted)."""
    v = np.ascontiguousarray(node_visits, np.int32)
    N = len(v)
    slot_of = np.zeros(N, np.int32)
    adm = np.zeros(max(min(cap_rows, N), 1), np.int32)
    n = lib().oracle_feat_fill(N, v, cap_rows, slot_of, adm.ctypes.data)
    return slot_of, adm[:n]


def adj_fill(indptr, indices, edge_counts, c_adj_bytes: int):
    """O-12 Algorithm 1 + Fig. 6.  Returns (indices_R, cached_len, cache_off, acache)."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    cnt = np.ascontiguousarray(edge_counts, np.int32)
    N, E = len(indptr) - 1, len(indices)
    R = np.zeros(max(E, 1), np.int32)
    cl = np.zeros(max(N, 1), np.int32)
    co = np.zeros(max(N, 1), np.int64)
    cap_e = min(c_adj_bytes // 4, E)
    ac = np.zeros(max(cap_e, 1), np.int32)
    n = lib().oracle_adj_fill(N, E, indptr, indices, cnt, c_adj_bytes, R, cl, co, ac)
    return R[:E], cl[:N], co[:N], ac[:n]


def mean_aggregate(bptr, bsrc, X, op: str = "mean"):
    """O-13 aggregation over a block (fp64): H[d] = mean (op="mean") or sum (op="sum") of
    X[bsrc[bptr[d]:bptr[d+1]]]."""
    bptr = np.ascontiguousarray(bptr, np.int32)
    bsrc = np.ascontiguousarray(bsrc, np.int32)
    X = np.ascontiguousarray(X, np.float32)
    n = len(bptr) - 1
    D = X.shape[1]
    H = np.zeros((max(n, 1), D), np.float64)
    if len(bsrc) == 0:
        bsrc = np.zeros(1, np.int32)
    lib().oracle_block_aggregate(bptr, bsrc, n, X, D, D, {"mean": 0, "sum": 1}[op], H)
    return H[:n]


def knapsack_fill(indptr, node_visits, edge_counts, C_bytes: int, row_bytes: int, cost_feat: float,
                  cost_adj: float):
    """O-14 unified-budget greedy knapsack (DUCATI-style).  Returns
    (slot_of, cached_len, bytes_used)."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    v = np.ascontiguousarray(node_visits, np.int32)
    c = np.ascontiguousarray(edge_counts, np.int32)
    N, E = len(indptr) - 1, len(c)
    slot = np.zeros(max(N, 1), np.int32)
    cl = np.zeros(max(N, 1), np.int32)
    if E == 0:
        c = np.zeros(1, np.int32)
    used = lib().oracle_knapsack_fill(N, E, indptr, v, c, C_bytes, row_bytes, cost_feat, cost_adj, slot, cl)
    return slot[:N], cl[:N], int(used)
