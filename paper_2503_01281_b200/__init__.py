"""Python binding of libdci (include/dci.h) — argument marshalling only.

Every step of the DCI hot path (sampling, dedup/relabel, feature route, gather, presample
counting, radix-select fills) runs in the CUDA kernels of ``libdci.so``; this module only
converts arguments, allocates output tensors with torch (device memory plumbing) and
passes torch's current CUDA stream.  There is no CPU fallback: if the extension is missing
or no CUDA device is present, the compute calls raise.

Names follow the C ABI: ``load_graph``, ``presample``, ``allocate``, ``fill``,
``sample_gather`` (+ ``sample_gather_host``), ``output_bounds``, ``workspace_create``,
``cache_state``, ``cache_info``; ``GroupCall`` is ``dci_sample_gather_many`` with its fixed
arguments marshalled once.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DCI_LIB", os.path.join(_HERE, "libdci.so"))  # override: build experiments
MAX_LAYERS = 8
MAX_FANOUT = 1024

STATUS = {0: "DCI_OK", 1: "DCI_EINVAL", 2: "DCI_ESTATE", 3: "DCI_ECUDA", 4: "DCI_ENOMEM", 5: "DCI_ESEED",
          6: "DCI_EDUP", 7: "DCI_ECAP", 8: "DCI_ERANGE"}
OK, EINVAL, ESTATE, ECUDA, ENOMEM, ESEED, EDUP, ECAP, ERANGE = range(9)

EXPORTED = ["dci_load_graph", "dci_destroy", "dci_output_bounds", "dci_workspace_create", "dci_workspace_destroy",
            "dci_sample_gather", "dci_sample_gather_host", "dci_sample_gather_many", "dci_sample_gather_many_host",
            "dci_presample", "dci_allocate", "dci_fill",
            "dci_cache_info_get", "dci_fill_times_get", "dci_cache_state", "dci_workspace_set_profiling", "dci_workspace_stage_ms",
            "dci_workspace_stats", "dci_mean_aggregate", "dci_block_aggregate", "dci_fill_partitioned", "dci_fill_knapsack", "dci_feature_partition_handle",
            "dci_attach_feature_partitions", "dci_launch_count", "dci_last_error", "dci_version"]
IPC_HANDLE_BYTES = 64


class DciError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str = ""):
        super().__init__(f"{where}: {STATUS.get(code, code)} {msg}")
        self.code = code


class dci_batch_out(C.Structure):
    _fields_ = [("frontier", C.c_void_p), ("frontier_cap", C.c_int64), ("sizes", C.c_void_p),
                ("bptr", C.c_void_p * MAX_LAYERS), ("bsrc", C.c_void_p * MAX_LAYERS),
                ("hop_cap", C.c_int64 * MAX_LAYERS), ("bsrc_cap", C.c_int64 * MAX_LAYERS),
                ("X", C.c_void_p), ("ldx", C.c_int64), ("counters", C.c_void_p), ("status", C.c_void_p)]


class dci_ws_stats(C.Structure):
    _fields_ = [("batches", C.c_uint64), ("seeds", C.c_uint64), ("frontier_rows", C.c_uint64),
                ("counters", C.c_uint64 * 4), ("timed_batches", C.c_uint64), ("sample_ms", C.c_double),
                ("gather_ms", C.c_double), ("gather_launches", C.c_uint64), ("rows_read", C.c_uint64),
                ("gather_bytes", C.c_uint64), ("host_rows_read", C.c_uint64), ("host_adj_sectors", C.c_uint64),
                ("gather_kinds", C.c_uint64 * 3), ("table_bytes", C.c_uint64), ("host_adj_runs", C.c_uint64)]


class dci_fill_times(C.Structure):
    _fields_ = [(k, C.c_float) for k in ("level2_ms", "adj_select_ms", "adj_copy_ms", "feat_select_ms",
                                         "feat_copy_ms", "total_ms")]


class dci_cache_info(C.Structure):
    _fields_ = [("state", C.c_int32), ("pitch", C.c_int32), ("N", C.c_int64), ("E", C.c_int64), ("D", C.c_int32),
                ("whole_fit", C.c_int32), ("c_adj", C.c_uint64), ("c_feat", C.c_uint64), ("adj_elems", C.c_int64),
                ("feat_rows", C.c_int64), ("feat_rows_total", C.c_int64), ("feat_partitions", C.c_int32),
                ("pad_", C.c_int32), ("presample_peak_bytes", C.c_uint64), ("launches", C.c_uint64)]


_lib = None


def lib():
    """Load libdci.so (built in-tree by __graft_entry__.build()); raise if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "dci_load_graph": [C.POINTER(C.c_void_p), C.c_int, i64, i64, vp, vp, vp, i32, C.c_uint32],
        "dci_destroy": [vp],
        "dci_output_bounds": [vp, i32, vp, i32, vp, vp, vp],
        "dci_workspace_create": [vp, i32, vp, i32, C.POINTER(C.c_void_p)],
        "dci_workspace_destroy": [vp],
        "dci_sample_gather": [vp, vp, vp, i32, vp, i32, u64, C.POINTER(dci_batch_out), vp],
        "dci_sample_gather_host": [vp, vp, vp, i32, vp, i32, u64, C.POINTER(dci_batch_out), vp, vp, vp, vp],
        "dci_sample_gather_many": [vp, i32, vp, vp, vp, vp, i32, u64, vp, vp],
        "dci_sample_gather_many_host": [vp, i32, vp, vp, vp, vp, i32, u64, vp, vp, vp],
        "dci_presample": [vp, vp, i64, i32, vp, i32, u64, vp, vp, vp, vp, vp],
        "dci_allocate": [vp, u64, vp, vp, i32, i64, i64, C.POINTER(u64), C.POINTER(u64)],
        "dci_fill": [vp, vp, vp, u64, u64, vp],
        "dci_fill_partitioned": [vp, vp, vp, u64, u64, i32, i32, vp],
        "dci_fill_knapsack": [vp, vp, vp, u64, C.c_double, C.c_double, vp],
        "dci_feature_partition_handle": [vp, vp],
        "dci_attach_feature_partitions": [vp, vp, i32],
        "dci_cache_info_get": [vp, C.POINTER(dci_cache_info)],
        "dci_fill_times_get": [vp, C.POINTER(dci_fill_times)],
        "dci_cache_state": [vp, vp, vp, vp, vp, vp, vp],
        "dci_workspace_set_profiling": [vp, i32],
        "dci_workspace_stage_ms": [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)],
        "dci_workspace_stats": [vp, C.POINTER(dci_ws_stats), i32],
        "dci_mean_aggregate": [vp, vp, vp, vp, vp, i64, i32, vp, i64, vp],
        "dci_block_aggregate": [vp, vp, vp, vp, vp, i64, i32, vp, i64, i32, vp],
        "dci_launch_count": [vp],
        "dci_last_error": [],
        "dci_version": [],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.dci_launch_count.restype = C.c_uint64
    L.dci_last_error.restype = C.c_char_p
    _lib = L
    return L


def _check(rc: int, where: str):
    if rc != OK:
        raise DciError(rc, where, lib().dci_last_error().decode(errors="replace"))


def _np_ptr(a):
    return a.ctypes.data


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _t_ptr(t):
    return None if t is None else t.data_ptr()


class Context:
    """Owns a dci_ctx (graph in pinned host memory + device directory + caches)."""

    def __init__(self, handle, N, E, D, device):
        self.handle, self.N, self.E, self.D, self.device = handle, N, E, D, device
        self._workspaces = weakref.WeakSet()

    def close(self):
        """Destroy the context (its live workspaces first: finalizers of garbage cycles run
        in arbitrary order, so a workspace may still exist when the context goes)."""
        if self.handle:
            for ws in list(self._workspaces):
                ws.close()
            lib().dci_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().dci_launch_count(self.handle))


ADOPT_HOST = 1  # DCI_ADOPT_HOST


def load_graph(indptr, indices, feats, device: int = 0, adopt: bool = False, D: int | None = None) -> Context:
    """dci_load_graph (S0).  indptr int64[N+1], indices int32[E], feats fp32[N, D]: host arrays
    (numpy or CPU torch); copied into pinned, device-mapped memory.

    adopt=True (DCI_ADOPT_HOST): indices and feats are registered IN PLACE (no copy; e.g. a
    node-shared shm segment, see parallel.shared_graph) and must stay alive as long as the
    context (the Context keeps references).  feats must then be [N, pitch] with pitch =
    round_up(D, 4) (pad columns zero); pass the true D when pitch != D."""
    ip = np.ascontiguousarray(_to_np(indptr), np.int64)
    if adopt:
        ix, ft = _to_np(indices), _to_np(feats)
        if not (ix.dtype == np.int32 and ix.flags.c_contiguous and ft.dtype == np.float32 and ft.flags.c_contiguous):
            raise TypeError("adopt=True needs C-contiguous int32 indices and float32 feats (no copies are made)")
        D = int(D if D is not None else ft.shape[1])
        if ft.shape[1] != (D + 3) // 4 * 4:
            raise ValueError(f"adopt=True: feats must be [N, round_up(D, 4)] = [N, {(D + 3) // 4 * 4}], "
                             f"got {ft.shape}")
    else:
        ix = np.ascontiguousarray(_to_np(indices), np.int32)
        ft = np.ascontiguousarray(_to_np(feats), np.float32)
        D = ft.shape[1]
    N, E = len(ip) - 1, len(ix)
    h = C.c_void_p()
    _check(lib().dci_load_graph(C.byref(h), device, N, E, _np_ptr(ip), _np_ptr(ix) if E else None, _np_ptr(ft),
                                D, ADOPT_HOST if adopt else 0), "dci_load_graph")
    ctx = Context(h, N, E, D, device)
    if adopt:
        ctx._adopted = (ix, ft)  # the registered memory must outlive the context
    return ctx


def _to_np(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return a.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(a)


def output_bounds(ctx: Context, B: int, fanouts):
    """dci_output_bounds: worst-case |F_h| (h=0..L), bsrc sizes per hop, feature pitch."""
    fan = np.ascontiguousarray(fanouts, np.int32)
    L = len(fan)
    fc = np.zeros(L + 1, np.int64)
    bc = np.zeros(L, np.int64)
    p = C.c_int32()
    _check(lib().dci_output_bounds(ctx.handle, B, _np_ptr(fan), L, _np_ptr(fc), _np_ptr(bc), C.byref(p)),
           "dci_output_bounds")
    return fc, bc, int(p.value)


class Workspace:
    def __init__(self, ctx: Context, max_batch: int, max_fanouts):
        fan = np.ascontiguousarray(max_fanouts, np.int32)
        h = C.c_void_p()
        _check(lib().dci_workspace_create(ctx.handle, max_batch, _np_ptr(fan), len(fan), C.byref(h)),
               "dci_workspace_create")
        self.handle, self.ctx, self.max_batch, self.fanouts = h, ctx, max_batch, tuple(int(f) for f in fan)
        ctx._workspaces.add(self)

    def close(self):
        if self.handle:
            lib().dci_workspace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on: bool = True):
        _check(lib().dci_workspace_set_profiling(self.handle, 1 if on else 0), "dci_workspace_set_profiling")

    def stats(self, reset: bool = False) -> dict:
        """dci_workspace_stats: running totals (batches, seeds, rows, counters, stage ms)."""
        st = dci_ws_stats()
        _check(lib().dci_workspace_stats(self.handle, C.byref(st), 1 if reset else 0), "dci_workspace_stats")
        return {"batches": st.batches, "seeds": st.seeds, "frontier_rows": st.frontier_rows,
                "counters": [int(c) for c in st.counters], "timed_batches": st.timed_batches,
                "sample_ms": st.sample_ms, "gather_ms": st.gather_ms, "gather_launches": st.gather_launches,
                "rows_read": st.rows_read, "gather_bytes": st.gather_bytes,
                "host_rows_read": st.host_rows_read, "host_adj_sectors": st.host_adj_sectors,
                "gather_kinds": [int(k) for k in st.gather_kinds], "table_bytes": int(st.table_bytes),
                "host_adj_runs": int(st.host_adj_runs)}

    def stage_ms(self):
        s, g = C.c_float(), C.c_float()
        _check(lib().dci_workspace_stage_ms(self.handle, C.byref(s), C.byref(g)), "dci_workspace_stage_ms")
        return float(s.value), float(g.value)


def workspace_create(ctx: Context, max_batch: int, max_fanouts) -> Workspace:
    return Workspace(ctx, max_batch, max_fanouts)


class BatchOut:
    """Caller-owned device output buffers of one batch (torch tensors on ctx.device)."""

    def __init__(self, ctx: Context, B: int, fanouts, with_x: bool = True, ldx: int | None = None):
        import torch
        fc, bc, pitch = output_bounds(ctx, B, fanouts)
        dev = torch.device("cuda", ctx.device)
        L = len(fanouts)
        self.L, self.D, self.pitch = L, ctx.D, pitch
        self.ldx = pitch if ldx is None else int(ldx)
        self.frontier = torch.empty(max(int(fc[L]), 1), dtype=torch.int32, device=dev)
        self.sizes = torch.zeros(L + 1, dtype=torch.int64, device=dev)
        self.bptr = [torch.empty(int(fc[h]) + 1, dtype=torch.int32, device=dev) for h in range(L)]
        self.bsrc = [torch.empty(max(int(bc[h]), 1), dtype=torch.int32, device=dev) for h in range(L)]
        self.X = torch.empty((max(int(fc[L]), 1), self.ldx), dtype=torch.float32, device=dev) if with_x else None
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        s = dci_batch_out()
        s.frontier = self.frontier.data_ptr()
        s.frontier_cap = int(fc[L])
        s.sizes = self.sizes.data_ptr()
        for h in range(L):
            s.bptr[h] = self.bptr[h].data_ptr()
            s.bsrc[h] = self.bsrc[h].data_ptr()
            s.hop_cap[h] = int(fc[h])
            s.bsrc_cap[h] = int(bc[h])
        s.X = _t_ptr(self.X)
        s.ldx = self.ldx
        s.counters = self.counters.data_ptr()
        s.status = self.status.data_ptr()
        self.struct = s
        self._streams = set()

    def record_stream(self, stream):
        """Once per stream: the caching allocator then waits for all work queued on `stream`
        before recycling these buffers, even if this BatchOut is dropped mid-flight."""
        key = stream.cuda_stream
        if key in self._streams:
            return
        for t in [self.frontier, self.sizes, self.counters, self.status, self.X] + self.bptr + self.bsrc:
            if t is not None:
                t.record_stream(stream)
        self._streams.add(key)

    def result(self):
        """Synchronise and return host copies trimmed to the batch's actual sizes."""
        import torch
        torch.cuda.synchronize(self.frontier.device)
        n = self.sizes.cpu().numpy()
        L = self.L
        bptr = [self.bptr[h][: n[h] + 1].cpu().numpy() for h in range(L)]
        bsrc = [self.bsrc[h][: int(bptr[h][-1])].cpu().numpy() for h in range(L)]
        out = {
            "F": self.frontier[: n[L]].cpu().numpy(),
            "sizes": n,
            "bptr": bptr,
            "bsrc": bsrc,
            "counters": self.counters.cpu().numpy().astype(np.uint64),
            "status": int(self.status.cpu().item()),
        }
        if self.X is not None:
            out["X"] = self.X[: n[L], : self.D].cpu().numpy()
        return out


def _device_i32(t, what, device=None):
    """Arguments passed to the ABI as device int32 pointers must be contiguous int32 CUDA tensors
    (the ABI sees only the pointer, so a wrong dtype or a strided view would be read as garbage)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
        raise TypeError(f"{what}: expected a contiguous int32 CUDA tensor, got "
                        f"{getattr(t, 'dtype', type(t))} on {getattr(t, 'device', '?')}")
    if device is not None and t.device.index != device:
        raise ValueError(f"{what}: tensor on cuda:{t.device.index}, context on cuda:{device}")


def _host_i32(t, what):
    import torch
    if not (isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
        raise TypeError(f"{what}: expected a contiguous int32 CPU (pinned) tensor")


def _counts_ok(ctx, node_visits, edge_counts):
    """Presample histograms: device int32[N] and int32[E]."""
    _device_i32(node_visits, "node_visits", ctx.device)
    if node_visits.numel() < ctx.N:
        raise ValueError("node_visits must hold N counts")
    if ctx.E:
        _device_i32(edge_counts, "edge_counts", ctx.device)
        if edge_counts.numel() < ctx.E:
            raise ValueError("edge_counts must hold E counts")


def _record(tensor, stream):
    """The batch reads `tensor` asynchronously on `stream`: tell torch's caching allocator, so a
    tensor the caller drops is not handed to another allocation before the batch has run."""
    if stream is not None and tensor.is_cuda:
        tensor.record_stream(stream)


def sample_gather(ctx: Context, ws: Workspace, seeds, fanouts, seed: int, out: BatchOut, stream=None):
    """dci_sample_gather (S5-S8), asynchronous on `stream` (default: torch current stream).
    seeds: int32 CUDA tensor on ctx.device."""
    import torch
    fan = np.ascontiguousarray(fanouts, np.int32)
    _device_i32(seeds, "seeds", ctx.device)
    st = torch.cuda.current_stream() if stream is None else stream
    _record(seeds, st)
    out.record_stream(st)
    _check(lib().dci_sample_gather(ctx.handle, ws.handle, seeds.data_ptr(), int(seeds.numel()), _np_ptr(fan),
                                   len(fan), seed, C.byref(out.struct), st.cuda_stream), "dci_sample_gather")


def sample_gather_many(ctx: Context, wss, seeds_list, fanouts, seed: int, outs, stream=None):
    """dci_sample_gather_many: n <= 32 (DCI_MAX_GROUP) batches (one workspace and one BatchOut each) sampled
    concurrently and gathered by ONE group gather launch (row mode or node sweep); asynchronous on `stream`."""
    import torch
    n = len(wss)
    if not n == len(seeds_list) == len(outs):
        raise ValueError("wss, seeds_list and outs must have the same length")
    for sd in seeds_list:
        _device_i32(sd, "seeds", ctx.device)
    fan = np.ascontiguousarray(fanouts, np.int32)
    st = torch.cuda.current_stream() if stream is None else stream
    for sd in seeds_list:
        _record(sd, st)
    for o in outs:
        o.record_stream(st)
    ws_arr = (C.c_void_p * n)(*[w.handle for w in wss])
    sd_arr = (C.c_void_p * n)(*[sd.data_ptr() for sd in seeds_list])
    b_arr = (C.c_int32 * n)(*[int(sd.numel()) for sd in seeds_list])
    out_arr = (dci_batch_out * n)(*[o.struct for o in outs])
    _check(lib().dci_sample_gather_many(ctx.handle, n, ws_arr, sd_arr, b_arr, _np_ptr(fan), len(fan), seed, out_arr,
                                        st.cuda_stream), "dci_sample_gather_many")


def _record_once(tensor, stream):
    """_record, once per (tensor, stream): the caching allocator keeps every stream a block was
    recorded on until the block is freed, so repeating the call for the same pair adds nothing
    (the streams already recorded ride on the tensor object)."""
    key = stream.cuda_stream
    seen = getattr(tensor, "_dci_streams", None)
    if seen is None:
        seen = set()
        tensor._dci_streams = seen
    if key not in seen:
        tensor.record_stream(stream)
        seen.add(key)


class GroupCall:
    """dci_sample_gather_many with its fixed arguments (workspaces, outputs, fan-outs) marshalled
    once: each call passes only the n seed tensors, so a group's host enqueue -- which every timed
    region waits on before the group's first kernel -- costs a few microseconds of Python instead
    of rebuilding four ctypes arrays.  Holds references to the workspaces and outputs.  One
    GroupCall is not for concurrent use from several host threads (its argument arrays are
    reused); the library has copied them when a call returns."""

    def __init__(self, ctx: Context, wss, fanouts, outs):
        if len(wss) != len(outs):
            raise ValueError("wss and outs must have the same length")
        self.ctx, self.wss, self.outs = ctx, list(wss), list(outs)
        self.n = len(self.wss)
        self.fan = np.ascontiguousarray(fanouts, np.int32)
        self.ws_arr = (C.c_void_p * self.n)(*[w.handle for w in self.wss])
        self.out_arr = (dci_batch_out * self.n)(*[o.struct for o in self.outs])
        self.sd_arr = (C.c_void_p * self.n)()
        self.b_arr = (C.c_int32 * self.n)()

    def __call__(self, seeds_list, seed: int, stream=None):
        """One group call on `stream` (default: torch current stream); seeds_list: n contiguous int32
        CUDA tensors on the context's device."""
        import torch
        if len(seeds_list) != self.n:
            raise ValueError(f"expected {self.n} seed tensors")
        st = torch.cuda.current_stream() if stream is None else stream
        for i, sd in enumerate(seeds_list):
            _device_i32(sd, "seeds", self.ctx.device)
            _record_once(sd, st)
            self.sd_arr[i] = sd.data_ptr()
            self.b_arr[i] = sd.numel()
        for o in self.outs:
            o.record_stream(st)
        _check(lib().dci_sample_gather_many(self.ctx.handle, self.n, self.ws_arr, self.sd_arr, self.b_arr,
                                            self.fan.ctypes.data, len(self.fan), seed, self.out_arr,
                                            st.cuda_stream), "dci_sample_gather_many")

    def host(self, seeds_host_list, seed: int, results_host=None, stream=None):
        """The dci_sample_gather_many_host form: pinned host seed tensors in, every batch's
        sizes / counters / status back in one copy into results_host (see result_buffer).  The
        copies are asynchronous: keep the seed tensors and results_host alive, and read the
        results, after synchronising `stream`."""
        import torch
        if len(seeds_host_list) != self.n:
            raise ValueError(f"expected {self.n} seed tensors")
        st = torch.cuda.current_stream() if stream is None else stream
        for i, sd in enumerate(seeds_host_list):
            _host_i32(sd, "seeds_host")
            self.sd_arr[i] = sd.data_ptr()
            self.b_arr[i] = sd.numel()
        for o in self.outs:
            o.record_stream(st)
        assert results_host is None or (results_host.shape[0] >= self.n and results_host.shape[-1] == RESULT_WORDS)
        _check(lib().dci_sample_gather_many_host(self.ctx.handle, self.n, self.ws_arr, self.sd_arr, self.b_arr,
                                                 self.fan.ctypes.data, len(self.fan), seed, self.out_arr,
                                                 results_host.data_ptr() if results_host is not None else None,
                                                 st.cuda_stream), "dci_sample_gather_many_host")


MAX_LAYERS = 8
RESULT_WORDS =MAX_LAYERS + 1 + 4 + 1  # dci_batch_result as int64 words: sizes[9], counters[4], status|pad


def result_buffer(n: int):
    """Pinned host buffer for n dci_batch_result records (int64 [n, RESULT_WORDS])."""
    import torch
    return torch.zeros((n, RESULT_WORDS), dtype=torch.int64).pin_memory()


def parse_results(results_host, L: int):
    """dci_batch_result records -> [{"sizes", "counters", "status"}] (after a stream sync)."""
    r = results_host.numpy()
    out = []
    for row in r:
        st = int(row[MAX_LAYERS + 5] & 0xFFFFFFFF)
        out.append({"sizes": row[: L + 1].copy(), "counters": row[MAX_LAYERS + 1: MAX_LAYERS + 5].astype(np.uint64),
                    "status": st - (1 << 32) if st >= 1 << 31 else st})
    return out


def sample_gather_many_host(ctx: Context, wss, seeds_host_list, fanouts, seed: int, outs, results_host=None,
                            stream=None):
    """dci_sample_gather_many_host: host (pinned) seeds in; every batch's sizes / counters /
    status come back in ONE copy into results_host (see result_buffer / parse_results), valid
    after synchronising `stream`."""
    n = len(wss)
    if not n == len(seeds_host_list) == len(outs):
        raise ValueError("wss, seeds_host_list and outs must have the same length")
    for sd in seeds_host_list:
        _host_i32(sd, "seeds_host")
    fan = np.ascontiguousarray(fanouts, np.int32)
    if stream is not None:
        for o in outs:
            o.record_stream(stream)
    ws_arr = (C.c_void_p * n)(*[w.handle for w in wss])
    sd_arr = (C.c_void_p * n)(*[sd.data_ptr() for sd in seeds_host_list])
    b_arr = (C.c_int32 * n)(*[int(sd.numel()) for sd in seeds_host_list])
    out_arr = (dci_batch_out * n)(*[o.struct for o in outs])
    assert results_host is None or (results_host.shape[0] >= n and results_host.shape[-1] == RESULT_WORDS)
    _check(lib().dci_sample_gather_many_host(ctx.handle, n, ws_arr, sd_arr, b_arr, _np_ptr(fan), len(fan), seed,
                                             out_arr, results_host.data_ptr() if results_host is not None else None,
                                             _stream_ptr(stream)), "dci_sample_gather_many_host")


def sample_gather_host(ctx: Context, ws: Workspace, seeds_host, fanouts, seed: int, out: BatchOut, sizes_host,
                       counters_host, status_host, stream=None):
    """dci_sample_gather_host: seeds from (pinned) host memory; sizes/counters/status copied back
    to host buffers (pinned torch tensors) on the same stream.  The host tensors must stay alive
    until the stream has been synchronised (the copies are asynchronous)."""
    import torch
    _host_i32(seeds_host, "seeds_host")
    fan = np.ascontiguousarray(fanouts, np.int32)
    if stream is not None:
        out.record_stream(stream)
    _check(lib().dci_sample_gather_host(ctx.handle, ws.handle, seeds_host.data_ptr(), int(seeds_host.numel()),
                                        _np_ptr(fan), len(fan), seed, C.byref(out.struct),
                                        sizes_host.data_ptr(), counters_host.data_ptr(), status_host.data_ptr(),
                                        _stream_ptr(stream)), "dci_sample_gather_host")


def mean_aggregate(ctx: Context, out: BatchOut, hop: int | None = None, H=None, stream=None, op: str = "mean"):
    """dci_block_aggregate (NEXT F2): mean ("avg", GCN) or sum (GraphSAGE "sum", Table III) over
    block `hop` (default the input layer L-1, whose sources are the rows of out.X).  Returns
    H [hop_cap, ldx] (device)."""
    import torch
    hop = out.L - 1 if hop is None else hop
    if hop != out.L - 1:
        raise ValueError("only the input-layer block has its source rows in out.X")
    if out.X is None:
        raise ValueError("out has no X")
    rows = out.bptr[hop].numel() - 1
    if H is None:
        H = torch.empty((max(rows, 1), out.ldx), dtype=torch.float32, device=out.X.device)
    st = torch.cuda.current_stream() if stream is None else stream
    out.record_stream(st)
    _record(H, st)
    _check(lib().dci_block_aggregate(ctx.handle, out.bptr[hop].data_ptr(), out.bsrc[hop].data_ptr(),
                                     out.sizes.data_ptr() + 8 * hop, out.X.data_ptr(), out.ldx, out.D,
                                     H.data_ptr(), H.shape[1], {"mean": 0, "sum": 1}[op], st.cuda_stream),
           "dci_block_aggregate")
    return H


def presample(ctx: Context, seeds, batch: int, fanouts, seed: int, node_visits, edge_counts, stream=None):
    """dci_presample (S1): accumulates into node_visits int32[N] / edge_counts int32[E] (CUDA
    tensors); returns host uint64 arrays (t_sample_ns, t_feature_ns), one entry per batch."""
    _device_i32(seeds, "seeds", ctx.device)
    _device_i32(node_visits, "node_visits", ctx.device)
    if ctx.E:
        _device_i32(edge_counts, "edge_counts", ctx.device)
    fan = np.ascontiguousarray(fanouts, np.int32)
    n = int(seeds.numel())
    nb = (n + batch - 1) // batch
    ts = np.zeros(max(nb, 1), np.uint64)
    tf = np.zeros(max(nb, 1), np.uint64)
    _check(lib().dci_presample(ctx.handle, seeds.data_ptr(), n, batch, _np_ptr(fan), len(fan), seed,
                               node_visits.data_ptr(), _t_ptr(edge_counts) if ctx.E else None, _np_ptr(ts),
                               _np_ptr(tf), _stream_ptr(stream)), "dci_presample")
    return ts[:nb], tf[:nb]


def allocate(ctx: Context | None, C_bytes: int, t_sample=(), t_feature=(), ratio=None):
    """dci_allocate (S2, Eq. 1).  C_bytes = 0 -> auto budget.  ratio=(num, den) overrides."""
    ts = np.ascontiguousarray(t_sample, np.uint64).reshape(-1)
    tf = np.ascontiguousarray(t_feature, np.uint64).reshape(-1)
    n = len(ts)
    if n == 0:
        ts = np.zeros(1, np.uint64)
        tf = np.zeros(1, np.uint64)
    num, den = (0, 0) if ratio is None else ratio
    a, f = C.c_uint64(), C.c_uint64()
    _check(lib().dci_allocate(ctx.handle if ctx else None, C_bytes, _np_ptr(ts), _np_ptr(tf), n, num, den,
                              C.byref(a), C.byref(f)), "dci_allocate")
    return int(a.value), int(f.value)


def fill(ctx: Context, node_visits, edge_counts, c_adj: int, c_feat: int, stream=None):
    """dci_fill (S3 + S4)."""
    _counts_ok(ctx, node_visits, edge_counts)
    _check(lib().dci_fill(ctx.handle, node_visits.data_ptr(), _t_ptr(edge_counts) if ctx.E else None, c_adj,
                          c_feat, _stream_ptr(stream)), "dci_fill")


def fill_partitioned(ctx: Context, node_visits, edge_counts, c_adj: int, c_feat: int, world: int, rank: int,
                     stream=None):
    """dci_fill_partitioned (NEXT F1): the feature cache spans `world` partitions (c_feat per
    partition); rank -1 = all partitions on this device (emulation)."""
    _counts_ok(ctx, node_visits, edge_counts)
    _check(lib().dci_fill_partitioned(ctx.handle, node_visits.data_ptr(), _t_ptr(edge_counts) if ctx.E else None,
                                      c_adj, c_feat, world, rank, _stream_ptr(stream)), "dci_fill_partitioned")


def fill_knapsack(ctx: Context, node_visits, edge_counts, C_bytes: int, cost_feat: float, cost_adj: float,
                  stream=None):
    """dci_fill_knapsack (NEXT F4): DUCATI-style unified-budget greedy fill (comparison)."""
    _counts_ok(ctx, node_visits, edge_counts)
    _check(lib().dci_fill_knapsack(ctx.handle, node_visits.data_ptr(), _t_ptr(edge_counts) if ctx.E else None,
                                   C_bytes, float(cost_feat), float(cost_adj), _stream_ptr(stream)),
           "dci_fill_knapsack")


def feature_partition_handle(ctx: Context) -> bytes:
    """dci_feature_partition_handle: 64-byte CUDA IPC handle of this device's partition."""
    buf = (C.c_char * IPC_HANDLE_BYTES)()
    _check(lib().dci_feature_partition_handle(ctx.handle, buf), "dci_feature_partition_handle")
    return bytes(buf)


def attach_feature_partitions(ctx: Context, handles):
    """dci_attach_feature_partitions: open the other ranks' partitions (rank-major handles)."""
    blob = b"".join(handles)
    buf = (C.c_char * len(blob)).from_buffer_copy(blob)
    _check(lib().dci_attach_feature_partitions(ctx.handle, buf, len(handles)), "dci_attach_feature_partitions")


def cache_info(ctx: Context) -> dict:
    info = dci_cache_info()
    _check(lib().dci_cache_info_get(ctx.handle, C.byref(info)), "dci_cache_info_get")
    return {k: getattr(info, k) for k, _ in dci_cache_info._fields_}


def fill_times(ctx: Context) -> dict:
    """dci_fill_times_get: stage times (ms) of the context's last fill."""
    t = dci_fill_times()
    _check(lib().dci_fill_times_get(ctx.handle, C.byref(t)), "dci_fill_times_get")
    return {k: float(getattr(t, k)) for k, _ in dci_fill_times._fields_}


def cache_state(ctx: Context) -> dict:
    """dci_cache_state: host copies of the directory cache fields, both caches and the current
    host CSC."""
    info = cache_info(ctx)
    N, E, pitch = info["N"], info["E"], info["pitch"]
    cl = np.zeros(N, np.int32)
    co = np.zeros(N, np.int64)
    so = np.zeros(N, np.int32)
    ac = np.zeros(max(info["adj_elems"], 1), np.int32)
    fc = np.zeros((max(info["feat_rows"], 1), pitch), np.float32)
    ix = np.zeros(max(E, 1), np.int32)
    _check(lib().dci_cache_state(ctx.handle, _np_ptr(cl), _np_ptr(co), _np_ptr(so), _np_ptr(ac), _np_ptr(fc),
                                 _np_ptr(ix)), "dci_cache_state")
    return {"cached_len": cl, "cache_off": co, "slot_of": so, "acache": ac[: info["adj_elems"]],
            "fcache": fc[: info["feat_rows"]], "indices_cur": ix[:E], "info": info}
