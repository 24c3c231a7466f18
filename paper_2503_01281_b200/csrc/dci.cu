// C-ABI of libdci (include/dci.h): context lifecycle, workspaces, presample (S1), Eq. (1)
// allocation (S2), fill (S3/S4, fill.cu) and the per-batch hot loop (S5-S8, sample.cu /
// gather.cu).  Host code only orchestrates: every step of the path runs in a kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <mutex>
#include <string>
#include <thread>
#include <vector>
#include <unordered_map>

#include "dci_internal.cuh"

namespace dci {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

dci_status fail(dci_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

dci_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? DCI_ENOMEM : DCI_ECUDA;
}

int occupancy_blocks(const void* kernel, int block, int cap) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  // cache the raw occupancy per kernel; the cap differs between calls
  auto it = cache.find(kernel);
  int n;
  if (it != cache.end()) {
    n = it->second;
  } else {
    n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, 0) != cudaSuccess || n < 1) n = 1;
    cache[kernel] = n;
  }
  return std::min(n, cap);
}

namespace {

// Run body(lo, hi) over [0, n) on up to hardware_concurrency host threads (load-time copies and
// validation of graphs with billions of edges; not on the per-batch path).
template <class F>
void parallel_for(int64_t n, int64_t grain, F body) {
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw, n / std::max<int64_t>(grain, 1)));
  if (nt <= 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo < hi) th.emplace_back(body, lo, hi);
  }
  for (auto& x : th) x.join();
}

bool gather_serial() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("DCI_GATHER_SERIAL");
    mode = (e && e[0] == '1') ? 1 : 0;
  }
  return mode == 1;
}

// TMA gather: DCI_GATHER_SERIAL=0 lets gathers of concurrent batches overlap (experiments)
bool gather_concurrent() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("DCI_GATHER_SERIAL");
    mode = (e && e[0] == '0') ? 1 : 0;
  }
  return mode == 1;
}

bool graph_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("DCI_GRAPH");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// |F_h| <= min(N, B * prod_{j<h} (1 + f_j)), hop j using fanouts[L-1-j] (reading C3).
void frontier_bounds(int64_t N, int64_t B, const int32_t* fan, int32_t L, int64_t* caps) {
  caps[0] = std::min<int64_t>(N, B);
  for (int h = 0; h < L; ++h) {
    const int64_t f = fan[L - 1 - h];
    const double est = (double)caps[h] * (double)(1 + f);
    caps[h + 1] = est >= (double)N ? N : std::min<int64_t>(N, caps[h] * (1 + f));
  }
}

dci_status check_fanouts(const int32_t* fanouts, int32_t L) {
  if (!fanouts || L < 1 || L > DCI_MAX_LAYERS) return fail(DCI_EINVAL, "L must be in [1, DCI_MAX_LAYERS]");
  for (int i = 0; i < L; ++i)
    if (fanouts[i] < 1 || fanouts[i] > DCI_MAX_FANOUT) return fail(DCI_EINVAL, "fan-out must be in [1, 1024]");
  return DCI_OK;
}

// Fold a timing record into the workspace totals (waits for its last event).
dci_status trec_fold(dci_workspace* ws, dci_workspace::TimeRec& r) {
  if (r.state & 1) {
    float ms = 0.f;
    DCI_CUDA(cudaEventSynchronize(r.e[1]));
    DCI_CUDA(cudaEventElapsedTime(&ms, r.e[0], r.e[1]));
    ws->acc_sample_ms += ms;
    ws->acc_timed += r.nb;
  }
  if (r.state & 2) {
    float ms = 0.f;
    DCI_CUDA(cudaEventSynchronize(r.e[3]));
    if (r.state & 4) {  // split gather: the two launches, without the wait between them
      float ms2 = 0.f;
      DCI_CUDA(cudaEventElapsedTime(&ms, r.e[2], r.e[4]));
      DCI_CUDA(cudaEventElapsedTime(&ms2, r.e[5], r.e[3]));
      ms += ms2;
      ws->acc_gather_launches += 2;
    } else {
      DCI_CUDA(cudaEventElapsedTime(&ms, r.e[2], r.e[3]));
      ws->acc_gather_launches += 1;
    }
    ws->acc_gather_ms += ms;
  }
  r.state = 0;
  return DCI_OK;
}

// Advance to the workspace's next timing record, folding the one it reuses (issued kTimeRing
// batches ago on this workspace, so normally long finished: no host stall).
dci_status trec_begin(dci_workspace* ws) {
  ws->trec_cur = (ws->trec_cur + 1) % dci_workspace::kTimeRing;
  return trec_fold(ws, ws->trec[ws->trec_cur]);
}

// Parameters of the last hop's relabel (a virtual hop L whose "previous hop" is hop L-1).
HopParams epilogue_params(dci_workspace* ws, int32_t L, const int32_t* fanouts, const dci_batch_out* out) {
  HopParams e{};
  e.F = out->frontier;
  e.hop = L;
  e.f = 1;
  e.prev_cand = ws->cand[(L - 1) & 1];
  e.prev_kcnt = ws->kcnt[(L - 1) & 1];
  e.prev_bptr = out->bptr[L - 1];
  e.prev_bsrc = out->bsrc[L - 1];
  e.prev_f = fanouts[0];
  return e;
}

// Argument checks of one batch (dci_sample_gather, _many, presample).
dci_status validate_batch(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds, int32_t B, const int32_t* fanouts,
                          int32_t L, const dci_batch_out* out) {
  if (ws->ctx != ctx) return fail(DCI_EINVAL, "workspace belongs to another context");
  dci_status st = check_fanouts(fanouts, L);
  if (st != DCI_OK) return st;
  if (!out || !out->frontier || !out->sizes || !out->counters || !out->status)
    return fail(DCI_EINVAL, "dci_batch_out has a null required pointer");
  if (B < 0 || B > ws->max_batch) return fail(DCI_EINVAL, "B exceeds the workspace's max_batch");
  if (B > 0 && !seeds) return fail(DCI_EINVAL, "seeds is null");
  if (L != ws->L) return fail(DCI_EINVAL, "L differs from the workspace's L");
  for (int i = 0; i < L; ++i)
    if (fanouts[i] > ws->max_fan[i]) return fail(DCI_EINVAL, "fan-out exceeds the workspace's max_fanouts");
  int64_t caps[DCI_MAX_LAYERS + 1];
  frontier_bounds(ctx->N, B, fanouts, L, caps);
  if (out->frontier_cap < caps[L]) return fail(DCI_ECAP, "frontier_cap < dci_output_bounds");
  for (int h = 0; h < L; ++h) {
    const int64_t f = fanouts[L - 1 - h];
    if (!out->bptr[h] || !out->bsrc[h]) return fail(DCI_EINVAL, "null bptr/bsrc");
    if (out->hop_cap[h] < caps[h] || out->bsrc_cap[h] < caps[h] * f)
      return fail(DCI_ECAP, "hop_cap/bsrc_cap < dci_output_bounds");
  }
  if (out->X && out->ldx < ctx->D) return fail(DCI_EINVAL, "ldx < D");
  return DCI_OK;
}

// Per-batch header (seeds pointer, B, seed, table epoch): pinned ring -> the workspace's device
// scalars, on stream s, ahead of the batch's kernels (which are a fixed CUDA graph).
dci_status stage_header(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds, int32_t B, uint64_t seed,
                        cudaStream_t s) {
  if (++ws->epoch == 0) {  // 2^32 batches on this workspace: clear the tag table once
    DCI_CUDA(cudaMemsetAsync(ws->pos_of, 0, ws->table_bytes, s));
    ws->epoch = 1;
  }
  const int slot = (int)(ws->calls++ % dci_workspace::kHdrRing);
  DCI_CUDA(cudaEventSynchronize(ws->hdr_ev[slot]));  // the copy that last used this slot is done
  BatchHeader* hh = ws->hdr_ring + slot;
  hh->seeds = seeds;
  hh->seed = seed;
  hh->B = B;
  hh->epoch = ws->epoch;
  DCI_CUDA(cudaMemcpyAsync(&ws->scal->hdr, hh, sizeof(BatchHeader), cudaMemcpyHostToDevice, s));
  DCI_CUDA(cudaEventRecord(ws->hdr_ev[slot], s));
  return DCI_OK;
}

// Enqueue one batch (shared by inference pass 0 and presample pass 1).
dci_status run_batch(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds, int32_t B, const int32_t* fanouts,
                     int32_t L, uint64_t seed, uint32_t pass, const dci_batch_out* out, int32_t* node_visits,
                     int32_t* edge_counts, cudaStream_t s) {
  dci_status st = validate_batch(ctx, ws, seeds, B, fanouts, L, out);
  if (st != DCI_OK) return st;
  DeviceGuard g(ctx->device);
  const bool prof = ws->profiling || pass == 1;
  dci_workspace::TimeRec* tr = nullptr;
  if (prof) {
    dci_status ts = trec_begin(ws);
    if (ts != DCI_OK) return ts;
    tr = &ws->trec[ws->trec_cur];
    tr->nb = 1;
  }
  st = stage_header(ctx, ws, seeds, B, seed, s);
  if (st != DCI_OK) return st;

  // ---- kernels: a CUDA graph per workspace, re-captured only when the signature changes ----
  struct Sig {
    int32_t L, pass, prof, serial, tma;
    int32_t fan[DCI_MAX_LAYERS];
    dci_batch_out out;
    const int32_t* nv;
    const int32_t* ec;
    const void* acache;
    const void* fcache;
    const void* uidx;
    const void* fbases;
    int32_t G;
    int32_t gather_bps;
  } sig;
  // TMA gather: the last hop's relabel runs as its own kernel; inference gathers are serialised
  // on the context's gather stream (one at a time at full bandwidth, beside other batches'
  // sampling).  Register-copy gather: relabel fused, gathers of concurrent batches overlap
  // unless DCI_GATHER_SERIAL=1.
  const bool tma = gather_uses_tma(ctx, out);
  const bool serial = pass == 0 && (tma ? !gather_concurrent() : gather_serial());
  memset(&sig, 0, sizeof(sig));
  sig.L = L;
  sig.pass = (int32_t)pass;
  sig.prof = prof ? 1 : 0;
  sig.serial = serial ? 1 : 0;
  sig.tma = tma ? 1 : 0;
  for (int i = 0; i < L; ++i) sig.fan[i] = fanouts[i];
  sig.out = *out;
  sig.nv = node_visits;
  sig.ec = edge_counts;
  sig.acache = ctx->d_acache;
  sig.fcache = ctx->d_fcache;
  sig.uidx = ctx->u_idx_cur;
  sig.fbases = ctx->d_fbases;
  sig.G = ctx->fpart_world;
  sig.gather_bps = gather_blocks_per_sm(ctx);
  static_assert(sizeof(Sig) <= sizeof(ws->graph_sig), "signature buffer too small");
  const bool use_graph = graph_mode();
  const bool need_capture =
      use_graph && !(ws->n_graphs && ws->graph_sig_len == sizeof(Sig) && !memcmp(ws->graph_sig, &sig, sizeof(Sig)));
  HopParams last{};
  last.f = fanouts[0];
  last.cand = ws->cand[(L - 1) & 1];
  last.kcnt = ws->kcnt[(L - 1) & 1];
  const HopParams epi = epilogue_params(ws, L, fanouts, out);
  // part 0: the L sampling hops (+ the last hop's relabel when the gather does not fuse it and
  // runs on the same stream); part 1: the route + gather kernel; part 2 (serial TMA gather only):
  // the last hop's relabel, on the sampling stream while the gather runs on the gather stream
  const bool relabel_apart = tma && serial;
  ws->in_group = 0;
  auto enqueue_part = [&](int part, cudaStream_t es) {
    if (part == 0) {
      HopParams prev{};
      for (int h = 0; h < L; ++h) {
        HopParams p{};
        p.F = out->frontier;
        p.hop = h;
        p.f = fanouts[L - 1 - h];
        p.pass = pass;
        p.cand = ws->cand[h & 1];
        p.kcnt = ws->kcnt[h & 1];
        if (h > 0) {
          p.prev_cand = prev.cand;
          p.prev_kcnt = prev.kcnt;
          p.prev_bptr = out->bptr[h - 1];
          p.prev_bsrc = out->bsrc[h - 1];
          p.prev_f = prev.f;
        }
        p.bptr = out->bptr[h];
        p.edge_counts = edge_counts;
        launch_sample_hop(ctx, &ws, &p, 1, es);
        launch_scan_hop(ctx, &ws, &p, 1, es);
        prev = p;
      }
      if (tma && !relabel_apart) launch_hop_epilogue(ctx, &ws, &epi, 1, es);
    } else if (part == 1) {
      launch_gather_fused(ctx, ws, L, out, last, node_visits, es);
    } else {
      launch_hop_epilogue(ctx, &ws, &epi, 1, es);
    }
  };
  const int nparts = relabel_apart ? 3 : 2;
  if (need_capture) {
    // one graph per part when profiling (stage events go between them) or when the gather runs
    // on the gather stream; else one graph
    const int ngraphs = (prof || serial) ? nparts : 1;
    for (int gi = 0; gi < 3; ++gi) {
      if (ws->graph_exec[gi]) cudaGraphExecDestroy(ws->graph_exec[gi]);
      ws->graph_exec[gi] = nullptr;
    }
    ws->n_graphs = 0;
    // the cached signature matches no batch until every graph of this shape is built (a failed
    // capture of graph gi >= 1 must not leave a signature that skips capture next time)
    ws->graph_sig_len = 0;
    for (int gi = 0; gi < ngraphs; ++gi) {
      const uint64_t launches0 = ctx->launches;
      DCI_CUDA(cudaStreamBeginCapture(ws->cap_stream, cudaStreamCaptureModeThreadLocal));
      if (ngraphs > 1) {
        enqueue_part(gi, ws->cap_stream);
      } else {
        enqueue_part(0, ws->cap_stream);
        enqueue_part(1, ws->cap_stream);
      }
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamEndCapture(ws->cap_stream, &graph);
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      ws->graph_kernels[gi] = ctx->launches - launches0;
      ctx->launches = launches0;  // counted when the graph actually runs
      e = cudaGraphInstantiate(&ws->graph_exec[gi], graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      ws->n_graphs = gi + 1;
    }
    memcpy(ws->graph_sig, &sig, sizeof(Sig));
    ws->graph_sig_len = sizeof(Sig);
  }
  auto run_part = [&](int part, cudaStream_t rs) -> cudaError_t {
    if (!use_graph) {
      enqueue_part(part, rs);
      return cudaSuccess;
    }
    if (ws->n_graphs > 1) {
      ctx->launches += ws->graph_kernels[part];
      return cudaGraphLaunch(ws->graph_exec[part], rs);
    }
    if (part == 0) {
      ctx->launches += ws->graph_kernels[0];
      return cudaGraphLaunch(ws->graph_exec[0], rs);
    }
    return cudaSuccess;  // single graph holds both parts
  };
  if (prof) DCI_CUDA(cudaEventRecord(tr->e[0], s));
  DCI_CUDA(run_part(0, s));
  if (prof) {
    DCI_CUDA(cudaEventRecord(tr->e[1], s));
    tr->state |= 1;
  }
  if (serial) {
    DCI_CUDA(cudaEventRecord(ws->ev_mid, s));
    DCI_CUDA(cudaStreamWaitEvent(ctx->gstream, ws->ev_mid, 0));
    if (prof) DCI_CUDA(cudaEventRecord(tr->e[2], ctx->gstream));
    DCI_CUDA(run_part(1, ctx->gstream));
    if (prof) DCI_CUDA(cudaEventRecord(tr->e[3], ctx->gstream));
    DCI_CUDA(cudaEventRecord(ws->ev_done, ctx->gstream));
    if (relabel_apart) DCI_CUDA(run_part(2, s));
    DCI_CUDA(cudaStreamWaitEvent(s, ws->ev_done, 0));
  } else {
    if (prof) DCI_CUDA(cudaEventRecord(tr->e[2], s));
    DCI_CUDA(run_part(1, s));
    if (prof) DCI_CUDA(cudaEventRecord(tr->e[3], s));
  }
  if (prof) tr->state |= 2;
  DCI_CUDA(cudaGetLastError());
  return DCI_OK;
}

void free_ctx(dci_ctx* c) {
  if (!c) return;
  if (c->pre_ws) dci_workspace_destroy(c->pre_ws);
  if (c->pre_out_mem) cudaFree(c->pre_out_mem);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  if (c->gather_ev) cudaEventDestroy(c->gather_ev);
  if (c->gather_q_ev) cudaEventDestroy(c->gather_q_ev);
  if (c->d_dir) cudaFree(c->d_dir);
  if (c->d_acache) cudaFree(c->d_acache);
  release_feature_partitions(c);
  if (c->d_fbases) cudaFree(c->d_fbases);
  if (c->d_fcache) cudaFree(c->d_fcache);
  if (c->h_idx_cur && c->h_idx_cur != c->h_idx_orig) cudaFreeHost(c->h_idx_cur);
  // adopted caller memory (DCI_ADOPT_HOST) is only unregistered, never freed
  if (c->h_idx_orig) (c->adopted_idx ? cudaHostUnregister(c->h_idx_orig) : cudaFreeHost(c->h_idx_orig));
  if (c->h_feats) (c->adopted_feats ? cudaHostUnregister(c->h_feats) : cudaFreeHost(c->h_feats));
  free(c->h_indptr);
  delete c;
}

}  // namespace
}  // namespace dci

using namespace dci;

extern "C" {

const char* dci_last_error(void) { return g_last_error.c_str(); }
int32_t dci_version(void) { return DCI_VERSION; }

dci_status dci_load_graph(dci_ctx** out, int device, int64_t N, int64_t E, const int64_t* indptr,
                          const int32_t* indices, const float* feats, int32_t D, uint32_t flags) {
  if (!out) return fail(DCI_EINVAL, "out is null");
  *out = nullptr;
  if ((flags & ~(uint32_t)DCI_ADOPT_HOST) != 0) return fail(DCI_EINVAL, "unknown flags");
  const bool adopt = (flags & DCI_ADOPT_HOST) != 0;
  if (N < 1 || N >= (1ll << 31)) return fail(DCI_EINVAL, "N must be in [1, 2^31)");
  if (E < 0 || E >= (1ll << 40)) return fail(DCI_EINVAL, "E must be in [0, 2^40)");
  if (D < 1) return fail(DCI_EINVAL, "D must be >= 1");
  if (!indptr || (E > 0 && !indices) || !feats) return fail(DCI_EINVAL, "null input pointer");
  // CSC invariants: monotone column pointers, ids in range
  if (indptr[0] != 0 || indptr[N] != E) return fail(DCI_EINVAL, "indptr[0] must be 0 and indptr[N] == E");
  for (int64_t v = 0; v < N; ++v) {
    if (indptr[v + 1] < indptr[v]) return fail(DCI_EINVAL, "indptr must be non-decreasing");
    if (indptr[v + 1] - indptr[v] >= (1ll << 31)) return fail(DCI_ERANGE, "a degree exceeds 2^31-1");
  }
  std::atomic<bool> bad_index{false};
  parallel_for(E, 1 << 24, [&](int64_t lo, int64_t hi) {
    bool bad = false;
    for (int64_t e = lo; e < hi; ++e) bad |= indices[e] < 0 || (int64_t)indices[e] >= N;
    if (bad) bad_index = true;
  });
  if (bad_index) return fail(DCI_EINVAL, "indices entry out of [0, N)");
  int ndev = 0;
  DCI_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(DCI_EINVAL, "bad device ordinal");
  DeviceGuard g(device);
  dci_ctx* c = new (std::nothrow) dci_ctx();
  if (!c) return fail(DCI_ENOMEM, "host allocation failed");
  c->device = device;
  c->N = N;
  c->E = E;
  c->D = D;
  c->pitch = (D + 3) / 4 * 4;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  auto bail = [&](dci_status s) {
    free_ctx(c);
    return s;
  };
  c->h_indptr = static_cast<int64_t*>(malloc(sizeof(int64_t) * (N + 1)));
  if (!c->h_indptr) return bail(fail(DCI_ENOMEM, "host allocation failed"));
  // the context's gather stream (group gathers and serial gathers run one at a time on it);
  // created here so concurrent callers with distinct workspaces never race on it
  if (cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->gather_ev, kCrossStreamEvent) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->gather_q_ev, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(DCI_ECUDA, "cudaStreamCreate(gather stream)"));
  memcpy(c->h_indptr, indptr, sizeof(int64_t) * (N + 1));
  cudaError_t e;
  const int64_t pitch = c->pitch;
  const size_t fbytes = sizeof(float) * (size_t)N * c->pitch;
  if (adopt) {
    // DCI_ADOPT_HOST: register the caller's buffers in place (pinned + mapped, portable), e.g. one
    // node-shared POSIX shm segment that every rank's context adopts; the library never writes them
    if (E > 0) {
      e = cudaHostRegister(const_cast<int32_t*>(indices), sizeof(int32_t) * (size_t)E,
                           cudaHostRegisterMapped | cudaHostRegisterPortable);
      if (e != cudaSuccess) return bail(cuda_fail(e, "cudaHostRegister(indices)"));
      c->h_idx_orig = const_cast<int32_t*>(indices);
      c->adopted_idx = true;
    }
    e = cudaHostRegister(const_cast<float*>(feats), fbytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaHostRegister(feats)"));
    c->h_feats = const_cast<float*>(feats);
    c->adopted_feats = true;
  }
  if (!c->adopted_idx) {
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_idx_orig), sizeof(int32_t) * std::max<int64_t>(E, 1),
                      cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaHostAlloc(indices)"));
    parallel_for(E, 1 << 24, [&](int64_t lo, int64_t hi) {
      memcpy(c->h_idx_orig + lo, indices + lo, sizeof(int32_t) * (hi - lo));
    });
  }
  c->h_idx_cur = c->h_idx_orig;
  if (!c->adopted_feats) {
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->h_feats), fbytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaHostAlloc(feats)"));
    parallel_for(N, 1 << 16, [&](int64_t lo, int64_t hi) {
      if (pitch == D) {
        memcpy(c->h_feats + lo * pitch, feats + lo * D, sizeof(float) * D * (hi - lo));
      } else {
        for (int64_t v = lo; v < hi; ++v) {
          memcpy(c->h_feats + v * pitch, feats + v * D, sizeof(float) * D);
          memset(c->h_feats + v * pitch + D, 0, sizeof(float) * (pitch - D));
        }
      }
    });
  }
  void* dp = nullptr;
  if ((e = cudaHostGetDevicePointer(&dp, c->h_idx_orig, 0)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaHostGetDevicePointer"));
  c->u_idx_orig = c->u_idx_cur = static_cast<const int32_t*>(dp);
  if ((e = cudaHostGetDevicePointer(&dp, c->h_feats, 0)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaHostGetDevicePointer"));
  c->u_feats = static_cast<const float*>(dp);
  if ((e = cudaMalloc(&c->d_dir, sizeof(DirEntry) * N)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(dir)"));
  int64_t* d_indptr = nullptr;
  if ((e = cudaMalloc(&d_indptr, sizeof(int64_t) * (N + 1))) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc"));
  cudaMemcpy(d_indptr, indptr, sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice);
  launch_build_directory(c, d_indptr, 0);
  e = cudaDeviceSynchronize();
  cudaFree(d_indptr);
  if (e != cudaSuccess) return bail(cuda_fail(e, "build directory"));
  c->state = DCI_STATE_LOADED;
  *out = c;
  return DCI_OK;
}

dci_status dci_destroy(dci_ctx* ctx) {
  if (!ctx) return DCI_OK;
  DeviceGuard g(ctx->device);
  cudaDeviceSynchronize();
  free_ctx(ctx);
  return DCI_OK;
}

dci_status dci_output_bounds(const dci_ctx* ctx, int32_t B, const int32_t* fanouts, int32_t L,
                             int64_t* frontier_caps, int64_t* bsrc_caps, int32_t* pitch) {
  if (!ctx || B < 0) return fail(DCI_EINVAL, "bad arguments");
  dci_status st = check_fanouts(fanouts, L);
  if (st != DCI_OK) return st;
  int64_t caps[DCI_MAX_LAYERS + 1];
  frontier_bounds(ctx->N, B, fanouts, L, caps);
  for (int h = 0; h < L; ++h)
    if (caps[h] * (fanouts[L - 1 - h] + 1) >= (1ll << 31))
      return fail(DCI_ERANGE, "batch too large: |F_h| * (f + 1) must stay < 2^31");
  for (int h = 0; h <= L; ++h)
    if (frontier_caps) frontier_caps[h] = caps[h];
  for (int h = 0; h < L; ++h)
    if (bsrc_caps) bsrc_caps[h] = caps[h] * fanouts[L - 1 - h];
  if (pitch) *pitch = ctx->pitch;
  return DCI_OK;
}

static dci_status workspace_create(dci_ctx* ctx, int32_t max_batch, const int32_t* max_fanouts, int32_t L,
                                   dci_workspace** out, bool user);

dci_status dci_workspace_create(dci_ctx* ctx, int32_t max_batch, const int32_t* max_fanouts, int32_t L,
                                dci_workspace** out) {
  return workspace_create(ctx, max_batch, max_fanouts, L, out, true);
}

static dci_status workspace_create(dci_ctx* ctx, int32_t max_batch, const int32_t* max_fanouts, int32_t L,
                                   dci_workspace** out, bool user) {
  if (!ctx || !out || max_batch < 1) return fail(DCI_EINVAL, "bad arguments");
  *out = nullptr;
  dci_status st = check_fanouts(max_fanouts, L);
  if (st != DCI_OK) return st;
  DeviceGuard g(ctx->device);
  dci_workspace* w = new (std::nothrow) dci_workspace();
  if (!w) return fail(DCI_ENOMEM, "host allocation failed");
  static std::atomic<uint64_t> next_uid{1};
  w->ctx = ctx;
  w->uid = next_uid++;
  w->device = ctx->device;
  w->max_batch = max_batch;
  w->L = L;
  for (int i = 0; i < L; ++i) w->max_fan[i] = max_fanouts[i];
  frontier_bounds(ctx->N, max_batch, max_fanouts, L, w->hop_cap);
  int64_t max_front = 0;
  for (int h = 0; h <= L; ++h) max_front = std::max(max_front, w->hop_cap[h]);
  for (int h = 0; h < L; ++h)
    if (w->hop_cap[h] * (max_fanouts[L - 1 - h] + 1) >= (1ll << 31)) {
      delete w;
      return fail(DCI_ERANGE, "batch too large: |F_h| * (f + 1) must stay < 2^31");
    }
  w->cand_cap = 0;
  w->tiles_cap = 0;
  for (int h = 0; h < L; ++h) {
    w->cand_cap = std::max(w->cand_cap, w->hop_cap[h] * max_fanouts[L - 1 - h]);
    w->tile_off[h] = w->tiles_cap;
    w->tiles_cap += (w->hop_cap[h] + kScanDsts - 1) / kScanDsts + 1;
  }
  w->tile_off[L] = w->tiles_cap;
  auto bail = [&](cudaError_t e, const char* what) {
    dci_workspace_destroy(w);
    return cuda_fail(e, what);
  };
  cudaError_t e;
  // position table layout (dci_internal.cuh): hashed when the dense table (8 N bytes) would be more
  // than 4x the hashed one (16 B x pow2 >= 2 x the frontier bound) -- papers100M-shaped graphs;
  // env DCI_TABLE=dense|hash overrides
  {
    static const int forced = [] {
      const char* v = getenv("DCI_TABLE");
      return !v ? 0 : (v[0] == 'd' ? 1 : (v[0] == 'h' ? 2 : 0));
    }();
    uint64_t cap = 1;
    while (cap < 2ull * (uint64_t)std::max<int64_t>(w->hop_cap[L], 1)) cap <<= 1;
    const uint64_t dense_b = 8ull * (uint64_t)ctx->N, hash_b = 16ull * cap;
    const bool hashed = cap <= (1ull << 31) && (forced == 2 || (forced == 0 && dense_b > 4 * hash_b));
    w->hmask = hashed ? (uint32_t)(cap - 1) : 0u;
    w->table_bytes = hashed ? hash_b : dense_b;
  }
  if ((e = cudaMalloc(&w->pos_of, w->table_bytes)) != cudaSuccess) return bail(e, "cudaMalloc(pos_of)");
  for (int i = 0; i < 2; ++i) {
    if ((e = cudaMalloc(&w->cand[i], sizeof(int32_t) * std::max<int64_t>(w->cand_cap, 1))) != cudaSuccess)
      return bail(e, "cudaMalloc(cand)");
    if ((e = cudaMalloc(&w->kcnt[i], sizeof(int32_t) * std::max<int64_t>(max_front, 1))) != cudaSuccess)
      return bail(e, "cudaMalloc(kcnt)");
  }
  if ((e = cudaMalloc(&w->nmask, sizeof(uint32_t) * std::max<int64_t>(max_front, 1))) != cudaSuccess)
    return bail(e, "cudaMalloc(nmask)");
  if ((e = cudaMalloc(&w->tile_state, sizeof(unsigned long long) * w->tiles_cap)) != cudaSuccess)
    return bail(e, "cudaMalloc(tile_state)");
  if ((e = cudaMalloc(&w->scal, sizeof(BatchScalars))) != cudaSuccess) return bail(e, "cudaMalloc(scal)");
  if ((e = cudaMalloc(&w->seeds_stage, sizeof(int32_t) * max_batch)) != cudaSuccess) return bail(e, "cudaMalloc");
  for (auto& r : w->trec)
    for (auto& ev : r.e)
      if ((e = cudaEventCreate(&ev)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaEventCreateWithFlags(&w->ev_mid, kCrossStreamEvent)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaEventCreateWithFlags(&w->ev_pre, kCrossStreamEvent)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaEventCreateWithFlags(&w->ev_done, kCrossStreamEvent)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaEventCreateWithFlags(&w->gseeds_ev, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaHostAlloc(reinterpret_cast<void**>(&w->hdr_ring), sizeof(BatchHeader) * dci_workspace::kHdrRing,
                         cudaHostAllocPortable)) != cudaSuccess)
    return bail(e, "cudaHostAlloc(header ring)");
  for (int i = 0; i < dci_workspace::kHdrRing; ++i)
    if ((e = cudaEventCreateWithFlags(&w->hdr_ev[i], cudaEventDisableTiming)) != cudaSuccess) return bail(e, "event");
  if ((e = cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking)) != cudaSuccess) return bail(e, "stream");
  cudaMemset(w->pos_of, 0, w->table_bytes);
  cudaMemset(w->tile_state, 0, sizeof(unsigned long long) * w->tiles_cap);
  cudaMemset(w->scal, 0, sizeof(BatchScalars));
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "workspace init");
  if (user) {
    w->live_ws = ctx->live_ws;
    ++*w->live_ws;
  }
  *out = w;
  return DCI_OK;
}

dci_status dci_workspace_destroy(dci_workspace* w) {
  if (!w) return DCI_OK;
  DeviceGuard g(w->device);
  cudaDeviceSynchronize();
  cudaFree(w->pos_of);
  for (int i = 0; i < 2; ++i) {
    cudaFree(w->cand[i]);
    cudaFree(w->kcnt[i]);
  }
  cudaFree(w->nmask);
  cudaFree(w->tile_state);
  cudaFree(w->scal);
  cudaFree(w->seeds_stage);
  for (auto& r : w->trec)
    for (auto& ev : r.e)
      if (ev) cudaEventDestroy(ev);
  for (int i = 0; i < dci_workspace::kHdrRing; ++i)
    if (w->hdr_ev[i]) cudaEventDestroy(w->hdr_ev[i]);
  if (w->ev_mid) cudaEventDestroy(w->ev_mid);
  if (w->ev_pre) cudaEventDestroy(w->ev_pre);
  if (w->ev_done) cudaEventDestroy(w->ev_done);

  if (w->hdr_ring) cudaFreeHost(w->hdr_ring);
  for (int i = 0; i < 3; ++i)
    if (w->graph_exec[i]) cudaGraphExecDestroy(w->graph_exec[i]);
  for (auto& c : w->gg) {
    if (c.exec) cudaGraphExecDestroy(c.exec);
    if (c.exec2) cudaGraphExecDestroy(c.exec2);
    free(c.sig);
  }
  if (w->ghdr_ring) cudaFreeHost(w->ghdr_ring);
  if (w->ghdr_dev) cudaFree(w->ghdr_dev);
  for (auto& ev : w->ghdr_ev)
    if (ev) cudaEventDestroy(ev);
  if (w->stage) cudaFree(w->stage);
  if (w->gseeds_host) cudaFreeHost(w->gseeds_host);
  if (w->gseeds_dev) cudaFree(w->gseeds_dev);
  if (w->gseeds_ev) cudaEventDestroy(w->gseeds_ev);
  if (w->live_ws) --*w->live_ws;
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  delete w;
  return DCI_OK;
}

dci_status dci_sample_gather(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds, int32_t B,
                             const int32_t* fanouts, int32_t L, uint64_t seed, const dci_batch_out* out,
                             void* stream) {
  if (!ctx || !ws) return fail(DCI_EINVAL, "null context/workspace");
  return run_batch(ctx, ws, seeds, B, fanouts, L, seed, 0, out, nullptr, nullptr,
                   static_cast<cudaStream_t>(stream));
}

dci_status dci_sample_gather_many(dci_ctx* ctx, int32_t n, dci_workspace* const* ws, const int32_t* const* seeds,
                                  const int32_t* B, const int32_t* fanouts, int32_t L, uint64_t seed,
                                  const dci_batch_out* outs, void* stream) {
  if (!ctx || !ws || !seeds || !B || !outs) return fail(DCI_EINVAL, "null argument");
  if (n < 1 || n > DCI_MAX_GROUP) return fail(DCI_EINVAL, "n must be in [1, DCI_MAX_GROUP]");
  for (int i = 0; i < n; ++i) {
    if (!ws[i] || ws[i]->ctx != ctx) return fail(DCI_EINVAL, "workspace null or of another context");
    for (int j = 0; j < i; ++j)
      if (ws[j] == ws[i]) return fail(DCI_EINVAL, "a workspace appears twice in one group");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ws[0]->staged = false;
  if (!gather_many_uses_tma(ctx, outs, n)) {
    // outputs that cannot take bulk stores: one batch after another on `stream`
    for (int i = 0; i < n; ++i) {
      dci_status st = run_batch(ctx, ws[i], seeds[i], B[i], fanouts, L, seed, 0, outs + i, nullptr, nullptr, s);
      if (st != DCI_OK) return st;
    }
    return DCI_OK;
  }
  for (int i = 0; i < n; ++i) {
    dci_status st = validate_batch(ctx, ws[i], seeds[i], B[i], fanouts, L, outs + i);
    if (st != DCI_OK) return st;
  }
  DeviceGuard g(ctx->device);
  dci_workspace* w0 = ws[0];
  const bool prof = w0->profiling != 0;
  dci_workspace::TimeRec* tr = nullptr;
  if (prof) {
    dci_status ts = trec_begin(w0);
    if (ts != DCI_OK) return ts;
    tr = &w0->trec[w0->trec_cur];
    tr->nb = n;
  }
  const bool use_graph = graph_mode();
  if (!use_graph) {
    for (int i = 0; i < n; ++i) {
      dci_status st = stage_header(ctx, ws[i], seeds[i], B[i], seed, s);
      if (st != DCI_OK) return st;
    }
  } else {
    // all n headers in ONE copy (pinned ring slot -> the first workspace's staging block); the
    // group's graph scatters them into the workspaces' scalars as its first node
    if (!w0->ghdr_ring) {  // first group on this workspace: all three resources or none
      BatchHeader* ring = nullptr;
      BatchHeader* dev = nullptr;
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&ring),
                                    sizeof(BatchHeader) * DCI_MAX_GROUP * dci_workspace::kGroupHdrRing,
                                    cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaMalloc(&dev, sizeof(BatchHeader) * DCI_MAX_GROUP);
      for (auto& ev : w0->ghdr_ev)
        if (e == cudaSuccess && !ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e != cudaSuccess) {
        if (ring) cudaFreeHost(ring);
        if (dev) cudaFree(dev);
        return cuda_fail(e, "group header staging");
      }
      w0->ghdr_dev = dev;
      w0->ghdr_ring = ring;
    }
    const int slot = (int)(w0->gcalls++ % dci_workspace::kGroupHdrRing);
    DCI_CUDA(cudaEventSynchronize(w0->ghdr_ev[slot]));  // the copy that last used this slot is done
    BatchHeader* hh = w0->ghdr_ring + (size_t)slot * DCI_MAX_GROUP;
    for (int i = 0; i < n; ++i) {
      if (++ws[i]->epoch == 0) {  // 2^32 batches on this workspace: clear the tag table once
        DCI_CUDA(cudaMemsetAsync(ws[i]->pos_of, 0, ws[i]->table_bytes, s));
        ws[i]->epoch = 1;
      }
      hh[i].seeds = seeds[i];
      hh[i].seed = seed;
      hh[i].B = B[i];
      hh[i].epoch = ws[i]->epoch;
    }
    DCI_CUDA(cudaMemcpyAsync(w0->ghdr_dev, hh, sizeof(BatchHeader) * n, cudaMemcpyHostToDevice, s));
    DCI_CUDA(cudaEventRecord(w0->ghdr_ev[slot], s));
  }
  // ---- the group's sampling: every hop of all n batches is ONE launch (hop, scan), captured as
  // a CUDA graph on the first workspace, re-captured when the group (workspaces, outputs,
  // fan-outs, caches) changes; the last hop's relabel follows the gather launch ----
  struct GroupSig {
    int32_t n, L, hs;
    int32_t fan[DCI_MAX_LAYERS];
    uint64_t ws[DCI_MAX_GROUP];  // workspace uids (a freed workspace's address may be reused)
    dci_batch_out out[DCI_MAX_GROUP];
    const void* acache;
    const void* uidx;
  };
  GroupSig* sig = new (std::nothrow) GroupSig;
  if (!sig) return fail(DCI_ENOMEM, "host allocation failed");
  std::unique_ptr<GroupSig> sig_guard(sig);
  memset(sig, 0, sizeof(GroupSig));
  sig->n = n;
  sig->L = L;
  for (int i = 0; i < L; ++i) sig->fan[i] = fanouts[i];
  for (int i = 0; i < n; ++i) {
    sig->ws[i] = ws[i]->uid;
    sig->out[i] = outs[i];
  }
  sig->acache = ctx->d_acache;
  sig->uidx = ctx->u_idx_cur;
  // hops [h0, h1) of the group (the parameters of every hop are built, so a range can start late)
  auto enqueue = [&](cudaStream_t es, int h0, int h1) {
    HopParams p[DCI_MAX_GROUP], prev[DCI_MAX_GROUP];
    for (int h = 0; h < h1; ++h) {
      for (int i = 0; i < n; ++i) {
        HopParams& q = p[i];
        q = HopParams{};
        q.F = outs[i].frontier;
        q.hop = h;
        q.f = fanouts[L - 1 - h];
        q.pass = 0;
        q.cand = ws[i]->cand[h & 1];
        q.kcnt = ws[i]->kcnt[h & 1];
        if (h > 0) {
          q.prev_cand = prev[i].cand;
          q.prev_kcnt = prev[i].kcnt;
          q.prev_bptr = outs[i].bptr[h - 1];
          q.prev_bsrc = outs[i].bsrc[h - 1];
          q.prev_f = prev[i].f;
        }
        q.bptr = outs[i].bptr[h];
      }
      if (h >= h0) {
        launch_sample_hop(ctx, ws, p, n, es);
        launch_newmask_sweep(ctx, ws, p, n, es);
        launch_scan_hop(ctx, ws, p, n, es);
      }
      for (int i = 0; i < n; ++i) prev[i] = p[i];
    }
  };
  // node sweep when the group's frontier bounds together reach N (Reddit-shaped: one batch's bound
  // alone is N); host-resident papers100M-shaped groups stay in row mode
  bool sweep = false;
  bool all_dense = true;
  for (int i = 0; i < n; ++i) all_dense &= ws[i]->hmask == 0;
  if (gather_sweep_enabled() && n >= 2 && all_dense) {
    int64_t grow = 1;
    for (int h = 0; h < L; ++h) grow = std::min<int64_t>(ctx->N, grow * (1 + (int64_t)fanouts[h]));
    int64_t cover = 0;
    for (int i = 0; i < n; ++i) cover += std::min<int64_t>(ctx->N, (int64_t)B[i] * grow);
    sweep = cover >= ctx->N;
    // host-resident feature rows: the sweep reads each MISS row once per group instead of once per
    // batch (and each hit row once), at the price of probing n tables for every node id.  Taken
    // when the host bytes a row-mode gather would move -- the frontier bound x the uncached share
    // of the rows x the row size, at ~50 GB/s -- exceed twice the probe bytes at ~6 TB/s
    // (M3 groups of 20 sweep anyway: 2.6 -> 4.0 M seeds/s; papers100M-shaped M4 needs this rule)
    if (!sweep && ctx->fcache_total_rows < ctx->N) {
      const double miss = 1.0 - (double)ctx->fcache_total_rows / (double)ctx->N;
      const double host_s = (double)cover * miss * 4.0 * (double)ctx->pitch / 50e9;
      const double probe_s = (double)ctx->N * (double)n * 8.0 / 6e12;
      sweep = host_s > 2.0 * probe_s;
    }
  }
  // alone: the previous group's gather had already finished when this group was enqueued, so
  // nothing is queued ahead of this group's gather
  const bool alone = !ctx->gather_q_valid || cudaEventQuery(ctx->gather_q_ev) == cudaSuccess;
  // Split gather (DCI_SPLIT_GATHER=1; off by default): when nothing else would run beside this
  // group's sampling (alone), its node-sweep gather is two launches -- the rows of F_{L-1} right
  // after hop L-2's scan, beside hop L-1's sampling and scan, then the rows added by hop L-1 -- to
  // hide the last hop's sampling.  Measured on M2 (groups of 20, one group per timed region): no
  // gain (10.72 vs 10.74 M seeds/s): the two launches take 1.71 ms against 1.44 ms for one (each
  // reads the shared rows, and the first shares the GPU with the sampler), which cancels the
  // ~0.3 ms of hidden sampling.  Pipelined groups (not alone) never split.
  const bool split = sweep && alone && L >= 2 && gather_split_enabled() && !gather_concurrent();
  // split schedule: hops [0, hs) before the wait for the previous group's gather, [hs, L) after
  const bool phased = group_phased();
  const bool split_sched = phased && group_split() && L >= 2;
  const int hs = (split || split_sched) ? L - 1 : 0;
  sig->hs = hs;
  // the relabel of every batch's last hop: needed by the caller, not by the gather, so it runs
  // on `stream` while the gather runs on the gather stream
  auto enqueue_epilogue = [&](cudaStream_t es) {
    HopParams p[DCI_MAX_GROUP];
    for (int i = 0; i < n; ++i) p[i] = epilogue_params(ws[i], L, fanouts, outs + i);
    launch_hop_epilogue(ctx, ws, p, n, es);
  };
  w0->in_group = 1;
  // two cached group graphs per first workspace (least recently used replaced): a caller that
  // alternates two group shapes (e.g. a full group and a shorter last one) never re-captures
  dci_workspace::GroupGraph* gg = nullptr;
  if (use_graph) {
    for (auto& c : w0->gg)
      if (c.exec && c.sig && c.sig_len == sizeof(GroupSig) && !memcmp(c.sig, sig, sizeof(GroupSig))) gg = &c;
    if (!gg) {
      gg = &w0->gg[0];
      for (auto& c : w0->gg)
        if (!c.exec || c.last_use < gg->last_use) gg = &c;
      if (gg->exec) cudaGraphExecDestroy(gg->exec);
      if (gg->exec2) cudaGraphExecDestroy(gg->exec2);
      gg->exec = gg->exec2 = nullptr;
      free(gg->sig);  // the entry matches no group until both graphs are built
      gg->sig = nullptr;
      gg->sig_len = 0;
      // part 1: the header scatter and hops [0, hs) (all hops when not split); part 2: [hs, L)
      for (int part = 0; part < (hs > 0 ? 2 : 1); ++part) {
        const uint64_t launches0 = ctx->launches;
        DCI_CUDA(cudaStreamBeginCapture(w0->cap_stream, cudaStreamCaptureModeThreadLocal));
        if (part == 0) {
          launch_scatter_headers(ctx, ws, w0->ghdr_dev, n, w0->cap_stream);
          enqueue(w0->cap_stream, 0, hs > 0 ? hs : L);
        } else {
          enqueue(w0->cap_stream, hs, L);
        }
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(w0->cap_stream, &graph);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
        (part == 0 ? gg->kernels : gg->kernels2) = ctx->launches - launches0;
        ctx->launches = launches0;
        e = cudaGraphInstantiate(part == 0 ? &gg->exec : &gg->exec2, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      }
      if (hs == 0) gg->kernels2 = 0;
      if (!gg->sig) gg->sig = malloc(sizeof(GroupSig));
      if (!gg->sig) return fail(DCI_ENOMEM, "host allocation failed");
      memcpy(gg->sig, sig, sizeof(GroupSig));
      gg->sig_len = sizeof(GroupSig);
    }
    gg->last_use = ++w0->gg_clock;
  }
  // Schedule of consecutive groups (DCI_PHASED): by default a group's sampling overlaps the
  // previous group's gather (+6 % seeds/s on M2 against alternating them, although each gather
  // launch runs ~3 % slower beside the sampler, exp60).  DCI_PHASED=1: a group
  // samples only after the previous group's gather has finished; DCI_PHASED=2: only its last hop
  // waits for it.
  if (phased && !split_sched && ctx->gather_ev_valid) DCI_CUDA(cudaStreamWaitEvent(s, ctx->gather_ev, 0));
  if (tr) DCI_CUDA(cudaEventRecord(tr->e[0], s));
  if (use_graph) {
    ctx->launches += gg->kernels;
    DCI_CUDA(cudaGraphLaunch(gg->exec, s));
  } else {
    enqueue(s, 0, hs > 0 ? hs : L);
  }
  // ---- the group's gather, on the context's gather stream (group gathers run one at a time;
  // DCI_GATHER_SERIAL=0 puts it on `stream` instead).  Node-sweep kernel: the bulk-copy one
  // (faster alone, 1.43 vs 1.55 ms on M2) when the gather runs by itself, else the register-copy
  // one, whose full SMs keep the next group's sampling from slowing it (exp r2-6) ----
  cudaStream_t gs = gather_concurrent() ? s : ctx->gstream;
  dci_batch_result* stage = nullptr;
  if (w0->want_stage) {
    if (!w0->stage) DCI_CUDA(cudaMalloc(&w0->stage, sizeof(dci_batch_result) * DCI_MAX_GROUP));
    stage = w0->stage;
    w0->staged = true;
  }
  auto gather_launch = [&](int32_t phase) -> dci_status {
    int kind = 0;
    dci_status gst = launch_gather_many(ctx, ws, outs, n, L, stage, sweep, alone, phase, gs, &kind);
    if (gst != DCI_OK) return gst;
    ++w0->kind_launches[kind];
    return DCI_OK;
  };
  if (split) {  // first launch: the rows of F_{L-1}, beside hop L-1's sampling and scan
    DCI_CUDA(cudaEventRecord(w0->ev_pre, s));
    DCI_CUDA(cudaStreamWaitEvent(gs, w0->ev_pre, 0));
    if (tr) DCI_CUDA(cudaEventRecord(tr->e[2], gs));
    dci_status gst = gather_launch(1);
    if (gst != DCI_OK) return gst;
    if (tr) DCI_CUDA(cudaEventRecord(tr->e[4], gs));
  }
  if (hs > 0) {
    if (split_sched && ctx->gather_ev_valid) DCI_CUDA(cudaStreamWaitEvent(s, ctx->gather_ev, 0));
    if (use_graph) {
      ctx->launches += gg->kernels2;
      DCI_CUDA(cudaGraphLaunch(gg->exec2, s));
    } else {
      enqueue(s, hs, L);
    }
  }
  if (tr) {
    DCI_CUDA(cudaEventRecord(tr->e[1], s));
    tr->state |= 1;
  }
  if (gs != s) {
    DCI_CUDA(cudaEventRecord(w0->ev_mid, s));
    DCI_CUDA(cudaStreamWaitEvent(gs, w0->ev_mid, 0));
  }
  if (tr) DCI_CUDA(cudaEventRecord(tr->e[split ? 5 : 2], gs));
  {
    dci_status gst = gather_launch(split ? 2 : 0);
    if (gst != DCI_OK) return gst;
    DCI_CUDA(cudaEventRecord(ctx->gather_q_ev, gs));
    ctx->gather_q_valid = true;
  }
  // the last hop's relabel beside the gather (default), or after it (DCI_EPI_AFTER=1, a measurement
  // knob: the relabel's random tag reads compete with the gather's writes)
  static const bool epi_after = [] {
    const char* e = getenv("DCI_EPI_AFTER");
    return e && e[0] == '1';
  }();
  if (epi_after && gs != s) {
    DCI_CUDA(cudaEventRecord(w0->ev_done, gs));
    DCI_CUDA(cudaStreamWaitEvent(s, w0->ev_done, 0));
  }
  enqueue_epilogue(s);
  if (phased) {
    DCI_CUDA(cudaEventRecord(ctx->gather_ev, gs));
    ctx->gather_ev_valid = true;
  }
  if (tr) {
    DCI_CUDA(cudaEventRecord(tr->e[3], gs));
    tr->state |= split ? 6 : 2;
  }
  if (gs != s) {
    DCI_CUDA(cudaEventRecord(w0->ev_done, gs));
    DCI_CUDA(cudaStreamWaitEvent(s, w0->ev_done, 0));
  }
  DCI_CUDA(cudaGetLastError());
  return DCI_OK;
}

dci_status dci_sample_gather_many_host(dci_ctx* ctx, int32_t n, dci_workspace* const* ws,
                                       const int32_t* const* seeds_host, const int32_t* B, const int32_t* fanouts,
                                       int32_t L, uint64_t seed, const dci_batch_out* outs,
                                       dci_batch_result* results_host, void* stream) {
  if (!ctx || !ws || !seeds_host || !B || !outs) return fail(DCI_EINVAL, "null argument");
  if (n < 1 || n > DCI_MAX_GROUP) return fail(DCI_EINVAL, "n must be in [1, DCI_MAX_GROUP]");
  if (L < 1 || L > DCI_MAX_LAYERS) return fail(DCI_EINVAL, "L must be in [1, DCI_MAX_LAYERS]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard g(ctx->device);
  const int32_t* dseeds[DCI_MAX_GROUP];
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (!ws[i]) return fail(DCI_EINVAL, "null workspace");
    if (B[i] < 0 || B[i] > ws[i]->max_batch) return fail(DCI_EINVAL, "B exceeds the workspace's max_batch");
    if (B[i] > 0 && !seeds_host[i]) return fail(DCI_EINVAL, "seeds_host is null");
    total += B[i];
  }
  // all seeds of the group in ONE host->device copy: packed into the first workspace's pinned
  // staging block (its previous copy has finished: event), then scattered by pointer offsets
  dci_workspace* w0 = ws[0];
  if (total > w0->gseeds_cap) {
    if (w0->gseeds_host) cudaFreeHost(w0->gseeds_host);
    if (w0->gseeds_dev) cudaFree(w0->gseeds_dev);
    w0->gseeds_host = nullptr;
    w0->gseeds_dev = nullptr;
    w0->gseeds_cap = 0;
    DCI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w0->gseeds_host), sizeof(int32_t) * total, cudaHostAllocDefault));
    DCI_CUDA(cudaMalloc(&w0->gseeds_dev, sizeof(int32_t) * total));
    w0->gseeds_cap = total;
  }
  if (total > 0) {
    DCI_CUDA(cudaEventSynchronize(w0->gseeds_ev));
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      if (B[i] > 0) memcpy(w0->gseeds_host + off, seeds_host[i], sizeof(int32_t) * B[i]);
      dseeds[i] = w0->gseeds_dev + off;
      off += B[i];
    }
    DCI_CUDA(cudaMemcpyAsync(w0->gseeds_dev, w0->gseeds_host, sizeof(int32_t) * total, cudaMemcpyHostToDevice, s));
    DCI_CUDA(cudaEventRecord(w0->gseeds_ev, s));
  } else {
    for (int i = 0; i < n; ++i) dseeds[i] = ws[i]->seeds_stage;
  }
  // the group gather's last block also writes every batch's results into the first workspace's
  // device staging block, so one copy brings them all back
  ws[0]->want_stage = results_host != nullptr;
  dci_status st = dci_sample_gather_many(ctx, n, ws, dseeds, B, fanouts, L, seed, outs, stream);
  const bool staged = ws[0]->want_stage && ws[0]->staged;
  ws[0]->want_stage = false;
  if (st != DCI_OK || !results_host) return st;
  if (staged) {
    DCI_CUDA(cudaMemcpyAsync(results_host, ws[0]->stage, sizeof(dci_batch_result) * n, cudaMemcpyDeviceToHost, s));
  } else {  // batch-by-batch fallback path: per-batch copies
    for (int i = 0; i < n; ++i) {
      DCI_CUDA(cudaMemcpyAsync(results_host[i].sizes, outs[i].sizes, sizeof(int64_t) * (L + 1),
                               cudaMemcpyDeviceToHost, s));
      DCI_CUDA(cudaMemcpyAsync(results_host[i].counters, outs[i].counters, sizeof(uint64_t) * 4,
                               cudaMemcpyDeviceToHost, s));
      DCI_CUDA(cudaMemcpyAsync(&results_host[i].status, outs[i].status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    }
  }
  return DCI_OK;
}

dci_status dci_sample_gather_host(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds_host, int32_t B,
                                  const int32_t* fanouts, int32_t L, uint64_t seed, const dci_batch_out* out,
                                  int64_t* sizes_host, uint64_t* counters_host, int32_t* status_host,
                                  void* stream) {
  if (!ctx || !ws) return fail(DCI_EINVAL, "null context/workspace");
  if (B < 0 || B > ws->max_batch) return fail(DCI_EINVAL, "B exceeds the workspace's max_batch");
  if (B > 0 && !seeds_host) return fail(DCI_EINVAL, "seeds_host is null");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard g(ctx->device);
  if (B > 0)
    DCI_CUDA(cudaMemcpyAsync(ws->seeds_stage, seeds_host, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s));
  dci_status st = run_batch(ctx, ws, ws->seeds_stage, B, fanouts, L, seed, 0, out, nullptr, nullptr, s);
  if (st != DCI_OK) return st;
  if (sizes_host)
    DCI_CUDA(cudaMemcpyAsync(sizes_host, out->sizes, sizeof(int64_t) * (L + 1), cudaMemcpyDeviceToHost, s));
  if (counters_host)
    DCI_CUDA(cudaMemcpyAsync(counters_host, out->counters, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost, s));
  if (status_host) DCI_CUDA(cudaMemcpyAsync(status_host, out->status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  return DCI_OK;
}

dci_status dci_presample(dci_ctx* ctx, const int32_t* seeds, int64_t num_seeds, int32_t batch,
                         const int32_t* fanouts, int32_t L, uint64_t seed, int32_t* node_visits,
                         int32_t* edge_counts, uint64_t* t_sample_ns, uint64_t* t_feature_ns, void* stream) {
  if (!ctx) return fail(DCI_EINVAL, "null context");
  if (ctx->state != DCI_STATE_LOADED) return fail(DCI_ESTATE, "dci_presample must run before dci_fill");
  if (batch < 1 || num_seeds < 0) return fail(DCI_EINVAL, "batch must be >= 1");
  if (num_seeds > 0 && !seeds) return fail(DCI_EINVAL, "seeds is null");
  if (!node_visits || (ctx->E > 0 && !edge_counts)) return fail(DCI_EINVAL, "null count array");
  dci_status st = check_fanouts(fanouts, L);
  if (st != DCI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DeviceGuard g(ctx->device);
  const int32_t B = (int32_t)std::min<int64_t>(batch, std::max<int64_t>(num_seeds, 1));
  // (re)create the internal presample workspace and outputs when the shape changes
  bool same = ctx->pre_ws && ctx->pre_B == B && ctx->pre_L == L;
  for (int i = 0; same && i < L; ++i) same = ctx->pre_fan[i] == fanouts[i];
  int64_t caps[DCI_MAX_LAYERS + 1];
  frontier_bounds(ctx->N, B, fanouts, L, caps);
  if (!same) {
    DCI_CUDA(cudaDeviceSynchronize());
    if (ctx->pre_ws) dci_workspace_destroy(ctx->pre_ws);
    ctx->pre_ws = nullptr;
    if (ctx->pre_out_mem) cudaFree(ctx->pre_out_mem);
    ctx->pre_out_mem = nullptr;
    st = workspace_create(ctx, B, fanouts, L, &ctx->pre_ws, false);
    if (st != DCI_OK) return st;
    size_t bytes = 0;
    auto take = [&](size_t n) {
      size_t off = bytes;
      bytes += (n + 255) / 256 * 256;
      return off;
    };
    size_t o_front = take(sizeof(int32_t) * caps[L]);
    size_t o_sizes = take(sizeof(int64_t) * (L + 1));
    size_t o_cnt = take(sizeof(uint64_t) * 4);
    size_t o_status = take(sizeof(int32_t));
    size_t o_bptr[DCI_MAX_LAYERS], o_bsrc[DCI_MAX_LAYERS];
    for (int h = 0; h < L; ++h) {
      o_bptr[h] = take(sizeof(int32_t) * (caps[h] + 1));
      o_bsrc[h] = take(sizeof(int32_t) * caps[h] * fanouts[L - 1 - h]);
    }
    size_t o_x = take(sizeof(float) * caps[L] * ctx->pitch);
    DCI_CUDA(cudaMalloc(&ctx->pre_out_mem, bytes));
    char* base = static_cast<char*>(ctx->pre_out_mem);
    dci_batch_out& o = ctx->pre_out;
    memset(&o, 0, sizeof(o));
    o.frontier = reinterpret_cast<int32_t*>(base + o_front);
    o.frontier_cap = caps[L];
    o.sizes = reinterpret_cast<int64_t*>(base + o_sizes);
    o.counters = reinterpret_cast<uint64_t*>(base + o_cnt);
    o.status = reinterpret_cast<int32_t*>(base + o_status);
    for (int h = 0; h < L; ++h) {
      o.bptr[h] = reinterpret_cast<int32_t*>(base + o_bptr[h]);
      o.bsrc[h] = reinterpret_cast<int32_t*>(base + o_bsrc[h]);
      o.hop_cap[h] = caps[h];
      o.bsrc_cap[h] = caps[h] * fanouts[L - 1 - h];
    }
    o.X = reinterpret_cast<float*>(base + o_x);
    o.ldx = ctx->pitch;
    ctx->pre_B = B;
    ctx->pre_L = L;
    for (int i = 0; i < L; ++i) ctx->pre_fan[i] = fanouts[i];
    // predicted peak per-batch workspace for the auto budget: outputs + scratch
    uint64_t ws_bytes = bytes + sizeof(unsigned long long) * (uint64_t)ctx->N +
                        sizeof(int32_t) * 2 * (uint64_t)(ctx->pre_ws->cand_cap + caps[L]);
    ctx->presample_peak = std::max<uint64_t>(ctx->presample_peak, ws_bytes);
  }
  int32_t status = 0;
  const int64_t nb = (num_seeds + batch - 1) / batch;
  for (int64_t b = 0; b < nb; ++b) {
    const int32_t nbat = (int32_t)std::min<int64_t>(batch, num_seeds - b * batch);
    st = run_batch(ctx, ctx->pre_ws, seeds + b * batch, nbat, fanouts, L, seed, 1, &ctx->pre_out, node_visits,
                   edge_counts, s);
    if (st != DCI_OK) return st;
    DCI_CUDA(cudaMemcpyAsync(&status, ctx->pre_out.status, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaStreamSynchronize(s));
    float ms_s = 0.f, ms_f = 0.f;
    const dci_workspace::TimeRec& pr = ctx->pre_ws->trec[ctx->pre_ws->trec_cur];
    DCI_CUDA(cudaEventElapsedTime(&ms_s, pr.e[0], pr.e[1]));
    DCI_CUDA(cudaEventElapsedTime(&ms_f, pr.e[1], pr.e[3]));
    if (t_sample_ns) t_sample_ns[b] = (uint64_t)llround((double)ms_s * 1e6);
    if (t_feature_ns) t_feature_ns[b] = (uint64_t)llround((double)ms_f * 1e6);
    if (status != DCI_OK) return fail((dci_status)status, "dci_presample: invalid or duplicate seed in a batch");
  }
  return DCI_OK;
}

dci_status dci_allocate(dci_ctx* ctx, uint64_t C, const uint64_t* t_sample_ns, const uint64_t* t_feature_ns,
                        int32_t n, int64_t ratio_num, int64_t ratio_den, uint64_t* c_adj, uint64_t* c_feat) {
  if (!c_adj || !c_feat || n < 0) return fail(DCI_EINVAL, "bad arguments");
  if (n > 0 && (!t_sample_ns || !t_feature_ns)) return fail(DCI_EINVAL, "null time arrays");
  if (C == 0) {
    // auto budget: what stays free for the caches once the fill is done.  Free device
    // memory now (the caller's inference workspaces and outputs, created before this call, are
    // already excluded: dci.h) + memory the fill gives back (current caches, the presample
    // workspace) - the fill's own temporaries - the 1 GiB reserve (C21).
    if (!ctx) return fail(DCI_EINVAL, "auto budget needs a context");
    DeviceGuard g(ctx->device);
    size_t free_b = 0, total_b = 0;
    DCI_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t held = (uint64_t)ctx->acache_len * 4 + (uint64_t)ctx->fcache_rows * 4 * ctx->pitch;
    const uint64_t pre = ctx->pre_ws ? ctx->presample_peak : 0;
    const uint64_t reserve = 1ull << 30;
    const uint64_t avail = (uint64_t)free_b + held + pre;
    const uint64_t need = fill_temp_bound(ctx->N, ctx->E) + reserve;
    C = avail > need ? avail - need : 0;
  }
  unsigned __int128 adj;
  if (ratio_den > 0) {
    if (ratio_num < 0 || ratio_num > ratio_den) return fail(DCI_EINVAL, "ratio must be in [0, 1]");
    adj = (unsigned __int128)C * (unsigned __int128)ratio_num / (unsigned __int128)ratio_den;
  } else {
    unsigned __int128 S = 0, F = 0;
    for (int32_t k = 0; k < n; ++k) {
      S += t_sample_ns[k];
      F += t_feature_ns[k];
    }
    adj = (S + F == 0) ? (unsigned __int128)(C / 2) : (unsigned __int128)C * S / (S + F);
  }
  *c_adj = (uint64_t)adj;
  *c_feat = C - (uint64_t)adj;
  return DCI_OK;
}

dci_status dci_fill(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts, uint64_t c_adj,
                    uint64_t c_feat, void* stream) {
  if (!ctx) return fail(DCI_EINVAL, "null context");
  if (!node_visits || (ctx->E > 0 && !edge_counts)) return fail(DCI_EINVAL, "null count array");
  DeviceGuard g(ctx->device);
  DCI_CUDA(cudaDeviceSynchronize());  // no batch may be in flight while caches change
  return fill_impl(ctx, node_visits, edge_counts, c_adj, c_feat, 1, 0, static_cast<cudaStream_t>(stream));
}

dci_status dci_fill_partitioned(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts,
                                uint64_t c_adj, uint64_t c_feat, int32_t world, int32_t rank, void* stream) {
  if (!ctx) return fail(DCI_EINVAL, "null context");
  if (!node_visits || (ctx->E > 0 && !edge_counts)) return fail(DCI_EINVAL, "null count array");
  if (world < 1 || world > dci_ctx::kMaxParts || rank < -1 || rank >= world)
    return fail(DCI_EINVAL, "need 1 <= world <= 16 and -1 <= rank < world");
  DeviceGuard g(ctx->device);
  DCI_CUDA(cudaDeviceSynchronize());
  return fill_impl(ctx, node_visits, edge_counts, c_adj, c_feat, world, rank, static_cast<cudaStream_t>(stream));
}

dci_status dci_fill_knapsack(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts, uint64_t C,
                             double cost_feat, double cost_adj, void* stream) {
  if (!ctx) return fail(DCI_EINVAL, "null context");
  if (!node_visits || (ctx->E > 0 && !edge_counts)) return fail(DCI_EINVAL, "null count array");
  if (!(cost_feat >= 0.0) || !(cost_adj >= 0.0)) return fail(DCI_EINVAL, "costs must be >= 0");
  DeviceGuard g(ctx->device);
  DCI_CUDA(cudaDeviceSynchronize());
  KnapsackPlan plan{C, cost_feat, cost_adj};
  return fill_impl(ctx, node_visits, edge_counts, 0, 0, 1, 0, static_cast<cudaStream_t>(stream), &plan);
}

dci_status dci_feature_partition_handle(dci_ctx* ctx, void* handle) {
  if (!ctx || !handle) return fail(DCI_EINVAL, "bad arguments");
  if (!ctx->d_fcache) return fail(DCI_ESTATE, "no feature partition on this device (fill first)");
  static_assert(sizeof(cudaIpcMemHandle_t) == DCI_IPC_HANDLE_BYTES, "IPC handle size");
  DeviceGuard g(ctx->device);
  cudaIpcMemHandle_t h;
  DCI_CUDA(cudaIpcGetMemHandle(&h, ctx->d_fcache));
  memcpy(handle, &h, sizeof(h));
  return DCI_OK;
}

dci_status dci_attach_feature_partitions(dci_ctx* ctx, const void* handles, int32_t world) {
  if (!ctx || !handles) return fail(DCI_EINVAL, "bad arguments");
  if (ctx->fpart_rank < 0 || world != ctx->fpart_world)
    return fail(DCI_ESTATE, "context was not filled with dci_fill_partitioned(world, rank >= 0)");
  DeviceGuard g(ctx->device);
  for (int p = 0; p < world; ++p) {
    if (p == ctx->fpart_rank) continue;
    if (ctx->ipc_opened[p]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)p * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    DCI_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->ipc_opened[p] = ptr;
    ctx->h_fbases[p] = static_cast<const float*>(ptr);
  }
  DCI_CUDA(cudaMemcpy(ctx->d_fbases, ctx->h_fbases, sizeof(float*) * dci_ctx::kMaxParts, cudaMemcpyHostToDevice));
  return DCI_OK;
}

dci_status dci_fill_times_get(const dci_ctx* ctx, dci_fill_times* out) {
  if (!ctx || !out) return fail(DCI_EINVAL, "null argument");
  out->level2_ms = ctx->fill_ms[0];
  out->adj_select_ms = ctx->fill_ms[1];
  out->adj_copy_ms = ctx->fill_ms[2];
  out->feat_select_ms = ctx->fill_ms[3];
  out->feat_copy_ms = ctx->fill_ms[4];
  out->total_ms = ctx->fill_ms[5];
  return DCI_OK;
}

dci_status dci_cache_info_get(const dci_ctx* ctx, dci_cache_info* info) {
  if (!ctx || !info) return fail(DCI_EINVAL, "bad arguments");
  info->state = ctx->state;
  info->pitch = ctx->pitch;
  info->N = ctx->N;
  info->E = ctx->E;
  info->D = ctx->D;
  info->whole_fit = ctx->whole_fit;
  info->c_adj = ctx->c_adj;
  info->c_feat = ctx->c_feat;
  info->adj_elems = ctx->acache_len;
  info->feat_rows = ctx->fcache_rows;
  info->feat_rows_total = ctx->fcache_total_rows;
  info->feat_partitions = ctx->fpart_world;
  info->presample_peak_bytes = ctx->presample_peak;
  info->launches = ctx->launches;
  return DCI_OK;
}

dci_status dci_cache_state(dci_ctx* ctx, int32_t* cached_len, int64_t* cache_off, int32_t* slot_of,
                           int32_t* acache, float* fcache, int32_t* indices_cur) {
  if (!ctx) return fail(DCI_EINVAL, "null context");
  DeviceGuard g(ctx->device);
  DCI_CUDA(cudaDeviceSynchronize());
  const int64_t N = ctx->N;
  if (cached_len || cache_off || slot_of) {
    DirEntry* h = static_cast<DirEntry*>(malloc(sizeof(DirEntry) * N));
    if (!h) return fail(DCI_ENOMEM, "host allocation failed");
    cudaError_t e = cudaMemcpy(h, ctx->d_dir, sizeof(DirEntry) * N, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      free(h);
      return cuda_fail(e, "copy directory");
    }
    for (int64_t v = 0; v < N; ++v) {
      if (cached_len) cached_len[v] = h[v].cached_len;
      if (cache_off) cache_off[v] = h[v].cache_off;
      if (slot_of) slot_of[v] = h[v].slot;
    }
    free(h);
  }
  if (acache && ctx->acache_len)
    DCI_CUDA(cudaMemcpy(acache, ctx->d_acache, sizeof(int32_t) * ctx->acache_len, cudaMemcpyDeviceToHost));
  if (fcache && ctx->fcache_rows)
    DCI_CUDA(cudaMemcpy(fcache, ctx->d_fcache, sizeof(float) * ctx->fcache_rows * ctx->pitch,
                        cudaMemcpyDeviceToHost));
  if (indices_cur && ctx->E) memcpy(indices_cur, ctx->h_idx_cur, sizeof(int32_t) * ctx->E);
  return DCI_OK;
}

dci_status dci_workspace_set_profiling(dci_workspace* ws, int32_t on) {
  if (!ws) return fail(DCI_EINVAL, "null workspace");
  ws->profiling = on ? 1 : 0;
  return DCI_OK;
}

dci_status dci_workspace_stage_ms(dci_workspace* ws, float* sample_ms, float* gather_ms) {
  if (!ws) return fail(DCI_EINVAL, "null workspace");
  const dci_workspace::TimeRec& r = ws->trec[ws->trec_cur];
  if ((r.state & 3) != 3) return fail(DCI_ESTATE, "no profiled batch recorded");
  DeviceGuard g(ws->device);
  DCI_CUDA(cudaEventSynchronize(r.e[3]));
  if (sample_ms) DCI_CUDA(cudaEventElapsedTime(sample_ms, r.e[0], r.e[1]));
  if (gather_ms) {
    if (r.state & 4) {  // split gather: both launches, without the wait between them
      float a = 0.f, b = 0.f;
      DCI_CUDA(cudaEventElapsedTime(&a, r.e[2], r.e[4]));
      DCI_CUDA(cudaEventElapsedTime(&b, r.e[5], r.e[3]));
      *gather_ms = a + b;
    } else {
      DCI_CUDA(cudaEventElapsedTime(gather_ms, r.e[2], r.e[3]));
    }
  }
  return DCI_OK;
}

dci_status dci_workspace_stats(dci_workspace* ws, dci_ws_stats* out, int32_t reset) {
  if (!ws || !out) return fail(DCI_EINVAL, "bad arguments");
  DeviceGuard g(ws->device);
  DCI_CUDA(cudaDeviceSynchronize());
  for (auto& r : ws->trec) {
    dci_status st = trec_fold(ws, r);
    if (st != DCI_OK) return st;
  }
  BatchScalars h;
  DCI_CUDA(cudaMemcpy(&h, ws->scal, sizeof(h), cudaMemcpyDeviceToHost));
  out->batches = h.acc_batches;
  out->seeds = h.acc_seeds;
  out->frontier_rows = h.acc_rows;
  for (int c = 0; c < 4; ++c) out->counters[c] = h.acc_counters[c];
  out->timed_batches = ws->acc_timed;
  out->sample_ms = ws->acc_sample_ms;
  out->gather_ms = ws->acc_gather_ms;
  out->gather_launches = ws->acc_gather_launches;
  out->rows_read = h.acc_rows_read;
  out->gather_bytes = h.acc_gather_bytes;
  out->host_rows_read = h.acc_host_rows;
  out->host_adj_sectors = h.acc_host_sectors;
  out->host_adj_runs = h.acc_host_runs;
  for (int k = 0; k < 3; ++k) out->gather_kinds[k] = ws->kind_launches[k];
  out->table_bytes = ws->table_bytes;
  if (reset) {
    h.acc_batches = h.acc_seeds = h.acc_rows = 0;
    h.acc_rows_read = h.acc_gather_bytes = 0;
    h.acc_host_rows = h.acc_host_sectors = h.acc_host_runs = 0;
    for (auto& k : ws->kind_launches) k = 0;
    for (int c = 0; c < 4; ++c) h.acc_counters[c] = 0;
    DCI_CUDA(cudaMemcpy(ws->scal, &h, sizeof(h), cudaMemcpyHostToDevice));
    ws->acc_timed = ws->acc_gather_launches = 0;
    ws->acc_sample_ms = ws->acc_gather_ms = 0.0;
  }
  return DCI_OK;
}

dci_status dci_block_aggregate(dci_ctx* ctx, const int32_t* bptr, const int32_t* bsrc, const int64_t* n_dst,
                               const float* Xsrc, int64_t ldx, int32_t D, float* H, int64_t ldh, int32_t op,
                               void* stream) {
  if (!ctx || !bptr || !bsrc || !n_dst || !Xsrc || !H) return fail(DCI_EINVAL, "null argument");
  if (D < 1 || ldx < D || ldh < D) return fail(DCI_EINVAL, "need D >= 1, ldx >= D, ldh >= D");
  if (op != DCI_AGG_MEAN && op != DCI_AGG_SUM) return fail(DCI_EINVAL, "op must be DCI_AGG_MEAN or DCI_AGG_SUM");
  DeviceGuard g(ctx->device);
  return launch_block_aggregate(ctx, bptr, bsrc, n_dst, Xsrc, ldx, D, H, ldh, op, static_cast<cudaStream_t>(stream));
}

dci_status dci_mean_aggregate(dci_ctx* ctx, const int32_t* bptr, const int32_t* bsrc, const int64_t* n_dst,
                              const float* Xsrc, int64_t ldx, int32_t D, float* H, int64_t ldh, void* stream) {
  return dci_block_aggregate(ctx, bptr, bsrc, n_dst, Xsrc, ldx, D, H, ldh, DCI_AGG_MEAN, stream);
}

uint64_t dci_launch_count(const dci_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
