/*
 * dci.h — C ABI of libdci, the B200-native (sm_100a) hot path of DCI (arXiv 2503.01281):
 * dual-cache mini-batch preparation for sampled GNN inference.
 *
 * Citation key: P:n = PAPER.md line n (the paper's LaTeX, /root/reference at build time);
 * O-k / Ck = oracle definition / reading k of DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Every call returns dci_status; no C++ exception crosses the ABI.  On failure a
 *    thread-local message is available from dci_last_error().
 *  - "host" pointers are ordinary CPU memory; "device" pointers are CUDA device memory of
 *    the context's device (e.g. torch tensors' data_ptr()).  `stream` is a cudaStream_t
 *    passed as void* (NULL = legacy default stream).
 *  - Sizes are element counts unless named *_bytes.  Node ids are int32 (N < 2^31).
 *  - A context belongs to one device.  Calls on one context are not thread-safe, except
 *    that distinct workspaces may run dci_sample_gather concurrently on distinct streams.
 *  - Asynchronous calls (dci_sample_gather*) never synchronise the host.  Per-batch data
 *    errors (bad seed id, duplicate seed) are reported through the device status word of
 *    dci_batch_out, not the return value.
 */
#ifndef DCI_H_
#define DCI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DCI_VERSION 100          /* 1.0.0 */
#define DCI_MAX_LAYERS 8         /* L <= 8 hops */
#define DCI_MAX_GROUP 32          /* batches per dci_sample_gather_many call */
#define DCI_MAX_FANOUT 1024      /* per-hop fan-out 1..1024 (<= 32: registers, else shared memory) */

typedef enum dci_status {
  DCI_OK = 0,
  DCI_EINVAL = 1,  /* bad argument (null pointer, size, fan-out, layout) */
  DCI_ESTATE = 2,  /* call not allowed in the context's current state */
  DCI_ECUDA = 3,   /* CUDA runtime error (message in dci_last_error) */
  DCI_ENOMEM = 4,  /* device or pinned host allocation failed */
  DCI_ESEED = 5,   /* a seed id is outside [0, N)                (device status word) */
  DCI_EDUP = 6,    /* a seed id appears twice in one batch       (device status word) */
  DCI_ECAP = 7,    /* an output buffer is smaller than dci_output_bounds requires */
  DCI_ERANGE = 8   /* a count/size exceeds a documented limit */
} dci_status;

typedef struct dci_ctx dci_ctx;

#define DCI_ADOPT_HOST 1u /* dci_load_graph flag: register the caller's host buffers in place */
typedef struct dci_workspace dci_workspace;

/* Context lifecycle states (dci_cache_info.state). */
enum { DCI_STATE_LOADED = 1, DCI_STATE_FILLED = 2 };

/* --------------------------------------------------------------------------------------
 * dci_load_graph — S0.  P:130-131 (CSC: Col_ptr / Row_index), P:147 + P:170 (host graph
 * reached through UVA on a miss).
 *  indptr  host int64[N+1]  CSC column pointers (Col_ptr): indptr[0]=0, non-decreasing,
 *                           indptr[N]=E.  Node v's in-neighbours are
 *                           indices[indptr[v] .. indptr[v+1]).
 *  indices host int32[E]    in-neighbour ids (Row_index), each in [0, N).
 *  feats   host fp32[N*D]   row-major node features.
 *  The library copies indices and feats into its own pinned, device-mapped host buffers
 *  (feature rows padded to pitch = round_up(D, 4) floats so every row is 16-byte aligned;
 *  the pad is zero) and builds the per-node device directory.  The caller's buffers may
 *  be freed on return.  Validates the CSC invariants (O(E) host pass) -> DCI_EINVAL.
 *  flags: 0, or DCI_ADOPT_HOST: indices and feats are NOT copied but registered in place
 *    (cudaHostRegister, mapped + portable) and read through UVA; feats must then already hold
 *    N rows of pitch = round_up(D, 4) floats (pad columns zero, 16-byte aligned rows).  The
 *    library never writes adopted memory (the fill's level-2 reordered CSC is its own buffer),
 *    so several contexts -- e.g. one rank per GPU -- may adopt one node-shared segment (P:52,
 *    papers100M stays host-resident).  The buffers must outlive the context;
 *    dci_destroy unregisters them.  Registration failure -> DCI_ECUDA.
 *  Limits: 1 <= N < 2^31, 0 <= E < 2^40, 1 <= D.  *out owns all device and pinned memory.
 * ------------------------------------------------------------------------------------ */
dci_status dci_load_graph(dci_ctx** out, int device, int64_t N, int64_t E, const int64_t* indptr,
                          const int32_t* indices, const float* feats, int32_t D, uint32_t flags);

dci_status dci_destroy(dci_ctx* ctx);

/* --------------------------------------------------------------------------------------
 * Output of one mini-batch (all pointers are DEVICE memory owned by the caller).
 * Hop h (0 = the seeds' hop) samples dst = F_h with fan-out fanouts[L-1-h] (DGL order,
 * C3) and produces the block CSR (bptr[h], bsrc[h]) over dst = F_h, src ids local to
 * F_{h+1}.  frontier holds F_L; every F_h is its prefix of length sizes[h] (C2, C6).
 *  frontier  int32[frontier_cap]       global node ids, first-occurrence order (O-6)
 *  sizes     int64[L+1]                |F_0| .. |F_L|
 *  bptr[h]   int32[hop_cap[h] + 1]     block row pointers (bptr[h][0] = 0)
 *  bsrc[h]   int32[bsrc_cap[h]]        block column ids (local ids into F_{h+1})
 *  X         fp32[frontier_cap * ldx]  X[i][0..D) = feats[F_L[i]] (O-7); columns
 *                                      [D, pitch) receive the zero pad when ldx >= pitch;
 *                                      may be NULL (sampling only)
 *  counters  uint64[4]                 {adj_hit, adj_miss, feat_hit, feat_miss} of this
 *                                      batch (O-9), overwritten
 *  status    int32[1]                  DCI_OK or DCI_ESEED / DCI_EDUP, overwritten
 * Capacities must be >= the values dci_output_bounds returns (checked on the host ->
 * DCI_ECAP), so the device path never truncates.
 * ------------------------------------------------------------------------------------ */
typedef struct dci_batch_out {
  int32_t* frontier;
  int64_t frontier_cap;
  int64_t* sizes;
  int32_t* bptr[DCI_MAX_LAYERS];
  int32_t* bsrc[DCI_MAX_LAYERS];
  int64_t hop_cap[DCI_MAX_LAYERS];
  int64_t bsrc_cap[DCI_MAX_LAYERS];
  float* X;
  int64_t ldx;
  uint64_t* counters;
  int32_t* status;
} dci_batch_out;

/* Worst-case sizes for a batch of B seeds: frontier_caps[h] = min(N, B*prod_{j<h}(1+f_j))
 * for h = 0..L (host int64[L+1]), bsrc_caps[h] = frontier_caps[h] * f_h (host int64[L]),
 * feature pitch in floats.  Pure host arithmetic. */
dci_status dci_output_bounds(const dci_ctx* ctx, int32_t B, const int32_t* fanouts, int32_t L,
                             int64_t* frontier_caps, int64_t* bsrc_caps, int32_t* pitch);

/* --------------------------------------------------------------------------------------
 * Workspace: per-stream scratch for one in-flight batch (epoch-tagged node->position table
 * of N uint64, candidate / count arrays, scan tile state, batch scalars, stage events).
 * Sized for batches of up to max_batch seeds with fan-outs up to max_fanouts[.] (L hops).
 * Use one workspace per concurrently in-flight batch (a dci_sample_gather_many group uses one
 * per batch of the group), and issue a workspace's batches in order on one stream (its scratch
 * is reused by the next batch).  The number of live workspaces also tells the library how many
 * single-batch calls are in flight: their register-copy gather takes 4 blocks per SM with one
 * live workspace, 2 with two or three, 1 with four or more (override: env DCI_GATHER_BPS).
 * Memory: 8 N bytes of position table + candidate arrays of max |F_h| * f_h int32 (x2) + small.
 * ------------------------------------------------------------------------------------ */
dci_status dci_workspace_create(dci_ctx* ctx, int32_t max_batch, const int32_t* max_fanouts, int32_t L,
                                dci_workspace** out);
dci_status dci_workspace_destroy(dci_workspace* ws);

/* --------------------------------------------------------------------------------------
 * dci_sample_gather — S5..S8, the per-batch hot loop.  P:116-117, P:128 (sampled
 * inference), P:170 (hit -> GPU memory, miss -> host memory through UVA)
 * (adjacency prefix-hit rule), P:200 (feature cache lookup).
 *  seeds  device int32[B] (unique ids in [0, N)); B >= 0, B <= the workspace's max_batch.
 *  fanouts host int32[L] (DGL order, each 1..1024, each <= the workspace's max_fanouts).
 *  seed   64-bit sampling seed; draws are Philox(ctr=(node, slot, hop, pass=0),
 *         key=seed) (O-2), so results do not depend on batch composition or GPU count.
 * Asynchronous on `stream`; enqueues only device work (no host sync, no allocation).
 * Allowed in both states: before dci_fill it samples the original CSC with no cache.
 * ------------------------------------------------------------------------------------ */
dci_status dci_sample_gather(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds, int32_t B,
                             const int32_t* fanouts, int32_t L, uint64_t seed, const dci_batch_out* out,
                             void* stream);

/* --------------------------------------------------------------------------------------
 * dci_sample_gather_many — the same S5..S8 for a group of n batches (1 <= n <= DCI_MAX_GROUP),
 * one workspace and one dci_batch_out per batch (distinct workspaces, all with the call's L).
 * Batch i samples seeds[i] (device int32[B[i]]).  Every sampling kernel covers all n batches
 * (one hop / scan launch per hop for the whole group, captured once as a CUDA graph on ws[0]);
 * then ONE feature-gather launch (Blackwell bulk copies, cp.async.bulk, through a shared-memory
 * ring) moves the rows of every batch on the context's gather stream, so group gathers run one at
 * a time while the next group samples.  When 2..32 batches together hold at least N rows -- or
 * part of the features live in host memory and the host bytes a row-by-row gather would move
 * outweigh probing every node id -- the gather sweeps node ids and reads each feature row ONCE
 * for all batches holding it, in node order (P:170's hit/miss sources unchanged).  Likewise a hop
 * samples by node sweep once its frontiers reach N nodes (N / 20 when part of the adjacency is
 * host-resident).  Sweeps need dense position tables (8 N bytes per workspace; DCI_TABLE=dense
 * forces them for large graphs).  Results are identical to n dci_sample_gather calls (O-6, O-7;
 * the draws do not depend on the batch, C4).  Asynchronous on `stream`: work enqueued on `stream`
 * before the call happens before the group, and work enqueued after it sees every output; issue
 * a workspace's groups in order on one stream, and a context's groups from one host thread (they
 * share its gather stream and, under DCI_PHASED=1/2, the schedule's event).  If an output cannot
 * take bulk stores (X NULL,
 * ldx % 4 != 0 or X not 16-byte aligned) the batches run one by one on `stream`.  Timing
 * (profiling on ws[0]): the group's sampling and its gather launch are each timed once and
 * booked on ws[0] (dci_workspace_stats).
 * Errors: as dci_sample_gather per batch; DCI_EINVAL for n out of range or a repeated workspace.
 * ------------------------------------------------------------------------------------ */
dci_status dci_sample_gather_many(dci_ctx* ctx, int32_t n, dci_workspace* const* ws, const int32_t* const* seeds,
                                  const int32_t* B, const int32_t* fanouts, int32_t L, uint64_t seed,
                                  const dci_batch_out* outs, void* stream);

/* Per-batch results copied back to the host by dci_sample_gather_many_host. */
typedef struct dci_batch_result {
  int64_t sizes[DCI_MAX_LAYERS + 1]; /* |F_0| .. |F_L| (entries past L unspecified) */
  uint64_t counters[4];              /* adj_hit, adj_miss, feat_hit, feat_miss */
  int32_t status;                    /* DCI_OK, DCI_ESEED or DCI_EDUP */
  int32_t pad_;
} dci_batch_result;

/* End-to-end group variant: seeds_host[i] HOST int32[B[i]] (pinned for overlap) copied to the
 * workspaces' staging buffers on `stream`, then dci_sample_gather_many, then ONE device->host
 * copy of all n results into results_host (HOST dci_batch_result[n], pinned for overlap), on
 * `stream`; valid once the stream has been synchronised. */
dci_status dci_sample_gather_many_host(dci_ctx* ctx, int32_t n, dci_workspace* const* ws,
                                       const int32_t* const* seeds_host, const int32_t* B, const int32_t* fanouts,
                                       int32_t L, uint64_t seed, const dci_batch_out* outs,
                                       dci_batch_result* results_host, void* stream);

/* End-to-end variant: seeds_host is HOST memory (pinned for full overlap); the call
 * enqueues the host->device copy of the seeds, the batch, and device->host copies of
 * sizes (int64[L+1]), counters (uint64[4]) and status (int32) into the given host buffers.
 * Asynchronous: the host buffers are valid after the stream is synchronised. */
dci_status dci_sample_gather_host(dci_ctx* ctx, dci_workspace* ws, const int32_t* seeds_host, int32_t B,
                                  const int32_t* fanouts, int32_t L, uint64_t seed, const dci_batch_out* out,
                                  int64_t* sizes_host, uint64_t* counters_host, int32_t* status_host,
                                  void* stream);

/* --------------------------------------------------------------------------------------
 * dci_presample — S1.  P:177 (pre-sampling batches), P:196 (t_sample, t_feature per
 * batch), P:200 (per-node visit counts), P:203 (per-element Counts, Fig. 6(a)).
 * Runs ceil(num_seeds / batch) batches (last one ragged) with pass = 1 over the ORIGINAL
 * CSC and no cache, and ACCUMULATES (+=) into the caller's device arrays:
 *   node_visits int32[N]: +1 per batch in which v is in F_L (C7)
 *   edge_counts int32[E]: +1 per (hop, batch) in which element e is sampled (C8)
 * and writes host uint64 t_sample_ns[nb], t_feature_ns[nb] (CUDA-event stage times of
 * each batch: hops S5-S6 vs route+gather S7-S8).  Synchronises `stream`.
 * Errors: DCI_EINVAL, DCI_ESTATE (after dci_fill), DCI_ESEED / DCI_EDUP (bad seeds).
 * ------------------------------------------------------------------------------------ */
dci_status dci_presample(dci_ctx* ctx, const int32_t* seeds, int64_t num_seeds, int32_t batch,
                         const int32_t* fanouts, int32_t L, uint64_t seed, int32_t* node_visits,
                         int32_t* edge_counts, uint64_t* t_sample_ns, uint64_t* t_feature_ns, void* stream);

/* --------------------------------------------------------------------------------------
 * dci_allocate — S2, Eq. (1).  Exact integer arithmetic (O-10):
 *   C_adj = floor(C * S / (S + F)), C_feat = C - C_adj, S = sum t_sample_ns, F = sum
 *   t_feature_ns; S + F == 0 -> C_adj = floor(C / 2).
 *   ratio_den > 0: C_adj = floor(C * ratio_num / ratio_den) instead (sweeps, C20).
 *   C == 0 ("auto"): C = free device memory + memory the fill releases (current
 *   caches, the presample workspace) - the fill's temporaries (<= 48 B/node + 24 B/element)
 *   - 1 GiB reserve (C21), floored at 0.  Create the inference workspaces and outputs BEFORE
 *   this call: they are then already excluded from the free memory the budget is cut from.
 * Postcondition: *c_adj + *c_feat == C.  Host-only.
 * ------------------------------------------------------------------------------------ */
dci_status dci_allocate(dci_ctx* ctx, uint64_t C, const uint64_t* t_sample_ns, const uint64_t* t_feature_ns,
                        int32_t n, int64_t ratio_num, int64_t ratio_den, uint64_t* c_adj, uint64_t* c_feat);

/* --------------------------------------------------------------------------------------
 * dci_fill — S3 + S4.  Feature fill P:200 (O-11): cap = min(N, floor(c_feat / (4*pitch)))
 * rows; admits the top-cap nodes by (visits desc, id asc) via a device radix select and
 * assigns slots in ascending id.  Adjacency fill, Algorithm 1 P:209-243 + Fig. 6
 * P:203-206 (O-12): per-node stable reorder of each run by count desc (level 2, always
 * applied to the host CSC), node order (total desc, id asc) (level 1) found by a weighted
 * radix select, node-major prefix of floor(c_adj / 4) elements (whole CSC if it fits).
 *  node_visits device int32[N], edge_counts device int32[E] (e.g. the presample output,
 *  allreduced across ranks).  Re-filling recomputes from the original CSC (idempotent).
 * Synchronises `stream`.  Device memory: caches + ~8E bytes temporarily.
 * ------------------------------------------------------------------------------------ */
dci_status dci_fill(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts, uint64_t c_adj,
                    uint64_t c_feat, void* stream);

/* --------------------------------------------------------------------------------------
 * dci_fill_knapsack — NEXT F4: the DUCATI-style comparison strategy (
 * simplified as in SPEC S:496-504, O-14): one budget C (bytes) over feature rows (value =
 * visits * cost_feat, size = 4*pitch) and adjacency elements (value = count * cost_adj, 4 B),
 * admitted greedily by value density (ties: feature first, then id), skipping items that no
 * longer fit.  The admitted elements of each node form a prefix of its level-2 order, so the
 * host CSC is reordered exactly as by dci_fill and the prefix hit rule holds.  cost_* are the
 * times saved per hit (any unit, only their ratio matters).  Synchronises `stream`.
 * ------------------------------------------------------------------------------------ */
dci_status dci_fill_knapsack(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts, uint64_t C,
                             double cost_feat, double cost_adj, void* stream);

/* --------------------------------------------------------------------------------------
 * NEXT F1 — NVLink-partitioned feature cache (BJ north_star: "a partitioned cache read over
 * NVLink peer access").  All `world` ranks fill with the same (allreduced) counts; the admitted
 * set is the top min(N, world * floor(c_feat / (4*pitch))) nodes (O-11 with that capacity,
 * slots in ascending id), and global slot s is stored on rank s % world at row s / world.
 * c_feat is the budget of ONE partition (one GPU).  The adjacency cache stays replicated.
 *  rank in [0, world): this device holds only its partition; exchange partitions with
 *    dci_feature_partition_handle (a 64-byte CUDA IPC handle of the local rows) and
 *    dci_attach_feature_partitions (all ranks' handles, rank-major) before sampling; hits on
 *    other partitions are then peer loads over NVLink (P2P through CUDA IPC mappings).
 *  rank == -1: all partitions live on this device (single-device emulation / testing).
 * A re-fill frees this rank's partition and closes the peers' mappings: exchange and attach
 * again (on every rank, after all ranks have filled) before the next batch.
 * Synchronises `stream`.  Errors: DCI_EINVAL (world not in 1..16, rank out of range).
 * ------------------------------------------------------------------------------------ */
#define DCI_IPC_HANDLE_BYTES 64
dci_status dci_fill_partitioned(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts,
                                uint64_t c_adj, uint64_t c_feat, int32_t world, int32_t rank, void* stream);
dci_status dci_feature_partition_handle(dci_ctx* ctx, void* handle /* DCI_IPC_HANDLE_BYTES */);
dci_status dci_attach_feature_partitions(dci_ctx* ctx, const void* handles /* world * 64 bytes */,
                                         int32_t world);

/* --------------------------------------------------------------------------------------
 * Introspection (parity tests).  Every output pointer is HOST memory and may be NULL.
 *  cached_len int32[N], cache_off int64[N] (element offset of v's prefix in acache),
 *  slot_of int32[N] (-1 = not cached; a global slot when partitioned), acache
 *  int32[info.adj_elems] (prefixes laid out in ascending node id), fcache
 *  fp32[info.feat_rows * pitch] (this device's rows; partition by partition when emulated),
 *  indices_cur int32[E] (the
 *  current host CSC: original before fill, level-2 reordered after).
 * ------------------------------------------------------------------------------------ */
typedef struct dci_cache_info {
  int32_t state;
  int32_t pitch;          /* floats per cached/host feature row */
  int64_t N, E;
  int32_t D;
  int32_t whole_fit;      /* 1 if the whole CSC is cached (Alg. 1 lines 1-3) */
  uint64_t c_adj, c_feat; /* bytes granted by the last fill */
  int64_t adj_elems;      /* elements in the adjacency cache */
  int64_t feat_rows;      /* feature-cache rows held on this device */
  int64_t feat_rows_total; /* rows over all feature partitions (== feat_rows unless partitioned) */
  int32_t feat_partitions; /* 1, or the partition count of dci_fill_partitioned */
  int32_t pad_;
  uint64_t presample_peak_bytes;
  uint64_t launches;      /* kernels this context has launched so far */
} dci_cache_info;

dci_status dci_cache_info_get(const dci_ctx* ctx, dci_cache_info* info);

/* Stage times of the last fill, in ms (CUDA events on the fill stream; -1 = stage not timed):
 * level 2 (per-node reorder, Alg. 1's element sort, incl. the reordered CSC back to the host),
 * adjacency selection (level-1 weighted radix select + prefix scan), adjacency copy (prefixes
 * into the cache), feature selection (top-k radix select + slot scan), feature copy (host rows
 * into HBM), total.  The knapsack fill (F4) reports level 2 and the total only.  P:316-330 and
 * P:371-376 make preprocessing time a headline; this splits it by step. */
typedef struct dci_fill_times {
  float level2_ms, adj_select_ms, adj_copy_ms, feat_select_ms, feat_copy_ms, total_ms;
} dci_fill_times;
dci_status dci_fill_times_get(const dci_ctx* ctx, dci_fill_times* out);
dci_status dci_cache_state(dci_ctx* ctx, int32_t* cached_len, int64_t* cache_off, int32_t* slot_of,
                           int32_t* acache, float* fcache, int32_t* indices_cur);

/* Stage times of the workspace's last batch, in ms (CUDA events recorded on the launch
 * streams around the sampling hops and around the gather launch; requires profiling on).
 * Timing uses a ring of event records per workspace, so it never blocks the host. */
dci_status dci_workspace_set_profiling(dci_workspace* ws, int32_t on);
dci_status dci_workspace_stage_ms(dci_workspace* ws, float* sample_ms, float* gather_ms);

/* Running totals of a workspace since its last reset (synchronises the device):
 * batches finished, seeds, sum of |F_L| (feature rows gathered), summed counters, and -
 * with profiling on - the number of event-timed batches and their summed sampling time
 * (hops S5-S6), the number of timed gather launches and their summed time (S7-S8; a
 * dci_sample_gather_many group has ONE launch, booked on its first workspace), in ms.
 * rows_read: feature rows the gather actually read (a node-sweep group reads each row once
 * for all its batches); gather_bytes: the gather's algorithmic bytes (row
 * reads + row writes + lookups), also booked on a group's first workspace.
 * host_rows_read: feature rows read from pinned host memory (misses; once per row in a node
 * sweep); host_adj_sectors: distinct 32-byte host sectors (the unit the GPU fetches from system
 * memory) read by adjacency misses (per dst node and hop; a node-sweep hop reads a node's
 * elements once for all batches).  Together they give the host-link bytes of the bench roofline
 * (T_roof = max(B_hbm/BW_hbm, B_host/BW_host, ...)).  Both are booked on the first
 * workspace of a launch.
 * reset != 0 zeroes the totals after reading them. */
typedef struct dci_ws_stats {
  uint64_t batches;
  uint64_t seeds;
  uint64_t frontier_rows;
  uint64_t counters[4];
  uint64_t timed_batches;
  double sample_ms;
  double gather_ms;
  uint64_t gather_launches;
  uint64_t rows_read;
  uint64_t gather_bytes;
  uint64_t host_rows_read;
  uint64_t host_adj_sectors;
  uint64_t gather_kinds[3]; /* group gathers this workspace led: row mode, node sweep with register
                               copies, node sweep with bulk copies */
  uint64_t table_bytes;     /* device bytes of the workspace's position table (dense 8 N, or hashed) */
  uint64_t host_adj_runs;   /* (dst, hop) runs with at least one adjacency miss: the random host requests
                               of the sampler (a run's sectors are contiguous); with host_rows_read the
                               request count of the bench's host-link request view */
} dci_ws_stats;

dci_status dci_workspace_stats(dci_workspace* ws, dci_ws_stats* out, int32_t reset);

/* --------------------------------------------------------------------------------------
 * dci_mean_aggregate — NEXT F2: the GraphSAGE mean aggregator the prepared mini-batch feeds
 * (BJ north_star's optional consumer; O-13):
 *   H[d][c] = (1/k_d) * sum_{j=bptr[d]}^{bptr[d+1]-1} Xsrc[bsrc[j]][c] for c < D, k_d = 0 -> 0,
 * for d < *n_dst.  All pointers DEVICE memory: bptr int32[n+1], bsrc int32[...], n_dst int64[1]
 * (e.g. out->sizes + h, so no host sync is needed), Xsrc fp32 rows of stride ldx (e.g. the
 * batch's X for the input layer h = L-1), H fp32 rows of stride ldh (caller-owned, >= n
 * rows).  fp32 accumulation in bsrc order.  Asynchronous on `stream`.
 * ------------------------------------------------------------------------------------ */
dci_status dci_mean_aggregate(dci_ctx* ctx, const int32_t* bptr, const int32_t* bsrc, const int64_t* n_dst,
                              const float* Xsrc, int64_t ldx, int32_t D, float* H, int64_t ldh, void* stream);

/* The same with the aggregator of Table III: DCI_AGG_MEAN ("avg", GCN) as above, or
 * DCI_AGG_SUM (GraphSAGE's "sum": H[d] = sum_j Xsrc[bsrc[j]], no 1/k_d). */
enum { DCI_AGG_MEAN = 0, DCI_AGG_SUM = 1 };
dci_status dci_block_aggregate(dci_ctx* ctx, const int32_t* bptr, const int32_t* bsrc, const int64_t* n_dst,
                               const float* Xsrc, int64_t ldx, int32_t D, float* H, int64_t ldh, int32_t op,
                               void* stream);

/* Kernels launched by this context so far (all workspaces). */
uint64_t dci_launch_count(const dci_ctx* ctx);

const char* dci_last_error(void);
int32_t dci_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DCI_H_ */
