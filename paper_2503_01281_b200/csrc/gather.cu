// S7 + S8 of the hot path.
//
// k_gather: one kernel per batch (dci_sample_gather, dci_presample):
//  - relabel of the last hop's candidates into its block CSR (table tag -> local id)
//  - feature-cache route inline through the remap table: slot = dir[F[i]].slot
//  - feature gather: X[i] = fcache[slot] on a hit (HBM -> HBM) or feats[v] on a
//    miss (pinned host -> HBM, UVA zero-copy), one warp per row, every lane issuing all of
//    its 16-byte loads before any store; the next row's (F, slot) lookups are prefetched
//  - presample: node_visits[v] += 1 (C7)
//  - the last block to finish publishes sizes / counters / status and resets the
//    workspace scalars for the next batch.
//
// k_gather_tma: one kernel per group of batches (dci_sample_gather_many): Blackwell bulk copies
// through a shared-memory ring, in row mode or node-sweep mode (see the kernel's comments).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "dci_internal.cuh"

namespace dci {

namespace {

// L2 policy for the streaming feature traffic (rows read once per batch, X written once):
// evict-first, so ~700 MB/batch of streaming bytes do not flush the small hot structures
// (directory, adjacency cache lines, position tables) out of the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ int4 ld_stream_v4(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// Pinned-host (UVA) row reads on a miss: a plain (L1-allocating) load.  Random host-row reads with
// L1::no_allocate loads stop at ~25.7 GB/s on this B200 whatever the row size, plain loads reach
// ~49.7 GB/s (tools/probe/hostreq_probe.cu, profiles/hostreq_probe.jsonl); host rows are
// read-only while kernels run, so L1 allocation is safe.
__device__ __forceinline__ int4 ld_host_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// a feature row's 16-byte word from the HBM cache (hit) or from pinned host memory (miss)
__device__ __forceinline__ int4 ld_row_v4(const int4* p, bool host, uint64_t pol) {
  return host ? ld_host_v4(p) : ld_stream_v4(p, pol);
}

__device__ __forceinline__ void st_v4(int4* p, const int4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

struct FusedArgs {
  const DirEntry* dir;
  unsigned long long* pos_of;
  uint32_t hmask;  // position table layout (dci_internal.cuh)
  BatchScalars* sc;
  int64_t N;
  int32_t L;
  const int32_t* F;
  // last hop (L-1) relabel
  const int32_t* last_cand;
  const int32_t* last_kcnt;
  const int32_t* last_bptr;
  int32_t* last_bsrc;
  int32_t last_f;
  unsigned long long* last_tiles;
  int64_t last_ntiles;
  // feature rows
  const float* fcache;
  const float* const* fbases;  // feature partitions (G > 1): slot s -> fbases[s % G] + (s / G) rows
  int32_t G;
  const float* hfeats;  // device alias of the pinned host feature table
  int32_t pitch;
  int32_t D;
  float* X;
  int64_t ldx;
  int32_t* node_visits;
  // publication
  int64_t* out_sizes;
  uint64_t* out_counters;
  int32_t* out_status;
};

// MODE 0: no X (route + counters only); 1: scalar copy of D floats; 2: int4 copy of pitch
// floats (ldx % 4 == 0, ldx >= pitch), VPL int4 per lane per pass.
template <int MODE, int VPL>
__global__ void __launch_bounds__(256) k_gather(FusedArgs a) {
  BatchScalars* sc = a.sc;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int32_t B = sc->hdr.B;
  {
    const int pf = a.last_f;
    const int64_t n_prev = (a.L == 1) ? (int64_t)B : sc->sizes[a.L - 1];
    const int64_t nq = n_prev * pf;
    for (int64_t q = tid; q < nq; q += nthreads) {
      const int64_t d = q / pf;
      const int s = (int)(q - d * pf);
      if (s < a.last_kcnt[d])
        a.last_bsrc[a.last_bptr[d] + s] =
            (int32_t)(0xFFFFFFFFu - (uint32_t)pt_tag(a.pos_of, a.hmask, a.last_cand[q], sc->hdr.epoch));
    }
    for (int64_t t = tid; t < a.last_ntiles; t += nthreads) a.last_tiles[t] = 0ull;
    if (tid == 0) sc->tickets[a.L - 1] = 0;
  }
  const int64_t n = sc->sizes[a.L];
  const uint64_t pol = policy_evict_first();
  const int64_t warp = tid >> 5;
  const int64_t nwarps = nthreads >> 5;
  uint32_t hits = 0, misses = 0;
  int64_t r = warp;
  int32_t v = -1, slot = -1;
  if (r < n) {
    v = a.F[r];
    if (v >= 0 && (int64_t)v < a.N) slot = __ldg(&a.dir[v].slot);
  }
  while (r < n) {
    const int64_t nxt = r + nwarps;
    int32_t vn = -1;
    if (nxt < n) vn = a.F[nxt];
    const bool ok = v >= 0 && (int64_t)v < a.N;
    if (ok) {
      const float* src;
      if (slot < 0)
        src = a.hfeats + (int64_t)v * a.pitch;
      else if (a.G == 1)
        src = a.fcache + (int64_t)slot * a.pitch;
      else  // partitioned cache: local or peer (NVLink) rows
        src = reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(a.fbases) +
                                                   slot % a.G)) +
              (int64_t)(slot / a.G) * a.pitch;
      if (MODE == 2) {
        const int row16 = a.pitch >> 2;
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(a.X + r * a.ldx);
        for (int c0 = 0; c0 < row16; c0 += 32 * VPL) {
          int4 buf[VPL];
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            const int idx = c0 + lane + 32 * j;
            if (idx < row16) buf[j] = ld_row_v4(s4 + idx, slot < 0, pol);
          }
#pragma unroll
          for (int j = 0; j < VPL; ++j) {
            const int idx = c0 + lane + 32 * j;
            if (idx < row16) st_v4(d4 + idx, buf[j], pol);
          }
        }
      } else if (MODE == 1) {
        float* dst = a.X + r * a.ldx;
        for (int c = lane; c < a.D; c += 32) dst[c] = src[c];
      }
      if (lane == 0) {
        if (slot >= 0)
          ++hits;
        else
          ++misses;
        if (a.node_visits) atomicAdd(a.node_visits + v, 1);
      }
    }
    int32_t sn = -1;
    if (vn >= 0 && (int64_t)vn < a.N) sn = __ldg(&a.dir[vn].slot);
    r = nxt;
    v = vn;
    slot = sn;
  }
  if (lane == 0 && (hits | misses)) {
    atomicAdd(&sc->counters[2], (unsigned long long)hits);
    atomicAdd(&sc->counters[3], (unsigned long long)misses);
  }
  // last block publishes the batch scalars and resets them for the next batch
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&sc->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    a.out_sizes[0] = B;
    for (int h = 1; h <= a.L; ++h) a.out_sizes[h] = __ldcg(&sc->sizes[h]);
    for (int c = 0; c < 4; ++c) {
      a.out_counters[c] = __ldcg(&sc->counters[c]);
      sc->counters[c] = 0;
    }
    *a.out_status = __ldcg(&sc->status);
    sc->acc_batches += 1;
    sc->acc_seeds += (unsigned long long)B;
    const unsigned long long rows = (unsigned long long)__ldcg(&sc->sizes[a.L]);
    sc->acc_rows += rows;
    if (MODE != 0) {
      sc->acc_rows_read += rows;
      sc->acc_gather_bytes += rows * (8ull * (unsigned long long)a.D + 4ull);
      sc->acc_host_rows += a.out_counters[3];  // every miss row is read from the host once
    }
    for (int c = 0; c < 4; ++c) sc->acc_counters[c] += a.out_counters[c];
    sc->status = 0;
    sc->done = 0;
  }
}

// ------------------------------------------------------------------------------------
// k_gather_tma: S7 + S8 with the Blackwell bulk-copy (TMA) engine instead of register copies.
// Each warp runs a K-slot shared-memory ring; a slot holds a chunk of R consecutive rows of F_L.
//  issue   lane 0 arms the slot's mbarrier with the chunk's bytes (expect_tx), then lane j of
//          the chunk issues cp.async.bulk global -> shared for its row (HBM cache row on a hit,
//          pinned host row through UVA on a miss), completing on the mbarrier
//  drain   wait on the mbarrier, then cp.async.bulk shared -> global into X (one bulk store of
//          R rows when X rows are contiguous, else one per row), committed as a bulk group;
//          a slot is refilled once its store has finished reading shared memory
// Row lookups (F[r] -> dir[F[r]].slot -> source address) are done 32 rows (one group) at a time
// by the 32 lanes and prefetched one group ahead, so the issuing lanes never wait on them.
// A handful of warps per SM keep ~150 KB of rows in flight, leaving the SM's registers and warps to
// the latency-bound sampling kernels of other batches.
// ------------------------------------------------------------------------------------
constexpr int kTmaMaxSlots = 16;
constexpr int kTmaMaxWarps = 8;
constexpr int kTmaMaxBatches = DCI_MAX_GROUP;
constexpr int kMaxDevices = 64;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TMA_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TMA_WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst), "r"(src),
               "r"(bytes), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct TmaArgs {
  int32_t hint;       // 1: evict-first L2 hint on rows and X, 0: evict-normal
  int32_t K;          // ring slots per warp
  int32_t R;          // rows per chunk (slot)
  int32_t row_bytes;  // 4 * pitch
  int32_t slot_bytes; // R * row_bytes
};

// One batch of a (multi-batch) TMA gather launch.
struct TmaBatch {
  const int32_t* F;       // F_L (global ids)
  const unsigned long long* pos_of;  // the workspace's node -> (epoch, local id) table
  BatchScalars* sc;       // the batch's workspace scalars (sizes[L], counters, status)
  float* X;
  int64_t ldx;            // floats
  int32_t out16;          // 16-byte words written per X row by the node sweep (whole 128-byte lines
                          // when ldx is a multiple of 32 floats and X is 128-byte aligned, else pitch)
  int32_t* node_visits;   // presample only
  int64_t* out_sizes;
  uint64_t* out_counters;
  int32_t* out_status;
};

struct TmaBatches {
  int32_t n;  // batches in this launch (<= kTmaMaxBatches)
  int32_t L;
  // node sweep only: 0 = every row of F_L; split group gather: 1 = the rows of F_{L-1} (local ids
  // < |F_{L-1}|, final once hop L-2's scan is done, so this launch runs beside hop L-1's sampling),
  // 2 = the rest (ids >= |F_{L-1}|, after hop L-1's scan)
  int32_t phase;
  int64_t N;
  const DirEntry* dir;
  const float* fcache;
  const float* const* fbases;
  int32_t G;
  int32_t pitch;
  int32_t D;
  const float* hfeats;
  dci_batch_result* stage;  // nullable: results of every batch, for one device->host copy
  TmaBatch b[kTmaMaxBatches];
};


// Shared end of a group gather launch (row mode and node sweep): per-batch feature hit/miss
// counts and the rows this block read are folded into the workspaces' scalars; the last block
// books the launch's algorithmic bytes on the first batch and publishes every
// batch's sizes / counters / status (and the staging record), then resets the scalars.
//  rows:  sum_b |F_L(b)| x (row read 4D + row write 4D + 4 B slot lookup)
//  sweep: N x (8 B tag probe per batch + 4 B slot lookup) + |union| x 4D + sum_b |F_L(b)| x 4D
__device__ __forceinline__ void group_epilogue(const TmaBatches& a, const unsigned (*s_cnt)[2], unsigned s_reads,
                                               unsigned s_host_rows, long long tot_rows, bool sweep) {
  // (a split gather's first launch books its bytes and folds its feature counts into the
  // scalars, but publishes nothing: the second launch publishes the batches' results)
  const int nb = a.n;
  if (threadIdx.x == 0 && s_reads) atomicAdd(&a.b[0].sc->launch_reads, (unsigned long long)s_reads);
  if (threadIdx.x == 0 && s_host_rows) atomicAdd(&a.b[0].sc->acc_host_rows, (unsigned long long)s_host_rows);
  if (threadIdx.x < nb) {
    const int i = threadIdx.x;
    if (s_cnt[i][0]) atomicAdd(&a.b[i].sc->counters[2], (unsigned long long)s_cnt[i][0]);
    if (s_cnt[i][1]) atomicAdd(&a.b[i].sc->counters[3], (unsigned long long)s_cnt[i][1]);
  }
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.b[0].sc->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    BatchScalars* sc0 = a.b[0].sc;
    const unsigned long long reads = __ldcg(&sc0->launch_reads);
    const unsigned long long tot = (unsigned long long)tot_rows;
    const unsigned long long rowb = 4ull * (unsigned long long)a.D;
    sc0->acc_rows_read += reads;
    sc0->acc_gather_bytes += sweep ? (unsigned long long)a.N * (8ull * nb + 4ull) + reads * rowb + tot * rowb
                                   : tot * (2ull * rowb + 4ull);
    sc0->launch_reads = 0;
    sc0->sweep_ticket = 0;
    if (a.phase == 1) sc0->done = 0;
  }
  __syncthreads();
  if (s_last && a.phase != 1 && threadIdx.x < nb) {
    __threadfence();
    const TmaBatch& tb = a.b[threadIdx.x];
    BatchScalars* sc = tb.sc;
    const int32_t B = sc->hdr.B;
    tb.out_sizes[0] = B;
    for (int h = 1; h <= a.L; ++h) tb.out_sizes[h] = __ldcg(&sc->sizes[h]);
    for (int c = 0; c < 4; ++c) {
      tb.out_counters[c] = __ldcg(&sc->counters[c]);
      sc->counters[c] = 0;
    }
    *tb.out_status = __ldcg(&sc->status);
    if (a.stage) {
      dci_batch_result& r = a.stage[threadIdx.x];
      for (int h = 0; h <= a.L; ++h) r.sizes[h] = tb.out_sizes[h];
      for (int c = 0; c < 4; ++c) r.counters[c] = tb.out_counters[c];
      r.status = *tb.out_status;
    }
    sc->acc_batches += 1;
    sc->acc_seeds += (unsigned long long)B;
    sc->acc_rows += (unsigned long long)__ldcg(&sc->sizes[a.L]);
    for (int c = 0; c < 4; ++c) sc->acc_counters[c] += tb.out_counters[c];
    sc->status = 0;
    if (threadIdx.x == 0) sc->done = 0;
  }
}

// ------------------------------------------------------------------------------------
// k_gather_sweep: node-sweep gather of a group (2..32 batches whose frontiers together cover the
// node set, e.g. Reddit-shaped graphs where one batch touches 61 % of all nodes).  The draws of a
// node do not depend on its batch (C4), so the batches of a group share most rows: instead of
// reading a feature row once per (batch, row), warps sweep node ids and look every node up in each
// batch's node -> local-id table (the epoch-tagged position table the sampler leaves behind: v is
// in batch b's F_L iff its tag carries b's epoch, and the tag's low word is then ~row).  A node
// present in any batch is read ONCE and written to every batch that holds it.  X is bit-identical
// to the row-mode gather.
//  probe  lane j of a warp owns node g + j: one coalesced 8-byte tag load per batch (a warp reads
//         256 contiguous bytes of each table) + its directory slot; the rows it holds go to a
//         per-warp shared-memory table (batch-major, conflict-free)
//  copy   the warp walks its present nodes two at a time: all lanes load both rows (16 B per lane,
//         register copies; HBM cache row on a hit, pinned host row through UVA on a miss) and store
//         each to every batch holding it.  Rows are written as whole 128-byte lines when the
//         output allows it (out16: zeros past the pitch): random-row writes of partial lines run
//         at ~4.0 TB/s on this B200, of whole lines at ~5.4-5.7 TB/s (tools/probe/scatter_probe.cu,
//         profiles/r02/scatter_probe.md).
// No per-lane arrays and no ring: ~40 registers, so many warps per SM hide the probe latency, and
// the SM's remaining registers are left to the next group's sampling kernels.
// ------------------------------------------------------------------------------------
constexpr int kSweepWarps = 8;
constexpr int kSweepMax = DCI_MAX_GROUP;  // 32-bit presence masks

// Per-launch batch table of a node sweep (shared memory): each batch's epoch and the local-id range
// [lo, hi) this launch writes (phase 0: all of F_L; split gather: 1 = F_{L-1}, 2 = the rest), and the
// rows the launch writes in all (for its algorithmic bytes).  |F_{L-1}| is final once hop L-2's
// scan has run: the hop L-1 sampling running beside a phase-1 launch only raises the tags of nodes
// outside F_{L-1} (candidate positions >= |F_{L-1}|), and its scan gives new nodes ids >= |F_{L-1}|.
// Ends with a block barrier.
__device__ __forceinline__ void sweep_init(const TmaBatches& a, uint32_t* s_ep, uint32_t* s_lo, uint32_t* s_hi,
                                           long long* s_tot) {
  const int nb = a.n;
  if (threadIdx.x < 32) {  // warp 0: lane b reads batch b; the rows written summed by shuffles
    long long rows = 0;
    if (threadIdx.x < nb) {
      const BatchScalars* sc = a.b[threadIdx.x].sc;
      s_ep[threadIdx.x] = __ldcg(&sc->hdr.epoch);
      const uint32_t nprev = a.L >= 2 ? (uint32_t)__ldcg(&sc->sizes[a.L - 1]) : (uint32_t)__ldcg(&sc->hdr.B);
      const long long nl = a.phase == 1 ? 0 : __ldcg(&sc->sizes[a.L]);
      s_lo[threadIdx.x] = a.phase == 2 ? nprev : 0u;
      s_hi[threadIdx.x] = a.phase == 1 ? nprev : 0xFFFFFFFFu;
      rows = a.phase == 0 ? nl : a.phase == 1 ? (long long)nprev : nl - (long long)nprev;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) rows += __shfl_xor_sync(0xffffffffu, rows, o);
    if (threadIdx.x == 0) *s_tot = rows;
  }
  __syncthreads();
}

// X row address of node j (lane index in the warp's group) in batch b
__device__ __forceinline__ int4* sweep_dst(const TmaBatches& a, const int* rt, int b, int j) {
  const TmaBatch& tb = a.b[b];
  return reinterpret_cast<int4*>(tb.X + (int64_t)rt[b * 32 + j] * tb.ldx);
}

// Row of one node (registers, VPL 16-byte words per lane per pass) -> every batch in mask m.  The
// destinations are taken two at a time, so the row-table (shared) and batch-table (constant) loads
// of the second overlap the first's stores.
template <int VPL>
__device__ __forceinline__ void sweep_store(const TmaBatches& a, const int* rt, int j, unsigned m, const int4 (&buf)[VPL],
                                            int c0, int lane, uint64_t pol) {
  while (m) {
    const int b1 = __ffs(m) - 1;
    m &= m - 1;
    const int b2 = m ? __ffs(m) - 1 : -1;
    if (m) m &= m - 1;
    int4* d1 = sweep_dst(a, rt, b1, j);
    const int o1 = a.b[b1].out16;
    int4* d2 = b2 >= 0 ? sweep_dst(a, rt, b2, j) : nullptr;
    const int o2 = b2 >= 0 ? a.b[b2].out16 : 0;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int idx = c0 + lane + 32 * k;
      if (idx < o1) st_v4(d1 + idx, buf[k], pol);
    }
    if (d2) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int idx = c0 + lane + 32 * k;
        if (idx < o2) st_v4(d2 + idx, buf[k], pol);
      }
    }
  }
}

// Two nodes (rows s1 -> mask m1, s2 -> m2; s2 may be null): both rows' loads are issued before
// any store.
template <int VPL>
__device__ __forceinline__ void sweep_copy(const TmaBatches& a, const int* rt, int row16, const char* s1, bool h1,
                                           unsigned m1, int j1, const char* s2, bool h2, unsigned m2, int j2,
                                           int lane, int out16max, uint64_t pol) {
  for (int c0 = 0; c0 < out16max; c0 += 32 * VPL) {
    int4 b1[VPL], b2[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int idx = c0 + lane + 32 * k;
      b1[k] = idx < row16 ? ld_row_v4(reinterpret_cast<const int4*>(s1) + idx, h1, pol) : make_int4(0, 0, 0, 0);
      b2[k] = (s2 && idx < row16) ? ld_row_v4(reinterpret_cast<const int4*>(s2) + idx, h2, pol)
                                  : make_int4(0, 0, 0, 0);
    }
    sweep_store<VPL>(a, rt, j1, m1, b1, c0, lane, pol);
    if (s2) sweep_store<VPL>(a, rt, j2, m2, b2, c0, lane, pol);
  }
}

// cp.async (LDGSTS) of 4/8 bytes global -> shared; src_bytes 0 fills zeros (a node past N)
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int VPL>
__global__ void __launch_bounds__(32 * kSweepWarps) k_gather_sweep(const __grid_constant__ TmaBatches a,
                                                                   int32_t out16max, int32_t hint) {
  // dynamic shared memory, per warp: tag stage [nb][32] u64 (the next group's probes, in flight
  // while the current group copies), slot stage [32] i32, row table [nb][32] i32
  extern __shared__ __align__(128) unsigned char s_dyn[];
  __shared__ uint32_t s_ep[kSweepMax];
  __shared__ uint32_t s_lo[kSweepMax], s_hi[kSweepMax];  // local-id range this launch writes
  __shared__ unsigned s_cnt[kSweepMax][2];
  __shared__ unsigned s_reads, s_host;
  __shared__ long long s_tot;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nb = a.n;
  if (threadIdx.x < 2 * kSweepMax) (&s_cnt[0][0])[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    s_reads = 0u;
    s_host = 0u;
  }
  sweep_init(a, s_ep, s_lo, s_hi, &s_tot);
  __syncthreads();
  unsigned char* mine = s_dyn + (size_t)wib * (nb * 32 * 12 + 128);
  unsigned long long* stag = reinterpret_cast<unsigned long long*>(mine);  // [nb][32]
  int* sslot = reinterpret_cast<int*>(mine + nb * 32 * 8);                 // [32]
  int* rt = sslot + 32;                                                     // [nb][32]
  const uint64_t pol = hint ? policy_evict_first() : policy_evict_normal();
  const int row16 = a.pitch >> 2;
  // dynamic schedule: a warp takes the next 32-node group from a ticket counter (in the first
  // batch's scalars), so blocks that start late (SMs held by kernels running beside the gather)
  // take fewer groups instead of running as a tail wave
  unsigned long long* ticket = &a.b[0].sc->sweep_ticket;
  auto take = [&]() -> int64_t {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1ull);
    return 32 * (int64_t)__shfl_sync(0xffffffffu, t, 0);
  };
  // probes of the group starting at node g: lane j copies node g + j's tag in every batch table
  // and its directory slot into the stage (zeros past N)
  auto prefetch = [&](int64_t g) {
    if (g >= a.N) return;
    const int64_t v = g + lane;
    const bool in = v < a.N;
    const int64_t vv = in ? v : 0;
    for (int b = 0; b < nb; ++b) cp_async8(stag + b * 32 + lane, a.b[b].pos_of + vv, in ? 8 : 0);
    cp_async4(sslot + lane, &a.dir[vv].slot, in ? 4 : 0);
  };
  unsigned reads = 0, host_reads = 0, hits = 0, misses = 0;  // lane b: batch b's feature hits / misses
  int64_t g = take();
  prefetch(g);
  cp_async_commit();
  while (g < a.N) {
    cp_async_wait_all();
    __syncwarp();
    const int64_t v = g + lane;
    const int32_t sl = v < a.N ? sslot[lane] : -1;
    unsigned mask = 0;
    for (int b = 0; b < nb; ++b) {
      const unsigned long long tg = stag[b * 32 + lane];
      const uint32_t row = 0xFFFFFFFFu - (uint32_t)tg;
      if ((uint32_t)(tg >> 32) == s_ep[b] && row >= s_lo[b] && row < s_hi[b]) {
        mask |= 1u << b;
        rt[b * 32 + lane] = (int)row;
      }
    }
    __syncwarp();  // the stage is consumed: the next group's probes may overwrite it
    const int64_t g_next = take();
    prefetch(g_next);
    cp_async_commit();
    const char* src = nullptr;
    if (mask) {
      if (sl < 0)
        src = reinterpret_cast<const char*>(a.hfeats + v * a.pitch);
      else if (a.G == 1)
        src = reinterpret_cast<const char*>(a.fcache + (int64_t)sl * a.pitch);
      else  // partitioned cache: local or peer (NVLink) rows
        src = reinterpret_cast<const char*>(
            reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(a.fbases) + sl % a.G)) +
            (int64_t)(sl / a.G) * a.pitch);
    }
    const unsigned hitm = __ballot_sync(0xffffffffu, sl >= 0);
    for (int b = 0; b < nb; ++b) {
      const unsigned inb = __ballot_sync(0xffffffffu, (mask >> b) & 1u);
      if (lane == b) {
        hits += __popc(inb & hitm);
        misses += __popc(inb & ~hitm);
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, mask != 0);
    reads += __popc(m);
    host_reads += __popc(m & ~hitm);
    while (m) {
      const int j1 = __ffs(m) - 1;
      m &= m - 1;
      const int j2 = m ? __ffs(m) - 1 : j1;
      const bool two = m != 0;
      if (m) m &= m - 1;
      const char* s1 = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), j1));
      const unsigned m1 = __shfl_sync(0xffffffffu, mask, j1);
      const char* s2 = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), j2));
      const unsigned m2 = __shfl_sync(0xffffffffu, mask, j2);
      const bool h1 = (hitm >> j1 & 1u) == 0, h2 = (hitm >> j2 & 1u) == 0;  // host rows (misses)
      sweep_copy<VPL>(a, rt, row16, s1, h1, m1, j1, two ? s2 : nullptr, h2, two ? m2 : 0u, j2, lane, out16max, pol);
    }
    __syncwarp();  // every lane is done with the row table before the next group rewrites it
    g = g_next;
  }
  cp_async_wait_all();
  if (lane < nb) {
    if (hits) atomicAdd(&s_cnt[lane][0], hits);
    if (misses) atomicAdd(&s_cnt[lane][1], misses);
  }
  if (lane == 0 && reads) atomicAdd(&s_reads, reads);
  if (lane == 0 && host_reads) atomicAdd(&s_host, host_reads);
  __syncthreads();
  group_epilogue(a, s_cnt, s_reads, s_host, s_tot, true);
}

// ------------------------------------------------------------------------------------
// k_gather_sweep_tma: the same node sweep with Blackwell bulk copies instead of register copies
// (DCI_SWEEP_KIND=tma).  A present node's row is loaded ONCE into a shared-memory ring slot
// (cp.async.bulk global -> shared, completing on the slot's mbarrier; HBM cache row on a hit,
// pinned host row through UVA on a miss), then the lanes of the warp store it to every batch that
// holds it IN PARALLEL -- lane b issues one cp.async.bulk shared -> global of the whole row into
// batch b's X.  Ring slots are line-padded (out16max words) with a zero tail, so whole-line X rows
// need no register work.  Probes as in k_gather_sweep (cp.async-prefetched tags, dynamic group
// tickets); a node's destination rows are copied into its slot's metadata when its load is
// issued, so the next group's probes may be processed while earlier slots still drain.
// Few warps and ~40 registers keep enough bytes in flight (the copies are asynchronous), which
// leaves the SMs' registers and warps to the next group's sampling kernels.
// ------------------------------------------------------------------------------------
constexpr int kSweepTmaMaxWarps = 8;
constexpr int kSweepTmaMaxSlots = 16;

struct SweepTmaArgs {
  int32_t W;           // warps per block
  int32_t K;           // ring slots per warp
  int32_t slot_bytes;  // out16max * 16 (128-byte multiple when lines are written)
  int32_t row_bytes;   // 4 * pitch: bytes loaded per row
  int32_t warp_bytes;  // dynamic shared memory per warp
  int32_t hint;
};

__global__ void __launch_bounds__(32 * kSweepTmaMaxWarps) k_gather_sweep_tma(const __grid_constant__ TmaBatches a,
                                                                           SweepTmaArgs t) {
  extern __shared__ __align__(128) unsigned char s_dyn[];
  __shared__ __align__(8) unsigned long long s_bar[kSweepTmaMaxWarps][kSweepTmaMaxSlots];
  __shared__ uint32_t s_ep[kSweepMax];
  __shared__ uint32_t s_lo[kSweepMax], s_hi[kSweepMax];  // local-id range this launch writes
  __shared__ unsigned s_cnt[kSweepMax][2];
  __shared__ unsigned s_reads, s_host;
  __shared__ long long s_tot;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nb = a.n;
  const int K = t.K;
  if (threadIdx.x < 2 * kSweepMax) (&s_cnt[0][0])[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    s_reads = 0u;
    s_host = 0u;
  }
  sweep_init(a, s_ep, s_lo, s_hi, &s_tot);
  // per warp: ring [K][slot_bytes] | tag stage [nb][32] u64 | slot stage [32] i32 | row table
  // [nb][32] i32 | slot metadata [K][1 + nb] i32 (mask, destination rows)
  unsigned char* mine = s_dyn + (size_t)wib * t.warp_bytes;
  unsigned char* ring = mine;
  unsigned long long* stag = reinterpret_cast<unsigned long long*>(mine + (size_t)K * t.slot_bytes);
  int* sslot = reinterpret_cast<int*>(stag + nb * 32);
  int* rt = sslot + 32;
  int* meta = rt + nb * 32;
  for (int i = lane; i < K * t.slot_bytes / 16; i += 32) reinterpret_cast<int4*>(ring)[i] = make_int4(0, 0, 0, 0);
  if (lane == 0) {
    for (int k = 0; k < K; ++k) mbar_init(smem_addr(&s_bar[wib][k]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero tails visible to bulk stores
  __syncthreads();
  const uint64_t pol = t.hint ? policy_evict_first() : policy_evict_normal();
  // lane b holds batch b's output row address base, stride and width (bulk stores are per lane)
  float* xb = nullptr;
  int64_t ldb = 0;
  uint32_t ob = 0;
  if (lane < nb) {
    xb = a.b[lane].X;
    ldb = a.b[lane].ldx;
    ob = (uint32_t)a.b[lane].out16 * 16u;
  }
  unsigned long long* ticket = &a.b[0].sc->sweep_ticket;
  auto take = [&]() -> int64_t {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(ticket, 1ull);
    return 32 * (int64_t)__shfl_sync(0xffffffffu, tk, 0);
  };
  auto prefetch = [&](int64_t g) {
    if (g >= a.N) return;
    const int64_t v = g + lane;
    const bool in = v < a.N;
    const int64_t vv = in ? v : 0;
    for (int b = 0; b < nb; ++b) cp_async8(stag + b * 32 + lane, a.b[b].pos_of + vv, in ? 8 : 0);
    cp_async4(sslot + lane, &a.dir[vv].slot, in ? 4 : 0);
  };
  unsigned reads = 0, host_reads = 0, hits = 0, misses = 0;
  int64_t g = take();
  prefetch(g);
  cp_async_commit();
  unsigned rem = 0, mask = 0;  // present lanes of the current group not yet issued; lane's mask
  const char* src = nullptr;
  bool done = false;
  // the current group's probes -> masks, row table, sources, counters; then prefetch the next
  auto next_group = [&]() {
    cp_async_wait_all();
    __syncwarp();
    const int64_t v = g + lane;
    const int32_t sl = v < a.N ? sslot[lane] : -1;
    mask = 0;
    for (int b = 0; b < nb; ++b) {
      const unsigned long long tg = stag[b * 32 + lane];
      const uint32_t row = 0xFFFFFFFFu - (uint32_t)tg;
      if ((uint32_t)(tg >> 32) == s_ep[b] && row >= s_lo[b] && row < s_hi[b]) {
        mask |= 1u << b;
        rt[b * 32 + lane] = (int)row;
      }
    }
    __syncwarp();
    const int64_t g_next = take();
    prefetch(g_next);
    cp_async_commit();
    src = nullptr;
    if (mask) {
      if (sl < 0)
        src = reinterpret_cast<const char*>(a.hfeats + v * a.pitch);
      else if (a.G == 1)
        src = reinterpret_cast<const char*>(a.fcache + (int64_t)sl * a.pitch);
      else
        src = reinterpret_cast<const char*>(
            reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(a.fbases) + sl % a.G)) +
            (int64_t)(sl / a.G) * a.pitch);
    }
    const unsigned hitm = __ballot_sync(0xffffffffu, sl >= 0);
    for (int b = 0; b < nb; ++b) {
      const unsigned inb = __ballot_sync(0xffffffffu, (mask >> b) & 1u);
      if (lane == b) {
        hits += __popc(inb & hitm);
        misses += __popc(inb & ~hitm);
      }
    }
    rem = __ballot_sync(0xffffffffu, mask != 0);
    reads += __popc(rem);
    host_reads += __popc(rem & ~hitm);
    g = g_next;
  };
  int64_t issued = 0, consumed = 0;
  // load the next present node's row into slot issued % K (false: the sweep is over)
  auto issue = [&]() -> bool {
    while (!rem) {
      if (done || g >= a.N) {
        done = true;
        return false;
      }
      next_group();
    }
    const int j = __ffs(rem) - 1;
    rem &= rem - 1;
    const int s = (int)(issued % K);
    const unsigned mj = __shfl_sync(0xffffffffu, mask, j);
    const char* sj = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), j));
    int* ms = meta + s * (1 + nb);
    if (lane < nb && ((mj >> lane) & 1u)) ms[1 + lane] = rt[lane * 32 + j];
    if (lane == 0) {
      ms[0] = (int)mj;
      const uint32_t bar = smem_addr(&s_bar[wib][s]);
      mbar_expect_tx(bar, (uint32_t)t.row_bytes);
      bulk_g2s(smem_addr(ring + (size_t)s * t.slot_bytes), sj, (uint32_t)t.row_bytes, bar, pol);
    }
    __syncwarp();
    ++issued;
    return true;
  };
  for (int k = 0; k < K; ++k)
    if (!issue()) break;
  while (consumed < issued) {
    const int s = (int)(consumed % K);
    mbar_wait(smem_addr(&s_bar[wib][s]), (uint32_t)((consumed / K) & 1));
    const int* ms = meta + s * (1 + nb);
    const unsigned mk = (unsigned)ms[0];
    if ((mk >> lane) & 1u)
      bulk_s2g(xb + (int64_t)ms[1 + lane] * ldb, smem_addr(ring + (size_t)s * t.slot_bytes), ob, pol);
    bulk_commit();
    ++consumed;
    bulk_wait_read1();  // stores of nodes < consumed - 1 have read their slots
    __syncwarp();
    if (issued < consumed - 1 + K) issue();
  }
  bulk_wait_all();
  cp_async_wait_all();
  if (lane < nb) {
    if (hits) atomicAdd(&s_cnt[lane][0], hits);
    if (misses) atomicAdd(&s_cnt[lane][1], misses);
  }
  if (lane == 0 && reads) atomicAdd(&s_reads, reads);
  if (lane == 0 && host_reads) atomicAdd(&s_host, host_reads);
  __syncthreads();
  group_epilogue(a, s_cnt, s_reads, s_host, s_tot, true);
}

__global__ void __launch_bounds__(32 * kTmaMaxWarps) k_gather_tma(const __grid_constant__ TmaBatches a, TmaArgs t) {
  extern __shared__ __align__(128) unsigned char s_ring[];
  __shared__ __align__(8) unsigned long long s_bar[kTmaMaxWarps][kTmaMaxSlots];
  __shared__ char* s_dst[kTmaMaxWarps][kTmaMaxSlots];   // X address of the chunk's first row
  __shared__ int s_nr[kTmaMaxWarps][kTmaMaxSlots];      // rows in the chunk
  __shared__ int s_ldb[kTmaMaxWarps][kTmaMaxSlots];     // X row stride in bytes; 0 = contiguous
  __shared__ long long s_pre[kTmaMaxBatches + 1];       // row prefix over the launch's batches
  __shared__ unsigned s_cnt[kTmaMaxBatches][2];         // feature hits / misses per batch
  __shared__ unsigned s_reads;                          // feature rows this block read
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int K = t.K, R = t.R, nb = a.n;
  const uint32_t ring = smem_addr(s_ring) + (uint32_t)(wib * K * t.slot_bytes);
  if (threadIdx.x < 32) {  // warp 0: lane b reads batch b, shuffle prefix sum
    const long long nl = threadIdx.x < nb ? __ldcg(&a.b[threadIdx.x].sc->sizes[a.L]) : 0;
    long long x = nl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)threadIdx.x >= o) x += y;
    }
    if ((int)threadIdx.x < nb) s_pre[threadIdx.x] = x - nl;
    if ((int)threadIdx.x == nb - 1) s_pre[nb] = x;
  }
  if (threadIdx.x < 2 * kTmaMaxBatches) (&s_cnt[0][0])[threadIdx.x] = 0u;
  if (threadIdx.x == 0) s_reads = 0u;
  if (lane == 0) {
    for (int s = 0; s < K; ++s) mbar_init(smem_addr(&s_bar[wib][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntot = s_pre[nb];
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const uint64_t pol = t.hint ? policy_evict_first() : policy_evict_normal();
  // balanced contiguous row ranges per warp over the concatenated batches
  const int64_t lo = ntot * gw / nw, hi = ntot * (gw + 1) / nw;

  // Row lookups, 32 rows (a group) at a time: lane j holds row grp + j.  Two-stage prefetch: the
  // frontier id of group +2 and the cache slot of group +1 are in flight while group 0 issues.
  struct Look {
    int32_t b;  // batch of the lane's row (-1: past the range)
    int64_t r;  // row within the batch
    int32_t v;
  };
  auto look_v = [&](int64_t grp) -> Look {
    Look l{-1, 0, -1};
    const int64_t gr = grp + lane;
    if (gr < hi) {
      int b = 0;
      while (b + 1 < nb && gr >= s_pre[b + 1]) ++b;
      l.b = b;
      l.r = gr - s_pre[b];
      l.v = __ldg(a.b[b].F + l.r);
    }
    return l;
  };
  auto look_slot = [&](const Look& l) -> int32_t {
    return (l.v >= 0 && (int64_t)l.v < a.N) ? __ldg(&a.dir[l.v].slot) : -1;
  };
  int64_t g_cur = lo;
  Look l_cur = look_v(g_cur);
  int32_t s_cur = look_slot(l_cur);
  Look l_nxt = look_v(g_cur + 32);
  int32_t s_nxt = look_slot(l_nxt);
  Look l_nn = look_v(g_cur + 64);
  const char* src_cur = nullptr;
  int rows_cur = 0;
  auto start_group = [&]() {
    rows_cur = g_cur < hi ? (int)(hi - g_cur < 32 ? hi - g_cur : 32) : 0;
    src_cur = nullptr;
    if (lane < rows_cur && l_cur.v >= 0 && (int64_t)l_cur.v < a.N) {
      if (s_cur < 0)
        src_cur = reinterpret_cast<const char*>(a.hfeats + (int64_t)l_cur.v * a.pitch);
      else if (a.G == 1)
        src_cur = reinterpret_cast<const char*>(a.fcache + (int64_t)s_cur * a.pitch);
      else  // partitioned cache: local or peer (NVLink) rows
        src_cur = reinterpret_cast<const char*>(
            reinterpret_cast<const float*>(
                __ldg(reinterpret_cast<const unsigned long long*>(a.fbases) + s_cur % a.G)) +
            (int64_t)(s_cur / a.G) * a.pitch);
      atomicAdd(&s_cnt[l_cur.b][s_cur >= 0 ? 0 : 1], 1u);
      if (a.b[l_cur.b].node_visits) atomicAdd(a.b[l_cur.b].node_visits + l_cur.v, 1);
    }
  };
  start_group();
  int off = 0;
  int64_t issued = 0, consumed = 0;
  // issue the next chunk (<= R rows of one batch) of this warp's range into slot issued % K
  auto issue = [&]() -> bool {
    if (g_cur >= hi) return false;
    const int b0 = __shfl_sync(0xffffffffu, l_cur.b, off);
    const unsigned same = __ballot_sync(0xffffffffu, lane >= off && lane < rows_cur && l_cur.b == b0);
    const int cnt = min(R, __popc(same));  // rows of one batch are consecutive
    const int s = (int)(issued % K);
    const uint32_t bar = smem_addr(&s_bar[wib][s]);
    // rows whose id is invalid (a bad seed; the batch status reports DCI_ESEED) are not loaded
    const unsigned valid = __ballot_sync(0xffffffffu, src_cur != nullptr && lane >= off && lane < off + cnt);
    const int64_t r0 = __shfl_sync(0xffffffffu, l_cur.r, off);
    if (lane == 0) {
      const TmaBatch& tb = a.b[b0];
      s_dst[wib][s] = reinterpret_cast<char*>(tb.X + r0 * tb.ldx);
      s_nr[wib][s] = cnt;
      s_ldb[wib][s] = tb.ldx == a.pitch ? 0 : (int)(tb.ldx * 4);
      mbar_expect_tx(bar, (uint32_t)__popc(valid) * (uint32_t)t.row_bytes);
      atomicAdd(&s_reads, (unsigned)__popc(valid));
    }
    __syncwarp();
    if ((valid >> lane) & 1u)
      bulk_g2s(ring + (uint32_t)(s * t.slot_bytes + (lane - off) * t.row_bytes), src_cur, (uint32_t)t.row_bytes, bar,
               pol);
    ++issued;
    off += cnt;
    if (off >= rows_cur) {  // next group of this warp's range
      off = 0;
      g_cur += 32;
      l_cur = l_nxt;
      s_cur = s_nxt;
      l_nxt = l_nn;
      s_nxt = look_slot(l_nxt);
      l_nn = look_v(g_cur + 64);
      start_group();
    }
    return true;
  };
  for (int k = 0; k < K; ++k)
    if (!issue()) break;
  while (consumed < issued) {
    const int s = (int)(consumed % K);
    mbar_wait(smem_addr(&s_bar[wib][s]), (uint32_t)((consumed / K) & 1));
    char* dst = s_dst[wib][s];
    const int nr = s_nr[wib][s];
    const int ldb = s_ldb[wib][s];
    const uint32_t slot_sm = ring + (uint32_t)(s * t.slot_bytes);
    if (ldb == 0) {
      if (lane == 0) bulk_s2g(dst, slot_sm, (uint32_t)(nr * t.row_bytes), pol);
    } else if (lane < nr) {
      bulk_s2g(dst + (int64_t)lane * ldb, slot_sm + (uint32_t)(lane * t.row_bytes), (uint32_t)t.row_bytes, pol);
    }
    bulk_commit();
    ++consumed;
    bulk_wait_read1();  // stores of chunks < consumed - 1 have finished reading their slots
    __syncwarp();
    if (issued < consumed - 1 + K) issue();
  }
  bulk_wait_all();
  __syncthreads();
  unsigned host_rows = 0;  // row mode reads every miss row once per batch
  for (int i = 0; i < nb; ++i) host_rows += s_cnt[i][1];
  group_epilogue(a, s_cnt, s_reads, host_rows, s_pre[nb], false);
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

}  // namespace

static int phased_mode() {
  static const int mode = [] {
    const char* e = getenv("DCI_PHASED");
    return !e ? 0 : e[0] == '1' ? 1 : e[0] == '2' ? 2 : 0;  // default: overlapped (exp60)
  }();
  return mode;
}
bool group_phased() { return phased_mode() != 0; }
// DCI_PHASED=2: only the last hop waits for the previous group's gather; the earlier (light)
// hops overlap it
bool group_split() { return phased_mode() == 2; }

bool gather_tma_mode() {
  static const int mode = [] {
    const char* e = getenv("DCI_GATHER");
    return (e && (e[0] == 't' || e[0] == 'T')) ? 1 : 0;  // "tma": single-batch calls use the TMA gather too
  }();
  return mode == 1;
}

// TMA gather configuration for rows of this context: W warps per block (1 block per SM), a ring of
// K slots of R rows per warp in dynamic shared memory; false when an output cannot take bulk
// stores (X null or not 16-byte aligned rows) or a row does not fit (register-copy kernel then).
static bool tma_config(const dci_ctx* ctx, const dci_batch_out* out, TmaArgs* t, int* warps, size_t* smem) {
  if (!out->X) return false;
  if ((out->ldx % 4) != 0 || out->ldx < ctx->pitch || (reinterpret_cast<uintptr_t>(out->X) % 16) != 0) return false;
  static const int W = std::max(1, std::min(kTmaMaxWarps, env_int("DCI_TMA_WARPS", 8)));
  static const int smem_kb = std::max(16, std::min(220, env_int("DCI_TMA_SMEM_KB", 200)));
  static const int chunk_target = env_int("DCI_TMA_CHUNK", 8192);
  static const int hint = env_int("DCI_TMA_HINT", 1);
  const int row_bytes = ctx->pitch * 4;
  int R = std::max(1, std::min(32, (chunk_target + row_bytes / 2) / row_bytes));
  const int ring = smem_kb * 1024 / W;
  int K = ring / (R * row_bytes);
  while (K < 4 && R > 1) {
    R = (R + 1) / 2;
    K = ring / (R * row_bytes);
  }
  K = std::min(K, kTmaMaxSlots);
  if (K < 3) return false;
  t->hint = hint;
  t->K = K;
  t->R = R;
  t->row_bytes = row_bytes;
  t->slot_bytes = R * row_bytes;
  *warps = W;
  *smem = (size_t)W * K * t->slot_bytes;
  return true;
}

bool gather_uses_tma(const dci_ctx* ctx, const dci_batch_out* out) {
  TmaArgs t;
  int w;
  size_t sm;
  return gather_tma_mode() && tma_config(ctx, out, &t, &w, &sm);
}

bool gather_many_uses_tma(const dci_ctx* ctx, const dci_batch_out* outs, int32_t n) {
  TmaArgs t;
  int w;
  size_t sm;
  for (int i = 0; i < n; ++i)
    if (!tma_config(ctx, outs + i, &t, &w, &sm)) return false;
  return true;
}

static TmaBatches tma_batches(const dci_ctx* ctx, int32_t L) {
  TmaBatches tb;
  memset(&tb, 0, sizeof(tb));
  tb.L = L;
  tb.N = ctx->N;
  tb.dir = ctx->d_dir;
  tb.fcache = ctx->d_fcache;
  tb.fbases = ctx->d_fbases;
  tb.G = ctx->fpart_world;
  tb.pitch = ctx->pitch;
  tb.D = ctx->D;
  tb.hfeats = ctx->u_feats;
  return tb;
}

// 16-byte words the node sweep writes per X row: whole 128-byte lines (zeros past the pitch) when
// the row stride is a multiple of 32 floats and X is 128-byte aligned, else the pitch
static int32_t sweep_out16(const dci_ctx* ctx, const dci_batch_out* out) {
  if (out->ldx % 32 == 0 && reinterpret_cast<uintptr_t>(out->X) % 128 == 0) return ((ctx->pitch + 31) / 32) * 8;
  return ctx->pitch / 4;
}

static void tma_add(TmaBatches* tb, const dci_ctx* ctx, dci_workspace* ws, const dci_batch_out* out,
                    int32_t* node_visits) {
  TmaBatch& b = tb->b[tb->n++];
  b.F = out->frontier;
  b.pos_of = ws->pos_of;
  b.sc = ws->scal;
  b.X = out->X;
  b.ldx = out->ldx;
  b.out16 = sweep_out16(ctx, out);
  b.node_visits = node_visits;
  b.out_sizes = out->sizes;
  b.out_counters = out->counters;
  b.out_status = out->status;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize applies to the current device only: remember, per
// device, the largest value set so far (a process-wide static skipped the second GPU)
static dci_status ensure_dyn_smem(const void* kernel, std::atomic<int>* set_for, int device, size_t smem) {
  if (device < 0 || device >= kMaxDevices) return fail(DCI_EINVAL, "device index out of range");
  int cur = set_for[device].load();
  if ((int)smem <= cur) return DCI_OK;
  DCI_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  while (cur < (int)smem && !set_for[device].compare_exchange_weak(cur, (int)smem)) {
  }
  return DCI_OK;
}

static dci_status tma_launch(dci_ctx* ctx, const TmaBatches& tb, const dci_batch_out* out0, cudaStream_t s) {
  TmaArgs t;
  int warps = 0;
  size_t smem = 0;
  tma_config(ctx, out0, &t, &warps, &smem);
  static std::atomic<int> smem_set[kMaxDevices];
  dci_status st = ensure_dyn_smem(reinterpret_cast<const void*>(k_gather_tma), smem_set, ctx->device, smem);
  if (st != DCI_OK) return st;
  static const int bps = std::max(1, std::min(4, env_int("DCI_TMA_BPS", 1)));
  // DCI_TMA_SMS: SMs the gather grid covers (default all; a measurement knob)
  static const int sms = env_int("DCI_TMA_SMS", 0);
  const int nsm = (sms > 0 && sms < ctx->num_sms) ? sms : ctx->num_sms;
  k_gather_tma<<<nsm * bps, 32 * warps, smem, s>>>(tb, t);
  ++ctx->launches;
  return DCI_OK;
}

template <int VPL>
static dci_status sweep_launch_v(dci_ctx* ctx, const TmaBatches& tb, int32_t out16max, cudaStream_t s) {
  static std::atomic<int> smem_set[kMaxDevices];
  const size_t smem = (size_t)kSweepWarps * ((size_t)tb.n * 32 * 12 + 128);
  const void* kern = reinterpret_cast<const void*>(k_gather_sweep<VPL>);
  dci_status st = ensure_dyn_smem(kern, smem_set, ctx->device, smem);
  if (st != DCI_OK) return st;
  static const int hint = env_int("DCI_TMA_HINT", 1);
  // grid: the blocks (of 8 warps) that are resident at once (register-limited: 3 per SM at VPL 5),
  // so no block waits for a second wave; DCI_SWEEP_BPS caps it (a measurement knob)
  int occ = 0;
  DCI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kSweepWarps, smem));
  static const int cap = env_int("DCI_SWEEP_BPS", 0);
  const int bps = std::max(1, cap > 0 ? std::min(cap, occ) : occ);
  // DCI_SWEEP_SMS: SMs' worth of blocks (default all; leaves the rest to sampling running beside it)
  static const int sms = env_int("DCI_SWEEP_SMS", 0);
  const int nsm = (sms > 0 && sms < ctx->num_sms) ? sms : ctx->num_sms;
  k_gather_sweep<VPL><<<nsm * bps, 32 * kSweepWarps, smem, s>>>(tb, out16max, hint);
  ++ctx->launches;
  return DCI_OK;
}

static dci_status sweep_tma_launch(dci_ctx* ctx, const TmaBatches& tb, int32_t out16max, cudaStream_t s) {
  // 8 warps x 4 slots measured best on M2 (1.43 ms per group of 20 alone; 4 x 6: 1.68 ms)
  static const int W = std::max(1, std::min(kSweepTmaMaxWarps, env_int("DCI_SWEEP_WARPS", 8)));
  static const int Kenv = std::max(2, std::min(kSweepTmaMaxSlots, env_int("DCI_SWEEP_SLOTS", 4)));
  static const int hint = env_int("DCI_TMA_HINT", 1);
  SweepTmaArgs t;
  t.W = W;
  t.slot_bytes = out16max * 16;
  t.row_bytes = tb.pitch * 4;
  t.hint = hint;
  const int nb = tb.n;
  auto warp_bytes = [&](int K) {
    const int b = K * t.slot_bytes + nb * 32 * 8 + 128 + nb * 32 * 4 + K * (1 + nb) * 4;
    return (b + 127) / 128 * 128;
  };
  int K = Kenv;
  while (K > 2 && (size_t)W * warp_bytes(K) > 220 * 1024) --K;
  t.K = K;
  t.warp_bytes = warp_bytes(K);
  const size_t smem = (size_t)W * t.warp_bytes;
  if (smem > 220 * 1024) return fail(DCI_ERANGE, "sweep gather: feature rows too wide for the TMA ring");
  static std::atomic<int> smem_set[kMaxDevices];
  dci_status st = ensure_dyn_smem(reinterpret_cast<const void*>(k_gather_sweep_tma), smem_set, ctx->device, smem);
  if (st != DCI_OK) return st;
  static const int sms = env_int("DCI_SWEEP_SMS", 0);
  const int nsm = (sms > 0 && sms < ctx->num_sms) ? sms : ctx->num_sms;
  k_gather_sweep_tma<<<nsm, 32 * W, smem, s>>>(tb, t);
  ++ctx->launches;
  return DCI_OK;
}

static dci_status sweep_launch(dci_ctx* ctx, const TmaBatches& tb, bool alone, cudaStream_t s, int* used) {
  int32_t out16max = 0;
  for (int i = 0; i < tb.n; ++i) out16max = std::max(out16max, tb.b[i].out16);
  // DCI_SWEEP_KIND: auto (default: bulk copies when the gather runs alone, register copies when the
  // next group's sampling will run beside it) | ldg | tma
  static const int kind = [] {
    const char* e = getenv("DCI_SWEEP_KIND");
    return !e ? 2 : (e[0] == 't' || e[0] == 'T') ? 1 : (e[0] == 'l' || e[0] == 'L') ? 0 : 2;
  }();
  if (kind == 1 || (kind == 2 && alone)) {
    *used = 2;
    return sweep_tma_launch(ctx, tb, out16max, s);
  }
  *used = 1;
  // 16-byte words per lane per pass over a row (rows longer than 32 * VPL words take several passes)
  if (out16max <= 32) return sweep_launch_v<1>(ctx, tb, out16max, s);
  if (out16max <= 64) return sweep_launch_v<2>(ctx, tb, out16max, s);
  if (out16max <= 96) return sweep_launch_v<3>(ctx, tb, out16max, s);
  return sweep_launch_v<5>(ctx, tb, out16max, s);
}

bool gather_sweep_enabled() {
  static const int sweep = env_int("DCI_SWEEP", 1);
  return sweep != 0;
}

bool gather_split_enabled() {
  static const int split = env_int("DCI_SPLIT_GATHER", 0);
  return split != 0;
}

dci_status launch_gather_many(dci_ctx* ctx, dci_workspace* const* ws, const dci_batch_out* outs, int32_t n,
                              int32_t L, dci_batch_result* stage, bool sweep, bool alone, int32_t phase,
                              cudaStream_t s, int* kind) {
  TmaBatches tb = tma_batches(ctx, L);
  tb.stage = stage;
  tb.phase = sweep ? phase : 0;
  if (phase != 0 && !(sweep && n >= 2 && n <= kSweepMax)) return fail(DCI_EINVAL, "split gather needs a node sweep");
  for (int i = 0; i < n; ++i) tma_add(&tb, ctx, ws[i], outs + i, nullptr);
  if (sweep && n >= 2 && n <= kSweepMax) return sweep_launch(ctx, tb, alone, s, kind);
  *kind = 0;
  return tma_launch(ctx, tb, outs, s);
}

int gather_blocks_per_sm(const dci_ctx* ctx) {
  static const int forced = [] {
    const char* e = getenv("DCI_GATHER_BPS");
    return e ? atoi(e) : 0;
  }();
  if (forced > 0) return forced;
  // measured on M2: 1 batch in flight -> 4, 2-3 -> 2, >= 4 -> 1
  const int w = ctx->live_ws->load();
  return w <= 1 ? 4 : (w <= 3 ? 2 : 1);
}

static FusedArgs fused_args(dci_ctx* ctx, dci_workspace* ws, int32_t L, const dci_batch_out* out,
                            const HopParams& last, int32_t* node_visits) {
  FusedArgs a;
  a.dir = ctx->d_dir;
  a.pos_of = ws->pos_of;
  a.hmask = ws->hmask;
  a.sc = ws->scal;
  a.N = ctx->N;
  a.L = L;
  a.F = out->frontier;
  a.last_cand = last.cand;
  a.last_kcnt = last.kcnt;
  a.last_bptr = out->bptr[L - 1];
  a.last_bsrc = out->bsrc[L - 1];
  a.last_f = last.f;
  a.last_tiles = ws->tile_state + ws->tile_off[L - 1];
  a.last_ntiles = ws->tile_off[L] - ws->tile_off[L - 1];
  a.fcache = ctx->d_fcache;
  a.fbases = ctx->d_fbases;
  a.G = ctx->fpart_world;
  a.hfeats = ctx->u_feats;
  a.pitch = ctx->pitch;
  a.D = ctx->D;
  a.X = out->X;
  a.ldx = out->ldx;
  a.node_visits = node_visits;
  a.out_sizes = out->sizes;
  a.out_counters = out->counters;
  a.out_status = out->status;
  return a;
}

bool launch_gather_fused(dci_ctx* ctx, dci_workspace* ws, int32_t L, const dci_batch_out* out,
                         const HopParams& last, int32_t* node_visits, cudaStream_t s) {
  const FusedArgs a = fused_args(ctx, ws, L, out, last, node_visits);
  if (gather_uses_tma(ctx, out)) {
    TmaBatches tb = tma_batches(ctx, L);
    tma_add(&tb, ctx, ws, out, node_visits);
    tma_launch(ctx, tb, out, s);  // (a failure surfaces at the next CUDA call on the stream)
    return false;  // relabel of the last hop not fused: launch_hop_epilogue
  }
  const int bps = gather_blocks_per_sm(ctx);
  auto go = [&](auto kern) { kern<<<persistent_grid(ctx, kern, 256, bps), 256, 0, s>>>(a); };
  const bool vec = out->X && (out->ldx % 4 == 0) && out->ldx >= ctx->pitch &&
                   (reinterpret_cast<uintptr_t>(out->X) % 16 == 0);
  if (!out->X)
    go(k_gather<0, 1>);
  else if (!vec)
    go(k_gather<1, 1>);
  else if (ctx->pitch <= 32 * 4 * 2)
    go(k_gather<2, 2>);
  else
    go(k_gather<2, 5>);
  ++ctx->launches;
  return true;
}

}  // namespace dci
