// S5-S6 of the hot path: per-hop neighbour sampling with the adjacency
// cache and per-hop dedup/relabel through an epoch-tagged
// node->position table plus a single-pass decoupled look-back scan (first-occurrence order,
// reading C6).  All launches use persistent, SM-count-sized grids that read the frontier size
// from device memory, so a batch never synchronises the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dci_internal.cuh"
#include "philox.cuh"

namespace dci {

namespace {

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Host-mapped (UVA) neighbour read: a plain global load that the GPU turns into a PCIe
// read request.  L1-allocating: random host reads through L1::no_allocate loads
// run at up to ~1.75x lower rates on this B200 (tools/probe/hostreq_probe.cu: 64 B requests 11.2
// vs 19.4 GB/s, 128 B 23 vs 42 GB/s); the host CSC is read-only while kernels run.
__device__ __forceinline__ int32_t ld_host_i32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ int32_t ld_keep_i32(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ int4 ld_keep_v4(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// One batch of a (multi-batch) hop launch.  A dci_sample_gather_many group runs every hop of all
// its batches as ONE launch over the concatenation of their frontiers; a single call is n = 1.
struct HopBatch {
  int32_t* F;                      // frontier (global ids); hop 0 reads the seeds from the header
  int32_t* cand;                   // [n_h * f]
  int32_t* kcnt;                   // [n_h]
  const int32_t* prev_cand;        // hop h-1 (relabelled by this hop's kernel)
  const int32_t* prev_kcnt;
  const int32_t* prev_bptr;
  int32_t* prev_bsrc;
  int32_t* bptr;                   // this hop's block row pointers (written by the scan)
  unsigned long long* pos_of;      // the workspace's node -> position tag table (dense or hashed)
  uint32_t* nmask;                 // [n_h] new-candidate slot masks of a node-sweep hop
  uint32_t hmask;                  // 0: dense table; else hashed capacity - 1 (pt_insert / pt_find)
  BatchScalars* sc;
  unsigned long long* tiles;       // this hop's scan tile state
  unsigned long long* prev_tiles;  // previous hop's scan tile state (cleared here)
  int64_t prev_ntiles;
};

struct HopLaunch {
  const DirEntry* dir;
  const int32_t* acache;
  const int32_t* uidx;  // device alias of the pinned host CSC (current order)
  int64_t N;
  int32_t hop, f, prev_f, n;
  uint32_t pass;
  int32_t elem_policy;  // L2 policy of adjacency-cache element loads: 0 evict-last, 1 normal (default), 2 evict-first
  int32_t dir_policy;   // L2 policy of directory-entry loads (same codes; default normal: evict-last measured
                        // 1 % slower on M2 and 3.6 % on M4s -- lines pinned in L2 crowd out the gather's)
  int32_t* edge_counts; // presample only (nullable, n = 1)
  int32_t precheck;     // read the tag before the atomicMax (DCI_PRECHECK=1; measured slower on M2)
  int32_t sweep;        // node-sweep sampling allowed (multi-batch hops covering >= sweep_min nodes)
  int64_t sweep_min;    // frontier total from which a hop sweeps (N, or N / 20 with host adjacency)
  int32_t nmask_on;     // a sweeping hop's new-candidate masks come from k_newmask_sweep (DCI_NMASK_SWEEP)
  HopBatch b[DCI_MAX_GROUP];
};

__device__ __forceinline__ uint64_t policy_by(int k) {
  uint64_t p;
  if (k == 0)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else if (k == 1)
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Per-launch batch table in shared memory: frontier prefix over the batches, epoch tags, seeds.
struct HopShared {
  long long pre[DCI_MAX_GROUP + 1];   // prefix of n_h(b)
  long long ppre[DCI_MAX_GROUP + 1];  // prefix of n_{h-1}(b) * f_{h-1} (relabel items)
  long long tpre[DCI_MAX_GROUP + 1];  // prefix of prev_ntiles(b)
  unsigned long long ehi[DCI_MAX_GROUP];
  unsigned long long seed[DCI_MAX_GROUP];
  const int32_t* Fin[DCI_MAX_GROUP];
  unsigned cnt[DCI_MAX_GROUP][2];     // adjacency hits / misses of this block, per batch
  unsigned host_sectors;              // distinct 32-byte host sectors its adjacency misses read
  unsigned host_runs;                 // (dst, hop) runs with at least one adjacency miss
  unsigned long long tbase[DCI_MAX_GROUP];  // epoch << 32 | ~n_h: a candidate's tag = tbase - (d f + slot)
  uint32_t nh[DCI_MAX_GROUP];         // n_h of each batch
  unsigned sweep_next;                // node sweep: the block's next node group (shared ticket)
  int all_ok;                         // no batch has a seed error (status set by hop 0)
};

// warp-inclusive prefix sum of 64-bit values (warp 0, all lanes)
__device__ __forceinline__ long long warp_incl_scan(long long x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// The launch's batch table in shared memory, built by warp 0 with lane b reading batch b's
// scalars (all batches' loads in flight at once; a serial loop in one thread cost ~2n dependent
// L2 round trips before every block could start) and shuffle prefix sums.
__device__ __forceinline__ void hop_shared_init(const HopLaunch& a, HopShared& S) {
  if (threadIdx.x < 32) {
    const int b = threadIdx.x;
    const bool in = b < a.n;
    long long nh = 0, pw = 0, tw = 0;
    int ok = 1;
    if (in) {
      const BatchScalars* sc = a.b[b].sc;
      const long long B = sc->hdr.B;
      nh = a.hop == 0 ? B : sc->sizes[a.hop];
      const long long np = a.hop == 0 ? 0 : (a.hop == 1 ? B : sc->sizes[a.hop - 1]);
      pw = np * a.prev_f;
      tw = a.b[b].prev_ntiles;
      S.ehi[b] = (unsigned long long)sc->hdr.epoch << 32;
      S.seed[b] = sc->hdr.seed;
      S.Fin[b] = a.hop == 0 ? sc->hdr.seeds : a.b[b].F;
      ok = __ldcg(&sc->status) == 0;
    }
    const long long ia = warp_incl_scan(nh, b), ip = warp_incl_scan(pw, b), it = warp_incl_scan(tw, b);
    if (in) {
      S.pre[b] = ia - nh;
      S.ppre[b] = ip - pw;
      S.tpre[b] = it - tw;
      S.nh[b] = (uint32_t)nh;
      S.tbase[b] = S.ehi[b] | (0xFFFFFFFFu - (uint32_t)nh);
    }
    if (b == a.n - 1) {
      S.pre[a.n] = ia;
      S.ppre[a.n] = ip;
      S.tpre[a.n] = it;
    }
    const int all_ok = __all_sync(0xffffffffu, ok);
    if (b == 0) {
      S.all_ok = all_ok;
      S.host_sectors = 0u;
      S.host_runs = 0u;
      S.sweep_next = 0u;
    }
  }
  if (threadIdx.x < 2 * DCI_MAX_GROUP) (&S.cnt[0][0])[threadIdx.x] = 0u;
  __syncthreads();
}

// Host-link traffic of the adjacency miss path (bench roofline): a sampled element
// that misses is a 4-byte zero-copy read of pinned host memory, and the GPU fetches system memory
// in 32-byte sectors, so misses of one (dst, hop) that fall in the same sector are served together.
// Ranks are sorted within a G-lane group, so the misses are its last lanes in address order: a miss
// lane opens a new sector unless the lane before it missed in the same sector, and the group's
// first miss lane opens its run (one contiguous stretch of the node's host run: the request view
// counts runs).  Adds the warp's counts to the caller's (warp-uniform) register totals, which are
// flushed once per thread block-wide at the end (no shared atomics in the sampling loops).
template <int G>
__device__ __forceinline__ void host_miss_counts(bool miss, int64_t elem, int gl, unsigned& sectors,
                                                 unsigned& runs) {
  const long long line = elem >> 3;  // 8 int32 per 32-byte sector
  const long long pl = __shfl_up_sync(0xffffffffu, line, 1, G);
  const bool pmiss = __shfl_up_sync(0xffffffffu, (int)miss, 1, G) != 0;
  const bool first = miss && (gl == 0 || !pmiss);
  sectors += __popc(__ballot_sync(0xffffffffu, miss && (first || pl != line)));
  runs += __popc(__ballot_sync(0xffffffffu, first));
}

__device__ __forceinline__ void host_miss_flush(HopShared& S, unsigned sectors, unsigned runs) {
  if ((threadIdx.x & 31) == 0) {
    if (sectors) atomicAdd(&S.host_sectors, sectors);
    if (runs) atomicAdd(&S.host_runs, runs);
  }
}

// batch of item q in a prefix table (n <= DCI_MAX_GROUP = 32: a linear scan over shared memory;
// the hot loops advance a running batch index instead, since their items only grow)
__device__ __forceinline__ int batch_of(const long long* pre, int n, long long q) {
  int b = 0;
  while (b + 1 < n && q >= pre[b + 1]) ++b;
  return b;
}

__device__ __forceinline__ void hop_shared_flush(const HopLaunch& a, HopShared& S) {
  __syncthreads();
  if (threadIdx.x < a.n) {
    BatchScalars* sc = a.b[threadIdx.x].sc;
    if (S.cnt[threadIdx.x][0]) atomicAdd(&sc->counters[0], (unsigned long long)S.cnt[threadIdx.x][0]);
    if (S.cnt[threadIdx.x][1]) atomicAdd(&sc->counters[1], (unsigned long long)S.cnt[threadIdx.x][1]);
  }
  if (threadIdx.x == 0 && S.host_sectors) atomicAdd(&a.b[0].sc->acc_host_sectors, (unsigned long long)S.host_sectors);
  if (threadIdx.x == 0 && S.host_runs) atomicAdd(&a.b[0].sc->acc_host_runs, (unsigned long long)S.host_runs);
}

// Fused extra work of every hop kernel: hop 0 writes the seeds into F and the position table
// (position = seed index); hop h >= 1 relabels hop h-1's candidates into its block CSR
// (tag -> final local id) and clears hop h-1's scan tile state and ticket.  With hop = L (no
// sampling: k_hop_epilogue) it relabels the last hop.
__device__ __forceinline__ void hop_prologue(const HopLaunch& a, const HopShared& S, int64_t tid, int64_t nthreads) {
  const int h = a.hop, n = a.n;
  if (h == 0) {
    const long long tot = S.pre[n];
    for (long long q = tid; q < tot; q += nthreads) {
      const int b = batch_of(S.pre, n, q);
      const int64_t d = q - S.pre[b];
      const HopBatch& hb = a.b[b];
      const int32_t s = S.Fin[b][d];
      hb.F[d] = s;
      if (s < 0 || (int64_t)s >= a.N)
        atomicCAS(&hb.sc->status, 0, (int32_t)DCI_ESEED);
      else
        atomicMax(pt_insert(hb.pos_of, hb.hmask, s, (uint32_t)(S.ehi[b] >> 32)), S.ehi[b] | (0xFFFFFFFFu - (uint32_t)d));
    }
    return;
  }
  // relabel of hop h-1 (its scan has completed: kernel boundary); final ids are tagged
  const int pf = a.prev_f;
  const long long ptot = S.ppre[n];
  // 4 independent items per thread and round, so their dependent loads (candidate -> tag) overlap
  constexpr int U = 4;
  int bh = 0;  // items only grow along a thread's loop: the batch index only advances
  for (long long q0 = tid; q0 < ptot; q0 += U * nthreads) {
    int bu[U];
    int64_t du[U];
    int su[U];
    int32_t ku[U], cu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long q = q0 + u * nthreads;
      ku[u] = 0;
      if (q < ptot) {
        while (bh + 1 < n && q >= S.ppre[bh + 1]) ++bh;
        bu[u] = bh;
        const HopBatch& hb = a.b[bu[u]];
        const uint32_t ql = (uint32_t)(q - S.ppre[bu[u]]);  // < 2^31 per batch (|F_h| * (f + 1) < 2^31)
        du[u] = ql / (uint32_t)pf;
        su[u] = (int)(ql - (uint32_t)du[u] * (uint32_t)pf);
        ku[u] = hb.prev_kcnt[du[u]];
        cu[u] = hb.prev_cand[ql];
      }
    }
    unsigned long long tu[U];
    int32_t pu[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (q0 + u * nthreads < ptot && su[u] < ku[u]) {
        const HopBatch& hb = a.b[bu[u]];
        tu[u] = pt_tag(hb.pos_of, hb.hmask, cu[u], (uint32_t)(S.ehi[bu[u]] >> 32));
        pu[u] = hb.prev_bptr[du[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * nthreads < ptot && su[u] < ku[u])
        a.b[bu[u]].prev_bsrc[pu[u] + su[u]] = (int32_t)(0xFFFFFFFFu - (uint32_t)tu[u]);
  }
  const long long ttot = S.tpre[n];
  for (long long t = tid; t < ttot; t += nthreads) {
    const int b = batch_of(S.tpre, n, t);
    a.b[b].prev_tiles[t - S.tpre[b]] = 0ull;
  }
  if (tid < n) a.b[tid].sc->tickets[h - 1] = 0;
}

// Rank selection of one dst group (O-4): lane gl of the group returns the gl-th smallest chosen
// rank (its output position is gl); deg <= f: ranks 0..deg-1 in order.  Must be called by the
// whole warp (shuffles); groups with floyd == false just return gl.
template <int G>
__device__ __forceinline__ int32_t select_rank(int gl, int lane, unsigned gmask, int f, int32_t deg, bool floyd,
                                               unsigned long long seed, uint32_t pass, uint32_t h, uint32_t v) {
  int32_t rank = gl;
  if (__any_sync(0xffffffffu, floyd)) {
    int32_t chosen = 0, j = 0;
    const bool draw = floyd && gl < f;
    if (draw) {
      j = deg - f + gl;
      const uint64_t u = philox_u64(seed, pass, h, v, (uint32_t)gl);
      chosen = (int32_t)__umul64hi(u, (uint64_t)(j + 1));
    }
    // Floyd: slot i keeps t_i unless an earlier slot already chose it, then takes j_i.  While
    // no earlier slot collided, chosen[k] = t_k, so slot i collides iff t_i repeats an earlier
    // t: when all of a group's draws are distinct (most groups when deg >> f) nothing changes,
    // and one __match_any_sync over (group, t) detects that.  Otherwise resolve in slot order.
    const unsigned long long key = draw ? (((unsigned long long)(lane / G) << 32) | (uint32_t)chosen)
                                        : (0xFFFFFFFF00000000ull | (unsigned)lane);
    const bool dup = __popc(__match_any_sync(0xffffffffu, key)) > 1;
    if (__any_sync(0xffffffffu, dup)) {
      for (int i = 1; i < f; ++i) {
        const int32_t ti = __shfl_sync(0xffffffffu, chosen, i, G);
        const unsigned coll = __ballot_sync(0xffffffffu, gl < i && chosen == ti) & gmask;
        if (gl == i && coll) chosen = j;
      }
    }
    // ascending order within the group: bitonic network over the G lanes (pads sort last)
    int32_t val = draw ? chosen : (floyd ? 0x7FFFFFFF : gl);
#pragma unroll
    for (int kk = 2; kk <= G; kk <<= 1) {
#pragma unroll
      for (int jj = kk >> 1; jj > 0; jj >>= 1) {
        const int32_t o = __shfl_xor_sync(0xffffffffu, val, jj, G);
        const bool keep_min = ((gl & jj) == 0) == ((gl & kk) == 0);
        val = keep_min ? min(val, o) : max(val, o);
      }
    }
    if (floyd) rank = val;
  }
  return rank;
}

// Whether a hop samples by node sweep (decided on the device: the frontier sizes are device data).
// k_sample_hop, k_newmask_sweep and k_scan_hop take the same decision from the same inputs (for
// h >= 1 the batches' status words and frontier sizes no longer change within the hop).
__device__ __forceinline__ bool hop_sweeps(const HopLaunch& a, long long total, int all_ok) {
  return a.f >= 3 && a.f <= 32 && a.hop >= 1 && all_ok && a.sweep && a.n >= 2 && total >= a.sweep_min &&
         a.edge_counts == nullptr;
}

// ------------------------------------------------------------------------------------
// Node-sweep sampling of a multi-batch hop (2+ batches whose frontiers together hold >= N nodes):
// the draws of (node v, hop h) do not depend on the batch (C4), so each node is sampled ONCE
// (one directory read, one selection, one element read per slot) and the result is written into
// every batch whose F_h holds v, at that batch's position d_b (v's tag in the batch's table:
// current epoch and id < |F_h(b)|).  The insertions into each batch's table and its candidate
// array are exactly those of the frontier-order loop, so the scan that follows sees the same
// state.  Cuts the hop's random element reads from sum_b |F_h(b)| * f to |union| * f.
// ------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void sample_sweep(const HopLaunch& a, HopShared& S, int64_t warp_id, int64_t nwarps,
                                             uint64_t keep, uint64_t epol) {
  constexpr int CH = DCI_MAX_GROUP / G;  // batches probed per lane (G >= 4)
  const int h = a.hop, f = a.f, n = a.n;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const int GPW = 32 / G;
  // the next node group's table probes and directory entry (contiguous: ids are consecutive)
  // are loaded while the current group samples and writes.  Schedule: each block owns a static
  // contiguous range of node groups and its warps take them one at a time from a shared-memory
  // ticket (taken one ahead).  A static stride over all warps left a long tail (a warp's work is a
  // sum of ~25 nodes present in 0..n batches: 12 % of the stall samples sat at the block barrier,
  // ncu r2i), and one global ticket counter measured slower still (226-617 us: contention on one
  // address, and too few chunks for 4.7 K warps); block ranges are sums of ~400 groups each.
  const int64_t ngroups = (a.N + GPW - 1) / GPW;
  const int64_t per_block = (ngroups + gridDim.x - 1) / gridDim.x;
  const int64_t g0 = (int64_t)blockIdx.x * per_block;
  const int64_t g1 = g0 + per_block < ngroups ? g0 + per_block : ngroups;
  auto take = [&]() -> int64_t {  // -> first node id of the warp's next group, or N when done
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(&S.sweep_next, 1u);
    const int64_t g = g0 + (int64_t)__shfl_sync(0xffffffffu, t, 0);
    return g < g1 ? g * GPW : a.N;
  };
  (void)warp_id;
  (void)nwarps;
  auto probe = [&](int64_t vb, unsigned long long* t, int4& x0, int4& x1) {
    const int64_t vv = vb + lane / G;
    x0 = make_int4(0, 0, 0, 0);
    x1 = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int bb = c * G + gl;
      t[c] = (vv < a.N && bb < n) ? __ldcg(a.b[bb].pos_of + vv) : 0ull;
    }
    if (vv < a.N) {
      const int4* ep = reinterpret_cast<const int4*>(a.dir + vv);
      x0 = ld_keep_v4(ep, keep);
      x1 = ld_keep_v4(ep + 1, keep);
    }
  };
  unsigned long long tc[CH], tn[CH];
  unsigned acc_h[CH], acc_m[CH];
  unsigned hsec = 0, hrun = 0;  // host sectors / runs of the adjacency misses (warp-uniform)
#pragma unroll
  for (int c = 0; c < CH; ++c) acc_h[c] = acc_m[c] = 0u;
  int4 e0, e1, e0n, e1n;
  int64_t vbase = take();
  probe(vbase, tc, e0, e1);
  while (vbase < a.N) {
    const int64_t vn = take();
    probe(vn, tn, e0n, e1n);
    const int64_t vv = vbase + lane / G;
    const bool in = vv < a.N;
    const int32_t v = (int32_t)vv;
    // which batches hold v in F_h, and where: lane gl probed batches gl, gl + G, ... (G >= 4, so
    // at most 4 per lane) and keeps the local ids for the write loop below
    unsigned pm = 0;
    uint32_t dd[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int bb = c * G + gl;
      bool pres = false;
      dd[c] = 0xFFFFFFFFu - (uint32_t)tc[c];
      if (c * G < n) {
        if (in && bb < n)
          pres = (tc[c] >> 32) == (S.ehi[bb] >> 32) && dd[c] < S.nh[bb];
        const unsigned bal = (__ballot_sync(0xffffffffu, pres) & gmask) >> gbase;
        pm |= bal << (c * G);
      }
    }
    if (!pm) {  // no batch holds v: nothing to sample (its directory entry is simply unused)
      e0 = make_int4(0, 0, 0, 0);
      e1 = make_int4(0, 0, 0, 0);
    }
    const int64_t host_off = ((int64_t)(uint32_t)e0.y << 32) | (uint32_t)e0.x;
    const int64_t cache_off = ((int64_t)(uint32_t)e0.w << 32) | (uint32_t)e0.z;
    const int32_t deg = e1.x;
    const int32_t cached_len = e1.y;
    const int k = deg < f ? deg : f;
    const bool floyd = deg > f;
    const int32_t rank = select_rank<G>(gl, lane, gmask, f, deg, floyd, S.seed[0], a.pass, (uint32_t)h, (uint32_t)v);
    const bool valid = pm && gl < k;
    int32_t x = -1;
    bool hit = false;
    if (valid) {
      hit = rank < cached_len;
      x = hit ? ld_keep_i32(a.acache + cache_off + rank, epol) : ld_host_i32(a.uidx + host_off + rank);
    }
    {  // read once for every batch holding v: its host sectors count once
      host_miss_counts<G>(valid && !hit, host_off + rank, gl, hsec, hrun);
    }
    // v's hits / misses, counted once per node and added to every batch holding v: lane gl keeps
    // the running counts of batches gl, gl + G, ... in registers (no per-sample shared atomics)
    {
      const unsigned vm = __ballot_sync(0xffffffffu, valid) & gmask;
      const unsigned hm = __ballot_sync(0xffffffffu, valid && hit) & gmask;
      const unsigned nh = __popc(hm), nm = __popc(vm) - nh;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if ((pm >> (c * G + gl)) & 1u) {
          acc_h[c] += nh;
          acc_m[c] += nm;
        }
    }
    // write the sample into every batch holding v (local id shuffled from the probing lane); the
    // loop runs over the batches holding ANY of the warp's nodes, not over all n
    for (unsigned um = __reduce_or_sync(0xffffffffu, pm); um; um &= um - 1) {
      const int bb = __ffs(um) - 1;
      const int cb = bb / G;
      uint32_t dsel = dd[0];
#pragma unroll
      for (int c = 1; c < CH; ++c)
        if (cb == c) dsel = dd[c];
      const uint32_t d = __shfl_sync(0xffffffffu, dsel, gbase + (bb & (G - 1)));
      if (!((pm >> bb) & 1u)) continue;
      const HopBatch& hb = a.b[bb];
      if (gl < f) hb.cand[(int64_t)d * f + gl] = x;
      if (gl == 0) hb.kcnt[d] = k;
      if (valid) {  // tag(n_h + d f + gl) = epoch << 32 | ~(n_h + d f + gl); no borrow: < 2^31
        const unsigned long long tag = S.tbase[bb] - (unsigned long long)(d * (uint32_t)f + (uint32_t)gl);
        if (!a.precheck || __ldcg(hb.pos_of + x) < tag) atomicMax(hb.pos_of + x, tag);
      }
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) tc[c] = tn[c];
    e0 = e0n;
    e1 = e1n;
    vbase = vn;
  }
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int bb = c * G + gl;
    if (bb < n) {
      if (acc_h[c]) atomicAdd(&S.cnt[bb][0], acc_h[c]);
      if (acc_m[c]) atomicAdd(&S.cnt[bb][1], acc_m[c]);
    }
  }
  host_miss_flush(S, hsec, hrun);
}

// ------------------------------------------------------------------------------------
// k_sample_hop<G>: one group of G lanes (G = next pow2 >= f) per dst node of F_h (of any batch of
// the launch: dst index q over the concatenated frontiers -> batch b, local dst d).
//  1. one broadcast 32 B directory load (host_off, cache_off, deg, cached_len)
//  2. k = min(deg, f); deg <= f -> ranks 0..deg-1; else Floyd's selection with lane i
//     drawing t_i = floor(u_i * (j_i + 1) / 2^64), j_i = deg - k + i, u_i =
//     Philox(v, i, hop, pass; seed) and a (f-1)-step shuffle/ballot collision resolution
//     (O-3, O-4)
//  3. ranks sorted in registers (position = #smaller ranks in the group)
//  4. element read: HBM cache iff rank < cached_len, else UVA host read
//  5. cand[d*f + pos] = neighbour, pads -1; kcnt[d] = k
//  6. insert into the batch's node->position table: atomicMax(tag(n_h + d*f + pos)), tag(p) =
//     epoch << 32 | ~p, so the table keeps each node's first (dst-major, rank-ascending)
//     occurrence and entries of earlier batches read as absent
//  7. presample: edge_counts[host_off + rank] += 1 (C8)
// Fused extra work: hop_prologue.
// ------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256) k_sample_hop(const __grid_constant__ HopLaunch a) {
  __shared__ HopShared S;
  hop_shared_init(a, S);
  const int h = a.hop;
  const int f = a.f;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  hop_prologue(a, S, tid, nthreads);
  const long long total = S.pre[a.n];

  const int GPW = 32 / G;
  const int64_t warp_id = tid >> 5;
  const int64_t nwarps = nthreads >> 5;
  const uint64_t keep = policy_by(a.dir_policy);
  const uint64_t epol = policy_by(a.elem_policy);
  // (not at hop 0: the seeds' table tags are written by this kernel's own prologue, so they are
  // not final until the kernel ends; from hop 1 on, F_h's tags were finalised by the last scan)
  // (and not when a batch has a seed error: a bad or repeated seed has no table slot of its own,
  // so the sweep would leave its candidate slots unwritten; frontier order fills them)
  if (G >= 4 && hop_sweeps(a, total, S.all_ok)) {
    if (a.nmask_on)  // the new-mask pass (next kernel) ORs into zeroed masks: one coalesced pass here
      for (long long q = tid, b = 0; q < total; q += nthreads) {
        while (b + 1 < a.n && q >= S.pre[b + 1]) ++b;  // q only grows: the batch only advances
        a.b[b].nmask[q - S.pre[b]] = 0u;
      }
    sample_sweep<(G >= 4 ? G : 4)>(a, S, warp_id, nwarps, keep, epol);
    hop_shared_flush(a, S);
    return;
  }
  // Software pipeline over this warp's dst groups: the frontier id of iteration i+2 and the
  // directory entry of iteration i+1 are in flight while iteration i draws, reads its elements and
  // inserts them, so the dependent F -> dir -> element chain costs one latency per iteration.
  const int64_t stride = nwarps * GPW;
  auto fetch_v = [&](int64_t db, int bb) -> int32_t {  // bb: a batch index <= that of db
    const int64_t qq = db + lane / G;
    if (qq >= total) return -1;
    while (bb + 1 < a.n && qq >= S.pre[bb + 1]) ++bb;
    return S.Fin[bb][qq - S.pre[bb]];
  };
  auto fetch_dir = [&](int32_t vv, int4& x0, int4& x1) {
    x0 = make_int4(0, 0, 0, 0);
    x1 = make_int4(0, 0, 0, 0);
    if (vv >= 0 && (int64_t)vv < a.N) {
      const int4* ep = reinterpret_cast<const int4*>(a.dir + vv);
      x0 = ld_keep_v4(ep, keep);
      x1 = ld_keep_v4(ep + 1, keep);
    }
  };
  int64_t dbase = warp_id * GPW;
  int b = 0;
  unsigned hsec = 0, hrun = 0;  // host sectors / runs of the adjacency misses (warp-uniform)
  int32_t v = fetch_v(dbase, 0);
  int4 e0, e1;
  fetch_dir(v, e0, e1);
  int32_t v_next = fetch_v(dbase + stride, 0);
  for (; dbase < total; dbase += stride) {
    int4 e0_next, e1_next;
    fetch_dir(v_next, e0_next, e1_next);
    const int32_t v_next2 = fetch_v(dbase + 2 * stride, b);
    const int64_t q = dbase + lane / G;
    const bool active = q < total;
    if (active)  // q only grows along a warp's loop: advance the batch index
      while (b + 1 < a.n && q >= S.pre[b + 1]) ++b;
    const HopBatch& hb = a.b[b];
    const int64_t d = q - S.pre[b];
    const int64_t n_h = S.pre[b + 1] - S.pre[b];
    const int64_t host_off = ((int64_t)(uint32_t)e0.y << 32) | (uint32_t)e0.x;
    const int64_t cache_off = ((int64_t)(uint32_t)e0.w << 32) | (uint32_t)e0.z;
    const int32_t deg = e1.x;
    const int32_t cached_len = e1.y;
    const int k = deg < f ? deg : f;
    const bool floyd = deg > f;

    const int32_t rank = select_rank<G>(gl, lane, gmask, f, deg, floyd, S.seed[b], a.pass, (uint32_t)h, (uint32_t)v);
    const int pos = gl;
    const bool valid = active && gl < k;
    host_miss_counts<G>(valid && rank >= cached_len, host_off + rank, gl, hsec, hrun);
    int32_t x = -1;
    const bool hit = valid && rank < cached_len;
    if (valid) {
      if (hit)
        x = ld_keep_i32(a.acache + cache_off + rank, epol);
      else
        x = ld_host_i32(a.uidx + host_off + rank);
    }
    {  // the group's hits / misses in one pair of shared atomics (its dst belongs to one batch)
      const unsigned vm = __ballot_sync(0xffffffffu, valid) & gmask;
      const unsigned hm = __ballot_sync(0xffffffffu, hit) & gmask;
      if (gl == 0 && vm) {
        if (hm) atomicAdd(&S.cnt[b][0], (unsigned)__popc(hm));
        if (vm != hm) atomicAdd(&S.cnt[b][1], (unsigned)__popc(vm & ~hm));
      }
    }
    if (active && gl < f) hb.cand[d * f + (valid ? pos : gl)] = x;
    if (active && gl == 0) hb.kcnt[d] = k;
    if (valid) {
      const unsigned long long tag = S.ehi[b] | (0xFFFFFFFFu - (uint32_t)(n_h + d * f + pos));
      unsigned long long* tp = pt_insert(hb.pos_of, hb.hmask, x, (uint32_t)(S.ehi[b] >> 32));
      if (!a.precheck || __ldcg(tp) < tag) atomicMax(tp, tag);
      if (a.edge_counts) atomicAdd(a.edge_counts + host_off + rank, 1);
    }
    v = v_next;
    e0 = e0_next;
    e1 = e1_next;
    v_next = v_next2;
  }
  host_miss_flush(S, hsec, hrun);
  hop_shared_flush(a, S);
}


// ------------------------------------------------------------------------------------
// k_sample_hop_wide: fan-outs 33..1024, one warp per dst, chosen ranks in shared memory.
// Floyd is resolved chunk by chunk: a lane's draw is first checked against every rank fixed by
// earlier chunks (parallel scan of shared memory), then the chunk's 32 slots are resolved in
// order with shuffles/ballots exactly as in k_sample_hop.  Ranks are then sorted ascending by
// a bitonic network in shared memory (padded to a power of two with INT_MAX).
// ------------------------------------------------------------------------------------
constexpr int kWideWarps = 4;

__global__ void __launch_bounds__(32 * kWideWarps) k_sample_hop_wide(const __grid_constant__ HopLaunch a) {
  extern __shared__ int32_t s_wide[];
  __shared__ HopShared S;
  hop_shared_init(a, S);
  const int h = a.hop;
  const int f = a.f;
  int fp2 = 1;
  while (fp2 < f) fp2 <<= 1;
  int32_t* chosen = s_wide + (threadIdx.x >> 5) * fp2;
  const int lane = threadIdx.x & 31;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  hop_prologue(a, S, tid, nthreads);
  const long long total = S.pre[a.n];
  const uint64_t keep = policy_by(a.dir_policy);
  const uint64_t epol = policy_by(a.elem_policy);
  unsigned hsec = 0, hrun = 0;  // host sectors / runs of the adjacency misses (warp-uniform)
  for (int64_t q = tid >> 5; q < total; q += nthreads >> 5) {
    const int b = batch_of(S.pre, a.n, q);
    const HopBatch& hb = a.b[b];
    const int64_t d = q - S.pre[b];
    const int64_t n_h = S.pre[b + 1] - S.pre[b];
    const int32_t v = S.Fin[b][d];
    int4 e0 = make_int4(0, 0, 0, 0), e1 = make_int4(0, 0, 0, 0);
    if (v >= 0 && (int64_t)v < a.N) {
      const int4* ep = reinterpret_cast<const int4*>(a.dir + v);
      e0 = ld_keep_v4(ep, keep);
      e1 = ld_keep_v4(ep + 1, keep);
    }
    const int64_t host_off = ((int64_t)(uint32_t)e0.y << 32) | (uint32_t)e0.x;
    const int64_t cache_off = ((int64_t)(uint32_t)e0.w << 32) | (uint32_t)e0.z;
    const int32_t deg = e1.x;
    const int32_t cached_len = e1.y;
    const int k = deg < f ? deg : f;
    if (deg > f) {
      for (int c0 = 0; c0 < f; c0 += 32) {
        const int i = c0 + lane;
        const bool in = i < f;
        int32_t t = 0, j = 0;
        bool coll_prev = false;
        if (in) {
          j = deg - f + i;
          const uint64_t u = philox_u64(S.seed[b], a.pass, (uint32_t)h, (uint32_t)v, (uint32_t)i);
          t = (int32_t)__umul64hi(u, (uint64_t)(j + 1));
          for (int m = 0; m < c0; ++m) coll_prev |= chosen[m] == t;
        }
        int32_t res = 0;
        for (int i2 = 0; i2 < 32; ++i2) {
          const int32_t ti = __shfl_sync(0xffffffffu, t, i2);
          const bool coll = __ballot_sync(0xffffffffu, lane < i2 && res == ti) != 0;
          if (lane == i2) res = (coll_prev || coll) ? j : t;
        }
        if (in) chosen[i] = res;
        __syncwarp();
      }
      for (int i = f + lane; i < fp2; i += 32) chosen[i] = 0x7FFFFFFF;
      __syncwarp();
      // bitonic sort of chosen[0..fp2) ascending
      for (int kk = 2; kk <= fp2; kk <<= 1) {
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          for (int i = lane; i < fp2; i += 32) {
            const int ixj = i ^ jj;
            if (ixj > i) {
              const int32_t x = chosen[i], y = chosen[ixj];
              const bool up = (i & kk) == 0;
              if ((x > y) == up) {
                chosen[i] = y;
                chosen[ixj] = x;
              }
            }
          }
          __syncwarp();
        }
      }
    }
    // element reads in sorted-rank order: pos -> rank (all lanes run every pass: the host-sector
    // count shuffles across the warp, carrying the previous pass's last miss sector)
    long long carry_line = -1;
    bool any_miss = false;  // this dst's run had a miss (one run per dst, warp-uniform)
    for (int base = 0; base < f; base += 32) {
      const int pos = base + lane;
      {
        const int32_t rk = pos < k ? (deg > f ? chosen[pos] : pos) : 0;
        const bool miss = pos < k && rk >= cached_len;
        const long long line = (host_off + rk) >> 3;  // 32-byte sector
        long long pl = __shfl_up_sync(0xffffffffu, line, 1);
        bool pmiss = __shfl_up_sync(0xffffffffu, (int)miss, 1) != 0;
        if (lane == 0) {
          pl = carry_line;
          pmiss = carry_line >= 0;
        }
        const unsigned opened = __ballot_sync(0xffffffffu, miss && (!pmiss || pl != line));
        const unsigned missm = __ballot_sync(0xffffffffu, miss);
        const long long last = __shfl_sync(0xffffffffu, line, 31);
        carry_line = (missm >> 31) & 1u ? last : -1;
        hsec += __popc(opened);
        any_miss |= missm != 0u;
      }
      if (pos >= f) continue;
      int32_t x = -1;
      if (pos < k) {
        const int32_t rank = deg > f ? chosen[pos] : pos;
        const bool hit = rank < cached_len;
        if (hit)
          x = ld_keep_i32(a.acache + cache_off + rank, epol);
        else
          x = ld_host_i32(a.uidx + host_off + rank);
        atomicAdd(&S.cnt[b][hit ? 0 : 1], 1u);
        const unsigned long long tag = S.ehi[b] | (0xFFFFFFFFu - (uint32_t)(n_h + d * f + pos));
        unsigned long long* tp = pt_insert(hb.pos_of, hb.hmask, x, (uint32_t)(S.ehi[b] >> 32));
        if (__ldcg(tp) < tag) atomicMax(tp, tag);
        if (a.edge_counts) atomicAdd(a.edge_counts + host_off + rank, 1);
      }
      hb.cand[d * f + pos] = x;
    }
    if (lane == 0) hb.kcnt[d] = k;
    hrun += any_miss ? 1u : 0u;
    __syncwarp();
  }
  host_miss_flush(S, hsec, hrun);
  hop_shared_flush(a, S);
}

// k_scatter_headers: a group's per-batch headers (seeds pointer, B, seed, epoch) arrive in ONE
// host->device copy into a staging block; this first node of the group's graph puts each into
// its workspace's scalars, where every kernel of the batch reads it.
struct HeaderScatter {
  const BatchHeader* src;
  BatchScalars* dst[DCI_MAX_GROUP];
  int32_t n;
};

__global__ void k_scatter_headers(const __grid_constant__ HeaderScatter a) {
  if ((int)threadIdx.x < a.n) a.dst[threadIdx.x]->hdr = a.src[threadIdx.x];
}

// k_hop_epilogue: the hop_prologue of a virtual hop L, i.e. the relabel of the last hop into its
// block CSR and the clear of its scan state (launched after the last scan; the gather of a
// group / TMA gather does not fuse it).
__global__ void __launch_bounds__(256) k_hop_epilogue(const __grid_constant__ HopLaunch a) {
  __shared__ HopShared S;
  hop_shared_init(a, S);
  hop_prologue(a, S, blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// ------------------------------------------------------------------------------------
// k_newmask_sweep: the new-candidate masks of a node-sweep hop, node-major.  After the hop's
// atomicMax insertions, a node v is NEW in batch b iff its tag carries b's epoch and a position
// p >= n_h (a candidate position of this hop: F_h's own entries hold final ids < n_h), and p is its
// FIRST occurrence, i.e. the candidate (d, s) = ((p - n_h) / f, (p - n_h) % f) that owns it -- the
// same test the scan otherwise makes per candidate (tag == own position).  Sweeping node ids reads
// every table once, coalesced (N x n x 8 B), instead of one random tag read per candidate
// (sum_b |F_h(b)| x f: 12 M per group of 20 on M2's last hop), and sets bit s of nmask_b[d].
// The hop kernel zeroed the masks (one coalesced pass).  Exits at once unless the hop swept.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_newmask_sweep(const __grid_constant__ HopLaunch a) {
  __shared__ HopShared S;
  hop_shared_init(a, S);
  if (!a.nmask_on || !hop_sweeps(a, S.pre[a.n], S.all_ok)) return;
  const int n = a.n, f = a.f;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = tid; v < a.N; v += nthreads) {
    for (int b0 = 0; b0 < n; b0 += 8) {
      unsigned long long t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = b0 + u < n ? __ldcg(a.b[b0 + u].pos_of + v) : 0ull;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + u;
        if (b >= n || (t[u] >> 32) != (S.ehi[b] >> 32)) continue;
        const uint32_t p = 0xFFFFFFFFu - (uint32_t)t[u];
        const uint32_t n_h = (uint32_t)(S.pre[b + 1] - S.pre[b]);
        if (p < n_h) continue;
        const uint32_t q = p - n_h;
        atomicOr(a.b[b].nmask + q / (uint32_t)f, 1u << (q % (uint32_t)f));
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// k_scan_hop: kScanItems consecutive dsts of F_h per thread (1: four per thread, a quarter of the
// look-back steps, measured slower -- fewer tiles leave the early hops' per-candidate tag reads
// less parallelism), kScanDsts dsts per tile, tiles taken by dynamic tickets (in-order =>
// deadlock-free look-back).  (Measured and not kept: a three-pass reduce-then-scan, 27 / 48 /
// 70 us against 14 / 26 / 65 us per hop of M2 -- the last scan's cost is its 2 M new-node appends
// (candidate read, F write, final-id tag write), not the look-back; and a warp-cooperative append,
// no change); a multi-batch launch numbers the tiles of all its
// batches consecutively (one ticket counter) and each batch's tiles look back only within it.
// Per dst: k (samples) and the bitmask of candidates that are the first occurrence of a node not
// yet in F (table tag == tag(n_h + q)).  One block scan + warp-parallel decoupled look-back over
// packed (k << 31 | nn):
//   bptr_h[d]            = sum of k over earlier dsts                 (block CSR)
//   new id of candidate  = n_h + (#new candidates before it)          (F_{h+1} append)
// and the owner of each new node rewrites its table tag to the final local id, which the
// next kernel uses to relabel.  Hop 0 also checks seed uniqueness (C22).
// ------------------------------------------------------------------------------------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanTile) k_scan_hop(const __grid_constant__ HopLaunch a) {
  const int h = a.hop;
  const int f = a.f;
  const int n = a.n;
  __shared__ long long s_pre[DCI_MAX_GROUP + 1];   // n_h(b) prefix
  __shared__ long long s_tpre[DCI_MAX_GROUP + 1];  // tile prefix
  __shared__ unsigned long long s_ehi[DCI_MAX_GROUP];
  __shared__ uint32_t s_ticket;
  __shared__ unsigned long long s_warp[kScanTile / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_nmask;  // the hop swept: new-candidate masks come from k_newmask_sweep
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < 32) {  // warp 0: lane b reads batch b (see hop_shared_init)
    const int b = threadIdx.x;
    const bool in = b < n;
    long long nh = 0, nt = 0;
    int ok = 1;
    if (in) {
      const BatchScalars* sc = a.b[b].sc;
      nh = h == 0 ? (long long)sc->hdr.B : sc->sizes[h];
      nt = (nh + kScanDsts - 1) / kScanDsts;
      s_ehi[b] = (unsigned long long)sc->hdr.epoch << 32;
      ok = __ldcg(&sc->status) == 0;
    }
    const long long ia = warp_incl_scan(nh, b), it = warp_incl_scan(nt, b);
    if (in) {
      s_pre[b] = ia - nh;
      s_tpre[b] = it - nt;
    }
    const int all_ok = __all_sync(0xffffffffu, ok);
    const long long acc = __shfl_sync(0xffffffffu, ia, n - 1);
    if (b == n - 1) {
      s_pre[n] = ia;
      s_tpre[n] = it;
    }
    if (b == 0) s_nmask = a.nmask_on && hop_sweeps(a, acc, all_ok) ? 1 : 0;
  }
  __syncthreads();
  const bool use_nmask = s_nmask != 0;
  // empty batches: no tiles; their block CSR and size are written here
  if (blockIdx.x == 0 && threadIdx.x < n && s_pre[threadIdx.x + 1] == s_pre[threadIdx.x]) {
    a.b[threadIdx.x].bptr[0] = 0;
    a.b[threadIdx.x].sc->sizes[h + 1] = 0;
  }
  const long long ntiles_all = s_tpre[n];
  unsigned int* ticket = &a.b[0].sc->tickets[h];
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket, 1u);
    __syncthreads();
    const long long gt = s_ticket;
    if (gt >= ntiles_all) break;
    int b = 0;  // batch of tile gt: binary search over the tile prefix (n <= 32)
#pragma unroll
    for (int step = 16; step; step >>= 1)
      if (b + step < n && gt >= s_tpre[b + step]) b += step;
    const HopBatch& hb = a.b[b];
    const int64_t tile = gt - s_tpre[b];
    const int64_t n_h = s_pre[b + 1] - s_pre[b];
    const int64_t ntiles = (n_h + kScanDsts - 1) / kScanDsts;
    const unsigned long long ehi = s_ehi[b];
    // this thread's kScanItems consecutive dsts of the tile
    const int64_t d0 = tile * kScanDsts + (int64_t)threadIdx.x * kScanItems;
    uint32_t kk[kScanItems], newmask[kScanItems], nwide[kScanItems];
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      kk[it] = 0;
      newmask[it] = 0;
      nwide[it] = 0;
    }
    if (use_nmask) {  // (f <= 32, h >= 1)
#pragma unroll
      for (int it = 0; it < kScanItems; ++it)
        if (d0 + it < n_h) {
          kk[it] = (uint32_t)hb.kcnt[d0 + it];
          newmask[it] = hb.nmask[d0 + it];
        }
    } else {
      for (int it = 0; it < kScanItems; ++it) {
        const int64_t d = d0 + it;
        if (d >= n_h) break;
        const uint32_t k = (uint32_t)hb.kcnt[d];
        kk[it] = k;
        const int32_t* c = hb.cand + d * f;
        const uint32_t base = (uint32_t)(n_h + d * f);
        // which of d's candidates own their node's first occurrence (8 loads in flight); a
        // 32-bit mask for f <= 32, else counted here and re-checked when appending
        uint32_t nm = 0, nw = 0;
        for (uint32_t s0 = 0; s0 < k; s0 += 8) {
          int32_t x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = (s0 + u < k) ? c[s0 + u] : -1;
          unsigned long long t[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            t[u] = x[u] >= 0 ? pt_tag(hb.pos_of, hb.hmask, x[u], (uint32_t)(ehi >> 32)) : 0ull;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (x[u] >= 0 && t[u] == (ehi | (0xFFFFFFFFu - (base + s0 + u)))) {
              if (f <= 32)
                nm |= 1u << (s0 + u);
              else
                ++nw;
            }
        }
        newmask[it] = nm;
        nwide[it] = nw;
        if (h == 0) {
          const int32_t sd = hb.F[d];
          if (sd >= 0 && (int64_t)sd < a.N &&
              pt_tag(hb.pos_of, hb.hmask, sd, (uint32_t)(ehi >> 32)) != (ehi | (0xFFFFFFFFu - (uint32_t)d)))
            atomicCAS(&hb.sc->status, 0, (int32_t)DCI_EDUP);
        }
      }
    }
    unsigned long long mine = 0;  // packed (k << 31 | nn) over the thread's dsts
#pragma unroll
    for (int it = 0; it < kScanItems; ++it)
      mine += ((unsigned long long)kk[it] << 31) | (f <= 32 ? (uint32_t)__popc(newmask[it]) : nwide[it]);
    // block exclusive scan of packed (k << 31 | nn)
    unsigned long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      unsigned long long w = (lane < kScanTile / 32) ? s_warp[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < kScanTile / 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      if (lane < kScanTile / 32) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned long long tile_total = s_warp[kScanTile / 32 - 1];
    const unsigned long long excl = incl - mine + (wid > 0 ? s_warp[wid - 1] : 0ull);
    // decoupled look-back within the batch, warp-parallel: 32 predecessors per round
    if (wid == 0) {
      unsigned long long prefix = 0;
      if (tile == 0) {
        if (lane == 0) st_volatile_u64(hb.tiles, kFlagIncl | tile_total);
      } else {
        if (lane == 0) st_volatile_u64(hb.tiles + tile, kFlagAgg | tile_total);
        int64_t base = tile - 1;
        for (;;) {
          const int64_t t = base - lane;
          unsigned long long st = t >= 0 ? ld_volatile_u64(hb.tiles + t) : kFlagIncl;
          while (__any_sync(0xffffffffu, (st & ~kValMask) == 0)) {
            if ((st & ~kValMask) == 0) st = ld_volatile_u64(hb.tiles + t);
          }
          const unsigned incl_mask = __ballot_sync(0xffffffffu, (st & ~kValMask) == kFlagIncl);
          const int stop = incl_mask ? (__ffs(incl_mask) - 1) : 31;
          unsigned long long v = (lane <= stop) ? (st & kValMask) : 0ull;
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          prefix += v;
          if (incl_mask) break;
          base -= 32;
        }
        if (lane == 0) st_volatile_u64(hb.tiles + tile, kFlagIncl | (prefix + tile_total));
      }
      if (lane == 0) {
        s_prefix = prefix;
        if (tile == ntiles - 1) {
          const unsigned long long tot = prefix + tile_total;
          hb.bptr[n_h] = (int32_t)(tot >> 31);
          hb.sc->sizes[h + 1] = n_h + (int64_t)(tot & ((1ull << 31) - 1));
        }
      }
    }
    __syncthreads();
    {
      unsigned long long pre = s_prefix + excl;
      for (int it = 0; it < kScanItems; ++it) {
        const int64_t d = d0 + it;
        if (d >= n_h) break;
        hb.bptr[d] = (int32_t)(pre >> 31);
        uint32_t nid = (uint32_t)(n_h + (int64_t)(pre & ((1ull << 31) - 1)));
        const int32_t* c = hb.cand + d * f;
        if (f <= 32) {
          for (uint32_t m = newmask[it]; m; m &= m - 1) {
            const int s = __ffs(m) - 1;
            const int32_t x = c[s];
            hb.F[nid] = x;
            *pt_find(hb.pos_of, hb.hmask, x, (uint32_t)(ehi >> 32)) = ehi | (0xFFFFFFFFu - nid);
            ++nid;
          }
        } else if (nwide[it]) {
          // only this candidate's owner rewrites its tag, so the check is stable (see above)
          const uint32_t base = (uint32_t)(n_h + d * f);
          for (uint32_t s = 0; s < kk[it]; ++s) {
            const int32_t x = c[s];
            unsigned long long* tp = x >= 0 ? pt_find(hb.pos_of, hb.hmask, x, (uint32_t)(ehi >> 32)) : nullptr;
            if (tp && __ldcg(tp) == (ehi | (0xFFFFFFFFu - (base + s)))) {
              hb.F[nid] = x;
              *tp = ehi | (0xFFFFFFFFu - nid);
              ++nid;
            }
          }
        }
        pre += ((unsigned long long)kk[it] << 31) | (f <= 32 ? (uint32_t)__popc(newmask[it]) : nwide[it]);
      }
    }
    __syncthreads();  // s_ticket / s_prefix reuse
  }
}

static HopLaunch hop_launch(dci_ctx* ctx, dci_workspace* const* ws, const HopParams* p, int32_t n) {
  static const int elem_policy = [] {
    const char* e = getenv("DCI_ELEM_POLICY");
    return e ? atoi(e) : 1;
  }();
  HopLaunch a;
  memset(&a, 0, sizeof(a));
  a.dir = ctx->d_dir;
  a.acache = ctx->d_acache;
  a.uidx = ctx->u_idx_cur;
  a.N = ctx->N;
  a.hop = p[0].hop;
  a.f = p[0].f;
  a.prev_f = p[0].prev_f;
  a.n = n;
  a.pass = p[0].pass;
  a.elem_policy = elem_policy;
  static const int dir_policy = [] {
    const char* e = getenv("DCI_DIR_POLICY");
    return e ? atoi(e) : 1;
  }();
  a.dir_policy = dir_policy;
  a.edge_counts = p[0].edge_counts;
  static const int precheck = [] {
    const char* e = getenv("DCI_PRECHECK");
    return e ? atoi(e) : 0;
  }();
  a.precheck = precheck;
  static const int sweep = [] {
    const char* e = getenv("DCI_SAMPLE_SWEEP");
    return e ? atoi(e) : 1;
  }();
  a.sweep = sweep;
  // a hop samples by node sweep once its frontiers together reach N nodes -- or N / 20 when part of
  // the adjacency lives in host memory: the sweep then also reads each node's host run once per
  // group, which outweighs probing every node id (M3 4.70 -> 5.13-5.19 M seeds/s, M4s 1.105 ->
  // 1.165 M; tools/exp/r3ll.sh).  DCI_SWEEP_FACTOR overrides the factor.
  static const double sweep_factor = [] {
    const char* e = getenv("DCI_SWEEP_FACTOR");
    return e ? atof(e) : -1.0;
  }();
  const double factor = sweep_factor >= 0 ? sweep_factor : (ctx->whole_fit ? 1.0 : 0.05);
  a.sweep_min = std::max<int64_t>(1, (int64_t)((double)ctx->N * factor));
  for (int i = 0; i < n; ++i)
    if (ws[i]->hmask) a.sweep = 0;  // the node sweep probes every node id: dense tables only
  static const int nmask_on = [] {
    const char* e = getenv("DCI_NMASK_SWEEP");
    return e ? atoi(e) : 1;
  }();
  a.nmask_on = nmask_on;
  for (int i = 0; i < n; ++i) {
    HopBatch& b = a.b[i];
    const int h = p[i].hop;
    b.F = p[i].F;
    b.cand = p[i].cand;
    b.kcnt = p[i].kcnt;
    b.prev_cand = p[i].prev_cand;
    b.prev_kcnt = p[i].prev_kcnt;
    b.prev_bptr = p[i].prev_bptr;
    b.prev_bsrc = p[i].prev_bsrc;
    b.bptr = p[i].bptr;
    b.pos_of = ws[i]->pos_of;
    b.nmask = ws[i]->nmask;
    b.hmask = ws[i]->hmask;
    b.sc = ws[i]->scal;
    b.tiles = h < ws[i]->L ? ws[i]->tile_state + ws[i]->tile_off[h] : nullptr;
    if (h > 0) {
      b.prev_tiles = ws[i]->tile_state + ws[i]->tile_off[h - 1];
      b.prev_ntiles = ws[i]->tile_off[h] - ws[i]->tile_off[h - 1];
    }
  }
  return a;
}

}  // namespace

void launch_sample_hop(dci_ctx* ctx, dci_workspace* const* ws, const HopParams* p, int32_t n, cudaStream_t s) {
  const HopLaunch a = hop_launch(ctx, ws, p, n);
  // resident blocks per SM of the sampling grids: 8 (the whole GPU).  (Round 1 used 2 when a group's
  // sampling overlapped the previous group's 1-block-per-SM gather; the round-2 node-sweep gather
  // fills the SMs itself, and 8 measured best both alone and overlapped: DESIGN.md §9.)
  static const int forced = [] {
    const char* e = getenv("DCI_SAMPLE_BPS");
    return e ? atoi(e) : 0;
  }();
  const int bps = forced > 0 ? forced : 8;
  // Grid: persistent (SM count x resident blocks), but no larger than the worst-case frontier of
  // this hop needs (small frontiers would otherwise start hundreds of idle blocks); the fused
  // relabel of hop h-1 (|F_{h-1}| * f_{h-1} items) is covered by the grid-stride loops either way.
  int64_t cap = 0;
  for (int i = 0; i < n; ++i) cap += ws[i]->hop_cap[p[0].hop];
  cap = std::max<int64_t>(cap, 1);
  auto sized = [&](int persistent, int64_t nodes_per_block) {
    const int64_t need = (cap + nodes_per_block - 1) / nodes_per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(persistent, need));
  };
  const int f = p[0].f;
  int gsz = 1;
  while (gsz < f) gsz <<= 1;
  auto go = [&](auto kern) {
    kern<<<sized(persistent_grid(ctx, kern, 256, bps), 256 / gsz), 256, 0, s>>>(a);
  };
  if (f > 32) {
    int fp2 = 1;
    while (fp2 < f) fp2 <<= 1;
    const size_t smem = (size_t)kWideWarps * fp2 * sizeof(int32_t);
    k_sample_hop_wide<<<sized(persistent_grid(ctx, k_sample_hop_wide, 32 * kWideWarps, 16), kWideWarps),
                        32 * kWideWarps, smem, s>>>(a);
  } else if (f <= 1)
    go(k_sample_hop<1>);
  else if (f <= 2)
    go(k_sample_hop<2>);
  else if (f <= 4)
    go(k_sample_hop<4>);
  else if (f <= 8)
    go(k_sample_hop<8>);
  else if (f <= 16)
    go(k_sample_hop<16>);
  else
    go(k_sample_hop<32>);
  ++ctx->launches;
}

void launch_scan_hop(dci_ctx* ctx, dci_workspace* const* ws, const HopParams* p, int32_t n, cudaStream_t s) {
  const HopLaunch a = hop_launch(ctx, ws, p, n);
  int64_t tiles = 0;
  for (int i = 0; i < n; ++i) tiles += (ws[i]->hop_cap[p[0].hop] + kScanDsts - 1) / kScanDsts;
  int64_t grid = persistent_grid(ctx, k_scan_hop, kScanTile, 8);
  if (tiles < grid) grid = tiles > 0 ? tiles : 1;
  k_scan_hop<<<(unsigned)grid, kScanTile, 0, s>>>(a);
  ++ctx->launches;
}

void launch_newmask_sweep(dci_ctx* ctx, dci_workspace* const* ws, const HopParams* p, int32_t n, cudaStream_t s) {
  const HopLaunch a = hop_launch(ctx, ws, p, n);
  if (!(a.nmask_on && n >= 2 && a.f >= 3 && a.f <= 32 && a.hop >= 1 && a.sweep && a.edge_counts == nullptr))
    return;
  // the frontiers' capacities bound their sizes: below N together, the hop cannot sweep (the
  // kernel would exit at once), so nothing is launched
  int64_t cap = 0;
  for (int i = 0; i < n; ++i) cap += ws[i]->hop_cap[p[i].hop];
  if (cap < a.sweep_min) return;
  const int64_t grid = std::min<int64_t>(persistent_grid(ctx, k_newmask_sweep, 256, 8), (ctx->N + 255) / 256);
  k_newmask_sweep<<<(unsigned)std::max<int64_t>(grid, 1), 256, 0, s>>>(a);
  ++ctx->launches;
}

void launch_scatter_headers(dci_ctx* ctx, dci_workspace* const* ws, const BatchHeader* src, int32_t n,
                            cudaStream_t s) {
  HeaderScatter a;
  memset(&a, 0, sizeof(a));
  a.src = src;
  a.n = n;
  for (int i = 0; i < n; ++i) a.dst[i] = ws[i]->scal;
  k_scatter_headers<<<1, 32, 0, s>>>(a);
  ++ctx->launches;
}

void launch_hop_epilogue(dci_ctx* ctx, dci_workspace* const* ws, const HopParams* p, int32_t n, cudaStream_t s) {
  const HopLaunch a = hop_launch(ctx, ws, p, n);
  int64_t items = 0;
  for (int i = 0; i < n; ++i) items += ws[i]->hop_cap[p[0].hop - 1] * p[0].prev_f;
  const int64_t need = std::max<int64_t>(1, (items + 255) / 256);
  // DCI_EPI_BLOCKS caps the grid (a measurement knob: the relabel runs beside the group gather)
  static const int cap = [] {
    const char* e = getenv("DCI_EPI_BLOCKS");
    return e ? atoi(e) : 0;
  }();
  int grid = (int)std::min<int64_t>(persistent_grid(ctx, k_hop_epilogue, 256, 8), need);
  if (cap > 0 && grid > cap) grid = cap;
  k_hop_epilogue<<<grid, 256, 0, s>>>(a);
  ++ctx->launches;
}

}  // namespace dci
