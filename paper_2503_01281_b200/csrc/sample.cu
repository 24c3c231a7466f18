// S5-S7 of the hot path: per-hop neighbour sampling with the adjacency
// cache, per-hop dedup/relabel via a node->position table and
// a single-pass decoupled look-back scan (first-occurrence order, reading C6), and the
// feature-cache route.  All launches use persistent, SM-count-sized grids
// that read the frontier size from device memory, so a batch never synchronises the host.
#include <cuda_runtime.h>

#include "dci_internal.cuh"
#include "philox.cuh"

namespace dci {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Host-mapped (UVA) neighbour read: a plain global load that the GPU turns into a PCIe
// read request.
__device__ __forceinline__ int32_t ld_host_i32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

struct SampleArgs {
  const DirEntry* dir;
  const int32_t* acache;
  const int32_t* uidx;  // device alias of the pinned host CSC (current order)
  int64_t N;
  int32_t* pos_of;
  BatchScalars* sc;
  HopParams p;
};

// ------------------------------------------------------------------------------------
// k_sample_hop<G>: one group of G lanes (G = next pow2 >= f) per dst node of F_h.
//  1. one broadcast 32 B directory load (host_off, cache_off, deg, cached_len)
//  2. k = min(deg, f); deg <= f -> ranks 0..deg-1; else Floyd's selection with lane i
//     drawing t_i = floor(u_i * (j_i + 1) / 2^64), j_i = deg - k + i, u_i =
//     Philox(v, i, hop, pass; seed) and a (f-1)-step shuffle/ballot collision resolution
//     (O-3, O-4)
//  3. ranks sorted in registers (position = #smaller ranks in the group)
//  4. element read: HBM cache iff rank < cached_len, else UVA host read
//  5. cand[d*f + pos] = neighbour, pads -1; kcnt[d] = k
//  6. insert into the node->position table: atomicMin(pos_of[x], n_h + d*f + pos), so the
//     table ends with each new node's first (dst-major, rank-ascending) occurrence
//  7. presample: edge_counts[host_off + rank] += 1 (C8)
// Fused extra work: hop 0 writes the seeds into F and the table (position = seed index);
// hop h >= 1 relabels hop h-1's candidates into its block CSR (bsrc[h-1]).
// ------------------------------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(256) k_sample_hop(SampleArgs a) {
  const HopParams& p = a.p;
  BatchScalars* sc = a.sc;
  const int h = p.hop;
  const int f = p.f;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int gbase = lane & ~(G - 1);
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;

  const int64_t n_h = (h == 0) ? (int64_t)p.B : sc->sizes[h];

  if (h == 0) {
    for (int64_t d = tid; d < p.B; d += nthreads) {
      const int32_t s = p.F_in[d];
      p.F[d] = s;
      if (s < 0 || (int64_t)s >= a.N)
        atomicCAS(&sc->status, 0, (int32_t)DCI_ESEED);
      else
        atomicMin(&a.pos_of[s], (int32_t)d);
    }
  } else {
    // relabel of hop h-1 (its scan has completed: kernel boundary)
    const int pf = p.prev_f;
    const int64_t n_prev = (h == 1) ? (int64_t)p.B : sc->sizes[h - 1];
    const int64_t nq = n_prev * pf;
    for (int64_t q = tid; q < nq; q += nthreads) {
      const int64_t d = q / pf;
      const int s = (int)(q - d * pf);
      if (s < p.prev_kcnt[d]) p.prev_bsrc[p.prev_bptr[d] + s] = a.pos_of[p.prev_cand[q]];
    }
  }

  const int GPW = 32 / G;
  const int64_t warp_id = tid >> 5;
  const int64_t nwarps = nthreads >> 5;
  uint32_t hits = 0, misses = 0;
  for (int64_t dbase = warp_id * GPW; dbase < n_h; dbase += nwarps * GPW) {
    const int64_t d = dbase + lane / G;
    const bool active = d < n_h;
    int32_t v = -1;
    int4 e0 = make_int4(0, 0, 0, 0), e1 = make_int4(0, 0, 0, 0);
    if (active) {
      v = p.F_in[d];
      if (v >= 0 && (int64_t)v < a.N) {
        const int4* ep = reinterpret_cast<const int4*>(a.dir + v);
        e0 = __ldg(ep);
        e1 = __ldg(ep + 1);
      }
    }
    const int64_t host_off = ((int64_t)(uint32_t)e0.y << 32) | (uint32_t)e0.x;
    const int64_t cache_off = ((int64_t)(uint32_t)e0.w << 32) | (uint32_t)e0.z;
    const int32_t deg = e1.x;
    const int32_t cached_len = e1.y;
    const int k = deg < f ? deg : f;
    const bool floyd = deg > f;

    int32_t rank = gl;
    int pos = gl;
    if (__any_sync(0xffffffffu, floyd)) {
      int32_t chosen = 0, j = 0;
      if (floyd && gl < f) {
        j = deg - f + gl;
        const uint64_t u = philox_u64(p.seed, p.pass, (uint32_t)h, (uint32_t)v, (uint32_t)gl);
        chosen = (int32_t)__umul64hi(u, (uint64_t)(j + 1));
      }
      // Floyd: slot i keeps t_i unless an earlier slot already chose it, then takes j_i.
      for (int i = 1; i < f; ++i) {
        const int32_t ti = __shfl_sync(0xffffffffu, chosen, i, G);
        const unsigned coll = __ballot_sync(0xffffffffu, gl < i && chosen == ti) & gmask;
        if (gl == i && coll) chosen = j;
      }
      // ascending order: position = number of smaller chosen ranks in the group
      int cnt = 0;
      for (int i = 0; i < f; ++i) {
        const int32_t c = __shfl_sync(0xffffffffu, chosen, i, G);
        cnt += (c < chosen) ? 1 : 0;
      }
      if (floyd) {
        rank = chosen;
        pos = cnt;
      }
    }

    const bool valid = active && gl < k;
    int32_t x = -1;
    if (valid) {
      if (rank < cached_len) {
        x = __ldg(a.acache + cache_off + rank);
        ++hits;
      } else {
        x = ld_host_i32(a.uidx + host_off + rank);
        ++misses;
      }
    }
    if (active && gl < f) p.cand[d * f + (valid ? pos : gl)] = x;
    if (active && gl == 0) p.kcnt[d] = k;
    if (valid) {
      const int32_t mypos = (int32_t)(n_h + d * f + pos);
      if (__ldcg(a.pos_of + x) > mypos) atomicMin(a.pos_of + x, mypos);
      if (p.edge_counts) atomicAdd(p.edge_counts + host_off + rank, 1);
    }
  }
  hits = __reduce_add_sync(0xffffffffu, hits);
  misses = __reduce_add_sync(0xffffffffu, misses);
  if (lane == 0 && (hits | misses)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->counters[0]), (unsigned long long)hits);
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->counters[1]), (unsigned long long)misses);
  }
}

// ------------------------------------------------------------------------------------
// k_scan_hop: one thread per dst of F_h, kScanTile dsts per tile, tiles taken by dynamic
// tickets (in-order => deadlock-free look-back).  Per dst: k (samples) and nn (candidates
// that are the first occurrence of a node not yet in F: pos_of[x] == n_h + q).  One block
// scan + decoupled look-back over packed (k << 31 | nn) gives
//   bptr_h[d]            = sum of k over earlier dsts                 (block CSR)
//   new id of candidate  = n_h + (#new candidates before it)          (F_{h+1} append)
// and the owner of each new node rewrites pos_of[x] to its final local id, which the next
// kernel uses to relabel.  Hop 0 also checks seed uniqueness (C22).
// ------------------------------------------------------------------------------------
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagIncl = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

struct ScanArgs {
  int32_t* pos_of;
  BatchScalars* sc;
  unsigned long long* tile_state;  // this hop's region
  int64_t N;
  HopParams p;
};

__global__ void __launch_bounds__(kScanTile) k_scan_hop(ScanArgs a) {
  const HopParams& p = a.p;
  BatchScalars* sc = a.sc;
  const int h = p.hop;
  const int f = p.f;
  const int64_t n_h = (h == 0) ? (int64_t)p.B : sc->sizes[h];
  const int64_t ntiles = (n_h + kScanTile - 1) / kScanTile;
  __shared__ uint32_t s_ticket;
  __shared__ unsigned long long s_warp[kScanTile / 32];
  __shared__ unsigned long long s_prefix;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  if (n_h == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.bptr[0] = 0;
      sc->sizes[h + 1] = 0;
    }
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_ticket = atomicAdd(&sc->tickets[h], 1u);
    __syncthreads();
    const int64_t tile = s_ticket;
    if (tile >= ntiles) break;
    const int64_t d = tile * kScanTile + threadIdx.x;
    uint32_t k = 0, nn = 0;
    if (d < n_h) {
      k = (uint32_t)p.kcnt[d];
      const int32_t* c = p.cand + d * f;
      const int32_t base = (int32_t)(n_h + d * f);
      for (uint32_t s = 0; s < k; ++s) nn += (__ldcg(a.pos_of + c[s]) == base + (int32_t)s) ? 1u : 0u;
      if (h == 0) {
        const int32_t sd = p.F[d];
        if (sd >= 0 && (int64_t)sd < a.N && __ldcg(a.pos_of + sd) != (int32_t)d)
          atomicCAS(&sc->status, 0, (int32_t)DCI_EDUP);
      }
    }
    // block exclusive scan of packed (k << 31 | nn)
    const unsigned long long mine = ((unsigned long long)k << 31) | nn;
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
    // decoupled look-back (thread 0)
    if (threadIdx.x == 0) {
      unsigned long long prefix = 0;
      if (tile == 0) {
        st_volatile_u64(a.tile_state, kFlagIncl | tile_total);
      } else {
        st_volatile_u64(a.tile_state + tile, kFlagAgg | tile_total);
        int64_t t = tile - 1;
        for (;;) {
          const unsigned long long s = ld_volatile_u64(a.tile_state + t);
          const unsigned long long flag = s & ~kValMask;
          if (flag == 0) continue;
          prefix += s & kValMask;
          if (flag == kFlagIncl) break;
          --t;
        }
        st_volatile_u64(a.tile_state + tile, kFlagIncl | (prefix + tile_total));
      }
      s_prefix = prefix;
      if (tile == ntiles - 1) {
        const unsigned long long tot = prefix + tile_total;
        p.bptr[n_h] = (int32_t)(tot >> 31);
        sc->sizes[h + 1] = n_h + (int64_t)(tot & ((1ull << 31) - 1));
      }
    }
    __syncthreads();
    if (d < n_h) {
      const unsigned long long pre = s_prefix + excl;
      p.bptr[d] = (int32_t)(pre >> 31);
      int32_t nid = (int32_t)(n_h + (int64_t)(pre & ((1ull << 31) - 1)));
      if (nn) {
        const int32_t* c = p.cand + d * f;
        const int32_t base = (int32_t)(n_h + d * f);
        for (uint32_t s = 0; s < k; ++s) {
          const int32_t x = c[s];
          if (__ldcg(a.pos_of + x) == base + (int32_t)s) {
            p.F[nid] = x;
            a.pos_of[x] = nid;
            ++nid;
          }
        }
      }
    }
    __syncthreads();  // s_ticket / s_prefix reuse
  }
}

// ------------------------------------------------------------------------------------
// k_route: relabel of the last hop + feature-cache route (S7).  For i < |F_L|:
// slot = dir[F[i]].slot; hit -> hit list (i, slot), miss -> miss list (i, v), appended
// with one atomic per warp (ballot + popc).  Presample: node_visits[v] += 1 (C7).
// ------------------------------------------------------------------------------------
struct RouteArgs {
  const DirEntry* dir;
  int32_t* pos_of;
  BatchScalars* sc;
  int64_t N;
  int32_t L;
  int32_t B;
  const int32_t* F;
  const int32_t* last_cand;
  const int32_t* last_kcnt;
  const int32_t* last_bptr;
  int32_t* last_bsrc;
  int32_t last_f;
  int64_t* hit_list;
  int64_t* miss_list;
  int32_t* node_visits;
};

__global__ void __launch_bounds__(256) k_route(RouteArgs a) {
  BatchScalars* sc = a.sc;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  {
    const int pf = a.last_f;
    const int64_t n_prev = (a.L == 1) ? (int64_t)a.B : sc->sizes[a.L - 1];
    const int64_t nq = n_prev * pf;
    for (int64_t q = tid; q < nq; q += nthreads) {
      const int64_t d = q / pf;
      const int s = (int)(q - d * pf);
      if (s < a.last_kcnt[d]) a.last_bsrc[a.last_bptr[d] + s] = a.pos_of[a.last_cand[q]];
    }
  }
  const int64_t n_L = sc->sizes[a.L];
  uint32_t hits = 0, misses = 0;
  const int64_t nwarps = nthreads >> 5;
  for (int64_t base = (tid >> 5) * 32; base < n_L; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t v = -1, slot = -1;
    bool ok = false;
    if (i < n_L) {
      v = a.F[i];
      ok = v >= 0 && (int64_t)v < a.N;
      if (ok) slot = __ldg(&a.dir[v].slot);
    }
    const bool is_hit = ok && slot >= 0;
    const bool is_miss = ok && slot < 0;
    const unsigned mh = __ballot_sync(0xffffffffu, is_hit);
    const unsigned mm = __ballot_sync(0xffffffffu, is_miss);
    uint32_t bh = 0, bm = 0;
    if (lane == 0) {
      if (mh) bh = atomicAdd(&sc->hit_count, (uint32_t)__popc(mh));
      if (mm) bm = atomicAdd(&sc->miss_count, (uint32_t)__popc(mm));
    }
    bh = __shfl_sync(0xffffffffu, bh, 0);
    bm = __shfl_sync(0xffffffffu, bm, 0);
    if (is_hit) a.hit_list[bh + __popc(mh & lanemask_lt())] = (i << 32) | (uint32_t)slot;
    if (is_miss) a.miss_list[bm + __popc(mm & lanemask_lt())] = (i << 32) | (uint32_t)v;
    if (ok && a.node_visits) atomicAdd(a.node_visits + v, 1);
    hits += is_hit ? 1u : 0u;
    misses += is_miss ? 1u : 0u;
  }
  hits = __reduce_add_sync(0xffffffffu, hits);
  misses = __reduce_add_sync(0xffffffffu, misses);
  if (lane == 0 && (hits | misses)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->counters[2]), (unsigned long long)hits);
    atomicAdd(reinterpret_cast<unsigned long long*>(&sc->counters[3]), (unsigned long long)misses);
  }
}

// ------------------------------------------------------------------------------------
// k_finish: publish sizes / counters / status to the caller's buffers, clear the
// node->position table over F_L (every key inserted this batch is in F_L), and reset the
// workspace scalars and scan tile state for the next batch.
// ------------------------------------------------------------------------------------
struct FinishArgs {
  int32_t* pos_of;
  BatchScalars* sc;
  unsigned long long* tile_state;
  int64_t tiles_total;
  int64_t N;
  int32_t L;
  int32_t B;
  const int32_t* F;
  int64_t* out_sizes;
  uint64_t* out_counters;
  int32_t* out_status;
};

__global__ void __launch_bounds__(256) k_finish(FinishArgs a) {
  BatchScalars* sc = a.sc;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_L = sc->sizes[a.L];
  for (int64_t i = tid; i < n_L; i += nthreads) {
    const int32_t v = a.F[i];
    if (v >= 0 && (int64_t)v < a.N) a.pos_of[v] = kPosEmpty;
  }
  for (int64_t i = tid; i < a.tiles_total; i += nthreads) a.tile_state[i] = 0ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.out_sizes[0] = a.B;
    for (int h = 1; h <= a.L; ++h) a.out_sizes[h] = sc->sizes[h];
    for (int c = 0; c < 4; ++c) {
      a.out_counters[c] = sc->counters[c];
      sc->counters[c] = 0;
    }
    *a.out_status = sc->status;
    sc->status = 0;
    for (int h = 0; h < DCI_MAX_LAYERS; ++h) sc->tickets[h] = 0;
    sc->hit_count = 0;
    sc->miss_count = 0;
  }
}

}  // namespace

void launch_sample_hop(dci_ctx* ctx, dci_workspace* ws, const HopParams& p, cudaStream_t s) {
  SampleArgs a{ctx->d_dir, ctx->d_acache, ctx->u_idx_cur, ctx->N, ws->pos_of, ws->scal, p};
  // sub-warp group width: next power of two >= f
  auto go = [&](auto kern) { kern<<<persistent_grid(ctx, kern, 256), 256, 0, s>>>(a); };
  if (p.f <= 1)
    go(k_sample_hop<1>);
  else if (p.f <= 2)
    go(k_sample_hop<2>);
  else if (p.f <= 4)
    go(k_sample_hop<4>);
  else if (p.f <= 8)
    go(k_sample_hop<8>);
  else if (p.f <= 16)
    go(k_sample_hop<16>);
  else
    go(k_sample_hop<32>);
  ++ctx->launches;
}

void launch_scan_hop(dci_ctx* ctx, dci_workspace* ws, const HopParams& p, cudaStream_t s) {
  ScanArgs a{ws->pos_of, ws->scal, ws->tile_state + ws->tile_off[p.hop], ctx->N, p};
  const int64_t tiles = (ws->hop_cap[p.hop] + kScanTile - 1) / kScanTile;
  int64_t grid = persistent_grid(ctx, k_scan_hop, kScanTile, 8);
  if (tiles < grid) grid = tiles > 0 ? tiles : 1;
  k_scan_hop<<<(unsigned)grid, kScanTile, 0, s>>>(a);
  ++ctx->launches;
}

void launch_route(dci_ctx* ctx, dci_workspace* ws, int32_t L, int32_t B, const int32_t* F, const int32_t* last_cand,
                  const int32_t* last_kcnt, const int32_t* last_bptr, int32_t* last_bsrc, int32_t last_f,
                  int32_t* node_visits, cudaStream_t s) {
  RouteArgs a{ctx->d_dir, ws->pos_of, ws->scal, ctx->N, L, B, F, last_cand, last_kcnt, last_bptr, last_bsrc,
              last_f, ws->hit_list, ws->miss_list, node_visits};
  k_route<<<persistent_grid(ctx, k_route, 256), 256, 0, s>>>(a);
  ++ctx->launches;
}

void launch_finish(dci_ctx* ctx, dci_workspace* ws, int32_t L, int32_t B, const dci_batch_out* out,
                   cudaStream_t s) {
  FinishArgs a{ws->pos_of, ws->scal, ws->tile_state, ws->tiles_cap, ctx->N, L, B, out->frontier, out->sizes,
               out->counters, out->status};
  k_finish<<<persistent_grid(ctx, k_finish, 256, 2), 256, 0, s>>>(a);
  ++ctx->launches;
}

}  // namespace dci
