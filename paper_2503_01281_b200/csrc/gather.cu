// S7 + S8 of the hot path, one kernel per batch:
//  - relabel of the last hop's candidates into its block CSR (table tag -> local id)
//  - feature-cache route inline through the remap table: slot = dir[F[i]].slot
//  - feature gather: X[i] = fcache[slot] on a hit (HBM -> HBM) or feats[v] on a
//    miss (pinned host -> HBM, UVA zero-copy), one warp per row, every lane issuing all of
//    its 16-byte loads before any store; the next row's (F, slot) lookups are prefetched
//  - presample: node_visits[v] += 1 (C7)
//  - the last block to finish publishes sizes / counters / status and resets the
//    workspace scalars for the next batch.
#include <cuda_runtime.h>

#include <cstdlib>

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

__device__ __forceinline__ int4 ld_stream_v4(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ void st_v4(int4* p, const int4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

struct FusedArgs {
  const DirEntry* dir;
  const unsigned long long* pos_of;
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
        a.last_bsrc[a.last_bptr[d] + s] = (int32_t)(0xFFFFFFFFu - (uint32_t)__ldcg(a.pos_of + a.last_cand[q]));
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
            if (idx < row16) buf[j] = ld_stream_v4(s4 + idx, pol);
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
    sc->acc_rows += (unsigned long long)__ldcg(&sc->sizes[a.L]);
    for (int c = 0; c < 4; ++c) sc->acc_counters[c] += a.out_counters[c];
    sc->status = 0;
    sc->done = 0;
  }
}

}  // namespace

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

void launch_gather_fused(dci_ctx* ctx, dci_workspace* ws, int32_t L, const dci_batch_out* out,
                         const HopParams& last, int32_t* node_visits, cudaStream_t s) {
  FusedArgs a;
  a.dir = ctx->d_dir;
  a.pos_of = ws->pos_of;
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
}

}  // namespace dci
