// S0 directory build and S3/S4 cache fills.
//  Feature fill (reading C11): top-cap nodes by key (visits desc, id asc) found by
//  an 8-pass MSB radix select over 64-bit keys (no sort), slots by an id-ordered scan.
//  Adjacency fill (Algorithm 1; Fig. 6): level 2 = per-node stable
//  counting sort of each run by access count (desc), applied to the host CSC; level 1 =
//  node order (total desc, id asc), realised by a WEIGHTED radix select (weight = degree)
//  that finds the node where the node-major prefix reaches floor(C_adj / 4) elements.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "dci_internal.cuh"

namespace dci {

namespace {

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void k_build_directory(const int64_t* __restrict__ indptr, int64_t N, DirEntry* dir) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    DirEntry e;
    e.host_off = indptr[v];
    e.cache_off = 0;
    e.deg = (int32_t)(indptr[v + 1] - indptr[v]);
    e.cached_len = 0;
    e.slot = -1;
    e.pad = 0;
    dir[v] = e;
  }
}

__global__ void k_max_i32(const int32_t* __restrict__ a, int64_t n, int32_t* out) {
  int32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, a[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ------------------------------------------------------------------------------------
// Level-2 reorder: one warp per node.  Stable LSD radix sort of the node's run by key
// b = cmax - count (ascending b == descending count; equal counts keep original order),
// 8-bit digits, npass passes (npass = 1 while cmax < 256).  Each pass: warp histogram in
// shared memory, warp exclusive scan, then a stable scatter in 32-element chunks where
// equal-digit lanes are ranked with __match_any_sync.  Nodes whose counts are all zero
// are copied unchanged.  Also writes node totals (Alg. 1 lines 5-8).
// ------------------------------------------------------------------------------------
constexpr int kL2Warps = 8;

struct Level2Args {
  const int64_t* indptr;
  int64_t N;
  const int32_t* idx_in;
  const int32_t* cnt;
  int32_t cmax;
  int npass;
  int32_t* idx_out;
  int32_t* tmp_idx[2];  // ping-pong scratch (npass > 1)
  uint32_t* tmp_key[2];
  int64_t* total;
  int32_t* range_err;
};

__global__ void __launch_bounds__(32 * kL2Warps) k_level2(Level2Args a) {
  __shared__ uint32_t s_hist[kL2Warps][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* hist = s_hist[wib];
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < a.N; v += nwarps) {
    const int64_t base = a.indptr[v];
    const int64_t deg = a.indptr[v + 1] - base;
    int64_t sum = 0;
    for (int64_t p = lane; p < deg; p += 32) sum += a.cnt[base + p];
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      a.total[v] = sum;
      if (sum >= (1ll << 32)) atomicExch(a.range_err, 1);
    }
    if (sum == 0) {
      for (int64_t p = lane; p < deg; p += 32) a.idx_out[base + p] = a.idx_in[base + p];
      continue;
    }
    for (int pass = 0; pass < a.npass; ++pass) {
      const int shift = 8 * pass;
      const bool first = pass == 0, last = pass == a.npass - 1;
      const int32_t* src_idx = first ? a.idx_in : a.tmp_idx[(pass - 1) & 1];
      const uint32_t* src_key = first ? nullptr : a.tmp_key[(pass - 1) & 1];
      int32_t* dst_idx = last ? a.idx_out : a.tmp_idx[pass & 1];
      uint32_t* dst_key = last ? nullptr : a.tmp_key[pass & 1];
      for (int b = lane; b < 256; b += 32) hist[b] = 0;
      __syncwarp();
      for (int64_t p = lane; p < deg; p += 32) {
        const uint32_t key = first ? (uint32_t)(a.cmax - a.cnt[base + p]) : src_key[base + p];
        atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncwarp();
      // exclusive scan of 256 buckets: lane owns buckets [8*lane, 8*lane + 8)
      uint32_t loc[8], run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        loc[j] = run;
        run += hist[lane * 8 + j];
      }
      uint32_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - run;
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j) hist[lane * 8 + j] = excl + loc[j];
      __syncwarp();
      for (int64_t p0 = 0; p0 < deg; p0 += 32) {
        const int64_t p = p0 + lane;
        const bool valid = p < deg;
        uint32_t key = 0;
        int32_t val = 0;
        if (valid) {
          key = first ? (uint32_t)(a.cmax - a.cnt[base + p]) : src_key[base + p];
          val = src_idx[base + p];
        }
        const uint32_t dig = valid ? ((key >> shift) & 255u) : (256u + lane);
        const unsigned peers = __match_any_sync(0xffffffffu, dig);
        const uint32_t rank = __popc(peers & lanemask_lt());
        uint32_t at = 0;
        if (valid) at = hist[dig] + rank;
        __syncwarp();
        if (valid && rank == 0) hist[dig] += __popc(peers);
        __syncwarp();
        if (valid) {
          dst_idx[base + at] = val;
          if (dst_key) dst_key[base + at] = key;
        }
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------------------------
// Weighted MSB radix select over 64-bit keys.  After pass p the top 8(p+1) bits of K* are
// known; `above` = total weight of keys strictly greater than every key sharing the
// known prefix.  K* is the largest key with W(keys >= K*) >= target.
// ------------------------------------------------------------------------------------
struct RSState {
  unsigned long long prefix;
  unsigned long long above;
  unsigned long long target;
  unsigned long long hist[256];
};

struct FeatKey {
  const int32_t* visits;
  __device__ __forceinline__ unsigned long long key(int64_t v) const {
    return ((unsigned long long)(uint32_t)visits[v] << 32) | (0xFFFFFFFFull - (unsigned long long)v);
  }
  __device__ __forceinline__ unsigned long long weight(int64_t) const { return 1ull; }
};

struct AdjKey {
  const int64_t* total;
  const int64_t* indptr;
  __device__ __forceinline__ unsigned long long key(int64_t v) const {
    return ((unsigned long long)total[v] << 32) | (0xFFFFFFFFull - (unsigned long long)v);
  }
  __device__ __forceinline__ unsigned long long weight(int64_t v) const {
    return (unsigned long long)(indptr[v + 1] - indptr[v]);
  }
};

template <class K>
__global__ void __launch_bounds__(256) k_rs_hist(K kf, int64_t N, int pass, RSState* st) {
  __shared__ unsigned long long h[256];
  for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int shift = 56 - 8 * pass;
  const unsigned long long hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
  const unsigned long long pre = st->prefix & hi_mask;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = kf.key(v);
    if ((k & hi_mask) == pre) {
      const unsigned long long w = kf.weight(v);
      if (w) atomicAdd(&h[(k >> shift) & 255ull], w);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x)
    if (h[b]) atomicAdd(&st->hist[b], h[b]);
}

__global__ void k_rs_select(int pass, RSState* st) {
  if (threadIdx.x != 0) return;
  const int shift = 56 - 8 * pass;
  unsigned long long cum = st->above;
  int b = 255;
  for (; b > 0; --b) {
    if (cum + st->hist[b] >= st->target) break;
    cum += st->hist[b];
  }
  st->above = cum;
  st->prefix |= (unsigned long long)b << shift;
  for (int i = 0; i < 256; ++i) st->hist[i] = 0;
}

// ------------------------------------------------------------------------------------
// Reduce-then-scan over node ids with a value functor (fill-time only, not the hot path).
// ------------------------------------------------------------------------------------
constexpr int kScanB = 256, kScanItems = 16, kScanChunk = kScanB * kScanItems;

template <class Op>
__global__ void __launch_bounds__(kScanB) k_chunk_sum(Op op, int64_t n, int64_t* sums) {
  __shared__ int64_t s[kScanB / 32];
  const int64_t c0 = blockIdx.x * (int64_t)kScanChunk;
  int64_t acc = 0;
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = c0 + threadIdx.x * kScanItems + j;
    if (i < n) acc += op.value(i);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < kScanB / 32; ++w) t += s[w];
    sums[blockIdx.x] = t;
  }
}

__global__ void k_scan_sums(int64_t* sums, int64_t nb, int64_t* total) {
  // one block of 1024: each thread scans a contiguous segment, then block scan of segments
  __shared__ int64_t seg[1024];
  const int64_t per = (nb + 1023) / 1024;
  const int64_t a = threadIdx.x * per, b = min(nb, a + per);
  int64_t t = 0;
  for (int64_t i = a; i < b; ++i) t += sums[i];
  seg[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < 1024; ++i) {
      const int64_t x = seg[i];
      seg[i] = run;
      run += x;
    }
    *total = run;
  }
  __syncthreads();
  int64_t run = seg[threadIdx.x];
  for (int64_t i = a; i < b; ++i) {
    const int64_t x = sums[i];
    sums[i] = run;
    run += x;
  }
}

template <class Op>
__global__ void __launch_bounds__(kScanB) k_chunk_scan_write(Op op, int64_t n, const int64_t* chunk_prefix) {
  __shared__ int64_t s[kScanB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t c0 = blockIdx.x * (int64_t)kScanChunk + threadIdx.x * (int64_t)kScanItems;
  int64_t vals[kScanItems];
  int64_t acc = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = c0 + j;
    vals[j] = (i < n) ? op.value(i) : 0;
    acc += vals[j];
  }
  int64_t incl = acc;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int w = 0; w < kScanB / 32; ++w) {
      const int64_t x = s[w];
      s[w] = run;
      run += x;
    }
  }
  __syncthreads();
  int64_t run = chunk_prefix[blockIdx.x] + s[wid] + incl - acc;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t i = c0 + j;
    if (i < n) op.write(i, run, vals[j]);
    run += vals[j];
  }
}

// feature admission: value = admitted ? 1 : 0; write slot + copy-list entry
struct FeatSlotOp {
  FeatKey kf;
  const RSState* st;  // nullptr: admit all
  DirEntry* dir;
  int64_t* list;
  __device__ __forceinline__ int64_t value(int64_t v) const {
    return (st == nullptr || kf.key(v) >= st->prefix) ? 1 : 0;
  }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t val) const {
    dir[v].slot = val ? (int32_t)excl : -1;
    if (val) list[excl] = (excl << 32) | v;
  }
};

// adjacency admission: value = cached_len; write cached_len + cache_off
struct AdjLenOp {
  AdjKey kf;
  const RSState* st;  // nullptr: whole fit
  unsigned long long cap_e;
  DirEntry* dir;
  __device__ __forceinline__ int64_t value(int64_t v) const {
    const int64_t deg = kf.indptr[v + 1] - kf.indptr[v];
    if (st == nullptr) return deg;
    const unsigned long long k = kf.key(v);
    if (k > st->prefix) return deg;
    if (k == st->prefix) return (int64_t)(cap_e - st->above);
    return 0;
  }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t val) const {
    dir[v].cached_len = (int32_t)val;
    dir[v].cache_off = excl;
  }
};

// knapsack adjacency: value = ties of node v (exclusive scan -> ties before v)
struct TieScanOp {
  const int32_t* ties;
  int64_t* ties_before;
  __device__ __forceinline__ int64_t value(int64_t v) const { return ties[v]; }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t) const { ties_before[v] = excl; }
};

// knapsack adjacency: cached_len = #count > cv + the node's share of the first cm ties
struct KnapAdjOp {
  const int32_t* gt;
  const int32_t* ties;
  const int64_t* ties_before;
  int64_t cm;
  DirEntry* dir;
  __device__ __forceinline__ int64_t value(int64_t v) const {
    const int64_t take = cm - ties_before[v];
    return (int64_t)gt[v] + (take <= 0 ? 0 : (take < ties[v] ? take : ties[v]));
  }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t val) const {
    dir[v].cached_len = (int32_t)val;
    dir[v].cache_off = excl;
  }
};

// knapsack features: tie rank among nodes with visits == fv
struct FeatTieOp {
  const int32_t* visits;
  int32_t fv;
  int64_t* rank;
  __device__ __forceinline__ int64_t value(int64_t v) const { return visits[v] == fv ? 1 : 0; }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t) const { rank[v] = excl; }
};

struct KnapFeatOp {
  const int32_t* visits;
  int32_t fv;
  int64_t fm;
  const int64_t* rank;
  DirEntry* dir;
  int64_t* list;
  __device__ __forceinline__ int64_t value(int64_t v) const {
    const int32_t x = visits[v];
    return (x > fv || (x == fv && rank[v] < fm)) ? 1 : 0;
  }
  __device__ __forceinline__ void write(int64_t v, int64_t excl, int64_t val) const {
    dir[v].slot = val ? (int32_t)excl : -1;
    if (val) list[excl] = (excl << 32) | v;
  }
};

__global__ void k_copy_prefixes(const int64_t* __restrict__ indptr, const DirEntry* __restrict__ dir, int64_t N,
                                const int32_t* __restrict__ idxR, int32_t* __restrict__ acache) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < N; v += nwarps) {
    const int32_t len = dir[v].cached_len;
    if (len == 0) continue;
    const int64_t off = dir[v].cache_off, base = indptr[v];
    for (int64_t p = lane; p < len; p += 32) acache[off + p] = idxR[base + p];
  }
}

__global__ void k_copy_rows_from_host(const int64_t* __restrict__ list, int64_t n, const float* __restrict__ src,
                                      int32_t pitch, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int row16 = pitch >> 2;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t ent = list[r];
    const int64_t slot = ent >> 32, v = ent & 0xffffffffll;
    const int4* s = reinterpret_cast<const int4*>(src + v * pitch);
    int4* d = reinterpret_cast<int4*>(dst + slot * pitch);
    for (int c = lane; c < row16; c += 32) d[c] = s[c];
  }
}

// Copy admitted rows host -> this device's partition(s).  Global slot s belongs to partition
// s % G at row s / G; rank >= 0 copies only its own partition's rows, rank = -1 (emulation)
// copies every partition into one buffer laid out partition by partition.
__global__ void k_copy_rows_partitioned(const int64_t* __restrict__ list, int64_t n, const float* __restrict__ src,
                                        int32_t pitch, float* __restrict__ dst, int32_t G, int32_t rank) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int row16 = pitch >> 2;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t ent = list[r];
    const int64_t slot = ent >> 32, v = ent & 0xffffffffll;
    const int32_t part = (int32_t)(slot % G);
    if (rank >= 0 && part != rank) continue;
    int64_t row = slot / G;
    if (rank < 0)
      for (int32_t q = 0; q < part; ++q) row += (n - q + G - 1) / G;  // rows of earlier partitions
    const int4* sp = reinterpret_cast<const int4*>(src + v * pitch);
    int4* dp = reinterpret_cast<int4*>(dst + row * pitch);
    for (int c = lane; c < row16; c += 32) dp[c] = sp[c];
  }
}

// ---- knapsack fill (NEXT F4) helpers ----
// histogram of small non-negative integers: block-private in shared memory when the value
// range fits (few bins receive millions of increments), merged with one atomic per bin
constexpr int kSmemBins = 4096;
__global__ void k_hist_i32(const int32_t* __restrict__ a, int64_t n, int32_t nbins, unsigned long long* hist) {
  __shared__ unsigned int sh[kSmemBins];
  const bool priv = nbins <= kSmemBins;
  if (priv)
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (priv)
      atomicAdd(&sh[a[i]], 1u);
    else
      atomicAdd(hist + a[i], 1ull);
  }
  __syncthreads();
  if (priv)
    for (int b = threadIdx.x; b < nbins; b += blockDim.x)
      if (sh[b]) atomicAdd(hist + b, (unsigned long long)sh[b]);
}

// per node: gt = #elements with count > cv, ties = #elements with count == cv
__global__ void k_node_level_counts(const int64_t* __restrict__ indptr, const int32_t* __restrict__ cnt, int64_t N,
                                    int32_t cv, int32_t* gt, int32_t* ties) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < N; v += nwarps) {
    int32_t g = 0, t = 0;
    for (int64_t e = indptr[v] + lane; e < indptr[v + 1]; e += 32) {
      const int32_t c = cnt[e];
      g += c > cv;
      t += c == cv;
    }
    g = __reduce_add_sync(0xffffffffu, g);
    t = __reduce_add_sync(0xffffffffu, t);
    if (lane == 0) {
      gt[v] = g;
      ties[v] = t;
    }
  }
}

__global__ void k_dir_reset_caches(DirEntry* dir, int64_t N) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    dir[v].cached_len = 0;
    dir[v].cache_off = 0;
    dir[v].slot = -1;
  }
}

template <class Op>
dci_status scan_nodes(dci_ctx* ctx, const Op& op, int64_t n, int64_t* d_total, cudaStream_t s) {
  const int64_t nb = (n + kScanChunk - 1) / kScanChunk;
  int64_t* sums = nullptr;
  DCI_CUDA(cudaMallocAsync(&sums, sizeof(int64_t) * (size_t)std::max<int64_t>(nb, 1), s));
  k_chunk_sum<<<(unsigned)nb, kScanB, 0, s>>>(op, n, sums);
  k_scan_sums<<<1, 1024, 0, s>>>(sums, nb, d_total);
  k_chunk_scan_write<<<(unsigned)nb, kScanB, 0, s>>>(op, n, sums);
  ctx->launches += 3;
  DCI_CUDA(cudaGetLastError());
  DCI_CUDA(cudaFreeAsync(sums, s));
  return DCI_OK;
}

template <class K>
dci_status radix_select(dci_ctx* ctx, const K& kf, int64_t N, unsigned long long target, RSState* d_st,
                        cudaStream_t s) {
  DCI_CUDA(cudaMemsetAsync(d_st, 0, sizeof(RSState), s));
  DCI_CUDA(cudaMemcpyAsync(&d_st->target, &target, sizeof(target), cudaMemcpyHostToDevice, s));
  for (int pass = 0; pass < 8; ++pass) {
    k_rs_hist<K><<<grid_for(ctx, 4), 256, 0, s>>>(kf, N, pass, d_st);
    k_rs_select<<<1, 32, 0, s>>>(pass, d_st);
    ctx->launches += 2;
  }
  DCI_CUDA(cudaGetLastError());
  return DCI_OK;
}

}  // namespace

void launch_build_directory(dci_ctx* ctx, const int64_t* d_indptr, cudaStream_t s) {
  k_build_directory<<<grid_for(ctx, 4), 256, 0, s>>>(d_indptr, ctx->N, ctx->d_dir);
  ++ctx->launches;
}

// Device temporaries of one fill: freed on every exit path.
struct TempAllocs {
  std::vector<void*> ptrs;
  template <class T>
  cudaError_t alloc(T** p, size_t bytes) {
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  void forget(const void* p) {  // ownership moved elsewhere
    for (auto& q : ptrs)
      if (q == p) q = nullptr;
  }
  ~TempAllocs() {
    for (void* q : ptrs)
      if (q) cudaFree(q);
  }
};

void release_feature_partitions(dci_ctx* ctx) {
  for (int p = 0; p < dci_ctx::kMaxParts; ++p) {
    if (ctx->ipc_opened[p]) cudaIpcCloseMemHandle(ctx->ipc_opened[p]);
    ctx->ipc_opened[p] = nullptr;
    ctx->h_fbases[p] = nullptr;
  }
}

// Host walk of the knapsack's density levels (O-14 order: density desc, feature before
// adjacency on ties, ids ascending inside a level), admitting whole levels while they fit.
// Result: features {visits > fv} + the first fm (by id) with visits == fv; adjacency
// {count > cv} + the first cm (by CSC position) with count == cv.  fv = -1 / cv = -1: all.
void knapsack_levels(const std::vector<unsigned long long>& hf, const std::vector<unsigned long long>& ha,
                     uint64_t C, int64_t R, double cf, double ca, int32_t* fv, int64_t* fm, int32_t* cv,
                     int64_t* cm, uint64_t* used) {
  int vi = (int)hf.size() - 1, ci = (int)ha.size() - 1;
  uint64_t left = C;
  bool fclosed = false, done = false;
  *fv = -1;
  *fm = 0;
  *cv = -1;
  *cm = 0;
  while (!done && (vi >= 0 || ci >= 0)) {
    const double df = vi >= 0 ? (double)vi * cf / (double)R : -1.0;
    const double da = ci >= 0 ? (double)ci * ca / 4.0 : -1.0;
    if (vi >= 0 && df >= da) {  // feature level (first on ties)
      if (!fclosed) {
        const unsigned long long need = hf[vi] * (unsigned long long)R;
        if (need <= left) {
          left -= need;
        } else {
          const int64_t m = (int64_t)(left / (uint64_t)R);
          left -= (uint64_t)m * (uint64_t)R;
          *fv = vi;
          *fm = m;
          fclosed = true;
        }
      }
      --vi;
    } else {
      const unsigned long long need = ha[ci] * 4ull;
      if (need <= left) {
        left -= need;
      } else {
        const int64_t m = (int64_t)(left / 4);
        left -= (uint64_t)m * 4;
        *cv = ci;
        *cm = m;
        done = true;  // fewer than 4 bytes left: nothing else fits
        if (!fclosed) {
          *fv = vi;  // lower feature levels were never reached
          *fm = 0;
        }
      }
      --ci;
    }
  }
  *used = C - left;
}

// Upper bound of the device temporaries one fill holds at its peak, next to the new caches
// (indptr + node totals + rank/list/tie arrays: <= 48 B per node; the original and reordered
// CSC copies: 8 B per element, plus 16 B per element of radix ping-pong when counts exceed 255).
// The auto budget (dci_allocate with C = 0) keeps this much free.
uint64_t fill_temp_bound(int64_t N, int64_t E) {
  return 48ull * (uint64_t)(N + 1) + 24ull * (uint64_t)E + (1ull << 20);
}

void release_presample(dci_ctx* ctx) {
  // presample is not allowed after a fill (DCI_ESTATE), so its workspace and outputs are freed
  // here: the auto budget counted their memory as available to the caches
  if (ctx->pre_ws) dci_workspace_destroy(ctx->pre_ws);
  ctx->pre_ws = nullptr;
  if (ctx->pre_out_mem) cudaFree(ctx->pre_out_mem);
  ctx->pre_out_mem = nullptr;
}

// CUDA events at the fill's stage boundaries (dci_fill_times): recorded on the fill stream, read
// once the fill has synchronised; destroyed on every exit path.
struct FillClock {
  cudaEvent_t e[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaStream_t s;
  explicit FillClock(cudaStream_t st) : s(st) {
    for (auto& x : e) cudaEventCreate(&x);
  }
  void mark(int i) {
    if (e[i]) cudaEventRecord(e[i], s);
  }
  float ms(int a, int b) const {
    float t = 0.f;
    return (e[a] && e[b] && cudaEventElapsedTime(&t, e[a], e[b]) == cudaSuccess) ? t : -1.f;
  }
  ~FillClock() {
    for (auto& x : e)
      if (x) cudaEventDestroy(x);
  }
};

dci_status fill_impl(dci_ctx* ctx, const int32_t* node_visits, const int32_t* edge_counts, uint64_t c_adj,
                     uint64_t c_feat, int32_t world, int32_t rank, cudaStream_t s, const KnapsackPlan* knap) {
  const int64_t N = ctx->N, E = ctx->E;
  release_presample(ctx);
  for (auto& t : ctx->fill_ms) t = -1.f;
  FillClock clk(s);
  clk.mark(0);
  const int64_t row_bytes = 4ll * ctx->pitch;
  // c_feat is the budget of ONE partition; the admitted set spans all `world` partitions
  const int64_t cap_part = (int64_t)std::min<uint64_t>((uint64_t)N, c_feat / (uint64_t)row_bytes);
  const int64_t cap_rows = std::min<int64_t>(N, cap_part * (int64_t)world);
  const uint64_t cap_e_raw = c_adj / 4;
  const bool whole_fit = (uint64_t)E <= cap_e_raw;
  const int64_t cap_e = whole_fit ? E : (int64_t)cap_e_raw;

  int64_t *d_indptr = nullptr, *d_total = nullptr, *d_sum = nullptr;
  int32_t *d_idx = nullptr, *d_idxR = nullptr, *d_scal = nullptr;
  RSState* d_st = nullptr;
  TempAllocs tmp;
  // If the fill stops part-way, leave a consistent "no cache" state behind.
  struct Rollback {
    dci_ctx* ctx;
    cudaStream_t s;
    bool armed = false, committed = false;
    ~Rollback() {
      if (!armed || committed) return;
      cudaStreamSynchronize(s);
      if (ctx->d_acache) cudaFree(ctx->d_acache);
      if (ctx->d_fcache) cudaFree(ctx->d_fcache);
      release_feature_partitions(ctx);
      ctx->d_acache = nullptr;
      ctx->d_fcache = nullptr;
      ctx->acache_len = ctx->fcache_rows = ctx->fcache_total_rows = 0;
      ctx->fpart_world = 1;
      ctx->fpart_rank = 0;
      k_dir_reset_caches<<<grid_for(ctx, 4), 256, 0, s>>>(ctx->d_dir, ctx->N);
      cudaStreamSynchronize(s);
    }
  } rollback{ctx, s};
  DCI_CUDA(tmp.alloc(&d_indptr, sizeof(int64_t) * (N + 1)));
  DCI_CUDA(tmp.alloc(&d_total, sizeof(int64_t) * std::max<int64_t>(N, 1)));
  DCI_CUDA(tmp.alloc(&d_sum, sizeof(int64_t)));
  DCI_CUDA(tmp.alloc(&d_idx, sizeof(int32_t) * std::max<int64_t>(E, 1)));
  DCI_CUDA(tmp.alloc(&d_idxR, sizeof(int32_t) * std::max<int64_t>(E, 1)));
  DCI_CUDA(tmp.alloc(&d_scal, sizeof(int32_t) * 4));
  DCI_CUDA(tmp.alloc(&d_st, sizeof(RSState)));
  DCI_CUDA(cudaMemcpyAsync(d_indptr, ctx->h_indptr, sizeof(int64_t) * (N + 1), cudaMemcpyHostToDevice, s));
  if (E) DCI_CUDA(cudaMemcpyAsync(d_idx, ctx->h_idx_orig, sizeof(int32_t) * E, cudaMemcpyHostToDevice, s));
  DCI_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(int32_t) * 4, s));

  // ---- level 2: per-node stable reorder by count desc (always applied, reading C17) ----
  if (E) {
    k_max_i32<<<grid_for(ctx, 4), 256, 0, s>>>(edge_counts, E, d_scal);
    ++ctx->launches;
  }
  int32_t h_scal[4] = {0, 0, 0, 0};
  DCI_CUDA(cudaMemcpyAsync(h_scal, d_scal, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost, s));
  DCI_CUDA(cudaStreamSynchronize(s));
  const int32_t cmax = h_scal[0];
  int npass = 1;
  while (npass < 4 && ((uint64_t)cmax >> (8 * npass)) != 0) ++npass;
  Level2Args l2{};
  l2.indptr = d_indptr;
  l2.N = N;
  l2.idx_in = d_idx;
  l2.cnt = edge_counts;
  l2.cmax = cmax;
  l2.npass = npass;
  l2.idx_out = d_idxR;
  l2.total = d_total;
  l2.range_err = d_scal + 1;
  if (npass > 1) {
    for (int i = 0; i < 2; ++i) {
      DCI_CUDA(tmp.alloc(&l2.tmp_idx[i], sizeof(int32_t) * E));
      DCI_CUDA(tmp.alloc(&l2.tmp_key[i], sizeof(uint32_t) * E));
    }
  }
  k_level2<<<grid_for(ctx, 8), 32 * kL2Warps, 0, s>>>(l2);
  ++ctx->launches;
  DCI_CUDA(cudaGetLastError());
  DCI_CUDA(cudaMemcpyAsync(h_scal, d_scal, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost, s));
  DCI_CUDA(cudaStreamSynchronize(s));
  if (h_scal[1]) return fail(DCI_ERANGE, "dci_fill: a node's total access count is >= 2^32");

  // reordered host CSC (pinned + mapped), separate from the original so refills restart
  // from the original order (idempotence)
  if (ctx->h_idx_cur == ctx->h_idx_orig) {
    int32_t* hb = nullptr;
    DCI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hb), sizeof(int32_t) * std::max<int64_t>(E, 1),
                           cudaHostAllocMapped | cudaHostAllocPortable));
    void* dp = nullptr;
    DCI_CUDA(cudaHostGetDevicePointer(&dp, hb, 0));
    ctx->h_idx_cur = hb;
    ctx->u_idx_cur = static_cast<const int32_t*>(dp);
  }
  if (E) DCI_CUDA(cudaMemcpyAsync(ctx->h_idx_cur, d_idxR, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
  clk.mark(1);  // level 2 done: reordered CSC on the host

  // ---- drop old caches, reset the directory's cache fields ----
  DCI_CUDA(cudaStreamSynchronize(s));
  rollback.armed = true;
  if (ctx->d_acache) cudaFree(ctx->d_acache);
  if (ctx->d_fcache) cudaFree(ctx->d_fcache);
  release_feature_partitions(ctx);
  ctx->d_acache = nullptr;
  ctx->d_fcache = nullptr;
  ctx->acache_len = 0;
  ctx->fcache_rows = 0;
  ctx->fcache_total_rows = 0;
  ctx->fpart_world = world;
  ctx->fpart_rank = rank;
  k_dir_reset_caches<<<grid_for(ctx, 4), 256, 0, s>>>(ctx->d_dir, N);
  ++ctx->launches;

  if (knap) {
    // ---- NEXT F4: unified-budget knapsack over feature rows and adjacency elements ----
    int32_t vmax = 0;
    DCI_CUDA(cudaMemsetAsync(d_scal, 0, sizeof(int32_t) * 4, s));
    k_max_i32<<<grid_for(ctx, 4), 256, 0, s>>>(node_visits, N, d_scal);
    ++ctx->launches;
    DCI_CUDA(cudaMemcpyAsync(&vmax, d_scal, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaStreamSynchronize(s));
    if (vmax > (1 << 20) || cmax > (1 << 20)) return fail(DCI_ERANGE, "knapsack fill: counts above 2^20");
    unsigned long long *d_hf = nullptr, *d_ha = nullptr;
    DCI_CUDA(tmp.alloc(&d_hf, sizeof(unsigned long long) * (vmax + 1)));
    DCI_CUDA(tmp.alloc(&d_ha, sizeof(unsigned long long) * (cmax + 1)));
    DCI_CUDA(cudaMemsetAsync(d_hf, 0, sizeof(unsigned long long) * (vmax + 1), s));
    DCI_CUDA(cudaMemsetAsync(d_ha, 0, sizeof(unsigned long long) * (cmax + 1), s));
    k_hist_i32<<<grid_for(ctx, 4), 256, 0, s>>>(node_visits, N, vmax + 1, d_hf);
    if (E) k_hist_i32<<<grid_for(ctx, 4), 256, 0, s>>>(edge_counts, E, cmax + 1, d_ha);
    ctx->launches += E ? 2 : 1;
    std::vector<unsigned long long> hf(vmax + 1), ha(cmax + 1);
    DCI_CUDA(cudaMemcpyAsync(hf.data(), d_hf, sizeof(unsigned long long) * (vmax + 1), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaMemcpyAsync(ha.data(), d_ha, sizeof(unsigned long long) * (cmax + 1), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaStreamSynchronize(s));
    if (!E) ha.assign(1, 0ull);
    int32_t fv, cv;
    int64_t fm, cm;
    uint64_t used;
    knapsack_levels(hf, ha, knap->C, row_bytes, knap->cost_feat, knap->cost_adj, &fv, &fm, &cv, &cm, &used);
    // adjacency: per-node counts above / at the cut level, ties before each node
    int32_t *d_gt = nullptr, *d_ties = nullptr;
    int64_t* d_tb = nullptr;
    DCI_CUDA(tmp.alloc(&d_gt, sizeof(int32_t) * std::max<int64_t>(N, 1)));
    DCI_CUDA(tmp.alloc(&d_ties, sizeof(int32_t) * std::max<int64_t>(N, 1)));
    DCI_CUDA(tmp.alloc(&d_tb, sizeof(int64_t) * std::max<int64_t>(N, 1)));
    k_node_level_counts<<<grid_for(ctx, 8), 256, 0, s>>>(d_indptr, edge_counts, N, cv, d_gt, d_ties);
    ++ctx->launches;
    dci_status r = scan_nodes(ctx, TieScanOp{d_ties, d_tb}, N, d_sum, s);
    if (r != DCI_OK) return r;
    r = scan_nodes(ctx, KnapAdjOp{d_gt, d_ties, d_tb, cv < 0 ? 0 : cm, ctx->d_dir}, N, d_sum, s);
    if (r != DCI_OK) return r;
    int64_t adj_elems = 0;
    DCI_CUDA(cudaMemcpyAsync(&adj_elems, d_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaStreamSynchronize(s));
    if (adj_elems > 0) {
      DCI_CUDA(cudaMalloc(&ctx->d_acache, sizeof(int32_t) * adj_elems));
      k_copy_prefixes<<<grid_for(ctx, 8), 256, 0, s>>>(d_indptr, ctx->d_dir, N, d_idxR, ctx->d_acache);
      ++ctx->launches;
    }
    ctx->acache_len = adj_elems;
    // features: tie ranks at the cut level, then admission + slots in ascending id
    int64_t* d_rank = nullptr;
    DCI_CUDA(tmp.alloc(&d_rank, sizeof(int64_t) * std::max<int64_t>(N, 1)));
    r = scan_nodes(ctx, FeatTieOp{node_visits, fv, d_rank}, N, d_sum, s);
    if (r != DCI_OK) return r;
    int64_t* d_list = nullptr;
    DCI_CUDA(tmp.alloc(&d_list, sizeof(int64_t) * std::max<int64_t>(N, 1)));
    r = scan_nodes(ctx, KnapFeatOp{node_visits, fv, fm, d_rank, ctx->d_dir, d_list}, N, d_sum, s);
    if (r != DCI_OK) return r;
    int64_t rows = 0;
    DCI_CUDA(cudaMemcpyAsync(&rows, d_sum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    DCI_CUDA(cudaStreamSynchronize(s));
    DCI_CUDA(cudaMalloc(&ctx->d_fcache, (size_t)row_bytes * std::max<int64_t>(rows, 1)));
    if (rows > 0) {
      k_copy_rows_from_host<<<grid_for(ctx, 8), 256, 0, s>>>(d_list, rows, ctx->u_feats, ctx->pitch,
                                                              ctx->d_fcache);
      ++ctx->launches;
    }
    ctx->fcache_rows = ctx->fcache_total_rows = rows;
    ctx->h_fbases[0] = ctx->d_fcache;
    if (!ctx->d_fbases) DCI_CUDA(cudaMalloc(&ctx->d_fbases, sizeof(float*) * dci_ctx::kMaxParts));
    DCI_CUDA(cudaMemcpyAsync(ctx->d_fbases, ctx->h_fbases, sizeof(float*) * dci_ctx::kMaxParts,
                             cudaMemcpyHostToDevice, s));
    DCI_CUDA(cudaGetLastError());
    DCI_CUDA(cudaStreamSynchronize(s));
    rollback.committed = true;
    clk.mark(5);
    ctx->fill_ms[0] = clk.ms(0, 1);
    ctx->fill_ms[5] = clk.ms(0, 5);
    ctx->whole_fit = adj_elems == E ? 1 : 0;
    ctx->c_adj = (uint64_t)adj_elems * 4;
    ctx->c_feat = (uint64_t)rows * (uint64_t)row_bytes;
    ctx->state = DCI_STATE_FILLED;
    return DCI_OK;
  }

  // ---- adjacency cache (Algorithm 1) ----
  AdjKey ak{d_total, d_indptr};
  if (cap_e > 0) {
    const RSState* stp = nullptr;
    if (!whole_fit) {
      dci_status r = radix_select(ctx, ak, N, (unsigned long long)cap_e, d_st, s);
      if (r != DCI_OK) return r;
      stp = d_st;
    }
    AdjLenOp op{ak, stp, (unsigned long long)cap_e, ctx->d_dir};
    dci_status r = scan_nodes(ctx, op, N, d_sum, s);
    if (r != DCI_OK) return r;
    clk.mark(2);
    if (whole_fit) {
      ctx->d_acache = d_idxR;  // the whole reordered CSC, cache_off == indptr
      tmp.forget(d_idxR);
      d_idxR = nullptr;
    } else {
      DCI_CUDA(cudaMalloc(&ctx->d_acache, sizeof(int32_t) * cap_e));
      k_copy_prefixes<<<grid_for(ctx, 8), 256, 0, s>>>(d_indptr, ctx->d_dir, N, d_idxR, ctx->d_acache);
      ++ctx->launches;
    }
    ctx->acache_len = cap_e;
  } else {
    clk.mark(2);
  }
  clk.mark(3);

  // ---- feature cache ----
  if (cap_rows > 0) {
    FeatKey fk{node_visits};
    const RSState* stp = nullptr;
    if (cap_rows < N) {
      dci_status r = radix_select(ctx, fk, N, (unsigned long long)cap_rows, d_st, s);
      if (r != DCI_OK) return r;
      stp = d_st;
    }
    int64_t* d_list = nullptr;
    DCI_CUDA(tmp.alloc(&d_list, sizeof(int64_t) * cap_rows));
    FeatSlotOp op{fk, stp, ctx->d_dir, d_list};
    dci_status r = scan_nodes(ctx, op, N, d_sum, s);
    if (r != DCI_OK) return r;
    clk.mark(4);
    // rows held on this device: all of them (world 1 or emulation), else this rank's share
    const int64_t local_rows = rank < 0 || world == 1 ? cap_rows : (cap_rows - rank + world - 1) / world;
    DCI_CUDA(cudaMalloc(&ctx->d_fcache, (size_t)row_bytes * std::max<int64_t>(local_rows, 1)));
    if (world == 1) {
      k_copy_rows_from_host<<<grid_for(ctx, 8), 256, 0, s>>>(d_list, cap_rows, ctx->u_feats, ctx->pitch,
                                                              ctx->d_fcache);
    } else {
      k_copy_rows_partitioned<<<grid_for(ctx, 8), 256, 0, s>>>(d_list, cap_rows, ctx->u_feats, ctx->pitch,
                                                                ctx->d_fcache, world, rank);
    }
    ++ctx->launches;
    DCI_CUDA(cudaStreamSynchronize(s));
    ctx->fcache_rows = local_rows;
    ctx->fcache_total_rows = cap_rows;
  } else {
    clk.mark(4);
  }
  // partition base pointers (peers are attached later through dci_attach_feature_partitions)
  int64_t off = 0;
  for (int p = 0; p < world; ++p) {
    const int64_t rows_p = (cap_rows - p + world - 1) / world;
    if (rank < 0)
      ctx->h_fbases[p] = ctx->d_fcache + off * ctx->pitch;
    else if (p == rank)
      ctx->h_fbases[p] = ctx->d_fcache;
    off += rows_p;
  }
  if (world == 1) ctx->h_fbases[0] = ctx->d_fcache;
  if (!ctx->d_fbases) DCI_CUDA(cudaMalloc(&ctx->d_fbases, sizeof(float*) * dci_ctx::kMaxParts));
  DCI_CUDA(cudaMemcpyAsync(ctx->d_fbases, ctx->h_fbases, sizeof(float*) * dci_ctx::kMaxParts,
                           cudaMemcpyHostToDevice, s));
  clk.mark(5);
  DCI_CUDA(cudaGetLastError());
  DCI_CUDA(cudaStreamSynchronize(s));
  rollback.committed = true;
  for (int i = 0; i < 5; ++i) ctx->fill_ms[i] = clk.ms(i, i + 1);
  ctx->fill_ms[5] = clk.ms(0, 5);
  ctx->whole_fit = whole_fit ? 1 : 0;
  ctx->c_adj = c_adj;
  ctx->c_feat = c_feat;
  ctx->state = DCI_STATE_FILLED;
  return DCI_OK;
}

}  // namespace dci
