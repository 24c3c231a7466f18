// Probe: the host link's random-read REQUEST rate (zero-copy UVA reads of pinned host memory) by
// access size and by pinned-region size, with enough reads in flight to saturate the link.
// Round 1's uva_rand4 probe kept one 4-byte read in flight per thread and measured 94 M reads/s;
// the sampler's adjacency misses reach far more (ncu: ~0.5 G sysmem requests/s on M4s's last hop),
// so that figure was a latency bound, not the link's.  Here every thread (S <= 32) or every group
// of S/16 lanes (S >= 64) keeps U = 8 independent reads in flight.
//
//   hostreq_probe [max_region_GB=64] > profiles/hostreq_probe.jsonl
//
// Every request of a launch goes to a DISTINCT S-byte slot (a bijective hash of its index over the
// power-of-two slot count, with at most half the slots touched), so no read is served by L2, and
// loads are the library's miss-path loads (ld.global.nc.L1::no_allocate).
// Output: one JSON line per (region, size): Mreq_per_s and payload GB/s (req x size / time).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include <algorithm>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)

// bijection of [0, 2^bits): odd multiplies and xorshifts, masked
__device__ __forceinline__ uint64_t perm(uint64_t x, int bits) {
  const uint64_t m = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  x = (x * 0x9E3779B97F4A7C15ull) & m;
  x ^= x >> (bits / 2 + 1);
  x = (x * 0xBF58476D1CE4E5B9ull) & m;
  x ^= x >> (bits / 2 + 1);
  return x & m;
}

// load kinds: 0 = ld.global.nc.L1::no_allocate (round 1's miss-path load), 1 = plain ld.global
// (L1-allocating; the library's miss-path load since round 2), 2 = ld.global.L1::no_allocate
// (coherent), 3 = ld.global.nc (read-only path, L1-allocating); plus TMA bulk copies ("bulk")
__device__ int g_kind_dummy;
template <int KIND>
__device__ __forceinline__ int ld32(const int* p) {
  int v;
  if (KIND == 0)
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (KIND == 1)
    asm volatile("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  else if (KIND == 3)
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <int KIND>
__device__ __forceinline__ int4 ld128(const int4* p) {
  int4 v;
  if (KIND == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 1)
    asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (KIND == 3)
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// S-byte random reads (S in {4, 16, 32}), one thread per read, U reads in flight per thread
template <int S, int U, int KIND>
__global__ void rand_small(const char* __restrict__ src, int bits, int iters, int* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    int v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t slot = perm(((uint64_t)(it * U + u)) * nthr + t, bits);
      const char* p = src + slot * S;
      if (S == 4) {
        v[u] = ld32<KIND>(reinterpret_cast<const int*>(p));
      } else if (S == 16) {
        const int4 x = ld128<KIND>(reinterpret_cast<const int4*>(p));
        v[u] = x.x ^ x.w;
      } else {  // 32: two 16-byte halves of one sector
        const int4 x = ld128<KIND>(reinterpret_cast<const int4*>(p));
        const int4 y = ld128<KIND>(reinterpret_cast<const int4*>(p) + 1);
        v[u] = x.x ^ y.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// S-byte random reads (S >= 64, multiple of 16) by groups of L = min(32, S/16) lanes, each lane
// reading S/(16 L) int4 of the request; U requests in flight per group
template <int S, int U, int KIND>
__global__ void rand_wide(const char* __restrict__ src, int bits, int iters, int* sink) {
  constexpr int L = (S / 16) < 32 ? (S / 16) : 32;
  constexpr int PER = S / 16 / L;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngrp = (uint64_t)gridDim.x * blockDim.x / L;
  const uint64_t grp = t / L;
  const int gl = (int)(t % L);
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    int v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t slot = perm(((uint64_t)(it * U + u)) * ngrp + grp, bits);
      const int4* p = reinterpret_cast<const int4*>(src + slot * S) + gl;
      v[u] = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int4 x = ld128<KIND>(p + k * L);
        v[u] ^= x.x ^ x.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678) sink[0] = acc;
}


// S-byte random reads by TMA bulk copies (cp.async.bulk global -> shared, mbarrier completion):
// lane 0 of each warp keeps U requests in flight in a U-slot ring (the row-mode group gather's
// miss path reads host rows this way)
template <int S, int U>
__global__ void rand_bulk(const char* __restrict__ src, int bits, int iters, int* sink) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) unsigned long long bar[8][U];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned char* mine = ring + (size_t)wib * U * S;
  if (lane == 0) {
    for (int u = 0; u < U; ++u)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[wib][u])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  int acc = 0;
  if (lane == 0) {
    const int total = iters * U;
    auto issue = [&](int k) {
      const int u = k % U;
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[wib][u]);
      const uint64_t slot = perm((uint64_t)k * nw + gw, bits);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(S) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(mine + (size_t)u * S)),
                   "l"(src + slot * S), "r"(S), "r"(b)
                   : "memory");
    };
    for (int k = 0; k < U && k < total; ++k) issue(k);
    for (int k = 0; k < total; ++k) {
      const int u = k % U;
      const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[wib][u]);
      const uint32_t par = (uint32_t)((k / U) & 1);
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(b),
                   "r"(par)
                   : "memory");
      acc ^= mine[(size_t)u * S];
      if (k + U < total) issue(k + U);
    }
  }
  if (acc == 0x12345678) sink[0] = acc;
}


// Mixed pattern (512-B rows, plain loads): a fraction hot_pct/100 of the requests go to the first
// 2^hot_bits slots (a compact "warm" sub-region), the rest to the whole region -- does a warm
// sub-region keep its translations while the rest of the requests thrash the TLB?
__global__ void rand_mixed512(const char* __restrict__ src, int bits, int hot_bits, int hot_pct, int iters, int* sink) {
  constexpr int S = 512, L = 32, U = 8;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngrp = (uint64_t)gridDim.x * blockDim.x / L;
  const uint64_t grp = t / L;
  const int gl = (int)(t % L);
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    int v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t idx = ((uint64_t)(it * U + u)) * ngrp + grp;
      const bool hot = (perm(idx ^ 0x5bd1e995ull, 20) % 100) < (uint64_t)hot_pct;
      const uint64_t slot = hot ? perm(idx, hot_bits) : perm(idx, bits);
      const int4 x = ld128<1>(reinterpret_cast<const int4*>(src + slot * S) + gl);
      v[u] = x.x ^ x.w;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int S, int KIND>
static double run(const char* src, size_t region, int* sink, int sms, double* mreq) {
  int bits = 0;
  while ((2ull << bits) <= region / S) ++bits;  // 2^bits slots of S bytes
  const int threads = 256;
  const int grid = sms * 8;
  constexpr int U = 8;
  const int per_group = S <= 32 ? 1 : ((S / 16) < 32 ? (S / 16) : 32);
  const double per_iter = (double)grid * threads / per_group * U;
  // at most half of the slots and ~16 M requests per launch
  int iters = (int)std::min(16.0, std::max(1.0, std::min((double)(1ull << bits) / 2, 16.0e6) / per_iter));
  const double nreq = per_iter * iters;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto launch = [&]() {
    if constexpr (S <= 32)
      rand_small<S, U, KIND><<<grid, threads>>>(src, bits, iters, sink);
    else
      rand_wide<S, U, KIND><<<grid, threads>>>(src, bits, iters, sink);
  };
  launch();  // warm-up (page-table walks of a fresh region)
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  *mreq = nreq / best / 1e3;
  return nreq * S / best / 1e6;  // payload GB/s
}


template <int S>
static double run_bulk_probe(const char* src, size_t region, int* sink, int sms, double* mreq) {
  int bits = 0;
  while ((2ull << bits) <= region / S) ++bits;
  constexpr int U = 8;
  const int warps = 8, grid = sms * 2;
  const size_t smem = (size_t)warps * U * S;
  CK(cudaFuncSetAttribute(rand_bulk<S, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const double per_iter = (double)grid * warps * U;
  const int iters = (int)std::min(64.0, std::max(1.0, std::min((double)(1ull << bits) / 2, 8.0e6) / per_iter));
  const double nreq = per_iter * iters;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  rand_bulk<S, U><<<grid, 32 * warps, smem>>>(src, bits, iters, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    rand_bulk<S, U><<<grid, 32 * warps, smem>>>(src, bits, iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  *mreq = nreq / best / 1e3;
  return nreq * S / best / 1e6;
}

int main(int argc, char** argv) {
  const double max_gb = argc > 1 ? atof(argv[1]) : 64.0;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = (size_t)(max_gb * (1ull << 30));
  void* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes; i += 4096) static_cast<char*>(h)[i] = (char)i;
  void* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  int* sink;
  CK(cudaMalloc(&sink, 64));
  const double regions[] = {0.5, 1, 2, 8, 32, 64};
  const bool mixed_only = argc > 2 && argv[2][0] == 'm';
  for (double gb : regions) {
    if (gb > max_gb || mixed_only) break;
    const size_t region = (size_t)(gb * (1ull << 30));
    const char* src = static_cast<const char*>(hd);
    double m, g;
#define ONEK(S, K)                                                                                          \
  g = run<S, K>(src, region, sink, sms, &m);                                                               \
  printf("{\"probe\":\"host_random_read\",\"region_GB\":%.1f,\"bytes\":%d,\"load\":\"%s\",\"Mreq_per_s\":%.1f," \
         "\"GBps\":%.2f}\n",                                                                                    \
         gb, S, K == 0 ? "nc.L1::no_allocate" : K == 1 ? "default" : K == 2 ? "L1::no_allocate" : "nc", m, g);                \
  fflush(stdout);
#define ONE(S) ONEK(S, 0) ONEK(S, 1) ONEK(S, 2) ONEK(S, 3)
    ONE(4) ONE(32) ONE(64) ONE(128) ONE(256) ONE(512) ONE(2048)
#define BULK(S)                                                                                                \
  g = run_bulk_probe<S>(src, region, sink, sms, &m);                                                           \
  printf("{\"probe\":\"host_random_read\",\"region_GB\":%.1f,\"bytes\":%d,\"load\":\"bulk\",\"Mreq_per_s\":%.1f," \
         "\"GBps\":%.2f}\n",                                                                                    \
         gb, S, m, g);                                                                                         \
  fflush(stdout);
    BULK(512) BULK(2048)
  }
  // mixed warm / cold pattern over the largest region
  {
    const size_t region = (size_t)(max_gb * (1ull << 30));
    int bits = 0;
    while ((2ull << bits) <= region / 512) ++bits;
    for (double hot_gb : {1.0, 2.0}) {
      int hb = 0;
      while ((2ull << hb) <= (size_t)(hot_gb * (1ull << 30)) / 512) ++hb;
      for (int pct : {0, 30, 50, 100}) {
        const int grid = sms * 8, threads = 256, iters = 4;
        const double nreq = (double)grid * threads / 32 * 8 * iters;
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        rand_mixed512<<<grid, threads>>>(static_cast<const char*>(hd), bits, hb, pct, iters, sink);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
          CK(cudaEventRecord(a));
          rand_mixed512<<<grid, threads>>>(static_cast<const char*>(hd), bits, hb, pct, iters, sink);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (ms < best) best = ms;
        }
        printf("{\"probe\":\"host_mixed_512\",\"region_GB\":%.1f,\"hot_GB\":%.1f,\"hot_pct\":%d,\"Mreq_per_s\":%.1f,"
               "\"GBps\":%.2f}\n", max_gb, hot_gb, pct, nreq / best / 1e3, nreq * 512 / best / 1e6);
        fflush(stdout);
      }
    }
  }
  CK(cudaFreeHost(h));
  return 0;
}
