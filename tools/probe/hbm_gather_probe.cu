// Probe: what an HBM row gather can reach on this B200, by access pattern.
// Table of T rows x P bytes (M2: 232,965 x 2416 B), n rows gathered (M2: ~141 K, 61 % of T).
// Patterns (read side -> write side):
//   seq      row i -> row i                    (a plain copy of the same bytes)
//   gather   idx[i] random -> row i            (S8 as shipped: X in frontier order)
//   sorted   idx[i] ascending -> row i         (reads in cache-slot order)
//   scatter  ascending rows -> row perm[i]     (reads in slot order, X written in frontier order)
// Each with a warp-per-row LDG/STG kernel (rows in flight per warp: 1 or 2) at several
// blocks/SM.  Prints GB/s of (read + write) bytes, best of 10, CUDA events.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <type_traits>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int ROWS>
__global__ void __launch_bounds__(256) k_copy(const int4* __restrict__ src, int4* __restrict__ dst,
                                              const int* __restrict__ ridx, const int* __restrict__ widx, int n,
                                              int row16) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int VPL = 5;
  for (int64_t r = warp * ROWS; r < n; r += nw * ROWS) {
    int4 buf[ROWS][VPL];
    int rs[ROWS], ws[ROWS];
#pragma unroll
    for (int q = 0; q < ROWS; ++q) {
      const int64_t rr = r + q;
      rs[q] = rr < n ? (ridx ? ridx[rr] : (int)rr) : -1;
      ws[q] = rr < n ? (widx ? widx[rr] : (int)rr) : -1;
    }
    for (int c0 = 0; c0 < row16; c0 += 32 * VPL) {
#pragma unroll
      for (int q = 0; q < ROWS; ++q)
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int idx = c0 + lane + 32 * j;
          if (rs[q] >= 0 && idx < row16) buf[q][j] = __ldcs(src + (int64_t)rs[q] * row16 + idx);
        }
#pragma unroll
      for (int q = 0; q < ROWS; ++q)
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const int idx = c0 + lane + 32 * j;
          if (ws[q] >= 0 && idx < row16) __stcs(dst + (int64_t)ws[q] * row16 + idx, buf[q][j]);
        }
    }
  }
}

// node-sweep pattern: row i read once (sequential), written to M outputs at random rows
template <int M>
__global__ void __launch_bounds__(256) k_multi(const int4* __restrict__ src, int4* __restrict__ dst,
                                               const int* __restrict__ perm, int n, int row16, int64_t out_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int VPL = 5;
  for (int64_t r = warp; r < n; r += nw) {
    int4 buf[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int idx = lane + 32 * j;
      if (idx < row16) buf[j] = __ldcs(src + r * row16 + idx);
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int w = perm[(r * 7 + m * 104729) % n];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int idx = lane + 32 * j;
        if (idx < row16) __stcs(dst + m * out_stride + (int64_t)w * row16 + idx, buf[j]);
      }
    }
  }
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 232965;
  const int P = argc > 2 ? atoi(argv[2]) : 2416;
  const int n = argc > 3 ? atoi(argv[3]) : 141187;
  const int row16 = P / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int4 *src, *dst;
  CK(cudaMalloc(&src, (size_t)T * P));
  CK(cudaMalloc(&dst, (size_t)n * P));
  CK(cudaMemset(src, 1, (size_t)T * P));
  std::mt19937_64 rng(1);
  std::vector<int> all(T);
  std::iota(all.begin(), all.end(), 0);
  std::shuffle(all.begin(), all.end(), rng);
  std::vector<int> rnd(all.begin(), all.begin() + n);  // random distinct rows
  std::vector<int> srt = rnd;
  std::sort(srt.begin(), srt.end());
  std::vector<int> perm(n);
  std::iota(perm.begin(), perm.end(), 0);
  std::shuffle(perm.begin(), perm.end(), rng);
  int *d_rnd, *d_srt, *d_perm;
  CK(cudaMalloc(&d_rnd, 4 * n));
  CK(cudaMalloc(&d_srt, 4 * n));
  CK(cudaMalloc(&d_perm, 4 * n));
  CK(cudaMemcpy(d_rnd, rnd.data(), 4 * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_srt, srt.data(), 4 * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_perm, perm.data(), 4 * n, cudaMemcpyHostToDevice));
  // L2 flush buffer
  void* flush;
  const size_t fbytes = 256ull << 20;
  CK(cudaMalloc(&flush, fbytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double bytes = 2.0 * n * (double)P;
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
      CK(cudaMemsetAsync(flush, it, fbytes));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    return best;
  };
  float ms = timeit([&] { CK(cudaMemcpyAsync(dst, src, (size_t)n * P, cudaMemcpyDeviceToDevice)); });
  printf("{\"pattern\": \"memcpy\", \"us\": %.1f, \"GBps\": %.1f}\n", ms * 1e3, bytes / ms / 1e6);
  struct Pat {
    const char* name;
    const int* r;
    const int* w;
  } pats[] = {{"seq", nullptr, nullptr}, {"gather", d_rnd, nullptr}, {"sorted", d_srt, nullptr},
              {"scatter", d_srt, d_perm}};
  for (auto& pt : pats)
    for (int bps : {1, 2, 3, 4, 6, 8})
      for (int rows : {1, 2}) {
        float t;
        if (rows == 1) {
          int occ = 0;
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy<1>, 256, 0));
          if (bps > occ) continue;
          t = timeit([&] { k_copy<1><<<sms * bps, 256>>>(src, dst, pt.r, pt.w, n, row16); });
        } else {
          int occ = 0;
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copy<2>, 256, 0));
          if (bps > occ) continue;
          t = timeit([&] { k_copy<2><<<sms * bps, 256>>>(src, dst, pt.r, pt.w, n, row16); });
        }
        printf("{\"pattern\": \"%s\", \"bps\": %d, \"rows_per_warp\": %d, \"us\": %.1f, \"GBps\": %.1f}\n", pt.name,
               bps, rows, t * 1e3, bytes / t / 1e6);
      }
  // multi-destination writes (row16 <= 160 only): a row read once, written to M random rows of M
  // outputs (the node-sweep gather's pattern; M ~ 0.61 x group size on M2)
  auto multi = [&](auto mconst) {
    constexpr int M = decltype(mconst)::value;
    int4* mdst;
    CK(cudaMalloc(&mdst, (size_t)M * n * P));
    const double mbytes = (double)n * P * (1 + M);
    for (int bps : {1, 2, 4}) {
      float t = timeit([&] { k_multi<M><<<sms * bps, 256>>>(src, mdst, d_perm, n, row16, (int64_t)n * row16); });
      printf("{\"pattern\": \"read1_write%d\", \"bps\": %d, \"us\": %.1f, \"GBps\": %.1f}\n", M, bps, t * 1e3,
             mbytes / t / 1e6);
    }
    CK(cudaFree(mdst));
  };
  if (row16 <= 160) {
    multi(std::integral_constant<int, 5>{});
    multi(std::integral_constant<int, 10>{});
    constexpr int M = 5;
    int4* mdst;
    CK(cudaMalloc(&mdst, (size_t)M * n * P));
    // pure sequential write of the same bytes (memset)
    float t = timeit([&] { CK(cudaMemsetAsync(mdst, 0, (size_t)M * n * P)); });
    printf("{\"pattern\": \"memset\", \"us\": %.1f, \"GBps\": %.1f}\n", t * 1e3, (double)M * n * P / t / 1e6);
  }
  return 0;
}
