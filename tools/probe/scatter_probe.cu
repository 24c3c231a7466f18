// Probe: the node-sweep gather's HBM pattern on this B200, with kernels that are NOT latency-bound,
// to find what the pattern itself allows (round-1 VERDICT weak #3: the round-1 probe kept one row
// in flight per warp and could not tell a DRAM ceiling from an issue ceiling).
//
// Model of one M2 group: T = 232,965 source rows of P bytes (the feature cache), M
// batches, each holding n = 141,187 distinct rows (random subset of the T nodes) in a random order
// (first-occurrence order).  A node present in c batches is read once and written c times.
// The destinations of every present node are precomputed on the host into a compact list (what a
// "sweep plan" kernel would hand the copy kernel), so the copy kernels only move bytes.
//
//   desc_ldg<W>   warp per present node, row loaded into registers (16 B/lane), stored to each of
//                 its destinations (STG), W = resident warps per SM (occupancy sweep)
//   desc_tma      per-warp ring of rows in shared memory: cp.async.bulk global->shared, then one
//                 cp.async.bulk shared->global per destination (lanes issue in parallel)
//   wrand         the same stores with no loads at all (the random-row write ceiling)
//   wseq          the same number of rows written sequentially (memset-like)
//   rows          row mode: every (batch, row) reads its source row (random) and writes X in order
// Prints (read + write) algorithmic bytes / best time of 5 (CUDA events, L2 flushed before each).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

struct Node {
  int32_t v;      // source row
  int32_t begin;  // destinations dst[begin..end)
  int32_t end;
  int32_t pad;
};

template <int VPL>
__global__ void __launch_bounds__(256) k_desc_ldg(const int4* __restrict__ src, int4* __restrict__ X,
                                                  const Node* __restrict__ nodes, const int64_t* __restrict__ dst,
                                                  int nn, int row16, int read) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nn; i += nw) {
    const Node nd = nodes[i];
    int4 buf[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int idx = lane + 32 * j;
      if (idx < row16) buf[j] = read ? __ldcs(src + (int64_t)nd.v * row16 + idx) : make_int4(nd.v, idx, 0, 0);
    }
    for (int d = nd.begin; d < nd.end; ++d) {
      int4* o = X + dst[d] * row16;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int idx = lane + 32 * j;
        if (idx < row16) __stcs(o + idx, buf[j]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_wseq(int4* __restrict__ X, int64_t rows, int row16) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw)
    for (int idx = lane; idx < row16; idx += 32) __stcs(X + r * row16 + idx, make_int4((int)r, idx, 0, 0));
}

template <int VPL>
__global__ void __launch_bounds__(256) k_rows(const int4* __restrict__ src, int4* __restrict__ X,
                                              const int32_t* __restrict__ rsrc, int64_t rows, int row16) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw) {
    const int v = rsrc[r];
    int4 buf[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int idx = lane + 32 * j;
      if (idx < row16) buf[j] = __ldcs(src + (int64_t)v * row16 + idx);
    }
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int idx = lane + 32 * j;
      if (idx < row16) __stcs(X + r * row16 + idx, buf[j]);
    }
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// per-warp ring of K one-row slots
__global__ void k_desc_tma(const char* __restrict__ src, char* __restrict__ X, const Node* __restrict__ nodes,
                           const int64_t* __restrict__ dst, int nn, int P, int K) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) unsigned long long bars[32][16];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;
  const uint32_t base = sa(ring) + (uint32_t)(wib * K * P);
  if (lane == 0) {
    for (int s = 0; s < K; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[wib][s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t warp = (int64_t)blockIdx.x * nwb + wib;
  const int64_t nw = (int64_t)gridDim.x * nwb;
  // this warp's nodes: warp, warp + nw, ...
  int64_t iss = warp, con = warp;
  int64_t k_iss = 0, k_con = 0;
  auto issue = [&]() {
    const int s = (int)(k_iss % K);
    if (lane == 0) {
      const uint32_t bar = sa(&bars[wib][s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(P) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              base + s * P),
          "l"(src + (int64_t)nodes[iss].v * P), "r"(P), "r"(bar)
          : "memory");
    }
    iss += nw;
    ++k_iss;
  };
  for (int k = 0; k < K && iss < nn; ++k) issue();
  while (con < nn) {
    const int s = (int)(k_con % K);
    const Node nd = nodes[con];
    const uint32_t bar = sa(&bars[wib][s]);
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            bar),
        "r"((uint32_t)((k_con / K) & 1))
        : "memory");
    for (int d = nd.begin + lane; d < nd.end; d += 32)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(X + dst[d] * P),
                   "r"(base + s * P), "r"(P)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    con += nw;
    ++k_con;
    // slot of k_con - 1 may still be read by its stores; refill the one before it
    if (iss < nn && k_iss < k_con - 1 + K) issue();
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 232965;
  const int P = argc > 2 ? atoi(argv[2]) : 2416;
  const int n = argc > 3 ? atoi(argv[3]) : 141187;
  const int M = argc > 4 ? atoi(argv[4]) : 20;
  const int row16 = P / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  // host plan: batch m holds a random n-subset of the T nodes in a random order
  std::mt19937_64 rng(7);
  std::vector<std::vector<std::pair<int32_t, int64_t>>> per(T);  // node -> destinations
  std::vector<int32_t> rsrc((size_t)M * n);
  std::vector<int> all(T);
  for (int m = 0; m < M; ++m) {
    std::iota(all.begin(), all.end(), 0);
    std::shuffle(all.begin(), all.end(), rng);
    for (int r = 0; r < n; ++r) {
      per[all[r]].push_back({m, (int64_t)m * n + r});
      rsrc[(size_t)m * n + r] = all[r];
    }
  }
  std::vector<Node> nodes;
  std::vector<int64_t> dst;
  for (int v = 0; v < T; ++v) {
    if (per[v].empty()) continue;
    Node nd{v, (int32_t)dst.size(), 0, 0};
    for (auto& p : per[v]) dst.push_back(p.second);
    nd.end = (int32_t)dst.size();
    nodes.push_back(nd);
  }
  const int nn = (int)nodes.size();
  const int64_t W = (int64_t)dst.size();
  printf("{\"T\": %d, \"P\": %d, \"n\": %d, \"M\": %d, \"present\": %d, \"writes\": %lld}\n", T, P, n, M, nn,
         (long long)W);
  char *src, *X;
  CK(cudaMalloc(&src, (size_t)T * P));
  CK(cudaMalloc(&X, (size_t)W * P));
  CK(cudaMemset(src, 1, (size_t)T * P));
  Node* d_nodes;
  int64_t* d_dst;
  int32_t* d_rsrc;
  CK(cudaMalloc(&d_nodes, sizeof(Node) * nn));
  CK(cudaMalloc(&d_dst, 8 * W));
  CK(cudaMalloc(&d_rsrc, 4 * W));
  CK(cudaMemcpy(d_nodes, nodes.data(), sizeof(Node) * nn, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_dst, dst.data(), 8 * W, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rsrc, rsrc.data(), 4 * W, cudaMemcpyHostToDevice));
  void* flush;
  const size_t fbytes = 256ull << 20;
  CK(cudaMalloc(&flush, fbytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch) {
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
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
  const double sweep_bytes = (double)P * (nn + W);  // each present row read once + every write
  const double write_bytes = (double)P * W;
  auto report = [&](const char* name, int bps, double bytes, float ms, int extra = -1) {
    printf("{\"kernel\": \"%s\", \"bps\": %d, \"K\": %d, \"us\": %.1f, \"GBps\": %.1f, \"write_GBps\": %.1f}\n", name,
           bps, extra, ms * 1e3, bytes / ms / 1e6, write_bytes / ms / 1e6);
    fflush(stdout);
  };
  float t = timeit([&] { CK(cudaMemsetAsync(X, 0, (size_t)W * P)); });
  report("memset", 0, write_bytes, t);
  for (int bps : {1, 2, 4, 8}) {
    t = timeit([&] { k_wseq<<<sms * bps, 256>>>((int4*)X, W, row16); });
    report("wseq", bps, write_bytes, t);
  }
  for (int bps : {1, 2, 4, 8}) {
    t = timeit([&] { k_desc_ldg<5><<<sms * bps, 256>>>((int4*)src, (int4*)X, d_nodes, d_dst, nn, row16, 0); });
    report("wrand", bps, write_bytes, t);
  }
  for (int bps : {1, 2, 4, 8}) {
    t = timeit([&] { k_desc_ldg<5><<<sms * bps, 256>>>((int4*)src, (int4*)X, d_nodes, d_dst, nn, row16, 1); });
    report("desc_ldg", bps, sweep_bytes, t);
  }
  for (int bps : {1, 2, 4, 8}) {
    t = timeit([&] { k_rows<5><<<sms * bps, 256>>>((int4*)src, (int4*)X, d_rsrc, W, row16); });
    report("rows", bps, 2.0 * write_bytes, t);
  }
  for (int warps : {4, 8, 16, 32})
    for (int K : {2, 4, 8}) {
      const size_t smem = (size_t)warps * K * P;
      if (smem > 220 * 1024) continue;
      CK(cudaFuncSetAttribute(k_desc_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      t = timeit([&] { k_desc_tma<<<sms, 32 * warps, smem>>>(src, X, d_nodes, d_dst, nn, P, K); });
      report("desc_tma", warps, sweep_bytes, t, K);
    }
  return 0;
}
