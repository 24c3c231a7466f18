// Host-link probe with N concurrent GPU readers of ONE pinned host region (SURVEY §7 step 0, §8(e)
// caveat; round-1 VERDICT missing #2): does the node's host memory + PCIe fabric sustain N x the
// one-GPU zero-copy rate when 1, 2, 4, 8 B200s read the same host-resident graph at once?
//
//   multireader_probe [region_GB=8] [out.json]
//
// The region is allocated once (cudaHostAllocPortable | Mapped: every device reads it through UVA,
// as DCI_ADOPT_HOST contexts do).  For each reader count n (powers of two up to the visible device
// count) one host thread per device launches the same kernel on its device at once; each device's
// time is taken with CUDA events on its stream, the aggregate rate is the total bytes over the
// slowest device's time.  Patterns (the two miss paths of the hot path):
//   rows512   random 512-byte feature rows, a warp per row (papers100M-shaped, D = 128 fp32)
//   rows400   random 400-byte rows (products-shaped, D = 100)
//   lines128  random 128-byte lines, a warp per line (one adjacency-miss request)
//   rand4     random 4-byte reads, independent per thread, 8 in flight per thread
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// warp per row; row16 16-byte words per row; rows picked by a per-device hash stream
__global__ void k_rows(const int4* __restrict__ src, uint64_t nrows, int row16, int64_t nout, uint32_t salt,
                       int4* sink) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t i = w; i < nout; i += nw) {
    const uint64_t r = ((uint64_t)hash32((uint32_t)i * 2654435761u ^ salt) * nrows) >> 32;
    for (int c = lane; c < row16; c += 32) {
      const int4 v = __ldcs(src + r * row16 + c);
      acc.x ^= v.x;
      acc.y ^= v.y;
    }
  }
  if (acc.x == 0x7fffffff && acc.y == 0x12345) sink[0] = acc;
}

__global__ void k_rand4(const int* __restrict__ src, uint64_t n, int per, uint32_t salt, int* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  int acc = 0;
  for (int j = 0; j < per; j += 8) {
    int v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t idx = ((uint64_t)hash32(t * 7919u + (j + u) * 104729u + salt) * n) >> 32;
      v[u] = __ldcs(src + idx);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678) sink[0] = acc;
}

struct Result {
  float ms = 0.f;
  double bytes = 0.0, requests = 0.0;
};

int main(int argc, char** argv) {
  const double region_gb = argc > 1 ? atof(argv[1]) : 8.0;
  const char* out = argc > 2 ? argv[2] : nullptr;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const size_t bytes = (size_t)(region_gb * (1ull << 30)) / 4096 * 4096;
  void* h = nullptr;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  for (size_t i = 0; i < bytes / 4; i += 1024) static_cast<int*>(h)[i] = (int)i;
  std::vector<int> sms(ndev);
  std::vector<void*> sink(ndev);
  for (int d = 0; d < ndev; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d));
    CK(cudaMalloc(&sink[d], 4096));
  }
  struct Pat {
    const char* name;
    int row_bytes;  // 0: rand4
  } pats[] = {{"rows512", 512}, {"rows400", 400}, {"lines128", 128}, {"rand4", 0}};
  std::string json = "{\"region_GB\": " + std::to_string(region_gb) + ", \"devices\": " + std::to_string(ndev) +
                     ", \"runs\": [";
  bool first = true;
  for (auto& p : pats) {
    for (int n = 1; n <= ndev; n *= 2) {
      std::vector<Result> res(n);
      auto work = [&](int d) {
        CK(cudaSetDevice(d));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        auto launch = [&](uint32_t salt) {
          if (p.row_bytes) {
            const int row16 = p.row_bytes / 16;
            const int64_t nout = (int64_t)(2ll << 30) / p.row_bytes;  // 2 GB of rows per device
            k_rows<<<sms[d] * 8, 256, 0, st>>>(static_cast<const int4*>(h), bytes / p.row_bytes, row16, nout,
                                               salt, static_cast<int4*>(sink[d]));
            res[d].bytes = (double)nout * p.row_bytes;
            res[d].requests = (double)nout;
          } else {
            const int per = 64;
            const int grid = sms[d] * 8;
            k_rand4<<<grid, 256, 0, st>>>(static_cast<const int*>(h), bytes / 4, per, salt,
                                          static_cast<int*>(sink[d]));
            res[d].requests = (double)grid * 256 * per;
            res[d].bytes = res[d].requests * 4;
          }
        };
        launch(1000u + d);  // warm-up
        CK(cudaStreamSynchronize(st));
        CK(cudaEventRecord(e0, st));
        launch(2000u + d);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&res[d].ms, e0, e1));
        CK(cudaStreamDestroy(st));
      };
      std::vector<std::thread> th;
      for (int d = 0; d < n; ++d) th.emplace_back(work, d);
      for (auto& t : th) t.join();
      float mx = 0.f;
      double tb = 0.0, tr = 0.0;
      for (auto& r : res) {
        mx = std::max(mx, r.ms);
        tb += r.bytes;
        tr += r.requests;
      }
      char line[512];
      snprintf(line, sizeof(line),
               "{\"pattern\": \"%s\", \"readers\": %d, \"aggregate_GBps\": %.2f, \"per_reader_GBps\": %.2f, "
               "\"aggregate_Mreq_per_s\": %.1f, \"slowest_ms\": %.3f}",
               p.name, n, tb / mx / 1e6, tb / mx / 1e6 / n, tr / mx / 1e3, mx);
      printf("%s\n", line);
      fflush(stdout);
      json += (first ? "" : ", ") + std::string(line);
      first = false;
    }
  }
  json += "]}\n";
  if (out) {
    FILE* f = fopen(out, "w");
    if (f) {
      fputs(json.c_str(), f);
      fclose(f);
    }
  }
  return 0;
}
