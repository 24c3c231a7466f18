// Box probe: host-link and HBM gather microbenchmarks.
// Not part of the product path; numbers feed DESIGN.md's roofline denominators.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void stream_read(const int4* __restrict__ src, int64_t n, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// random 4-byte reads: each thread does `per` dependent-free random reads
__global__ void rand_read4(const int* __restrict__ src, int64_t n, int per, int* sink) {
  int acc = 0;
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int j = 0; j < per; ++j) {
    uint64_t idx = ((uint64_t)hash32(t * 7919u + j * 104729u) * (uint64_t)n) >> 32;
    acc ^= src[idx];
  }
  if (acc == 0x12345678) sink[0] = acc;
}

// random row gather: warp per row, row_bytes multiple of 16
__global__ void rand_rows(const int4* __restrict__ src, int64_t nrows, int row16, int64_t nout,
                          int4* __restrict__ dst) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < nout; i += nw) {
    uint64_t r = ((uint64_t)hash32((uint32_t)i * 2654435761u + 12345u) * (uint64_t)nrows) >> 32;
    const int4* s = src + r * row16;
    int4* d = dst + i * row16;
    for (int c = lane; c < row16; c += 32) d[c] = s[c];
  }
}

static float time_kernel(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  launch(arg); CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch(arg);
  CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

struct SArgs { const int4* src; int64_t n; int4* sink; int grid; };
static void l_stream(void* p) { SArgs* a = (SArgs*)p; stream_read<<<a->grid, 512>>>(a->src, a->n, a->sink); }
struct RArgs { const int* src; int64_t n; int per; int* sink; int grid; };
static void l_rand4(void* p) { RArgs* a = (RArgs*)p; rand_read4<<<a->grid, 256>>>(a->src, a->n, a->per, a->sink); }
struct GArgs { const int4* src; int64_t nrows; int row16; int64_t nout; int4* dst; int grid; };
static void l_rows(void* p) { GArgs* a = (GArgs*)p; rand_rows<<<a->grid, 256>>>(a->src, a->nrows, a->row16, a->nout, a->dst); }

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)4 << 30;  // 4 GiB host buffer
  void* h; CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes / 4; i += 1024) ((int*)h)[i] = (int)i;
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  void* d; CK(cudaMalloc(&d, bytes));
  void* sink; CK(cudaMalloc(&sink, 1 << 20));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  float ms;
  // memcpy H2D / D2H
  CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
  CK(cudaEventRecord(a)); CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice)); CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
  printf("{\"probe\":\"memcpy_h2d\",\"GBps\":%.2f}\n", bytes / ms / 1e6);
  CK(cudaEventRecord(a)); CK(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost)); CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
  printf("{\"probe\":\"memcpy_d2h\",\"GBps\":%.2f}\n", bytes / ms / 1e6);
  // zero-copy streaming read
  for (int occ : {1, 2, 4, 8}) {
    SArgs s{(const int4*)hd, (int64_t)(bytes / 16), (int4*)sink, sms * occ};
    ms = time_kernel(l_stream, &s, 3);
    printf("{\"probe\":\"uva_stream_read16\",\"grid\":%d,\"GBps\":%.2f}\n", s.grid, bytes / ms / 1e6);
  }
  // HBM streaming read
  {
    SArgs s{(const int4*)d, (int64_t)(bytes / 16), (int4*)sink, sms * 4};
    ms = time_kernel(l_stream, &s, 5);
    printf("{\"probe\":\"hbm_stream_read16\",\"GBps\":%.2f}\n", bytes / ms / 1e6);
  }
  // random 4B reads host vs device
  for (int occ : {4, 8, 16}) {
    RArgs r{(const int*)hd, (int64_t)(bytes / 4), 16, (int*)sink, sms * occ};
    ms = time_kernel(l_rand4, &r, 3);
    double nreq = (double)r.grid * 256 * r.per;
    printf("{\"probe\":\"uva_rand4\",\"grid\":%d,\"Mreq_per_s\":%.1f,\"GBps_useful\":%.3f}\n", r.grid, nreq / ms / 1e3, nreq * 4 / ms / 1e6);
  }
  {
    RArgs r{(const int*)d, (int64_t)(bytes / 4), 16, (int*)sink, sms * 8};
    ms = time_kernel(l_rand4, &r, 5);
    double nreq = (double)r.grid * 256 * r.per;
    printf("{\"probe\":\"hbm_rand4\",\"Mreq_per_s\":%.1f}\n", nreq / ms / 1e3);
  }
  // random row gathers: 400 B (products), 512 B (papers), 2416 B (reddit pitch)
  int rows_b[3] = {400, 512, 2416};
  for (int k = 0; k < 3; ++k) {
    int row16 = rows_b[k] / 16;
    int64_t nrows = bytes / rows_b[k];
    int64_t nout = (256 << 20) / rows_b[k];
    for (int src_host = 0; src_host < 2; ++src_host) {
      for (int occ : {4, 8}) {
        GArgs g{(const int4*)(src_host ? hd : d), nrows, row16, nout, (int4*)((char*)d + ((size_t)2 << 30)), sms * occ};
        ms = time_kernel(l_rows, &g, src_host ? 2 : 5);
        double by = (double)nout * rows_b[k];
        printf("{\"probe\":\"%s_rows\",\"row_bytes\":%d,\"grid\":%d,\"GBps_read\":%.2f,\"GBps_rw\":%.2f}\n",
               src_host ? "uva" : "hbm", rows_b[k], g.grid, by / ms / 1e6, 2 * by / ms / 1e6);
      }
    }
  }
  return 0;
}
