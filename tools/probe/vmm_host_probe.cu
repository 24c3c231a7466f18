// Probe: does host memory allocated through the CUDA virtual-memory API (cuMemCreate with a
// CU_MEM_LOCATION_TYPE_HOST_NUMA location, mapped with the allocation's granularity) lift the
// random-request rate the GPU reaches over a large pinned region?  hostreq_probe.cu found random
// 512-B reads through UVA over cudaHostAlloc memory stopping at ~69 M requests/s for a 64 GB region
// (address translation), while 2-KB requests still moved 51.5 GB/s.  If the VMM mapping uses larger
// GPU pages, the translation limit should move.
//
//   vmm_host_probe [region_GB=64] > profiles/r02/vmm_host_probe.jsonl
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                            \
    }                                                                                     \
  } while (0)
#define CU(x)                                                                   \
  do {                                                                          \
    CUresult r = (x);                                                           \
    if (r != CUDA_SUCCESS) {                                                    \
      const char* m = nullptr;                                                  \
      cuGetErrorString(r, &m);                                                  \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, m ? m : "?"); \
      printf("{\"probe\":\"vmm_host\",\"error\":\"%s: %s\"}\n", #x, m ? m : "?"); \
      exit(0);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint64_t perm(uint64_t x, int bits) {
  const uint64_t m = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  x = (x * 0x9E3779B97F4A7C15ull) & m;
  x ^= x >> (bits / 2 + 1);
  x = (x * 0xBF58476D1CE4E5B9ull) & m;
  x ^= x >> (bits / 2 + 1);
  return x & m;
}

// S-byte random reads (S >= 64), groups of min(32, S/16) lanes, U requests in flight per group
template <int S>
__global__ void rand_rows(const char* __restrict__ src, int bits, int iters, int* sink) {
  constexpr int L = (S / 16) < 32 ? (S / 16) : 32, PER = S / 16 / L, U = 8;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t ngrp = (uint64_t)gridDim.x * blockDim.x / L, grp = t / L;
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
        int4 x;
        asm volatile("ld.global.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(p + k * L));
        v[u] ^= x.x ^ x.w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int S>
static void run(const char* src, size_t region, int* sink, int sms, const char* kind, double gb) {
  int bits = 0;
  while ((2ull << bits) <= region / S) ++bits;
  const int grid = sms * 8, threads = 256;
  constexpr int L = (S / 16) < 32 ? (S / 16) : 32;
  const double per_iter = (double)grid * threads / L * 8;
  const int iters = (int)(std::max(1.0, std::min(16.0, 8.0e6 / per_iter)));
  const double nreq = per_iter * iters;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  rand_rows<S><<<grid, threads>>>(src, bits, iters, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(a));
    rand_rows<S><<<grid, threads>>>(src, bits, iters, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  printf("{\"probe\":\"vmm_host\",\"alloc\":\"%s\",\"region_GB\":%.1f,\"bytes\":%d,\"Mreq_per_s\":%.1f,\"GBps\":%.2f}\n",
         kind, gb, S, nreq / best / 1e3, nreq * S / best / 1e6);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const double max_gb = argc > 1 ? atof(argv[1]) : 64.0;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* sink;
  CK(cudaMalloc(&sink, 64));
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = 0;
  size_t gmin = 0, grec = 0;
  CU(cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CU(cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("{\"probe\":\"vmm_host\",\"granularity_min\":%zu,\"granularity_recommended\":%zu}\n", gmin, grec);
  fflush(stdout);
  const size_t gran = grec > gmin ? grec : gmin;
  size_t bytes = (size_t)(max_gb * (1ull << 30));
  bytes = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CU(cuMemCreate(&h, bytes, &prop, 0));
  CUdeviceptr ptr = 0;
  CU(cuMemAddressReserve(&ptr, bytes, gran, 0, 0));
  CU(cuMemMap(ptr, bytes, 0, h, 0));
  CUmemAccessDesc acc[2];
  memset(acc, 0, sizeof(acc));
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc[0].location.id = 0;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  acc[1].location.id = 0;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUresult r2 = cuMemSetAccess(ptr, bytes, acc, 2);
  const bool host_access = r2 == CUDA_SUCCESS;
  if (!host_access) CU(cuMemSetAccess(ptr, bytes, acc, 1));
  printf("{\"probe\":\"vmm_host\",\"host_access\":%s}\n", host_access ? "true" : "false");
  fflush(stdout);
  CK(cudaMemset(reinterpret_cast<void*>(ptr), 1, bytes));  // touch every page from the GPU
  CK(cudaDeviceSynchronize());
  if (host_access) {  // the CPU sees the same virtual address
    volatile unsigned char* c = reinterpret_cast<volatile unsigned char*>(ptr);
    printf("{\"probe\":\"vmm_host\",\"cpu_reads\":%d}\n", (int)c[bytes / 2]);
  }
  const double regions[] = {2, 8, 32, 64};
  for (double gb : regions) {
    if (gb > max_gb) break;
    const size_t region = (size_t)(gb * (1ull << 30));
    const char* src = reinterpret_cast<const char*>(ptr);
    run<512>(src, region, sink, sms, "vmm_host_numa", gb);
    run<128>(src, region, sink, sms, "vmm_host_numa", gb);
    run<2048>(src, region, sink, sms, "vmm_host_numa", gb);
  }
  CU(cuMemUnmap(ptr, bytes));
  CU(cuMemRelease(h));
  CU(cuMemAddressFree(ptr, bytes));
  return 0;
}
