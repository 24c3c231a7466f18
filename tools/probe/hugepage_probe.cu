// Probe: random 512 B host-row reads (UVA) as a function of the host region size, for
// cudaHostAlloc'ed memory vs mmap + madvise(MADV_HUGEPAGE) + cudaHostRegister.  Decides how
// dci_load_graph should allocate the host-resident feature table (papers100M-shaped: 57 GB).
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

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

__global__ void ldg_rows(const int4* __restrict__ src, int64_t nrows, int row16, int64_t nout, int4* __restrict__ dst) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < nout; i += nw) {
    uint64_t h = ((uint64_t)hash32((uint32_t)i * 2654435761u + 12345u) << 32) | hash32((uint32_t)i ^ 0x9e3779b9u);
    uint64_t r = h % (uint64_t)nrows;
    const int4* s = src + r * row16;
    int4* d = dst + (i % 1000000) * row16;
    for (int c = lane; c < row16; c += 32) d[c] = s[c];
  }
}

static double run(const void* hd, size_t bytes, int rb, int sms, void* d) {
  const int64_t nrows = bytes / rb, nout = ((int64_t)1 << 30) / rb;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(a));
    ldg_rows<<<sms * 8, 256>>>((const int4*)hd, nrows, rb / 16, nout, (int4*)d);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
  }
  return nout * (double)rb / ms / 1e6;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* d;
  CK(cudaMalloc(&d, (size_t)1 << 30));
  size_t sizes_gb[4] = {1, 8, 32, 64};
  for (int si = 0; si < 4; ++si) {
    size_t bytes = sizes_gb[si] << 30;
    // (a) cudaHostAlloc
    void* h = nullptr;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 1, bytes);
    void* hd;
    CK(cudaHostGetDevicePointer(&hd, h, 0));
    double g1 = run(hd, bytes, 512, sms, d);
    CK(cudaFreeHost(h));
    // (b) mmap + THP + cudaHostRegister
    void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (m == MAP_FAILED) {
      perror("mmap");
      return 1;
    }
    int adv = madvise(m, bytes, MADV_HUGEPAGE);
    memset(m, 1, bytes);
    CK(cudaHostRegister(m, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    CK(cudaHostGetDevicePointer(&hd, m, 0));
    double g2 = run(hd, bytes, 512, sms, d);
    CK(cudaHostUnregister(m));
    munmap(m, bytes);
    printf("{\"probe\":\"host_region\",\"GB\":%zu,\"row_bytes\":512,\"hostalloc_GBps\":%.2f,\"thp_register_GBps\":%.2f,"
           "\"madvise_rc\":%d}\n",
           sizes_gb[si], g1, g2, adv);
    fflush(stdout);
  }
  return 0;
}
