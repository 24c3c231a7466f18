// Does the allocation kind of an output buffer change HBM write bandwidth on this B200?  ncu
// reports that the node-sweep gather's X stores (PyTorch allocations) are "sent to the L2
// compression unit" with 0 % success (the features are incompressible).  This probe writes
// INCOMPRESSIBLE data (a hash of the address) into a 6.8 GB buffer allocated three ways --
// cudaMalloc, cuMemCreate without compression, cuMemCreate with generic compression -- with the
// gather's two write patterns: sequential rows and whole-line rows at random positions
// (2432-byte rows, M2 group-of-20 sizes), and a memset for reference.
//
//   compress_probe [rows=2823740] [row_bytes=2432]   -> one JSON line per (allocation, kernel)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)
#define CU(x)                                                  \
  do {                                                         \
    CUresult r = (x);                                          \
    if (r != CUDA_SUCCESS) {                                   \
      const char* s = nullptr;                                 \
      cuGetErrorString(r, &s);                                 \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, s);    \
      return nullptr;                                          \
    }                                                          \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ int4 noise(uint64_t i) {
  const uint32_t a = hash32((uint32_t)i ^ 0x9e3779b9u), b = hash32(a + (uint32_t)(i >> 32));
  return make_int4((int)a, (int)b, (int)hash32(b), (int)hash32(a ^ 0x85ebca6bu));
}

// rows in order, a warp per row, 16-byte stores
__global__ void k_wseq(int4* X, int64_t rows, int row16) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < rows; r += nw)
    for (int c = lane; c < row16; c += 32) X[r * row16 + c] = noise(r * row16 + c);
}

// row r goes to position perm(r) (a bijective hash of r mod rows), a warp per row
__global__ void k_wrand(int4* X, int64_t rows, int row16) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < rows; r += nw) {
    const int64_t p = (r * 2654435761ll) % rows;  // a bijection: the multiplier is a prime not dividing rows
    for (int c = lane; c < row16; c += 32) X[p * row16 + c] = noise(r * row16 + c);
  }
}

static void* vmm_alloc(size_t bytes, bool compress, size_t* out_size) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  prop.allocFlags.compressionType = compress ? CU_MEM_ALLOCATION_COMP_GENERIC : CU_MEM_ALLOCATION_COMP_NONE;
  size_t gran = 0;
  CU(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CU(cuMemCreate(&h, sz, &prop, 0));
  if (compress) {
    CUmemAllocationProp got = {};
    CU(cuMemGetAllocationPropertiesFromHandle(&got, h));
    fprintf(stderr, "compressible allocation granted: %d\n", (int)got.allocFlags.compressionType);
  }
  CUdeviceptr p = 0;
  CU(cuMemAddressReserve(&p, sz, 0, 0, 0));
  CU(cuMemMap(p, sz, 0, h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(p, sz, &acc, 1));
  *out_size = sz;
  return (void*)p;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 2823740;
  const int P = argc > 2 ? atoi(argv[2]) : 2432;
  const int row16 = P / 16;
  const size_t bytes = (size_t)rows * P;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  int sms = 0, comp = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cuDeviceGetAttribute(&comp, CU_DEVICE_ATTRIBUTE_GENERIC_COMPRESSION_SUPPORTED, 0);
  printf("{\"rows\": %lld, \"row_bytes\": %d, \"GB\": %.2f, \"generic_compression_supported\": %d}\n", (long long)rows, P,
         bytes / 1e9, comp);
  void* flush;
  const size_t fbytes = 256ull << 20;
  CK(cudaMalloc(&flush, fbytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int kind = 0; kind < 3; ++kind) {
    const char* kname = kind == 0 ? "cudaMalloc" : kind == 1 ? "vmm_nocomp" : "vmm_generic";
    void* X = nullptr;
    size_t vsz = 0;
    if (kind == 0)
      CK(cudaMalloc(&X, bytes));
    else
      X = vmm_alloc(bytes, kind == 2, &vsz);
    if (!X) {
      printf("{\"alloc\": \"%s\", \"error\": \"allocation failed\"}\n", kname);
      continue;
    }
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
    float t = timeit([&] { CK(cudaMemsetAsync(X, 0, bytes)); });
    printf("{\"alloc\": \"%s\", \"kernel\": \"memset0\", \"GBps\": %.1f}\n", kname, bytes / t / 1e6);
    for (int bps : {2, 8}) {
      t = timeit([&] { k_wseq<<<sms * bps, 256>>>((int4*)X, rows, row16); });
      printf("{\"alloc\": \"%s\", \"kernel\": \"wseq\", \"bps\": %d, \"GBps\": %.1f}\n", kname, bps, bytes / t / 1e6);
      t = timeit([&] { k_wrand<<<sms * bps, 256>>>((int4*)X, rows, row16); });
      printf("{\"alloc\": \"%s\", \"kernel\": \"wrand\", \"bps\": %d, \"GBps\": %.1f}\n", kname, bps, bytes / t / 1e6);
    }
    fflush(stdout);
    if (kind == 0)
      CK(cudaFree(X));
    else {
      cuMemUnmap((CUdeviceptr)X, vsz);
      cuMemAddressFree((CUdeviceptr)X, vsz);
    }
  }
  return 0;
}
