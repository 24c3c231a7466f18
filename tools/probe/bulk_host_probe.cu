// Probe: random host-row reads through UVA, warp LDG vs TMA bulk copy (cp.async.bulk
// global->shared with mbarrier).  Decides how S8 should read feature-cache misses.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));    \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// LDG: warp per row, 16 B per lane
__global__ void ldg_rows(const int4* __restrict__ src, int64_t nrows, int row16, int64_t nout, int4* __restrict__ dst) {
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

// TMA bulk: one elected lane per warp, ring of Q slots; rows go host -> smem -> HBM
template <int Q>
__global__ void bulk_rows(const char* __restrict__ src, int64_t nrows, int row_bytes, int64_t nout, char* __restrict__ dst) {
  extern __shared__ __align__(128) unsigned char smem[];
  if ((threadIdx.x & 31) != 0) return;
  const int warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * Q;
  const int slot_bytes = (row_bytes + 127) & ~127;
  unsigned char* slots = smem + W * Q * 8 + (size_t)warp * Q * slot_bytes;
  for (int s = 0; s < Q; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(1) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t stride = (int64_t)gridDim.x * W, first = (int64_t)blockIdx.x * W + warp;
  const int64_t nm = first < nout ? (nout - first + stride - 1) / stride : 0;
  auto issue = [&](int64_t j) {
    const int64_t i = first + j * stride;
    uint64_t r = ((uint64_t)hash32((uint32_t)i * 2654435761u + 12345u) * (uint64_t)nrows) >> 32;
    const int s = (int)(j % Q);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(row_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(slots + (size_t)s * slot_bytes)),
                 "l"(src + r * row_bytes), "r"(row_bytes), "r"(smem_u32(&bars[s]))
                 : "memory");
  };
  for (int64_t j = 0; j < Q && j < nm; ++j) issue(j);
  for (int64_t i = 0; i < nm; ++i) {
    const int s = (int)(i % Q);
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_u32(&bars[s])),
        "r"((uint32_t)((i / Q) & 1))
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (first + i * stride) * row_bytes),
                 "r"(smem_u32(slots + (size_t)s * slot_bytes)), "r"(row_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (i >= 1 && i - 1 + Q < nm) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(i - 1 + Q);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)8 << 30;
  void* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < bytes / 4; i += 1024) ((int*)h)[i] = (int)i;
  void* hd;
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  void* d;
  CK(cudaMalloc(&d, (size_t)1 << 30));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaFuncSetAttribute(bulk_rows<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(bulk_rows<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  CK(cudaFuncSetAttribute(bulk_rows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  int rows_b[4] = {400, 512, 1024, 2416};
  for (int k = 0; k < 4; ++k) {
    const int rb = rows_b[k];
    const int64_t nrows = bytes / rb, nout = ((int64_t)512 << 20) / rb;
    for (int mode = 0; mode < 4; ++mode) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        if (mode == 0) {
          ldg_rows<<<sms * 8, 256>>>((const int4*)hd, nrows, rb / 16, nout, (int4*)d);
        } else {
          const int W = 8;
          const int Q = mode == 1 ? 4 : (mode == 2 ? 8 : 16);
          const int slot = (rb + 127) & ~127;
          size_t sm = (size_t)W * Q * (8 + slot);
          if (sm > 227 * 1024) continue;
          if (Q == 4) bulk_rows<4><<<sms, 32 * W, sm>>>((const char*)hd, nrows, rb, nout, (char*)d);
          if (Q == 8) bulk_rows<8><<<sms, 32 * W, sm>>>((const char*)hd, nrows, rb, nout, (char*)d);
          if (Q == 16) bulk_rows<16><<<sms, 32 * W, sm>>>((const char*)hd, nrows, rb, nout, (char*)d);
        }
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        CK(cudaEventElapsedTime(&ms, a, b));
      }
      printf("{\"probe\":\"host_rows\",\"mode\":\"%s\",\"row_bytes\":%d,\"GBps\":%.2f,\"Mrows_per_s\":%.1f}\n",
             mode == 0 ? "ldg" : (mode == 1 ? "bulk_q4" : (mode == 2 ? "bulk_q8" : "bulk_q16")), rb,
             nout * (double)rb / ms / 1e6, nout / ms / 1e3);
    }
  }
  return 0;
}
