// NEXT F2: mean / sum aggregator over one sampled block — the consumer
// the prepared mini-batch feeds ("each vertex transforms the features from its
// neighbours by aggregating them"; BJ north_star's optional consumer, reading C23).
//   mean: H[d][c] = (1 / k_d) * sum_{j in block row d} Xsrc[bsrc[j]][c] (k_d = 0 -> 0); sum: no 1/k_d
// One warp per dst row, float4 lanes across the row, fp32 accumulation in bsrc order (the
// oracle accumulates in fp64; DESIGN.md §4 states the tolerance).  HBM-bound gather-reduce.
#include <cuda_runtime.h>

#include "dci_internal.cuh"

namespace dci {

namespace {

struct AggArgs {
  const int32_t* bptr;
  const int32_t* bsrc;
  const int64_t* n_dst;
  const float* X;
  int64_t ldx;
  int32_t D;
  float* H;
  int64_t ldh;
  int32_t op;  // 0 mean, 1 sum
};

template <int VPL>
__global__ void __launch_bounds__(256) k_mean_aggregate_v4(AggArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = *a.n_dst;
  const int D4 = (a.D + 3) >> 2;
  for (int64_t d = warp; d < n; d += nwarps) {
    const int32_t j0 = a.bptr[d], j1 = a.bptr[d + 1];
    for (int c0 = 0; c0 < D4; c0 += 32 * VPL) {
      float4 acc[VPL];
#pragma unroll
      for (int t = 0; t < VPL; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int32_t j = j0; j < j1; ++j) {
        const float4* src = reinterpret_cast<const float4*>(a.X + (int64_t)__ldg(a.bsrc + j) * a.ldx);
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          const int c = c0 + lane + 32 * t;
          if (c < D4) {
            const float4 x = __ldg(src + c);
            acc[t].x += x.x;
            acc[t].y += x.y;
            acc[t].z += x.z;
            acc[t].w += x.w;
          }
        }
      }
      const float k = (float)(j1 - j0);
      float4* dst = reinterpret_cast<float4*>(a.H + d * a.ldh);
#pragma unroll
      for (int t = 0; t < VPL; ++t) {
        const int c = c0 + lane + 32 * t;
        if (c < D4) {
          float4 h = acc[t];
          if (a.op == 0)
            h = j1 > j0 ? make_float4(acc[t].x / k, acc[t].y / k, acc[t].z / k, acc[t].w / k)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
          dst[c] = h;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_mean_aggregate_scalar(AggArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = *a.n_dst;
  for (int64_t d = warp; d < n; d += nwarps) {
    const int32_t j0 = a.bptr[d], j1 = a.bptr[d + 1];
    for (int c = lane; c < a.D; c += 32) {
      float acc = 0.f;
      for (int32_t j = j0; j < j1; ++j) acc += __ldg(a.X + (int64_t)__ldg(a.bsrc + j) * a.ldx + c);
      a.H[d * a.ldh + c] = a.op == 1 ? acc : (j1 > j0 ? acc / (float)(j1 - j0) : 0.f);
    }
  }
}

}  // namespace

dci_status launch_block_aggregate(dci_ctx* ctx, const int32_t* bptr, const int32_t* bsrc, const int64_t* n_dst,
                                  const float* X, int64_t ldx, int32_t D, float* H, int64_t ldh, int32_t op,
                                  cudaStream_t s) {
  AggArgs a{bptr, bsrc, n_dst, X, ldx, D, H, ldh, op};
  const int64_t D4x4 = (int64_t)((D + 3) / 4) * 4;
  const bool vec = ldx % 4 == 0 && ldh % 4 == 0 && ldx >= D4x4 && ldh >= D4x4 &&
                   reinterpret_cast<uintptr_t>(X) % 16 == 0 && reinterpret_cast<uintptr_t>(H) % 16 == 0;
  auto go = [&](auto kern) { kern<<<persistent_grid(ctx, kern, 256), 256, 0, s>>>(a); };
  const int D4 = (D + 3) / 4;
  if (!vec)
    go(k_mean_aggregate_scalar);
  else if (D4 <= 32)
    go(k_mean_aggregate_v4<1>);
  else if (D4 <= 64)
    go(k_mean_aggregate_v4<2>);
  else if (D4 <= 160)
    go(k_mean_aggregate_v4<5>);
  else
    go(k_mean_aggregate_v4<8>);
  ++ctx->launches;
  DCI_CUDA(cudaGetLastError());
  return DCI_OK;
}

}  // namespace dci
