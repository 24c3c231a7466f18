// S8 feature gather: X[i] = fcache[slot] on a feature-cache hit (HBM -> HBM) and
// X[i] = feats[v] on a miss (pinned host -> HBM through UVA zero-copy).  One warp per
// row; every lane issues all of its 16-byte loads for the row before any store, so each
// warp keeps a whole row (up to 32*VPL*16 B) in flight; the grid is persistent (a multiple
// of the SM count) and walks the route list written by k_route.
#include <cuda_runtime.h>

#include "dci_internal.cuh"

namespace dci {

namespace {

__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

struct GatherArgs {
  const int64_t* list;        // packed (row i << 32 | source row)
  const uint32_t* count;      // device list length
  const float* src;           // fcache (hits) or the mapped host feature table (misses)
  int32_t pitch;              // floats per source row (multiple of 4)
  float* X;
  int64_t ldx;                // floats per X row
  int32_t D;
};

// Vector path: ldx % 4 == 0 and ldx >= pitch -> copy whole pitch rows as int4.
template <int VPL>
__global__ void __launch_bounds__(256) k_gather_v4(GatherArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = *a.count;
  const int row16 = a.pitch >> 2;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t ent = __ldg(a.list + r);
    const int64_t i = ent >> 32;
    const int64_t srow = ent & 0xffffffffll;
    const int4* src = reinterpret_cast<const int4*>(a.src + srow * a.pitch);
    int4* dst = reinterpret_cast<int4*>(a.X + i * a.ldx);
    for (int c0 = 0; c0 < row16; c0 += 32 * VPL) {
      int4 buf[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int idx = c0 + lane + 32 * j;
        if (idx < row16) buf[j] = ld_stream_v4(src + idx);
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int idx = c0 + lane + 32 * j;
        if (idx < row16) st_v4(dst + idx, buf[j]);
      }
    }
  }
}

// Scalar path for any ldx >= D (e.g. an unpadded X with D % 4 != 0).
__global__ void __launch_bounds__(256) k_gather_scalar(GatherArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n = *a.count;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t ent = __ldg(a.list + r);
    const int64_t i = ent >> 32;
    const int64_t srow = ent & 0xffffffffll;
    const float* src = a.src + srow * a.pitch;
    float* dst = a.X + i * a.ldx;
    for (int c = lane; c < a.D; c += 32) dst[c] = src[c];
  }
}

}  // namespace

void launch_gather(dci_ctx* ctx, dci_workspace* ws, bool hits, const int32_t* /*F*/, int32_t /*L*/, float* X,
                   int64_t ldx, cudaStream_t s) {
  GatherArgs a;
  a.list = hits ? ws->hit_list : ws->miss_list;
  a.count = hits ? &ws->scal->hit_count : &ws->scal->miss_count;
  a.src = hits ? ctx->d_fcache : ctx->u_feats;
  a.pitch = ctx->pitch;
  a.X = X;
  a.ldx = ldx;
  a.D = ctx->D;
  const bool vec = (ldx % 4 == 0) && ldx >= ctx->pitch && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  if (!vec) {
    k_gather_scalar<<<persistent_grid(ctx, k_gather_scalar, 256), 256, 0, s>>>(a);
  } else if (ctx->pitch <= 32 * 4 * 2) {
    k_gather_v4<2><<<persistent_grid(ctx, k_gather_v4<2>, 256), 256, 0, s>>>(a);
  } else {
    k_gather_v4<5><<<persistent_grid(ctx, k_gather_v4<5>, 256), 256, 0, s>>>(a);
  }
  ++ctx->launches;
}

}  // namespace dci
