// Counter-based Philox4x32-10 for the sampling draws (BASELINE.json north_star: "a
// counter-based Philox draw keyed by (seed, layer, node, slot)"; reading C4).
// Salmon et al., SC'11.  Device-only; written independently of oracle/.
#pragma once
#include <stdint.h>

namespace dci {

__device__ __forceinline__ uint2 philox_draw_u32x2(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint2(c0, c1);
}

// 64-bit uniform for (node v, slot i, hop, pass) under a 64-bit seed: ctr = (v, i, hop,
// pass), key = (seed_lo, seed_hi), u = r1 << 32 | r0.
__device__ __forceinline__ uint64_t philox_u64(uint64_t seed, uint32_t pass, uint32_t hop, uint32_t v,
                                               uint32_t i) {
  uint2 r = philox_draw_u32x2(v, i, hop, pass, (uint32_t)seed, (uint32_t)(seed >> 32));
  return ((uint64_t)r.y << 32) | r.x;
}

}  // namespace dci
