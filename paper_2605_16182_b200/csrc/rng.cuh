// Counter-based RNG streams on the device. Every draw is a pure function of
// (seed; walk, hop, ordinal), so walks are independent of scheduling,
// tiering and GPU count (rng.hpp:15-21).
//
//  * SplitMix: the reference's CounterRng (rng.hpp:8-13, :25, :27-39),
//    bit-identical, so walks match the UNMODIFIED reference.
//  * Philox4x32-10: counter = (lo32 walk, lo32 hop, lo32 ordinal,
//    hi32 walk ^ hi32 hop ^ hi32 ordinal), key = (lo32 seed, hi32 seed),
//    bits = out.y << 32 | out.x — the function of the oracle's Philox shadow
//    header (oracle/philox_shadow/timewalk/rng.hpp).
#pragma once

#include "common.cuh"

namespace twg {

__host__ __device__ __forceinline__ u64 mix64(u64 x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Rng {
  int kind;    // TWG_RNG_*
  u64 key;     // splitmix: mix64(seed ^ 0x6a09e667f3bcc909); philox: seed

  static Rng make(int kind, u64 seed) {
    Rng r;
    r.kind = kind;
    r.key = kind == TWG_RNG_PHILOX ? seed : mix64(seed ^ 0x6a09e667f3bcc909ULL);
    return r;
  }

  __device__ __forceinline__ u64 bits(u64 walk, u64 hop, u64 ordinal) const {
    if (kind == TWG_RNG_PHILOX) {
      u32 c0 = static_cast<u32>(walk), c1 = static_cast<u32>(hop), c2 = static_cast<u32>(ordinal);
      u32 c3 = static_cast<u32>(walk >> 32) ^ static_cast<u32>(hop >> 32) ^ static_cast<u32>(ordinal >> 32);
      u32 k0 = static_cast<u32>(key), k1 = static_cast<u32>(key >> 32);
#pragma unroll
      for (int r = 0; r < 10; ++r) {
        const u32 lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const u32 lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      return (static_cast<u64>(c1) << 32) | c0;
    }
    u64 h = mix64(key ^ walk);
    h = mix64(h ^ hop);
    return mix64(h ^ ordinal);
  }

  // rng.hpp:36-39: 53 random bits, exact conversion
  __device__ __forceinline__ double uniform(u64 walk, u64 hop, u64 ordinal) const {
    return __dmul_rn(__ull2double_rn(bits(walk, hop, ordinal) >> 11), 0x1.0p-53);
  }
};

}  // namespace twg
