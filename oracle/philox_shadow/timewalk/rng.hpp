#pragma once
// TEST INFRASTRUCTURE ONLY. Shadow of the reference's `timewalk/rng.hpp`
// (rng.hpp:22-43) used to build the "Philox oracle": the unmodified reference
// sources compiled with this directory FIRST on the include path, so every
// CounterRng draw in walk_engine.cpp (:88, :211, :350, :381) comes from
// Philox4x32-10 keyed by (seed; walk, hop, ordinal) instead of splitmix.
// Same class name and member signatures; mix64 is kept for any other user.
// The product's device Philox (paper_2605_16182_b200/csrc/rng.cuh) implements
// the identical function, so walks are bit-exact against this oracle.

#include <cstdint>

namespace timewalk {

constexpr std::uint64_t mix64(std::uint64_t x) noexcept {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

class CounterRng {
 public:
  CounterRng() = default;
  explicit CounterRng(std::uint64_t seed) : key_(seed) {}

  /// Philox4x32-10. counter = (lo32 walk, lo32 hop, lo32 ordinal,
  /// hi32 walk ^ hi32 hop ^ hi32 ordinal), key = (lo32 seed, hi32 seed);
  /// result = (out.y << 32) | out.x.
  [[nodiscard]] std::uint64_t bits(std::uint64_t walk, std::uint64_t hop,
                                   std::uint64_t ordinal) const noexcept {
    std::uint32_t c0 = static_cast<std::uint32_t>(walk);
    std::uint32_t c1 = static_cast<std::uint32_t>(hop);
    std::uint32_t c2 = static_cast<std::uint32_t>(ordinal);
    std::uint32_t c3 = static_cast<std::uint32_t>(walk >> 32) ^
                       static_cast<std::uint32_t>(hop >> 32) ^
                       static_cast<std::uint32_t>(ordinal >> 32);
    std::uint32_t k0 = static_cast<std::uint32_t>(key_);
    std::uint32_t k1 = static_cast<std::uint32_t>(key_ >> 32);
    for (int r = 0; r < 10; ++r) {
      const std::uint64_t p0 = static_cast<std::uint64_t>(0xD2511F53u) * c0;
      const std::uint64_t p1 = static_cast<std::uint64_t>(0xCD9E8D57u) * c2;
      const std::uint32_t hi0 = static_cast<std::uint32_t>(p0 >> 32), lo0 = static_cast<std::uint32_t>(p0);
      const std::uint32_t hi1 = static_cast<std::uint32_t>(p1 >> 32), lo1 = static_cast<std::uint32_t>(p1);
      c0 = hi1 ^ c1 ^ k0;
      c1 = lo1;
      c2 = hi0 ^ c3 ^ k1;
      c3 = lo0;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    return (static_cast<std::uint64_t>(c1) << 32) | c0;
  }

  [[nodiscard]] double uniform(std::uint64_t walk, std::uint64_t hop,
                               std::uint64_t ordinal) const noexcept {
    return static_cast<double>(bits(walk, hop, ordinal) >> 11) * 0x1.0p-53;
  }

 private:
  std::uint64_t key_{0};
};

}  // namespace timewalk
