#pragma once
// Counter-based RNG (reference: proj/include/trioalign/rng.hpp:12-43).  The
// dataset generator and the seeded tests depend on its exact bytes, so the
// stream derivation, the SplitMix64 finalizer constants, the fixed-point
// bounded draw and the 53-bit unit draw are the reference's.  The engine's
// parallel generator (csrc/core/dataset.cpp) uses the same recipe per
// triplet stream (seed, index + 1).
#include <cstdint>

namespace trioalign {

class CounterRng {
 public:
  explicit CounterRng(uint64_t seed, uint64_t stream = 0)
      : key_(finalize(seed ^ kGolden) ^ finalize(stream ^ kMul1)) {}

  // value(n) = finalize(key + n * golden), n = 1, 2, ...
  uint64_t next() {
    ++counter_;
    return finalize(key_ + counter_ * kGolden);
  }

  // uniform in [0, n): high 64 bits of next() * n (0 when n == 0)
  uint64_t below(uint64_t n) {
    if (n == 0) return 0;
    const unsigned __int128 wide = static_cast<unsigned __int128>(next()) * n;
    return static_cast<uint64_t>(wide >> 64);
  }

  // uniform in [lo, hi] (inclusive)
  int64_t range(int64_t lo, int64_t hi) { return lo + static_cast<int64_t>(below(static_cast<uint64_t>(hi - lo + 1))); }

  // uniform in [0, 1) with 53 random bits
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

  char base() { return "ACGT"[below(4)]; }

 private:
  static constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
  static constexpr uint64_t kMul1 = 0xbf58476d1ce4e5b9ull;
  static constexpr uint64_t kMul2 = 0x94d049bb133111ebull;

  static uint64_t finalize(uint64_t z) {
    z ^= z >> 30;
    z *= kMul1;
    z ^= z >> 27;
    z *= kMul2;
    return z ^ (z >> 31);
  }

  uint64_t key_;
  uint64_t counter_ = 0;
};

}  // namespace trioalign
