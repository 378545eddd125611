// Counter-based RNG shared by the host C++ layer and the sm_100a kernels.
//
// Same algorithm and constants as the reference's RngStream
// (/root/reference/proj/include/dtsim/rng.hpp:10-61): a splitmix64 finaliser,
// fork(label) sub-streams, bits(a, b, c) = three chained mixes, uniform =
// ((bits >> 11) + 0.5) * 2^-53.  Integer-only up to the final exact
// int->double conversion, so device and host draws are bit-identical.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define DTG_HD __host__ __device__ __forceinline__
#else
#define DTG_HD inline
#endif

namespace dtg {

DTG_HD std::uint64_t rng_mix(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

DTG_HD std::uint64_t rng_fork(std::uint64_t seed, std::uint64_t label) {
  return rng_mix(seed ^ rng_mix(label ^ 0x8e9b5c1d3a7f2406ULL));
}

DTG_HD std::uint64_t rng_bits(std::uint64_t seed, std::uint64_t a,
                              std::uint64_t b, std::uint64_t c) {
  std::uint64_t h = rng_mix(seed ^ rng_mix(a));
  h = rng_mix(h ^ rng_mix(b ^ 0x6a09e667f3bcc909ULL));
  h = rng_mix(h ^ rng_mix(c ^ 0xbb67ae8584caa73bULL));
  return h;
}

/// bits(a, b, c) split into its three chained stages, so a common prefix can be
/// reused across many draws: bits(a, b, c) == rng_final(rng_prefix2(
/// rng_prefix1(seed, a), b), c).
DTG_HD std::uint64_t rng_prefix1(std::uint64_t seed, std::uint64_t a) {
  return rng_mix(seed ^ rng_mix(a));
}
DTG_HD std::uint64_t rng_prefix2(std::uint64_t h1, std::uint64_t b) {
  return rng_mix(h1 ^ rng_mix(b ^ 0x6a09e667f3bcc909ULL));
}
DTG_HD std::uint64_t rng_final(std::uint64_t h2, std::uint64_t c) {
  return rng_mix(h2 ^ rng_mix(c ^ 0xbb67ae8584caa73bULL));
}
DTG_HD double rng_unit(std::uint64_t bits) {
  return (static_cast<double>(bits >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/// Uniform strictly inside (0, 1).
DTG_HD double rng_uniform(std::uint64_t seed, std::uint64_t a, std::uint64_t b,
                          std::uint64_t c) {
  return (static_cast<double>(rng_bits(seed, a, b, c) >> 11) + 0.5) *
         (1.0 / 9007199254740992.0);
}

/// Sub-stream labels (rng.hpp:53-61).
namespace lane {
constexpr std::uint64_t kParamSample = 1;
constexpr std::uint64_t kVirtualCoin = 2;
constexpr std::uint64_t kGumbelLink = 3;
constexpr std::uint64_t kGumbelMerge = 4;
constexpr std::uint64_t kObsNoise = 5;
constexpr std::uint64_t kObsCoverage = 6;
constexpr std::uint64_t kIteration = 7;
}  // namespace lane

/// Host-side stream object with the reference RngStream interface.
class RngStream {
 public:
  explicit RngStream(std::uint64_t seed) : seed_(seed) {}
  RngStream fork(std::uint64_t label) const {
    return RngStream(rng_fork(seed_, label));
  }
  std::uint64_t bits(std::uint64_t a, std::uint64_t b = 0,
                     std::uint64_t c = 0) const {
    return rng_bits(seed_, a, b, c);
  }
  double uniform(std::uint64_t a, std::uint64_t b = 0,
                 std::uint64_t c = 0) const {
    return rng_uniform(seed_, a, b, c);
  }
  double uniform_in(double lo, double hi, std::uint64_t a, std::uint64_t b = 0,
                    std::uint64_t c = 0) const {
    return lo + (hi - lo) * uniform(a, b, c);
  }
  std::uint64_t seed() const { return seed_; }

 private:
  std::uint64_t seed_;
};

}  // namespace dtg
