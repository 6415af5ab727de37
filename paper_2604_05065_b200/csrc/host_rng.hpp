// Seeded host randomness, bit-identical to the reference generator
// (/root/reference/proj/include/aplicur/rng.hpp:12-78): splitmix64 seed
// derivation over std::mt19937_64, 53-bit uniforms, Box-Muller without spare
// caching, unbiased rejection sampling, low-bit Rademacher signs.  Device
// kernels never draw random numbers: the embedding S and the spectral probes
// are generated here and uploaded.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

#include "apc_internal.hpp"

namespace apc {

inline std::uint64_t splitmix(std::uint64_t z) {  // rng.hpp:15-20
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

enum class Stream : std::uint64_t { sketch = 1, probes = 2, problem = 3, rhs = 4, user = 5 };

class HostRng {
 public:
  explicit HostRng(std::uint64_t seed) : eng_(splitmix(seed)) {}
  HostRng(std::uint64_t root, Stream s, std::uint64_t index = 0)
      : eng_(splitmix(splitmix(root ^ (0x51ed2701a3c5e1bdULL * static_cast<std::uint64_t>(s))) +
                      index)) {}

  std::uint64_t bits() { return eng_(); }
  double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double gaussian() {
    const double a = 1.0 - uniform();
    const double b = uniform();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586476925286766559 * b);
  }
  std::uint64_t below(std::uint64_t n) {
    require(n > 0, APC_INVALID_ARGUMENT, "Rng::below: n must be positive");
    const std::uint64_t lim = ~std::uint64_t{0} - (~std::uint64_t{0} % n);
    std::uint64_t v;
    do {
      v = eng_();
    } while (v >= lim);
    return v % n;
  }
  double sign() { return (eng_() & 1ULL) ? 1.0 : -1.0; }

 private:
  std::mt19937_64 eng_;
};

}  // namespace apc
