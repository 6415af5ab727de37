// Seeded host randomness, bit-identical to the reference generator
// (/root/reference/proj/include/aplicur/rng.hpp:12-78): splitmix64 seed
// derivation over std::mt19937_64, 53-bit uniforms, Box-Muller without spare
// caching, unbiased rejection sampling, low-bit Rademacher signs.  Device
// kernels never draw random numbers: the embedding S and the spectral probes
// are generated here and uploaded.
#pragma once

#include <algorithm>
#include <exception>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

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

  // the same distributions as pure functions of the raw 64-bit draws, so a
  // stream consumed in a fixed pattern can be generated sequentially (fast)
  // and transformed in parallel with identical results
  static double uniform_of(std::uint64_t d) { return static_cast<double>(d >> 11) * 0x1.0p-53; }
  static double gaussian_of(std::uint64_t d1, std::uint64_t d2) {
    const double a = 1.0 - uniform_of(d1);
    const double b = uniform_of(d2);
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586476925286766559 * b);
  }
  // below(n) when the first draw is accepted (rejection probability < n / 2^64)
  static bool below_accepts(std::uint64_t d, std::uint64_t n) {
    return d < ~std::uint64_t{0} - (~std::uint64_t{0} % n);
  }

 private:
  std::mt19937_64 eng_;
};

// run f(begin, end) over [0, n) on the host's cores (a persistent worker pool,
// host_pool.cpp) when the total work (n * unit_cost, rough flop units) is
// worth it; exceptions thrown by f are rethrown on the calling thread.
// NOTE: this header is compiled both by nvcc (.cu) and g++ (.cpp).  Closure
// types of capturing lambdas are not guaranteed to have the same layout
// under both front ends while inline instantiations are merged by the
// linker, so callers in shared headers pass named functors, never lambdas.
int host_pool_workers();
void host_pool_run(i64 n, int nt, void (*fn)(void*, i64, i64), void* ctx);

template <class F>
void host_range_invoke(void* ctx, i64 b, i64 e) {
  (*static_cast<const F*>(ctx))(b, e);
}

template <class F>
void host_parallel_for(i64 n, const F& f, i64 unit_cost = 1) {
  static const bool serial = std::getenv("APC_HOST_SERIAL") != nullptr;
  const i64 nt = std::min<i64>(host_pool_workers() + 1, n);
  if (serial || n * unit_cost < 30000 || nt < 2) {
    f(i64{0}, n);
    return;
  }
  host_pool_run(n, static_cast<int>(nt), &host_range_invoke<F>, const_cast<void*>(static_cast<const void*>(&f)));
}

// n Gaussians of the stream (each consumes exactly two draws), transformed in parallel
struct GaussFromRaw {
  const std::uint64_t* raw;
  double* out;
  double scale;
  bool scaled;
  void operator()(i64 b, i64 e) const {
    for (i64 i = b; i < e; ++i) {
      const double g = HostRng::gaussian_of(raw[2 * i], raw[2 * i + 1]);
      out[i] = scaled ? scale * g : g;
    }
  }
};

inline void fill_gaussians(HostRng& rng, double* out, i64 n, double scale = 1.0, bool scaled = false) {
  std::vector<std::uint64_t> raw(static_cast<size_t>(2 * n));
  for (auto& d : raw) d = rng.bits();
  host_parallel_for(n, GaussFromRaw{raw.data(), out, scale, scaled}, 64);
}

}  // namespace apc
