// The raw 64-bit stream of std::mt19937_64 generated on the device.
//
// HostRng (host_rng.hpp, rng.hpp:12-78) seeds std::mt19937_64; the sketch
// embedding consumes millions of its draws strictly in order, which on the
// host is a sequential 3-5 ns/draw loop.  MT19937-64's twist of its 312-word
// state splits into two data-parallel halves (words 0..155 read only old
// words; words 156..311 read old words and the new first half), so one CTA
// regenerates the state 312 words at a time and tempers them in parallel.
// The seeding (the standard's linear recurrence) runs on the host, and a
// replica of the whole engine is checked against std::mt19937_64 once per
// process before the device stream is trusted (mt64_device_ok()).
#include <cstdint>
#include <random>
#include <vector>

#include "apc_internal.hpp"
#include "rng_dev.hpp"

namespace apc {
namespace {

constexpr int kN = 312, kM = 156;
constexpr std::uint64_t kA = 0xB5026F5AA96619E9ULL;
constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;

__host__ __device__ __forceinline__ std::uint64_t temper(std::uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__host__ __device__ __forceinline__ std::uint64_t twist_word(std::uint64_t cur, std::uint64_t next, std::uint64_t far) {
  const std::uint64_t y = (cur & kUpper) | (next & kLower);
  return far ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
}

// std::mt19937_64::seed(value) (the standard's initialisation recurrence)
void seed_state(std::uint64_t seed, std::uint64_t* mt) {
  mt[0] = seed;
  for (int i = 1; i < kN; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
}

// host replica of the engine (checked against the standard library)
struct Replica {
  std::uint64_t mt[kN];
  int idx = kN;
  explicit Replica(std::uint64_t seed) { seed_state(seed, mt); }
  std::uint64_t next() {
    if (idx >= kN) {
      std::uint64_t nw[kN];
      for (int k = 0; k < kN - kM; ++k) nw[k] = twist_word(mt[k], mt[k + 1], mt[k + kM]);
      for (int k = kN - kM; k < kN - 1; ++k) nw[k] = twist_word(mt[k], mt[k + 1], nw[k + kM - kN]);
      nw[kN - 1] = twist_word(mt[kN - 1], nw[0], nw[kM - 1]);
      for (int k = 0; k < kN; ++k) mt[k] = nw[k];
      idx = 0;
    }
    return temper(mt[idx++]);
  }
};

// one CTA: twist the state (two parallel halves), temper, store 312 draws
__global__ void __launch_bounds__(kN) mt64_stream_kernel(const std::uint64_t* __restrict__ state0, long long count,
                                                       std::uint64_t* __restrict__ out) {
  __shared__ std::uint64_t mt[kN];
  const int k = threadIdx.x;
  mt[k] = state0[k];
  __syncthreads();
  for (long long base = 0; base < count; base += kN) {
    // words 0..155: old words only
    std::uint64_t v = 0;
    if (k < kN - kM) v = twist_word(mt[k], mt[k + 1], mt[k + kM]);
    __syncthreads();
    if (k < kN - kM) mt[k] = v;
    __syncthreads();
    // words 156..311: old words and the new first half
    if (k >= kN - kM) v = twist_word(mt[k], k + 1 < kN ? mt[k + 1] : mt[0], mt[k + kM - kN]);
    __syncthreads();
    if (k >= kN - kM) mt[k] = v;
    __syncthreads();
    if (base + k < count) out[base + k] = temper(mt[k]);
  }
}

}  // namespace

bool mt64_device_ok() {
  static const bool ok = [] {
    for (std::uint64_t seed : {0ULL, 1ULL, 5489ULL, 0x9e3779b97f4a7c15ULL, 20260417ULL}) {
      std::mt19937_64 ref(seed);
      Replica rep(seed);
      for (int i = 0; i < 4 * kN + 7; ++i)
        if (ref() != rep.next()) return false;
    }
    return true;
  }();
  return ok;
}

void mt64_stream_device(apc_ctx* ctx, std::uint64_t seed, i64 count, std::uint64_t* d_out) {
  std::uint64_t st[kN];
  seed_state(seed, st);
  DBuf<std::uint64_t> d_st(kN);
  APC_CUDA(cudaMemcpyAsync(d_st.p, st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream));
  mt64_stream_kernel<<<1, kN, 0, ctx->stream>>>(d_st.p, count, d_out);
  ctx->launches++;
  APC_CUDA(cudaGetLastError());
  APC_CUDA(cudaStreamSynchronize(ctx->stream));  // d_st goes out of scope
}

}  // namespace apc
