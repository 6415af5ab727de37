// Device generation of the std::mt19937_64 raw stream (rng_dev.cu).
#pragma once

#include <cstdint>

#include "apc_internal.hpp"

namespace apc {

// true once the host replica of the engine matched std::mt19937_64 (checked
// once per process); callers fall back to the host stream otherwise
bool mt64_device_ok();
// the first `count` outputs of std::mt19937_64(seed) into d_out (device)
void mt64_stream_device(apc_ctx* ctx, std::uint64_t seed, i64 count, std::uint64_t* d_out);

}  // namespace apc
