// Host-side problem instance behind the opaque apc_problem handle: a
// generated BASELINE input (problems.cpp) or a Matrix Market file (io.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "apc_internal.hpp"

struct apc_problem {
  apc::i64 m = 0, n = 0;
  bool sparse = false;
  std::vector<double> dense;                 // column-major
  std::vector<std::int64_t> colptr, rowidx;  // CSC (reference layout)
  std::vector<double> vals;
  std::vector<double> b;
};
