// Phase-boundary vector helpers (vec.cu).
#pragma once

#include "apc_internal.hpp"

namespace apc {

struct VecWork {
  double mu = 0.0;
  DBuf<double> ax, part, scalar;
  VecWork(apc_mat& a, double mu);
};

// rhs = [b; 0] - A_mu x on the local rows (+ tail); returns ||rhs||^2 summed
// over ranks.  rhs may be null (norm only).
double residual(apc_mat& a, VecWork& w, const double* x, const double* b_local, double* rhs);
void axpy(apc_ctx* ctx, double* x, const double* d, long long n);

}  // namespace apc
