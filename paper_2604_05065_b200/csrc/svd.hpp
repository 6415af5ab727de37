// Device one-sided Jacobi SVD of a small square matrix (svd.cu).
#pragma once

#include "host_dense.hpp"

namespace apc {

// sigma (n, nonincreasing) and V (n x n, column-major) of the n x n matrix M
void device_jacobi_svd(apc_ctx* ctx, i64 n, const Vec& M, Vec& sigma, Vec& V);

}  // namespace apc
