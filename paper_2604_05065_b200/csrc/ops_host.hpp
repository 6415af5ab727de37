// Host-callable operator entry points (implemented in ops.cu).
#pragma once

#include <vector>

#include "apc_internal.hpp"

namespace apc {

// A x -> y (local rows), optional mu-tail: y[mloc + j] = mu * x[j]
void op_fwd(apc_mat& a, double mu, bool augmented, const double* x, double* y);
// A^T u -> y (local contribution), optional + mu * u[mloc + j]
void op_adj(apc_mat& a, double mu, bool augmented, const double* u, double* y);
// device CSR build from host CSC (matrix upload)
void upload_csc(apc_mat& a, const long long* colptr, const long long* rowidx, const double* val);

}  // namespace apc
