// Fused dense operator pair of one LSQR iteration (dense_pair.cu):
//   u <- A z - alpha * u/beta,  ||u||^2,  g = A^T u
// with A read from HBM ONCE.  Replaces dense_fwd_kernel + dense_adj_kernel
// (Matrix::matvec + Matrix::matvec_transpose, matrix.hpp:151-195, as lsqr_solve
// calls them back to back, lsqr.hpp:139-150) for matrices of 64 MB or more.
#pragma once

#include "apc_internal.hpp"

namespace apc {

struct LsqrState;

// true when `a` is dense, large enough and the panel copy could be built
// (built on the first call; APC_DENSE_PAIR=0 turns the path off, =1 forces it
// for every shape the kernel supports)
bool dense_pair_ready(apc_mat& a);
// u (mloc, in/out), g (n + 1: A^T u and ||u||^2), st == nullptr: u <- A z
void launch_dense_pair(apc_mat& a, const double* z, double* u, const LsqrState* st, double* g, const int* done);
// *out = ||y||^2 (one CTA, fixed order): the unfused leg of apc_op_pair_dev
void pair_norm2(apc_ctx* ctx, const double* y, long long m, double* out);

}  // namespace apc
