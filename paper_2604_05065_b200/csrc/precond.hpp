// Preconditioner construction (precond.cpp).
#pragma once

#include <functional>
#include <vector>

#include "host_dense.hpp"
#include "lsqr.hpp"

namespace apc {

// QrAccumulator (preconditioner.hpp:424-509): growing thin QR of R^T with one
// re-orthogonalisation pass per appended block.  Q lives on the device (the
// projections are cuBLAS GEMMs); the block factorisation is Householder on the
// host for small blocks and CholeskyQR2 on the device for tall ones.  T is
// small and stays on the host.
struct DevQrAcc {
  apc_ctx* ctx = nullptr;
  i64 rows = 0, k = 0, cap = 0;
  DBuf<double> q;  // rows x cap, column-major (first k columns valid)
  Vec t;           // k x k upper
  // append the b columns of the device block c (rows x b, column-major)
  void append(i64 m, i64 b, const double* c);
  void clear() { rows = k = 0; t.clear(); }
};

Vec gram_factor_sparse(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va);
// the same factor from the device rows of R (row-major l x n); the sparse host
// routine above is its fallback for a non-positive pivot
Vec gram_factor_rows_dev(apc_ctx* ctx, i64 n, i64 l, const double* r_rm, const std::vector<i64>& cp,
                         const std::vector<i64>& ri, const Vec& va);

struct BuildInputs {
  apc_ctx* ctx = nullptr;
  int variant = 0;  // 0 svd, 1 svd_free
  bool implicit = false;
  i64 m = 0, n = 0, l = 0;  // m: target rows (C's rows)
  double mu = 0.0, target_level = 0.0;
  std::function<Vec(const Vec&, i64)> core_solve_rm;  // U B for a row-major l x ncols B (DeviceCur, on the device)
  const Vec* block = nullptr;  // intersection A(I, J), l x l
  const Vec* t_r = nullptr;    // T_R (l x l upper)
  const double* q_dev = nullptr;  // explicit Q_R on the device (n x l, ld = n)
  Vec gram;                       // C^T C (l x l), from the device
  std::function<Vec()> c_dense;   // C densified on the host (QR fallback only)
  // R = A(I, :) as CSC of R^T (implicit)
  std::vector<i64> r_ptr, r_idx;
  Vec r_val;
};

struct PrecondInfo {
  double sigma_hat = 1.0, sigma_floor = 0.0;
  Vec sigma_cur, sigma_reg;
};

void build_precond(const BuildInputs& in, PrecondDev& p, PrecondInfo& info);

}  // namespace apc
