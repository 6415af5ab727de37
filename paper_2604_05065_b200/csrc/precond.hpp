// Preconditioner construction (precond.cpp).
#pragma once

#include <vector>

#include "host_dense.hpp"
#include "lsqr.hpp"

namespace apc {

// QrAccumulator (preconditioner.hpp:424-509): growing thin QR of R^T with one
// re-orthogonalisation pass per appended block.
struct QrAcc {
  i64 rows = 0, k = 0;
  Vec q, t;  // rows x k, k x k
  void append(i64 m, i64 b, Vec newcols);
  void clear() { rows = k = 0; q.clear(); t.clear(); }
};

Vec gram_factor_dense(i64 m, i64 k, const Vec& c);
Vec gram_factor_sparse(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va);

struct BuildInputs {
  apc_ctx* ctx = nullptr;
  int variant = 0;  // 0 svd, 1 svd_free
  bool implicit = false;
  i64 m = 0, n = 0, l = 0;
  double mu = 0.0, target_level = 0.0;
  const CoreFactorH* core = nullptr;
  const Vec* block = nullptr;  // intersection A(I, J), l x l
  const Vec* t_r = nullptr;    // T_R (l x l upper)
  const Vec* q_r = nullptr;    // explicit Q_R (n x l)
  // C = A(:, J)
  bool c_sparse = false;
  Vec c_dense;
  std::vector<i64> c_ptr, c_idx;
  Vec c_val;
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
