// Preconditioner construction per rebuild (preconditioner.hpp:138-396,
// 424-592) and its upload as the device form I + B K B^T / I + R^T G R that
// the LSQR loop applies (lsqr.cu).  The l x l algebra (Gram factors, core
// spectrum, middle operators) runs on the host with the restated reference
// routines; it is not index-affecting, so only the x / iteration
// parity bar applies to it.
#include <cmath>

#include "cur.hpp"
#include "precond.hpp"

namespace apc {

namespace {

double col_norm(i64 m, const double* c) {
  double s = 0.0;
  for (i64 i = 0; i < m; ++i) s += c[i] * c[i];
  return std::sqrt(s);
}

// chol_gram of a sparse CSC block (dense_factor.hpp:210-228)
Vec chol_gram_sparse(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va) {
  require(k >= 1, APC_INVALID_ARGUMENT, "chol_gram: empty matrix");
  Vec g(static_cast<size_t>(k * k), 0.0), work(static_cast<size_t>(m), 0.0);
  for (i64 j = 0; j < k; ++j) {
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) work[ri[p]] = va[p];
    for (i64 i = 0; i <= j; ++i) {
      double s = 0.0;
      for (i64 p = cp[i]; p < cp[i + 1]; ++p) s += va[p] * work[ri[p]];
      g[j * k + i] = s;
      g[i * k + j] = s;
    }
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) work[ri[p]] = 0.0;
  }
  return chol_upper(k, g, "chol_gram: non-positive pivot");
}

Vec densify_csc(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va) {
  Vec d(static_cast<size_t>(m * k), 0.0);
  for (i64 j = 0; j < k; ++j)
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) d[j * m + ri[p]] = va[p];
  return d;
}

// QrAccumulator::factor_checked (preconditioner.hpp:486-505)
QT factor_checked(i64 m, i64 k, Vec e, double scale) {
  Householder f = householder(m, k, std::move(e));
  for (i64 j = 0; j < k; ++j)
    if (std::fabs(f.a[j * m + j]) <= 1e-12 * scale)
      fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", j);
  QT r;
  r.m = m;
  r.k = k;
  r.q = thin_q(f);
  r.t = upper_of(f);
  normalise_signs(m, k, r.q, r.t);
  return r;
}

void upload_vec(apc_ctx* ctx, DBuf<double>& d, const Vec& h) {
  d.alloc(std::max<i64>(1, static_cast<i64>(h.size())));
  if (!h.empty())
    APC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
}

// host CSC (columns = rows of R) -> device CSR(R) (l x n) and CSR(R^T) (n x l)
void upload_r(apc_ctx* ctx, i64 n, i64 l, const std::vector<i64>& cp, const std::vector<i64>& ri,
              const Vec& va, PrecondDev& p) {
  const i64 nnz = cp[l];
  std::vector<int> rptr(l + 1), ridx(nnz);
  for (i64 i = 0; i <= l; ++i) rptr[i] = static_cast<int>(cp[i]);
  for (i64 q = 0; q < nnz; ++q) ridx[q] = static_cast<int>(ri[q]);
  // transpose: row j of R^T lists (i, R(i, j)) for i ascending
  std::vector<int> tptr(n + 1, 0), tidx(nnz);
  Vec tval(nnz);
  for (i64 q = 0; q < nnz; ++q) tptr[ri[q] + 1]++;
  for (i64 j = 0; j < n; ++j) tptr[j + 1] += tptr[j];
  std::vector<int> pos(tptr.begin(), tptr.end() - 1);
  for (i64 i = 0; i < l; ++i)
    for (i64 q = cp[i]; q < cp[i + 1]; ++q) {
      const int at = pos[ri[q]]++;
      tidx[at] = static_cast<int>(i);
      tval[at] = va[q];
    }
  auto up_i = [&](DBuf<int>& d, const std::vector<int>& h) {
    d.alloc(std::max<i64>(1, static_cast<i64>(h.size())));
    APC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
  };
  p.R.rows = l;
  p.R.cols = n;
  p.R.nnz = nnz;
  up_i(p.R.ptr, rptr);
  up_i(p.R.idx, ridx);
  upload_vec(ctx, p.R.val, va);
  p.RT.rows = n;
  p.RT.cols = l;
  p.RT.nnz = nnz;
  up_i(p.RT.ptr, tptr);
  up_i(p.RT.idx, tidx);
  upload_vec(ctx, p.RT.val, tval);
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// G = T^{-1} K T^{-T} for an implicit basis Q = R^T T^{-1} (l x l, T upper)
Vec conjugate_by_tinv(i64 l, const Vec& t, const Vec& K) {
  // X = T^{-1} K  (column by column), then G = X T^{-T} = (T^{-1} X^T)^T
  Vec X = K;
  for (i64 j = 0; j < l; ++j) tri_solve(l, t.data(), X.data() + j * l, false);
  Vec Xt = transpose(l, l, X);
  for (i64 j = 0; j < l; ++j) tri_solve(l, t.data(), Xt.data() + j * l, false);
  return transpose(l, l, Xt);
}

}  // namespace

// ---------------------------------------------------------------------------
void QrAcc::append(i64 m, i64 b, Vec c) {  // preconditioner.hpp:435-476
  require(b >= 1, APC_INVALID_ARGUMENT, "QrAccumulator: empty block");
  double scale = 0.0;
  for (i64 j = 0; j < b; ++j) scale = std::max(scale, col_norm(m, c.data() + j * m));
  if (k == 0) {
    QT qr = factor_checked(m, b, std::move(c), scale);
    rows = m;
    k = b;
    q = std::move(qr.q);
    t = std::move(qr.t);
    return;
  }
  require(m == rows, APC_DIMENSION_MISMATCH, "QrAccumulator: row count mismatch");
  const Vec qt = transpose(m, k, q);
  Vec p1 = matmul(k, m, b, qt, c);
  Vec qp = matmul(m, k, b, q, p1);
  Vec e = c;
  for (size_t s = 0; s < e.size(); ++s) e[s] -= qp[s];
  Vec p2 = matmul(k, m, b, qt, e);
  Vec qp2 = matmul(m, k, b, q, p2);
  for (size_t s = 0; s < e.size(); ++s) e[s] -= qp2[s];
  QT qr = factor_checked(m, b, std::move(e), scale);
  const i64 n0 = k, nt = k + b;
  Vec qn(static_cast<size_t>(m * nt));
  std::copy(q.begin(), q.end(), qn.begin());
  std::copy(qr.q.begin(), qr.q.end(), qn.begin() + m * n0);
  Vec tn(static_cast<size_t>(nt * nt), 0.0);
  for (i64 j = 0; j < n0; ++j)
    for (i64 i = 0; i <= j; ++i) tn[j * nt + i] = t[j * n0 + i];
  for (i64 j = 0; j < b; ++j)
    for (i64 i = 0; i < n0; ++i) tn[(n0 + j) * nt + i] = p1[j * n0 + i] + p2[j * n0 + i];
  for (i64 j = 0; j < b; ++j)
    for (i64 i = 0; i <= j; ++i) tn[(n0 + j) * nt + n0 + i] = qr.t[j * b + i];
  q = std::move(qn);
  t = std::move(tn);
  k = nt;
}

// gram_factor (preconditioner.hpp:143-150): Cholesky of C^T C, QR fallback
Vec gram_factor_dense(i64 m, i64 k, const Vec& c) {
  try {
    return chol_gram_dense(m, k, c.data());
  } catch (const Status& s) {
    if (s.code != APC_NOT_POSITIVE) throw;
    return thin_qr(m, k, c).t;
  }
}

Vec gram_factor_sparse(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va) {
  try {
    return chol_gram_sparse(m, k, cp, ri, va);
  } catch (const Status& s) {
    if (s.code != APC_NOT_POSITIVE) throw;
    return thin_qr(m, k, densify_csc(m, k, cp, ri, va)).t;
  }
}

// ---------------------------------------------------------------------------
void build_precond(const BuildInputs& in, PrecondDev& p, PrecondInfo& info) {
  const i64 l = in.l, n = in.n;
  require(l >= 1, APC_INVALID_ARGUMENT, "build_svd_precond: empty factors");
  apc_ctx* ctx = in.ctx;
  p = PrecondDev();
  p.n = n;
  p.l = l;
  // T_C = gram_factor(C)
  Vec t_c = in.c_sparse ? gram_factor_sparse(in.m, l, in.c_ptr, in.c_idx, in.c_val)
                        : gram_factor_dense(in.m, l, in.c_dense);
  Vec K;
  if (in.variant == 0) {
    // SVD form: M = T_C U T_R^T, small_svd(M) (preconditioner.hpp:158-192)
    Vec ut = in.core->solve_matrix(l, transpose(l, l, *in.t_r));
    Vec mm = matmul(l, l, l, t_c, ut);
    SvdH s = small_svd(l, l, mm);
    info.sigma_cur = s.sigma;
    info.sigma_reg.resize(l);
    for (i64 i = 0; i < l; ++i) info.sigma_reg[i] = std::sqrt(s.sigma[i] * s.sigma[i] + in.mu * in.mu);
    info.sigma_hat = info.sigma_reg.back();
    info.sigma_floor = info.sigma_cur.empty() ? 0.0 : info.sigma_cur.back();  // smallest_cur_sigma
    Vec d(l);
    for (i64 i = 0; i < l; ++i) d[i] = info.sigma_hat / info.sigma_reg[i] - 1.0;
    if (!in.implicit) {
      // V = Q_R V_M (explicit, n x l), K = diag(d)
      p.kind = 1;
      upload_vec(ctx, p.B, matmul(n, l, l, *in.q_r, s.v));
      K.assign(static_cast<size_t>(l * l), 0.0);
      for (i64 i = 0; i < l; ++i) K[i * l + i] = d[i];
      upload_vec(ctx, p.Kf, K);
      upload_vec(ctx, p.Ka, K);
    } else {
      // V = R^T T_R^{-1} V_M: G = W diag(d) W^T with W = T_R^{-1} V_M
      p.kind = 2;
      Vec W = s.v;
      for (i64 j = 0; j < l; ++j) tri_solve(l, in.t_r->data(), W.data() + j * l, false);
      Vec G(static_cast<size_t>(l * l), 0.0);
      for (i64 j = 0; j < l; ++j)
        for (i64 i = 0; i < l; ++i) {
          double acc = 0.0;
          for (i64 t = 0; t < l; ++t) acc += W[t * l + i] * d[t] * W[t * l + j];
          G[j * l + i] = acc;
        }
      upload_r(ctx, n, l, in.r_ptr, in.r_idx, in.r_val, p);
      upload_vec(ctx, p.Kf, G);
      upload_vec(ctx, p.Ka, G);
    }
  } else {
    // SVD-free: P^{-1} = sigma_hat Q_R M^{-1} Q_R^T + (I - Q_R Q_R^T),
    // M^{-1} = T_R^{-T} B T_C^{-1}  (preconditioner.hpp:279-318)
    info.sigma_hat = in.target_level;
    info.sigma_floor = in.target_level;
    Vec Minv(static_cast<size_t>(l * l), 0.0);
    Vec e(l), bw(l);
    for (i64 kcol = 0; kcol < l; ++kcol) {
      std::fill(e.begin(), e.end(), 0.0);
      e[kcol] = 1.0;
      tri_solve(l, t_c.data(), e.data(), false);
      for (i64 i = 0; i < l; ++i) {
        double acc = 0.0;
        for (i64 t = 0; t < l; ++t) acc += (*in.block)[t * l + i] * e[t];
        bw[i] = acc;
      }
      tri_solve(l, in.t_r->data(), bw.data(), true);
      for (i64 i = 0; i < l; ++i) Minv[kcol * l + i] = bw[i];
    }
    Vec Kf(static_cast<size_t>(l * l)), Ka(static_cast<size_t>(l * l));
    for (i64 j = 0; j < l; ++j)
      for (i64 i = 0; i < l; ++i) {
        Kf[j * l + i] = info.sigma_hat * Minv[j * l + i] - (i == j ? 1.0 : 0.0);
        Ka[j * l + i] = info.sigma_hat * Minv[i * l + j] - (i == j ? 1.0 : 0.0);
      }
    // the device keeps the middle operators row-major (warp per output row)
    if (!in.implicit) {
      p.kind = 1;
      upload_vec(ctx, p.B, *in.q_r);
      upload_vec(ctx, p.Kf, transpose(l, l, Kf));
      upload_vec(ctx, p.Ka, transpose(l, l, Ka));
    } else {
      p.kind = 2;
      upload_r(ctx, n, l, in.r_ptr, in.r_idx, in.r_val, p);
      upload_vec(ctx, p.Kf, transpose(l, l, conjugate_by_tinv(l, *in.t_r, Kf)));
      upload_vec(ctx, p.Ka, transpose(l, l, conjugate_by_tinv(l, *in.t_r, Ka)));
    }
  }
  p.sigma_hat = info.sigma_hat;
  p.sigma_floor = info.sigma_floor;
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace apc
