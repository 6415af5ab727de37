// Preconditioner construction per rebuild (preconditioner.hpp:138-396,
// 424-592) and its upload as the device form I + B K B^T / I + R^T G R that
// the LSQR loop applies (lsqr.cu).  Everything runs on the device: the tall
// products (C^T C, Q^T c, Q p, Q_R V_M) on the DMMA GEMM (blas.cu), the l x l
// algebra (Cholesky of the Gram matrices, the core solve U T_R^T, the core
// spectrum by Jacobi, the middle operators' triangular solves and products)
// on dense_small.cu / svd.cu / the CoreFactor kernels.  The host keeps the
// l^2 bookkeeping (transposes, diagonal scalings) and two rare fallbacks: QR
// when a Gram matrix is not positive definite, Householder for a small
// nearly dependent QrAccumulator block.  None of it is index-affecting
// (SURVEY.md G8): only the x / iteration parity bar applies.
#include <cmath>
#include <memory>

#include "blas.hpp"
#include "cur.hpp"
#include "dense_small.hpp"
#include "precond.hpp"
#include "svd.hpp"

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

}  // namespace

// T_R with T_R^T T_R = R R^T from the device rows of R (row-major l x n ==
// column-major n x l): Gram by the DMMA SYRK, Cholesky on the device; a
// non-positive pivot falls back to the host QR of the sparse rows
Vec gram_factor_rows_dev(apc_ctx* ctx, i64 n, i64 l, const double* r_rm, const std::vector<i64>& cp,
                         const std::vector<i64>& ri, const Vec& va) {
  require(l >= 1, APC_INVALID_ARGUMENT, "chol_gram: empty matrix");
  DBuf<double> G(l * l);
  dsyrk_t(ctx, l, n, 1.0, r_rm, n, 0.0, G.p, l);
  if (dpotrf_upper_dev(ctx, l, G.p) >= 0) return gram_factor_sparse(n, l, cp, ri, va);
  Vec t(static_cast<size_t>(l * l));
  copy_sync(ctx->stream, t.data(), G.p, sizeof(double) * l * l, cudaMemcpyDeviceToHost);
  return t;
}

namespace {

Vec densify_csc(i64 m, i64 k, const std::vector<i64>& cp, const std::vector<i64>& ri, const Vec& va) {
  Vec d(static_cast<size_t>(m * k), 0.0);
  for (i64 j = 0; j < k; ++j)
    for (i64 p = cp[j]; p < cp[j + 1]; ++p) d[j * m + ri[p]] = va[p];
  return d;
}

void upload_vec(apc_ctx* ctx, DBuf<double>& d, const Vec& h) {
  d.alloc(std::max<i64>(1, static_cast<i64>(h.size())));
  if (!h.empty())
    APC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
}

Vec download_vec(apc_ctx* ctx, const double* d, i64 n) {
  Vec h(static_cast<size_t>(n));
  copy_sync(ctx->stream, h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  return h;
}

// host CSC (columns = rows of R) -> device CSR(R) (l x n) and CSR(R^T) (n x l)
void upload_r(apc_ctx* ctx, i64 n, i64 l, const std::vector<i64>& cp, const std::vector<i64>& ri,
              const Vec& va, PrecondDev& p) {
  const i64 nnz = cp[l];
  std::vector<int> rptr(l + 1), ridx(nnz);
  for (i64 i = 0; i <= l; ++i) rptr[i] = static_cast<int>(cp[i]);
  for (i64 q = 0; q < nnz; ++q) ridx[q] = static_cast<int>(ri[q]);
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
    if (!h.empty())
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
Vec conjugate_by_tinv(apc_ctx* ctx, i64 l, const Vec& t, const Vec& K) {
  const Vec X = dtri_solve_cols(ctx, l, t, K, l, false);
  const Vec Xt = dtri_solve_cols(ctx, l, t, transpose(l, l, X), l, false);
  return transpose(l, l, Xt);
}

// mirror an upper-filled square matrix into a full symmetric one
void symmetrize_upper(i64 n, Vec& g) {
  for (i64 j = 0; j < n; ++j)
    for (i64 i = j + 1; i < n; ++i) g[j * n + i] = g[i * n + j];
}

// upper R with R^T R = e^T e for a device block (CholeskyQR, e <- e R^{-1})
Vec cholqr_step(apc_ctx* ctx, i64 m, i64 b, double* e) {
  DBuf<double> G(b * b);
  dsyrk_t(ctx, b, m, 1.0, e, m, 0.0, G.p, b);
  const int bad = dpotrf_upper_dev(ctx, b, G.p);  // G <- R (upper), on the device
  if (bad >= 0) fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", bad);
  dtrsm_right_upper(ctx, m, b, G.p, b, e, m);
  Vec r = download_vec(ctx, G.p, b * b);
  return r;
}

}  // namespace

// ---------------------------------------------------------------------------
void DevQrAcc::append(i64 m, i64 b, const double* c) {  // preconditioner.hpp:435-476
  require(b >= 1, APC_INVALID_ARGUMENT, "QrAccumulator: empty block");
  cudaStream_t st = ctx->stream;
  // incoming column scale (max column norm of the new block)
  Vec ch = download_vec(ctx, c, m * b);
  double scale = 0.0;
  for (i64 j = 0; j < b; ++j) scale = std::max(scale, col_norm(m, ch.data() + j * m));
  if (k > 0) require(m == rows, APC_DIMENSION_MISMATCH, "QrAccumulator: row count mismatch");
  DBuf<double> e(m * b);
  APC_CUDA(cudaMemcpyAsync(e.p, c, sizeof(double) * m * b, cudaMemcpyDeviceToDevice, st));
  Vec p1(static_cast<size_t>(k * b), 0.0), p2(static_cast<size_t>(k * b), 0.0);
  if (k > 0) {  // two projection passes: e = c - Q Q^T c, then once more
    DBuf<double> P(k * b);
    dgemm(ctx, true, false, k, b, m, 1.0, q.p, m, e.p, m, 0.0, P.p, k);
    dgemm(ctx, false, false, m, b, k, -1.0, q.p, m, P.p, k, 1.0, e.p, m);
    p1 = download_vec(ctx, P.p, k * b);
    dgemm(ctx, true, false, k, b, m, 1.0, q.p, m, e.p, m, 0.0, P.p, k);
    dgemm(ctx, false, false, m, b, k, -1.0, q.p, m, P.p, k, 1.0, e.p, m);
    p2 = download_vec(ctx, P.p, k * b);
  }
  // factor the block: CholeskyQR2 on the device; a small block whose Gram
  // matrix is not numerically positive definite (condition number beyond
  // ~1e8) goes to Householder on the host, which still tells a nearly
  // dependent block (|R_jj| <= 1e-12 scale) from a merely ill-conditioned one
  Vec rb;
  const bool small = static_cast<double>(m) * b * b <= 2e8;
  DBuf<double> e0;
  if (small) {
    e0.alloc(m * b);
    APC_CUDA(cudaMemcpyAsync(e0.p, e.p, sizeof(double) * m * b, cudaMemcpyDeviceToDevice, st));
  }
  bool done = false;
  try {
    Vec r1 = cholqr_step(ctx, m, b, e.p);
    Vec r2 = cholqr_step(ctx, m, b, e.p);
    rb = dmatmul(ctx, b, b, b, r2, r1);
    done = true;
  } catch (const Status& s) {
    if (!small || s.code != APC_RANK_DEFICIENT) throw;
  }
  if (done) {
    for (i64 j = 0; j < b; ++j)
      if (std::fabs(rb[j * b + j]) <= 1e-12 * scale) fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", j);
  } else {
    Vec eh = download_vec(ctx, e0.p, m * b);
    Householder f = householder(m, b, std::move(eh));
    for (i64 j = 0; j < b; ++j)
      if (std::fabs(f.a[j * m + j]) <= 1e-12 * scale) fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", j);
    Vec qe = thin_q(f);
    rb = upper_of(f);
    normalise_signs(m, b, qe, rb);
    APC_CUDA(cudaMemcpyAsync(e.p, qe.data(), sizeof(double) * m * b, cudaMemcpyHostToDevice, st));
    APC_CUDA(cudaStreamSynchronize(st));
  }
  // Q <- [Q, q_e]
  if (k + b > cap) {
    const i64 ncap = std::max(2 * cap, k + b);
    DBuf<double> nq(m * ncap);
    if (k > 0) APC_CUDA(cudaMemcpyAsync(nq.p, q.p, sizeof(double) * m * k, cudaMemcpyDeviceToDevice, st));
    q = std::move(nq);
    cap = ncap;
  }
  APC_CUDA(cudaMemcpyAsync(q.p + m * k, e.p, sizeof(double) * m * b, cudaMemcpyDeviceToDevice, st));
  // T <- [[T, p1 + p2], [0, R_e]]
  const i64 nt = k + b;
  Vec tn(static_cast<size_t>(nt * nt), 0.0);
  for (i64 j = 0; j < k; ++j)
    for (i64 i = 0; i <= j; ++i) tn[j * nt + i] = t[j * k + i];
  for (i64 j = 0; j < b; ++j)
    for (i64 i = 0; i < k; ++i) tn[(k + j) * nt + i] = p1[j * k + i] + p2[j * k + i];
  for (i64 j = 0; j < b; ++j)
    for (i64 i = 0; i <= j; ++i) tn[(k + j) * nt + k + i] = rb[j * b + i];
  t = std::move(tn);
  rows = m;
  k = nt;
  APC_CUDA(cudaStreamSynchronize(st));
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
  // T_C = gram_factor(C): Cholesky of the device Gram, QR fallback (preconditioner.hpp:143-150)
  Vec t_c;
  std::unique_ptr<ProfScope> ps(new ProfScope("pre.chol"));
  try {
    t_c = dchol_upper(ctx, l, in.gram, "chol_gram: non-positive pivot");
  } catch (const Status& s) {
    if (s.code != APC_NOT_POSITIVE) throw;
    t_c = thin_qr(in.m, l, in.c_dense()).t;
  }
  if (in.variant == 0) {
    // SVD form: M = T_C U T_R^T, small_svd(M) (preconditioner.hpp:158-192)
    ps.reset(new ProfScope("pre.core_matmul"));
    // U T_R^T on the device: T_R's column-major bytes are T_R^T row-major;
    // the row-major result transposed is the column-major product
    Vec ut = transpose(l, l, in.core_solve_rm(*in.t_r, l));
    Vec mm = dmatmul(ctx, l, l, l, t_c, ut);
    ps.reset(new ProfScope("pre.svd"));
    require(l <= 4096, APC_INVALID_ARGUMENT, "small_svd: dimension exceeds the small-problem cap");
    SvdH s;
    s.m = s.n = l;
    device_jacobi_svd(ctx, l, mm, s.sigma, s.v);  // parallel-order one-sided Jacobi (svd.cu)
    ps.reset(new ProfScope("pre.G"));
    info.sigma_cur = s.sigma;
    info.sigma_reg.resize(l);
    for (i64 i = 0; i < l; ++i) info.sigma_reg[i] = std::sqrt(s.sigma[i] * s.sigma[i] + in.mu * in.mu);
    info.sigma_hat = info.sigma_reg.back();
    info.sigma_floor = info.sigma_cur.empty() ? 0.0 : info.sigma_cur.back();  // smallest_cur_sigma
    Vec d(l);
    for (i64 i = 0; i < l; ++i) d[i] = info.sigma_hat / info.sigma_reg[i] - 1.0;
    if (!in.implicit) {
      // V = Q_R V_M (explicit, n x l, on the device), K = diag(d)
      p.kind = 1;
      DBuf<double> vm;
      upload_vec(ctx, vm, s.v);
      p.B.alloc(n * l);
      dgemm(ctx, false, false, n, l, l, 1.0, in.q_dev, n, vm.p, l, 0.0, p.B.p, n);
      Vec K(static_cast<size_t>(l * l), 0.0);
      for (i64 i = 0; i < l; ++i) K[i * l + i] = d[i];
      upload_vec(ctx, p.Kf, K);
      upload_vec(ctx, p.Ka, K);
      APC_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
      // V = R^T T_R^{-1} V_M: G = W diag(d) W^T with W = T_R^{-1} V_M (symmetric)
      p.kind = 2;
      const Vec W = dtri_solve_cols(ctx, l, *in.t_r, s.v, l, false);
      Vec WD = W;
      for (i64 t = 0; t < l; ++t)
        for (i64 i = 0; i < l; ++i) WD[t * l + i] *= d[t];
      Vec G = dmatmul(ctx, l, l, l, WD, transpose(l, l, W));
      upload_r(ctx, n, l, in.r_ptr, in.r_idx, in.r_val, p);
      upload_vec(ctx, p.Kf, G);
      upload_vec(ctx, p.Ka, G);
    }
  } else {
    // SVD-free: P^{-1} = sigma_hat Q_R M^{-1} Q_R^T + (I - Q_R Q_R^T),
    // M^{-1} = T_R^{-T} B T_C^{-1}  (preconditioner.hpp:279-318)
    info.sigma_hat = in.target_level;
    info.sigma_floor = in.target_level;
    // M^{-1} = T_R^{-T} A(I,J) T_C^{-1}: triangular solves and the product on the device
    Vec eye(static_cast<size_t>(l * l), 0.0);
    for (i64 i = 0; i < l; ++i) eye[i * l + i] = 1.0;
    const Vec tcinv = dtri_solve_cols(ctx, l, t_c, eye, l, false);
    const Vec Minv = dtri_solve_cols(ctx, l, *in.t_r, dmatmul(ctx, l, l, l, *in.block, tcinv), l, true);
    Vec Kf(static_cast<size_t>(l * l)), Ka(static_cast<size_t>(l * l));
    for (i64 j = 0; j < l; ++j)
      for (i64 i = 0; i < l; ++i) {
        Kf[j * l + i] = info.sigma_hat * Minv[j * l + i] - (i == j ? 1.0 : 0.0);
        Ka[j * l + i] = info.sigma_hat * Minv[i * l + j] - (i == j ? 1.0 : 0.0);
      }
    // the device keeps the middle operators row-major (warp per output row)
    if (!in.implicit) {
      p.kind = 1;
      p.B.alloc(n * l);
      APC_CUDA(cudaMemcpyAsync(p.B.p, in.q_dev, sizeof(double) * n * l, cudaMemcpyDeviceToDevice, ctx->stream));
      upload_vec(ctx, p.Kf, transpose(l, l, Kf));
      upload_vec(ctx, p.Ka, transpose(l, l, Ka));
    } else {
      p.kind = 2;
      upload_r(ctx, n, l, in.r_ptr, in.r_idx, in.r_val, p);
      upload_vec(ctx, p.Kf, transpose(l, l, conjugate_by_tinv(ctx, l, *in.t_r, Kf)));
      upload_vec(ctx, p.Ka, transpose(l, l, conjugate_by_tinv(ctx, l, *in.t_r, Ka)));
    }
  }
  p.sigma_hat = info.sigma_hat;
  p.sigma_floor = info.sigma_floor;
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace apc
