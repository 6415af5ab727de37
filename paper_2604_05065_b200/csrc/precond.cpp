// Preconditioner construction per rebuild (preconditioner.hpp:138-396,
// 424-592) and its upload as the device form I + B K B^T / I + R^T G R that
// the LSQR loop applies (lsqr.cu).  The tall products (C^T C, Q^T c, Q p,
// Q_R V_M) run on the device through cuBLAS; the l x l algebra (Cholesky of
// the Gram matrix, core spectrum, middle operators) runs on the host with the
// restated reference routines.  None of it is index-affecting:
// only the x / iteration parity bar applies.
#include <cmath>
#include <memory>

#include "blas.hpp"
#include "cur.hpp"
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
Vec conjugate_by_tinv(i64 l, const Vec& t, const Vec& K) {
  Vec X = K;
  for (i64 j = 0; j < l; ++j) tri_solve(l, t.data(), X.data() + j * l, false);
  Vec Xt = transpose(l, l, X);
  for (i64 j = 0; j < l; ++j) tri_solve(l, t.data(), Xt.data() + j * l, false);
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
  Vec g = download_vec(ctx, G.p, b * b);
  symmetrize_upper(b, g);
  Vec r;
  try {
    r = chol_upper(b, g, "QrAccumulator: dependent block");
  } catch (const Status& s) {
    fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", s.index);
  }
  DBuf<double> R(b * b);
  upload_vec(ctx, R, r);
  dtrsm_right_upper(ctx, m, b, R.p, b, e, m);
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
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
  // factor the block: Householder on the host when small, CholeskyQR2 on the device otherwise
  Vec rb;
  if (static_cast<double>(m) * b * b <= 2e8) {
    Vec eh = download_vec(ctx, e.p, m * b);
    Householder f = householder(m, b, std::move(eh));
    for (i64 j = 0; j < b; ++j)
      if (std::fabs(f.a[j * m + j]) <= 1e-12 * scale) fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", j);
    Vec qe = thin_q(f);
    rb = upper_of(f);
    normalise_signs(m, b, qe, rb);
    APC_CUDA(cudaMemcpyAsync(e.p, qe.data(), sizeof(double) * m * b, cudaMemcpyHostToDevice, st));
    APC_CUDA(cudaStreamSynchronize(st));
  } else {
    Vec r1 = cholqr_step(ctx, m, b, e.p);
    Vec r2 = cholqr_step(ctx, m, b, e.p);
    rb = matmul(b, b, b, r2, r1);
    for (i64 j = 0; j < b; ++j)
      if (std::fabs(rb[j * b + j]) <= 1e-12 * scale) fail(APC_RANK_DEFICIENT, "QrAccumulator: dependent block", j);
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
    t_c = chol_upper(l, in.gram, "chol_gram: non-positive pivot");
  } catch (const Status& s) {
    if (s.code != APC_NOT_POSITIVE) throw;
    t_c = thin_qr(in.m, l, in.c_dense()).t;
  }
  if (in.variant == 0) {
    // SVD form: M = T_C U T_R^T, small_svd(M) (preconditioner.hpp:158-192)
    ps.reset(new ProfScope("pre.core_matmul"));
    Vec ut = in.core->solve_matrix(l, transpose(l, l, *in.t_r));
    Vec mm = matmul(l, l, l, t_c, ut);
    ps.reset(new ProfScope("pre.svd"));
    require(l <= 4096, APC_INVALID_ARGUMENT, "small_svd: dimension exceeds the small-problem cap");
    SvdH s;
    if (l > 96) {  // parallel-order Jacobi on the device; serial cyclic on the host for small cores
      s.m = s.n = l;
      device_jacobi_svd(ctx, l, mm, s.sigma, s.v);
    } else {
      s = small_svd(l, l, mm);
    }
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
      Vec W = s.v;
      for (i64 j = 0; j < l; ++j) tri_solve(l, in.t_r->data(), W.data() + j * l, false);
      Vec WD = W;
      for (i64 t = 0; t < l; ++t)
        for (i64 i = 0; i < l; ++i) WD[t * l + i] *= d[t];
      Vec G = matmul(l, l, l, WD, transpose(l, l, W));
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
      p.B.alloc(n * l);
      APC_CUDA(cudaMemcpyAsync(p.B.p, in.q_dev, sizeof(double) * n * l, cudaMemcpyDeviceToDevice, ctx->stream));
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
