// Host-side small dense factorisations used between device kernels: the l x l
// intersection-block factor, the l x l preconditioner cores and the one-sided
// Jacobi SVD.  Each routine keeps the reference's operation order (no FMA:
// the library is built with -ffp-contract=off), because the core factor feeds
// index-selecting arithmetic (E^row, E^col) that must stay bit-identical.
//
// Restates /root/reference/proj/include/aplicur/dense_factor.hpp:31-447 and
// CoreFactor (cur.hpp:53-197).  Column-major storage throughout.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <vector>

#include "apc_internal.hpp"
#include "host_rng.hpp"

namespace apc {

using Vec = std::vector<double>;

// Householder QR in place (dense_factor.hpp:40-72): R in the upper triangle of
// a, unit reflector j in column j of hh (rows j..m-1).
struct Householder {
  i64 m = 0, k = 0;
  Vec a, hh;
};

struct HhTrailing {  // columns j+1+[b, e) <- (I - 2 v v^T) columns (named functor: see host_parallel_for)
  double* a;
  const double* v;
  i64 m, j;
  void operator()(i64 b, i64 e) const {
    for (i64 jj = j + 1 + b; jj < j + 1 + e; ++jj) {
      double* c = a + jj * m;
      double d = 0.0;
      for (i64 i = j; i < m; ++i) d += v[i] * c[i];
      d *= 2.0;
      for (i64 i = j; i < m; ++i) c[i] -= d * v[i];
    }
  }
};

inline Householder householder(i64 m, i64 k, Vec buf) {
  Householder f;
  f.m = m;
  f.k = k;
  f.a = std::move(buf);
  f.hh.assign(static_cast<size_t>(m * k), 0.0);
  for (i64 j = 0; j < k; ++j) {
    double* col = f.a.data() + j * m;
    double nrm2 = 0.0;
    for (i64 i = j; i < m; ++i) nrm2 += col[i] * col[i];
    const double nrm = std::sqrt(nrm2);
    double* v = f.hh.data() + j * m;
    if (nrm == 0.0) continue;
    const double alpha = col[j] >= 0.0 ? -nrm : nrm;
    for (i64 i = j; i < m; ++i) v[i] = col[i];
    v[j] -= alpha;
    double vn2 = 0.0;
    for (i64 i = j; i < m; ++i) vn2 += v[i] * v[i];
    const double vn = std::sqrt(vn2);
    if (vn == 0.0) continue;
    for (i64 i = j; i < m; ++i) v[i] /= vn;
    col[j] = alpha;
    for (i64 i = j + 1; i < m; ++i) col[i] = 0.0;
    // trailing columns are independent: same per-column chain on any core
    host_parallel_for(k - j - 1, HhTrailing{f.a.data(), v, m, j}, m - j);
  }
  return f;
}

inline void reflect_qt(const Householder& f, double* y) {  // y <- Q^T y
  for (i64 j = 0; j < f.k; ++j) {
    const double* v = f.hh.data() + j * f.m;
    double d = 0.0;
    for (i64 i = j; i < f.m; ++i) d += v[i] * y[i];
    d *= 2.0;
    for (i64 i = j; i < f.m; ++i) y[i] -= d * v[i];
  }
}

inline void reflect_q(const Householder& f, double* y) {  // y <- Q y
  for (i64 j = f.k - 1; j >= 0; --j) {
    const double* v = f.hh.data() + j * f.m;
    double d = 0.0;
    for (i64 i = j; i < f.m; ++i) d += v[i] * y[i];
    d *= 2.0;
    for (i64 i = j; i < f.m; ++i) y[i] -= d * v[i];
  }
}

inline Vec thin_q(const Householder& f) {  // dense_factor.hpp:96-106
  Vec q(static_cast<size_t>(f.m * f.k), 0.0), col(static_cast<size_t>(f.m));
  for (i64 j = 0; j < f.k; ++j) {
    std::fill(col.begin(), col.end(), 0.0);
    col[j] = 1.0;
    reflect_q(f, col.data());
    std::copy(col.begin(), col.end(), q.begin() + j * f.m);
  }
  return q;
}

struct QT {  // thin QR: q (m x k), t (k x k) upper with nonnegative diagonal
  i64 m = 0, k = 0;
  Vec q, t;
};

// sign-normalise T's diagonal (dense_factor.hpp:184-189)
inline void normalise_signs(i64 m, i64 k, Vec& q, Vec& t) {
  for (i64 j = 0; j < k; ++j)
    if (t[j * k + j] < 0.0) {
      for (i64 jj = j; jj < k; ++jj) t[jj * k + j] = -t[jj * k + j];
      for (i64 i = 0; i < m; ++i) q[j * m + i] = -q[j * m + i];
    }
}

inline Vec upper_of(const Householder& f) {
  Vec t(static_cast<size_t>(f.k * f.k), 0.0);
  for (i64 j = 0; j < f.k; ++j)
    for (i64 i = 0; i <= j; ++i) t[j * f.k + i] = f.a[j * f.m + i];
  return t;
}

// thin_qr (dense_factor.hpp:166-191)
inline QT thin_qr(i64 m, i64 k, Vec buf) {
  require(m >= k && k >= 1, APC_INVALID_ARGUMENT, "thin_qr: need m >= k >= 1");
  Householder f = householder(m, k, std::move(buf));
  double mx = 0.0;
  for (i64 j = 0; j < k; ++j) mx = std::max(mx, std::fabs(f.a[j * m + j]));
  const double tol = 1e-13 * mx;
  for (i64 j = 0; j < k; ++j)
    if (std::fabs(f.a[j * m + j]) <= tol)
      fail(APC_RANK_DEFICIENT, "thin_qr: numerically rank-deficient column", j);
  QT r;
  r.m = m;
  r.k = k;
  r.q = thin_q(f);
  r.t = upper_of(f);
  normalise_signs(m, k, r.q, r.t);
  return r;
}

// upper Cholesky of a k x k Gram matrix (dense_factor.hpp:229-244)
inline Vec chol_upper(i64 k, const Vec& g, const char* what) {
  Vec t(static_cast<size_t>(k * k), 0.0);
  for (i64 j = 0; j < k; ++j) {
    for (i64 i = 0; i < j; ++i) {
      double s = g[j * k + i];
      for (i64 r = 0; r < i; ++r) s -= t[i * k + r] * t[j * k + r];
      t[j * k + i] = s / t[i * k + i];
    }
    double s = g[j * k + j];
    for (i64 r = 0; r < j; ++r) s -= t[j * k + r] * t[j * k + r];
    if (!(s > 0.0)) fail(APC_NOT_POSITIVE, what, j);
    t[j * k + j] = std::sqrt(s);
  }
  return t;
}

// chol_gram of a dense m x k block (dense_factor.hpp:195-209)
inline Vec chol_gram_dense(i64 m, i64 k, const double* c) {
  require(k >= 1, APC_INVALID_ARGUMENT, "chol_gram: empty matrix");
  Vec g(static_cast<size_t>(k * k), 0.0);
  for (i64 j = 0; j < k; ++j)
    for (i64 i = 0; i <= j; ++i) {
      const double* ci = c + i * m;
      const double* cj = c + j * m;
      double s = 0.0;
      for (i64 r = 0; r < m; ++r) s += ci[r] * cj[r];
      g[j * k + i] = s;
      g[i * k + j] = s;
    }
  return chol_upper(k, g, "chol_gram: non-positive pivot");
}

// triangular solves against upper T (dense_factor.hpp:406-424)
inline void tri_solve(i64 k, const double* t, double* x, bool transpose) {
  if (!transpose) {
    for (i64 i = k - 1; i >= 0; --i) {
      double s = x[i];
      for (i64 j = i + 1; j < k; ++j) s -= t[j * k + i] * x[j];
      const double d = t[i * k + i];
      if (d == 0.0) fail(APC_SINGULAR, "tri_solve: zero diagonal", i);
      x[i] = s / d;
    }
  } else {
    for (i64 i = 0; i < k; ++i) {
      double s = x[i];
      for (i64 j = 0; j < i; ++j) s -= t[i * k + j] * x[j];
      const double d = t[i * k + i];
      if (d == 0.0) fail(APC_SINGULAR, "tri_solve: zero diagonal", i);
      x[i] = s / d;
    }
  }
}

// column-major C = A (m x k) * B (k x n), per-column sequential chains that
// skip zero B entries (matmul -> Matrix::matvec, matrix.hpp:151-162,351-361)
// (columns are independent, so they run on the host's cores: same bits)
struct MatmulCols {  // named functor: see the note at host_parallel_for
  i64 m, k;
  const double* a;
  const double* b;
  double* c;
  void operator()(i64 j0, i64 j1) const {
    for (i64 j = j0; j < j1; ++j) {
      double* cc = c + j * m;
      for (i64 t = 0; t < k; ++t) {
        const double x = b[j * k + t];
        if (x == 0.0) continue;
        const double* ac = a + t * m;
        for (i64 i = 0; i < m; ++i) cc[i] += x * ac[i];
      }
    }
  }
};

inline Vec matmul(i64 m, i64 k, i64 n, const Vec& a, const Vec& b) {
  Vec c(static_cast<size_t>(m * n), 0.0);
  host_parallel_for(n, MatmulCols{m, k, a.data(), b.data(), c.data()}, m * k);
  return c;
}

inline Vec transpose(i64 m, i64 n, const Vec& a) {
  Vec t(static_cast<size_t>(m * n));
  for (i64 j = 0; j < n; ++j)
    for (i64 i = 0; i < m; ++i) t[i * n + j] = a[j * m + i];
  return t;
}

// ---------------------------------------------------------------------------
// one-sided Jacobi SVD (dense_factor.hpp:249-402)
// ---------------------------------------------------------------------------
struct SvdH {
  i64 m = 0, n = 0;
  Vec u;      // m x k
  Vec sigma;  // k, nonincreasing
  Vec v;      // n x k
};

inline bool jacobi(i64 p, i64 n, Vec& w, Vec& v) {
  const double tol = 1.0e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (i64 j1 = 0; j1 < n - 1; ++j1)
      for (i64 j2 = j1 + 1; j2 < n; ++j2) {
        double* c1 = w.data() + j1 * p;
        double* c2 = w.data() + j2 * p;
        double a = 0.0, b = 0.0, c = 0.0;
        for (i64 i = 0; i < p; ++i) {
          a += c1[i] * c1[i];
          b += c2[i] * c2[i];
          c += c1[i] * c2[i];
        }
        if (std::fabs(c) <= tol * std::sqrt(a * b) || c == 0.0) continue;
        rotated = true;
        const double zeta = (b - a) / (2.0 * c);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + tt * tt);
        const double sn = cs * tt;
        for (i64 i = 0; i < p; ++i) {
          const double x = c1[i], y = c2[i];
          c1[i] = cs * x - sn * y;
          c2[i] = sn * x + cs * y;
        }
        double* v1 = v.data() + j1 * n;
        double* v2 = v.data() + j2 * n;
        for (i64 i = 0; i < n; ++i) {
          const double x = v1[i], y = v2[i];
          v1[i] = cs * x - sn * y;
          v2[i] = sn * x + cs * y;
        }
      }
    if (!rotated) return true;
  }
  return false;
}

inline SvdH small_svd(i64 m, i64 n, const Vec& mat) {
  require(m >= 1 && n >= 1, APC_INVALID_ARGUMENT, "small_svd: empty matrix");
  require(std::max(m, n) <= 4096, APC_INVALID_ARGUMENT,
          "small_svd: dimension exceeds the small-problem cap");
  if (m < n) {
    SvdH s = small_svd(n, m, transpose(m, n, mat));
    SvdH r;
    r.m = m;
    r.n = n;
    r.u = std::move(s.v);
    r.sigma = std::move(s.sigma);
    r.v = std::move(s.u);
    return r;
  }
  const bool pre = m > n;
  Householder qr;
  Vec w;
  i64 p = m;
  if (pre) {
    qr = householder(m, n, mat);
    p = n;
    w.assign(static_cast<size_t>(n * n), 0.0);
    for (i64 j = 0; j < n; ++j)
      for (i64 i = 0; i <= j; ++i) w[j * n + i] = qr.a[j * m + i];
  } else {
    w = mat;
  }
  Vec v(static_cast<size_t>(n * n), 0.0);
  for (i64 j = 0; j < n; ++j) v[j * n + j] = 1.0;
  if (n > 1 && !jacobi(p, n, w, v)) fail(APC_NO_CONVERGENCE, "small_svd: Jacobi sweep cap reached");
  Vec sig(static_cast<size_t>(n));
  for (i64 j = 0; j < n; ++j) {
    double s = 0.0;
    for (i64 i = 0; i < p; ++i) s += w[j * p + i] * w[j * p + i];
    sig[j] = std::sqrt(s);
  }
  std::vector<i64> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), i64{0});
  std::stable_sort(ord.begin(), ord.end(), [&](i64 a, i64 b) { return sig[a] > sig[b]; });
  SvdH r;
  r.m = m;
  r.n = n;
  r.sigma.resize(static_cast<size_t>(n));
  Vec us(static_cast<size_t>(p * n), 0.0);
  r.v.resize(static_cast<size_t>(n * n));
  std::vector<i64> nulls;
  for (i64 jj = 0; jj < n; ++jj) {
    const i64 j = ord[jj];
    r.sigma[jj] = sig[j];
    for (i64 i = 0; i < n; ++i) r.v[jj * n + i] = v[j * n + i];
    if (sig[j] > 0.0) {
      for (i64 i = 0; i < p; ++i) us[jj * p + i] = w[j * p + i] / sig[j];
    } else {
      nulls.push_back(jj);
    }
  }
  for (i64 jj : nulls) {
    for (i64 cand = 0; cand < p; ++cand) {
      Vec e(static_cast<size_t>(p), 0.0);
      e[cand] = 1.0;
      for (int pass = 0; pass < 2; ++pass)
        for (i64 j2 = 0; j2 < n; ++j2) {
          const double* uc = us.data() + j2 * p;
          double d = 0.0;
          for (i64 i = 0; i < p; ++i) d += uc[i] * e[i];
          for (i64 i = 0; i < p; ++i) e[i] -= d * uc[i];
        }
      double nr = 0.0;
      for (double x : e) nr += x * x;
      nr = std::sqrt(nr);
      if (nr > 0.5) {
        for (i64 i = 0; i < p; ++i) us[jj * p + i] = e[i] / nr;
        break;
      }
    }
  }
  if (pre) {
    r.u.assign(static_cast<size_t>(m * n), 0.0);
    Vec col(static_cast<size_t>(m));
    for (i64 j = 0; j < n; ++j) {
      std::fill(col.begin(), col.end(), 0.0);
      for (i64 i = 0; i < n; ++i) col[i] = us[j * n + i];
      reflect_q(qr, col.data());
      std::copy(col.begin(), col.end(), r.u.begin() + j * m);
    }
  } else {
    r.u = std::move(us);
  }
  return r;
}

// ---------------------------------------------------------------------------
// CoreFactor: factor of the l x l intersection block A(I, J) (cur.hpp:53-197)
// ---------------------------------------------------------------------------
struct LuTrailing {  // rows k+1+[b, e) of the LU elimination step k (independent rows)
  double* lu;
  i64 l, k;
  double piv;
  void operator()(i64 b, i64 e) const {
    for (i64 i = k + 1 + b; i < k + 1 + e; ++i) {
      const double fac = lu[k * l + i] / piv;
      lu[k * l + i] = fac;
      for (i64 j = k + 1; j < l; ++j) lu[j * l + i] -= fac * lu[j * l + k];
    }
  }
};

struct CoreFactorH {
  i64 l = 0;
  int kind = 0;  // 0 Householder QR, 1 LU with partial pivoting
  Householder qr;
  Vec lu;
  std::vector<i64> perm;

  static CoreFactorH build(i64 l, const Vec& block, int kind) {
    require(l >= 1, APC_INVALID_ARGUMENT, "CoreFactor: square nonempty block required");
    CoreFactorH f;
    f.l = l;
    f.kind = kind;
    if (kind == 0) {
      f.qr = householder(l, l, block);
      double dmin = std::numeric_limits<double>::infinity(), dmax = 0.0;
      for (i64 j = 0; j < l; ++j) {
        const double d = std::fabs(f.qr.a[j * l + j]);
        dmin = std::min(dmin, d);
        dmax = std::max(dmax, d);
      }
      if (!(dmin > 1e-14 * dmax))
        fail(APC_SINGULAR, "CoreFactor: intersection block numerically singular");
      return f;
    }
    f.lu = block;
    f.perm.resize(static_cast<size_t>(l));
    std::iota(f.perm.begin(), f.perm.end(), i64{0});
    double dmax = 0.0, dmin = std::numeric_limits<double>::infinity();
    for (i64 k = 0; k < l; ++k) {
      i64 best = k;
      double bm = -1.0;
      for (i64 i = k; i < l; ++i) {
        const double mg = std::fabs(f.lu[k * l + i]);
        if (mg > bm) {
          bm = mg;
          best = i;
        }
      }
      if (best != k) {
        for (i64 j = 0; j < l; ++j) std::swap(f.lu[j * l + k], f.lu[j * l + best]);
        std::swap(f.perm[k], f.perm[best]);
      }
      const double piv = f.lu[k * l + k];
      dmax = std::max(dmax, std::fabs(piv));
      dmin = std::min(dmin, std::fabs(piv));
      if (piv == 0.0) fail(APC_SINGULAR, "CoreFactor: intersection block numerically singular");
      host_parallel_for(l - k - 1, LuTrailing{f.lu.data(), l, k, piv}, l - k);
    }
    if (!(dmin > 1e-14 * dmax))
      fail(APC_SINGULAR, "CoreFactor: intersection block numerically singular");
    return f;
  }

  void solve(double* x) const {  // x <- A(I,J)^{-1} x
    Vec y(x, x + l);
    if (kind == 0) {
      reflect_qt(qr, y.data());
      for (i64 i = l - 1; i >= 0; --i) {
        double s = y[i];
        for (i64 j = i + 1; j < l; ++j) s -= qr.a[j * l + i] * y[j];
        y[i] = s / qr.a[i * l + i];
      }
    } else {
      for (i64 i = 0; i < l; ++i) y[i] = x[perm[i]];
      for (i64 i = 1; i < l; ++i)
        for (i64 j = 0; j < i; ++j) y[i] -= lu[j * l + i] * y[j];
      for (i64 i = l - 1; i >= 0; --i) {
        for (i64 j = i + 1; j < l; ++j) y[i] -= lu[j * l + i] * y[j];
        y[i] /= lu[i * l + i];
      }
    }
    std::copy(y.begin(), y.end(), x);
  }

  void solve_transpose(double* x) const {  // x <- A(I,J)^{-T} x
    Vec y(x, x + l);
    if (kind == 0) {
      for (i64 i = 0; i < l; ++i) {
        double s = y[i];
        for (i64 j = 0; j < i; ++j) s -= qr.a[i * l + j] * y[j];
        y[i] = s / qr.a[i * l + i];
      }
      reflect_q(qr, y.data());
      std::copy(y.begin(), y.end(), x);
    } else {
      for (i64 i = 0; i < l; ++i) {
        for (i64 j = 0; j < i; ++j) y[i] -= lu[i * l + j] * y[j];
        y[i] /= lu[i * l + i];
      }
      for (i64 i = l - 1; i >= 0; --i)
        for (i64 j = i + 1; j < l; ++j) y[i] -= lu[i * l + j] * y[j];
      for (i64 i = 0; i < l; ++i) x[perm[i]] = y[i];
    }
  }

  // columns are independent: parallel over the host's cores, same bits
  struct SolveCols {  // named functor: see the note at host_parallel_for
    const CoreFactorH* f;
    double* b;
    bool transpose;
    void operator()(i64 j0, i64 j1) const {
      for (i64 j = j0; j < j1; ++j) {
        if (transpose) f->solve_transpose(b + j * f->l);
        else f->solve(b + j * f->l);
      }
    }
  };
  Vec solve_matrix(i64 ncols, Vec b) const {
    host_parallel_for(ncols, SolveCols{this, b.data(), false}, 3 * l * l);
    return b;
  }
  Vec solve_matrix_transpose(i64 ncols, Vec b) const {
    host_parallel_for(ncols, SolveCols{this, b.data(), true}, 3 * l * l);
    return b;
  }
};

}  // namespace apc
