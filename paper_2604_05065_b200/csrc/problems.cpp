// Seeded synthetic inputs for the five BASELINE configurations
// (/root/repo/BASELINE.json "configs"; made concrete in SURVEY.md 8(d)).
// The paper's experiments use no public dataset; these generators stand in
// with the stated shapes and value distributions.  Inputs are generated once
// on the host and the same bytes feed both the CPU oracle and the GPU.
//
// Streams (problem seed P_k = 20260415 + k by default):
//   C1 dense U diag(s) V^T  : Rng(P, problem) -> U, V Gaussians; Rng(P, rhs) -> x*, noise
//   C2 sparse 10/row        : Rng(P, problem, 0) col scales, (P, problem, 1) rows,
//                             (P, problem, 2) empty-column fill; Rng(P, rhs) -> b
//   C3 dense RBF            : Rng(P, problem) points; Rng(P, rhs) -> x*, noise
//   C4 dense G/sqrt(m)+UsV^T: Rng(P, problem, j) column j of G; Rng(P, user, 0/1) U, V
//   C5 sparse Zipf(1.1)     : Rng(P, problem, 0) permutation, (P, problem, 1) col scales,
//                             (P, problem, 2 + blk) rows of block blk; Rng(P, rhs) -> b
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "apc_internal.hpp"
#include "host_dense.hpp"
#include "host_rng.hpp"

#include "problem.hpp"

namespace apc {

namespace {

int hw_threads() {
  unsigned t = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(1u, std::min(t, 64u)));
}

template <class F>
void parallel_for(i64 n, F f) {
  const int nt = hw_threads();
  std::vector<std::thread> th;
  const i64 chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const i64 b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// dense y = A x, column axpy order (matrix.hpp:156-162)
void dense_matvec(i64 m, i64 n, const Vec& a, const double* x, double* y) {
  std::fill(y, y + m, 0.0);
  for (i64 j = 0; j < n; ++j) {
    const double xj = x[j];
    if (xj == 0.0) continue;
    const double* col = a.data() + j * m;
    for (i64 i = 0; i < m; ++i) y[i] += xj * col[i];
  }
}

// CSC from per-row column lists (rows ascending => rows sorted within columns)
void csc_from_rows(apc_problem& p, const std::vector<std::vector<std::int32_t>>& rcols,
                   const std::vector<std::vector<double>>& rvals) {
  const i64 m = p.m, n = p.n;
  p.colptr.assign(n + 1, 0);
  for (i64 i = 0; i < m; ++i)
    for (auto c : rcols[i]) p.colptr[c + 1]++;
  for (i64 j = 0; j < n; ++j) p.colptr[j + 1] += p.colptr[j];
  const i64 nnz = p.colptr[n];
  p.rowidx.resize(nnz);
  p.vals.resize(nnz);
  std::vector<std::int64_t> pos(p.colptr.begin(), p.colptr.end() - 1);
  for (i64 i = 0; i < m; ++i)
    for (size_t q = 0; q < rcols[i].size(); ++q) {
      const i64 c = rcols[i][q];
      const i64 at = pos[c]++;
      p.rowidx[at] = i;
      p.vals[at] = rvals[i][q];
    }
}

// ---- C1 -------------------------------------------------------------------
void gen_c1(apc_problem& p, std::uint64_t P) {
  const i64 m = p.m, n = p.n;
  require(m >= n && n >= 2, APC_INVALID_ARGUMENT, "C1: need m >= n >= 2");
  HostRng rng(P, Stream::problem);
  Vec g1(static_cast<size_t>(m * n)), g2(static_cast<size_t>(n * n));
  for (auto& x : g1) x = rng.gaussian();
  for (auto& x : g2) x = rng.gaussian();
  QT u = thin_qr(m, n, std::move(g1));
  QT v = thin_qr(n, n, std::move(g2));
  for (i64 j = 0; j < n; ++j) {
    const double s = std::pow(10.0, -6.0 * static_cast<double>(j) / static_cast<double>(n - 1));
    for (i64 i = 0; i < m; ++i) u.q[j * m + i] *= s;
  }
  p.dense = matmul(m, n, n, u.q, transpose(n, n, v.q));
  HostRng rr(P, Stream::rhs);
  Vec xs(static_cast<size_t>(n));
  for (auto& x : xs) x = rr.gaussian();
  p.b.resize(static_cast<size_t>(m));
  dense_matvec(m, n, p.dense, xs.data(), p.b.data());
  for (i64 i = 0; i < m; ++i) p.b[i] += 1e-4 * rr.gaussian();
}

// ---- C2 -------------------------------------------------------------------
void gen_c2(apc_problem& p, std::uint64_t P, int per_row, double decades) {
  const i64 m = p.m, n = p.n;
  require(per_row <= n, APC_INVALID_ARGUMENT, "C2: more nonzeros per row than columns");
  p.sparse = true;
  Vec scale(static_cast<size_t>(n));
  HostRng rs(P, Stream::problem, 0);
  for (auto& s : scale) s = std::pow(10.0, -decades * rs.uniform());
  HostRng rp(P, Stream::problem, 1);
  std::vector<std::vector<std::int32_t>> rc(static_cast<size_t>(m));
  std::vector<std::vector<double>> rv(static_cast<size_t>(m));
  std::vector<char> used(static_cast<size_t>(n), 0);
  std::vector<i64> colcount(static_cast<size_t>(n), 0);
  for (i64 i = 0; i < m; ++i) {
    auto& c = rc[i];
    c.reserve(per_row + 1);
    while (static_cast<int>(c.size()) < per_row) {
      const i64 j = static_cast<i64>(rp.below(static_cast<std::uint64_t>(n)));
      if (used[j]) continue;  // redraw duplicates
      used[j] = 1;
      c.push_back(static_cast<std::int32_t>(j));
    }
    std::sort(c.begin(), c.end());
    for (auto j : c) used[j] = 0;
    rv[i].resize(c.size());
    for (size_t q = 0; q < c.size(); ++q) {
      rv[i][q] = rp.gaussian() * scale[c[q]];
      colcount[c[q]]++;
    }
  }
  HostRng re(P, Stream::problem, 2);
  for (i64 j = 0; j < n; ++j) {
    if (colcount[j] > 0) continue;
    const i64 i = static_cast<i64>(re.below(static_cast<std::uint64_t>(m)));
    auto& c = rc[i];
    auto it = std::lower_bound(c.begin(), c.end(), static_cast<std::int32_t>(j));
    const size_t at = static_cast<size_t>(it - c.begin());
    c.insert(it, static_cast<std::int32_t>(j));
    rv[i].insert(rv[i].begin() + static_cast<std::ptrdiff_t>(at), re.gaussian() * scale[j]);
  }
  csc_from_rows(p, rc, rv);
  HostRng rr(P, Stream::rhs);
  p.b.resize(static_cast<size_t>(m));
  for (auto& x : p.b) x = rr.gaussian();
}

// ---- C3 -------------------------------------------------------------------
void gen_c3(apc_problem& p, std::uint64_t P) {
  const i64 m = p.m, n = p.n, d = 8;
  require(n <= m, APC_INVALID_ARGUMENT, "C3: centers are the first n points (n <= m)");
  HostRng rng(P, Stream::problem);
  Vec pts(static_cast<size_t>(m * d));
  for (auto& x : pts) x = rng.gaussian();
  p.dense.assign(static_cast<size_t>(m * n), 0.0);
  const double den = 2.0 * 1.5 * 1.5;
  parallel_for(n, [&](i64 jb, i64 je) {
    for (i64 j = jb; j < je; ++j) {
      const double* c = pts.data() + j * d;
      double* col = p.dense.data() + j * m;
      for (i64 i = 0; i < m; ++i) {
        const double* q = pts.data() + i * d;
        double s = 0.0;
        for (i64 k = 0; k < d; ++k) {
          const double t = q[k] - c[k];
          s += t * t;
        }
        col[i] = std::exp(-s / den);
      }
    }
  });
  HostRng rr(P, Stream::rhs);
  Vec xs(static_cast<size_t>(n));
  for (auto& x : xs) x = rr.gaussian();
  p.b.assign(static_cast<size_t>(m), 0.0);
  // y = A x* (per-row chains are independent: parallel over row blocks keeps
  // the column-ascending order of each row's sum)
  parallel_for(m, [&](i64 ib, i64 ie) {
    for (i64 j = 0; j < n; ++j) {
      const double xj = xs[j];
      if (xj == 0.0) continue;
      const double* col = p.dense.data() + j * m;
      for (i64 i = ib; i < ie; ++i) p.b[i] += xj * col[i];
    }
  });
  for (i64 i = 0; i < m; ++i) p.b[i] += 1e-3 * rr.gaussian();
}

// ---- C4 -------------------------------------------------------------------
void gen_c4(apc_problem& p, std::uint64_t P, i64 k) {
  const i64 m = p.m, n = p.n;
  require(k <= std::min(m, n), APC_INVALID_ARGUMENT, "C4: planted rank exceeds shape");
  Vec gu(static_cast<size_t>(m * k)), gv(static_cast<size_t>(n * k));
  {
    HostRng ru(P, Stream::user, 0), rv(P, Stream::user, 1);
    for (auto& x : gu) x = ru.gaussian();
    for (auto& x : gv) x = rv.gaussian();
  }
  QT u = thin_qr(m, k, std::move(gu));
  QT v = thin_qr(n, k, std::move(gv));
  Vec s(static_cast<size_t>(k));
  for (i64 t = 0; t < k; ++t)
    s[t] = k == 1 ? 100.0 : std::pow(10.0, 4.0 + (2.0 - 4.0) * static_cast<double>(t) / static_cast<double>(k - 1));
  p.dense.assign(static_cast<size_t>(m * n), 0.0);
  const double isq = 1.0 / std::sqrt(static_cast<double>(m));
  parallel_for(n, [&](i64 jb, i64 je) {
    for (i64 j = jb; j < je; ++j) {
      HostRng rg(P, Stream::problem, static_cast<std::uint64_t>(j));
      double* col = p.dense.data() + j * m;
      for (i64 i = 0; i < m; ++i) col[i] = rg.gaussian() * isq;
      for (i64 t = 0; t < k; ++t) {  // + U(:,t) s_t V(j,t), t ascending
        const double c = s[t] * v.q[t * n + j];
        const double* uc = u.q.data() + t * m;
        for (i64 i = 0; i < m; ++i) col[i] += c * uc[i];
      }
    }
  });
  HostRng rr(P, Stream::rhs);
  p.b.resize(static_cast<size_t>(m));
  for (auto& x : p.b) x = rr.gaussian();
}

// ---- C5 -------------------------------------------------------------------
void gen_c5(apc_problem& p, std::uint64_t P, int per_row, double zipf_s, double decades) {
  const i64 m = p.m, n = p.n;
  require(per_row <= n, APC_INVALID_ARGUMENT, "C5: more nonzeros per row than columns");
  p.sparse = true;
  std::vector<std::int32_t> perm(static_cast<size_t>(n));
  for (i64 j = 0; j < n; ++j) perm[j] = static_cast<std::int32_t>(j);
  HostRng rperm(P, Stream::problem, 0);
  for (i64 i = n - 1; i >= 1; --i) {
    const i64 j = static_cast<i64>(rperm.below(static_cast<std::uint64_t>(i + 1)));
    std::swap(perm[i], perm[j]);
  }
  Vec scale(static_cast<size_t>(n));
  HostRng rs(P, Stream::problem, 1);
  for (auto& s : scale) s = std::pow(10.0, -decades * rs.uniform());
  Vec cdf(static_cast<size_t>(n));
  double acc = 0.0;
  for (i64 z = 1; z <= n; ++z) {
    acc += std::pow(static_cast<double>(z), -zipf_s);
    cdf[z - 1] = acc;
  }
  for (auto& c : cdf) c /= acc;
  constexpr i64 kBlock = 65536;
  const i64 nblocks = (m + kBlock - 1) / kBlock;
  std::vector<std::vector<std::int32_t>> bc(static_cast<size_t>(nblocks));
  std::vector<std::vector<double>> bv(static_cast<size_t>(nblocks));
  parallel_for(nblocks, [&](i64 b0, i64 b1) {
    std::vector<char> used(static_cast<size_t>(n), 0);
    std::vector<std::int32_t> row;
    for (i64 blk = b0; blk < b1; ++blk) {
      HostRng r(P, Stream::problem, 2 + static_cast<std::uint64_t>(blk));
      const i64 rb = blk * kBlock, re = std::min(m, rb + kBlock);
      auto& oc = bc[blk];
      auto& ov = bv[blk];
      oc.reserve(static_cast<size_t>((re - rb) * per_row));
      ov.reserve(static_cast<size_t>((re - rb) * per_row));
      for (i64 i = rb; i < re; ++i) {
        row.clear();
        while (static_cast<int>(row.size()) < per_row) {
          const double u = r.uniform();
          i64 z = static_cast<i64>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
          if (z >= n) z = n - 1;
          const std::int32_t c = perm[z];
          if (used[c]) continue;
          used[c] = 1;
          row.push_back(c);
        }
        std::sort(row.begin(), row.end());
        for (auto c : row) {
          used[c] = 0;
          oc.push_back(c);
          ov.push_back(r.gaussian() * scale[c]);
        }
      }
    }
  });
  // CSC by counting sort over columns (rows ascending within each column)
  p.colptr.assign(static_cast<size_t>(n + 1), 0);
  for (const auto& oc : bc)
    for (auto c : oc) p.colptr[c + 1]++;
  for (i64 j = 0; j < n; ++j) p.colptr[j + 1] += p.colptr[j];
  const i64 nnz = p.colptr[n];
  p.rowidx.resize(static_cast<size_t>(nnz));
  p.vals.resize(static_cast<size_t>(nnz));
  std::vector<std::int64_t> pos(p.colptr.begin(), p.colptr.end() - 1);
  for (i64 blk = 0; blk < nblocks; ++blk) {
    const i64 rb = blk * kBlock;
    const auto& oc = bc[blk];
    const auto& ov = bv[blk];
    for (size_t q = 0; q < oc.size(); ++q) {
      const i64 i = rb + static_cast<i64>(q) / per_row;
      const i64 at = pos[oc[q]]++;
      p.rowidx[at] = i;
      p.vals[at] = ov[q];
    }
  }
  HostRng rr(P, Stream::rhs);
  p.b.resize(static_cast<size_t>(m));
  for (auto& x : p.b) x = rr.gaussian();
}

}  // namespace

apc_problem* generate_problem(int config, i64 m, i64 n, std::uint64_t seed) {
  static const i64 dm[6] = {0, 4000, 200000, 100000, 50000, 8000000};
  static const i64 dn[6] = {0, 500, 20000, 10000, 50000, 400000};
  require(config >= 1 && config <= 5, APC_INVALID_ARGUMENT, "problem: config must be 1..5");
  auto* p = new apc_problem();
  p->m = m > 0 ? m : dm[config];
  p->n = n > 0 ? n : dn[config];
  const std::uint64_t P = seed ? seed : 20260415ULL + static_cast<std::uint64_t>(config);
  try {
    switch (config) {
      case 1: gen_c1(*p, P); break;
      case 2: gen_c2(*p, P, 10, 4.0); break;
      case 3: gen_c3(*p, P); break;
      case 4: gen_c4(*p, P, std::max<i64>(1, std::min<i64>(200, std::min(p->m, p->n) / 2))); break;
      default: gen_c5(*p, P, static_cast<int>(std::min<i64>(16, p->n)), 1.1, 3.0); break;
    }
  } catch (...) {
    delete p;
    throw;
  }
  return p;
}

}  // namespace apc

extern "C" {

int apc_problem_info(const apc_problem* p, int64_t* m, int64_t* n, int* sparse, int64_t* nnz) {
  if (m) *m = p->m;
  if (n) *n = p->n;
  if (sparse) *sparse = p->sparse ? 1 : 0;
  if (nnz) *nnz = p->sparse ? (p->colptr.empty() ? 0 : p->colptr.back()) : p->m * p->n;
  return APC_OK;
}

const double* apc_problem_dense(const apc_problem* p) { return p->sparse ? nullptr : p->dense.data(); }

int apc_problem_csc(const apc_problem* p, const int64_t** colptr, const int64_t** rowidx,
                    const double** vals) {
  if (!p->sparse) return APC_INVALID_ARGUMENT;
  *colptr = p->colptr.data();
  *rowidx = p->rowidx.data();
  *vals = p->vals.data();
  return APC_OK;
}

const double* apc_problem_b(const apc_problem* p) { return p->b.data(); }

int apc_problem_free(apc_problem* p) {
  delete p;
  return APC_OK;
}

}  // extern "C"
