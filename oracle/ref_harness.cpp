// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C-ABI wrapper around the *unmodified* APLICUR reference (header-only C++20,
// /root/reference/proj/include/aplicur/*.hpp).  Nothing from the reference is
// copied here: this translation unit #includes the reference headers in place
// and is compiled by oracle/Makefile into oracle/_ref/libaplicur_ref.so with
// the reference's own flags (-O3 -DNDEBUG -std=gnu++20, no -march, plus
// -ffp-contract=off; see /root/reference/proj/CMakeLists.txt:3-11).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load this library, and only as the checker or the CPU baseline.
// The product path (paper_2604_05065_b200/) never links or calls it.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

// The Gaussian-sketch CUR path has no public entry in the reference
// (cur.hpp:40-42, 220-221: init hard-wires SparseSignEmbedding; the ctor is
// private, cur.hpp:339).  To drive CurState with a GaussianEmbedding sketch
// without copying the class, open its private members for this TU only.
#define private public
#include "aplicur/cur.hpp"
#include "aplicur/dense_factor.hpp"
#include "aplicur/lsqr.hpp"
#include "aplicur/matrix.hpp"
#include "aplicur/matrix_market.hpp"
#include "aplicur/operators.hpp"
#include "aplicur/preconditioner.hpp"
#include "aplicur/problems.hpp"
#include "aplicur/rng.hpp"
#include "aplicur/sketch.hpp"
#include "aplicur/solver.hpp"
#undef private

using namespace aplicur;

namespace {

thread_local std::string g_err;

int fail_code(const Error& e) {
  g_err = e.what();
  return 1 + static_cast<int>(e.kind());
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    return fail_code(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

}  // namespace

extern "C" {

// Problem description: dense column-major (sparse == 0) or CSC with int64
// indices (the reference storage, matrix.hpp:18,31-34,66-94).
struct RefProblem {
  std::int64_t m, n;
  std::int32_t sparse;
  const double* dense;
  const std::int64_t* colptr;
  const std::int64_t* rowidx;
  const double* vals;
};

struct RefConfig {  // mirrors SolverConfig, solver.hpp:29-45
  std::int64_t block;
  double eps_cur, eps_lsqr, nu_prec, nu_lsqr, mu;
  std::int32_t variant;  // 0 svd, 1 svd_free
  std::int64_t sketch_xi, probe_count, lsqr_cap, max_rank;
  std::uint64_t seed;
  std::int32_t core;  // 0 qr, 1 lu
  std::int64_t trace_sample_stride, outer_cap;
};

// Output buffers owned by the caller; *_cap are capacities, counts written back.
struct RefOut {
  double* x;                 // n
  std::int32_t status;       // SolveStatus
  double final_rho, final_relres;
  std::uint64_t sketch_applications, system_matvecs;
  std::int64_t* row_idx;     // cap_idx
  std::int64_t* col_idx;     // cap_idx
  std::int64_t n_idx, cap_idx;
  double* rho_hist;          // cap_rho
  std::int64_t n_rho, cap_rho;
  // per phase: rank, lsqr_iters, reason, rho, sigma_hat, relres_at_end, t_lsqr_ms
  std::int64_t* ph_rank;
  std::int64_t* ph_iters;
  std::int32_t* ph_reason;
  double* ph_rho;
  double* ph_sigma_hat;
  double* ph_relres;
  double* ph_t_lsqr_ms;
  double* ph_t_total_ms;
  std::int64_t n_ph, cap_ph;
  // trace rows: phase, iter, phibar, matvecs
  std::int32_t* tr_phase;
  std::int64_t* tr_iter;
  double* tr_phibar;
  std::uint64_t* tr_matvecs;
  double* tr_relres;  // sampled true residual (NaN where not sampled)
  std::int64_t n_tr, cap_tr;
  double wall_ms;
};

const char* ref_last_error() { return g_err.c_str(); }

}  // extern "C"

namespace {

Matrix make_matrix(const RefProblem* p) {
  if (!p->sparse) {
    std::vector<double> v(p->dense, p->dense + p->m * p->n);
    return Matrix::dense(p->m, p->n, std::move(v));
  }
  std::vector<Triplet> trips;
  trips.reserve(static_cast<std::size_t>(p->colptr[p->n]));
  for (Index j = 0; j < p->n; ++j)
    for (Index k = p->colptr[j]; k < p->colptr[j + 1]; ++k)
      trips.push_back({p->rowidx[k], j, p->vals[k]});
  return Matrix::sparse(p->m, p->n, std::move(trips));
}

SolverConfig make_config(const RefConfig* c) {
  SolverConfig s;
  s.block = c->block;
  s.eps_cur = c->eps_cur;
  s.eps_lsqr = c->eps_lsqr;
  s.nu_prec = c->nu_prec;
  s.nu_lsqr = c->nu_lsqr;
  s.mu = c->mu;
  s.variant = c->variant == 0 ? PrecondVariant::svd : PrecondVariant::svd_free;
  s.sketch_xi = c->sketch_xi;
  s.probe_count = c->probe_count;
  s.lsqr_cap = c->lsqr_cap;
  s.max_rank = c->max_rank;
  s.seed = c->seed;
  s.core = c->core == 0 ? CoreFactorKind::qr : CoreFactorKind::lu;
  s.trace_sample_stride = c->trace_sample_stride;
  s.outer_cap = c->outer_cap;
  return s;
}

void fill_out(const SolveResult& r, RefOut* o) {
  std::copy(r.x.begin(), r.x.end(), o->x);
  o->status = static_cast<std::int32_t>(r.status);
  o->final_rho = r.final_rho;
  o->final_relres = r.final_relres;
  o->sketch_applications = r.sketch_applications;
  o->system_matvecs = r.system_matvecs;
  o->n_idx = static_cast<std::int64_t>(r.row_indices.size());
  for (std::int64_t k = 0; k < std::min(o->n_idx, o->cap_idx); ++k) {
    o->row_idx[k] = r.row_indices[k];
    o->col_idx[k] = r.col_indices[k];
  }
  o->n_rho = static_cast<std::int64_t>(r.rho_history.size());
  for (std::int64_t k = 0; k < std::min(o->n_rho, o->cap_rho); ++k) o->rho_hist[k] = r.rho_history[k];
  o->n_ph = static_cast<std::int64_t>(r.phases.size());
  for (std::int64_t k = 0; k < std::min(o->n_ph, o->cap_ph); ++k) {
    const PhaseReport& p = r.phases[k];
    o->ph_rank[k] = p.rank;
    o->ph_iters[k] = p.lsqr_iters;
    o->ph_reason[k] = static_cast<std::int32_t>(p.reason);
    o->ph_rho[k] = p.rho;
    o->ph_sigma_hat[k] = p.sigma_hat;
    o->ph_relres[k] = p.relres_at_end;
    o->ph_t_lsqr_ms[k] = p.t_lsqr_ms;
    o->ph_t_total_ms[k] = p.t_augment_ms + p.t_factor_ms + p.t_precond_ms + p.t_lsqr_ms;
  }
  o->n_tr = static_cast<std::int64_t>(r.trace.rows.size());
  for (std::int64_t k = 0; k < std::min(o->n_tr, o->cap_tr); ++k) {
    const LsqrTraceRow& t = r.trace.rows[k];
    o->tr_phase[k] = t.phase;
    o->tr_iter[k] = t.iter;
    o->tr_phibar[k] = t.phibar;
    o->tr_matvecs[k] = t.matvecs;
    o->tr_relres[k] = t.true_relres;
  }
}

}  // namespace

extern "C" {

// ---- RNG (rng.hpp:38-78) ----------------------------------------------------
// kind: 0 next_u64, 1 uniform, 2 gaussian, 3 below(bound), 4 sign.
// stream < 0 uses Rng(seed), else Rng(seed, RngStream(stream), index).
int ref_rng(std::uint64_t seed, std::int32_t stream, std::uint64_t index, std::int32_t kind,
            std::uint64_t bound, std::int64_t count, void* out) {
  return guarded([&] {
    Rng rng = stream < 0 ? Rng(seed) : Rng(seed, static_cast<RngStream>(stream), index);
    for (std::int64_t i = 0; i < count; ++i) {
      switch (kind) {
        case 0: static_cast<std::uint64_t*>(out)[i] = rng.next_u64(); break;
        case 1: static_cast<double*>(out)[i] = rng.uniform(); break;
        case 2: static_cast<double*>(out)[i] = rng.gaussian(); break;
        case 3: static_cast<std::uint64_t*>(out)[i] = rng.below(bound); break;
        default: static_cast<double*>(out)[i] = rng.sign(); break;
      }
    }
  });
}

std::uint64_t ref_mix64(std::uint64_t x) { return detail::mix64(x); }

// ---- matrix products (matrix.hpp:151-195, 365-392) --------------------------
int ref_matvec(const RefProblem* p, double mu, std::int32_t augmented, std::int32_t transpose,
               const double* x, double* y) {
  return guarded([&] {
    Matrix a = make_matrix(p);
    Index m = a.rows(), n = a.cols();
    if (augmented) {
      AugmentedOperator aug(a, mu);
      if (!transpose)
        aug.matvec({x, static_cast<std::size_t>(n)}, {y, static_cast<std::size_t>(m + n)});
      else
        aug.matvec_transpose({x, static_cast<std::size_t>(m + n)}, {y, static_cast<std::size_t>(n)});
      return;
    }
    if (!transpose)
      a.matvec({x, static_cast<std::size_t>(n)}, {y, static_cast<std::size_t>(m)});
    else
      a.matvec_transpose({x, static_cast<std::size_t>(m)}, {y, static_cast<std::size_t>(n)});
  });
}

// ---- sketching (sketch.hpp:18-197, cur.hpp:219-221) --------------------------
// Embedding rows/signs exactly as the reference generated them (read through
// the public column() accessor, sketch.hpp:58-63).
int ref_sparse_sign(std::int64_t s, std::int64_t m, std::int64_t xi, std::uint64_t seed,
                    std::int64_t* rows, std::int8_t* signs, double* scale) {
  return guarded([&] {
    SparseSignEmbedding e(s, m, xi, seed);
    std::vector<std::pair<Index, double>> col;
    Index x = e.sparsity();
    for (Index c = 0; c < m; ++c) {
      e.column(c, col);
      for (Index q = 0; q < x; ++q) {
        rows[c * x + q] = col[q].first;
        signs[c * x + q] = col[q].second > 0 ? 1 : -1;
      }
    }
    *scale = e.scale();
  });
}

// Y = S * A (augmented == 0) or S * [A; mu I]; emb_seed is the embedding seed
// (CurState::init uses mix64(seed ^ 0x5ce7c3a1b2d4f688), cur.hpp:220).
int ref_sketch_sparse_sign(const RefProblem* p, double mu, std::int32_t augmented, std::int64_t s,
                           std::int64_t xi, std::uint64_t emb_seed, double* y) {
  return guarded([&] {
    Matrix a = make_matrix(p);
    Matrix out;
    if (augmented) {
      AugmentedOperator aug(a, mu);
      SparseSignEmbedding e(s, aug.rows(), xi, emb_seed);
      out = e.apply_to_augmented(aug);
    } else {
      SparseSignEmbedding e(s, a.rows(), xi, emb_seed);
      out = e.apply(a);
    }
    auto d = out.dense_data();
    std::copy(d.begin(), d.end(), y);
  });
}

int ref_gaussian_embedding(std::int64_t s, std::int64_t m, std::uint64_t emb_seed, double* S) {
  return guarded([&] {
    GaussianEmbedding g(s, m, emb_seed);
    Matrix sm = g.to_matrix();
    auto d = sm.dense_data();
    std::copy(d.begin(), d.end(), S);
  });
}

int ref_sketch_gaussian(const RefProblem* p, std::int64_t s, std::uint64_t emb_seed, double* y) {
  return guarded([&] {
    Matrix a = make_matrix(p);
    GaussianEmbedding g(s, a.rows(), emb_seed);
    Matrix out = g.apply(a);
    auto d = out.dense_data();
    std::copy(d.begin(), d.end(), y);
  });
}

// ---- LUPP pivot order (dense_factor.hpp:119-157) -----------------------------
int ref_lupp(const double* w, std::int64_t rows, std::int64_t cols, std::int64_t max_pivots,
             std::int64_t* order, double* mags, std::int64_t* nsteps) {
  return guarded([&] {
    Matrix a = Matrix::dense(rows, cols, std::vector<double>(w, w + rows * cols));
    PivotOrder piv = lu_partial_pivot(a, max_pivots);
    *nsteps = static_cast<std::int64_t>(piv.order.size());
    for (std::size_t k = 0; k < piv.order.size(); ++k) {
      order[k] = piv.order[k];
      mags[k] = piv.magnitudes[k];
    }
  });
}

// ---- spectral estimate (sketch.hpp:209-229) ----------------------------------
int ref_spectral_norm_estimate(const double* e, std::int64_t rows, std::int64_t cols,
                               std::int64_t r, std::uint64_t seed, double* rho) {
  return guarded([&] {
    Matrix em = Matrix::dense(rows, cols, std::vector<double>(e, e + rows * cols));
    *rho = spectral_norm_estimate(em, r, seed);
  });
}

// ---- full solver (solver.hpp:162-448) ----------------------------------------
int ref_solve(const RefProblem* p, const double* b, const RefConfig* cfg, std::int32_t plain,
              RefOut* out) {
  return guarded([&] {
    ProblemInstance prob;
    prob.a = make_matrix(p);
    prob.b.assign(b, b + p->m);
    prob.mu = cfg->mu;
    SolverConfig sc = make_config(cfg);
    auto t0 = std::chrono::steady_clock::now();
    SolveResult r = plain ? plain_lsqr_solve(prob, sc) : aplicur_solve(prob, sc);
    out->wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fill_out(r, out);
  });
}

// ---- CurState stepping (cur.hpp:209-315) -------------------------------------
// Drives init/augment/refresh for `steps` augments and records I, J, rho after
// each step, plus the sketch Y.  gaussian != 0 replaces the sketch by
// GaussianEmbedding(s, rows, mix64(seed ^ 0x5ce7c3a1b2d4f688)).apply(A): the
// documented test-side Gaussian shim; everything else runs the
// reference CurState verbatim.  Target is the plain matrix A.
// Per step k: added[k], and indices appended to I/J; rho_hist[k].
int ref_cur_steps(const RefProblem* p, std::int64_t block, std::uint64_t seed, std::int64_t xi,
                  std::int64_t probes, std::int32_t core, std::int32_t gaussian, std::int64_t steps,
                  double* y_out, std::int64_t* added, std::int64_t* iidx, std::int64_t* jidx,
                  double* rho_hist, std::int64_t* nsteps_done, double* eres_out) {
  return guarded([&] {
    Matrix a = make_matrix(p);
    CurTarget tgt(a);
    CurState st = CurState::init(tgt, block, seed, xi, probes,
                                 core == 0 ? CoreFactorKind::qr : CoreFactorKind::lu);
    if (gaussian) {
      Index s = st.embedding().rows();
      GaussianEmbedding g(s, a.rows(), detail::mix64(seed ^ 0x5ce7c3a1b2d4f688ULL));
      st.y_ = g.apply(a);
      st.eres_ = st.y_;
      st.ztol_ = 1e-14 * st.y_.frob_norm();
    }
    if (y_out) {
      auto d = st.y_.dense_data();
      std::copy(d.begin(), d.end(), y_out);
    }
    std::int64_t done = 0;
    Index pos = 0;
    for (std::int64_t k = 0; k < steps; ++k) {
      if (st.rank() >= std::min(a.rows(), a.cols())) break;
      AugmentOutcome o = st.augment();
      added[k] = o.added;
      if (o.added == 0) {
        rho_hist[k] = st.rho();
        ++done;
        break;
      }
      try {
        st.refresh();
      } catch (const Error& e) {
        if (e.kind() != ErrorKind::singular) throw;
        st.rollback_last_augment();
        added[k] = -1;  // singular core: rolled back
        ++done;
        break;
      }
      for (Index q = pos; q < st.rank(); ++q) {
        iidx[q] = st.row_indices()[q];
        jidx[q] = st.col_indices()[q];
      }
      pos = st.rank();
      rho_hist[k] = st.rho();
      ++done;
    }
    *nsteps_done = done;
    if (eres_out) {
      auto d = st.eres_.dense_data();
      std::copy(d.begin(), d.end(), eres_out);
    }
  });
}

// ---- CPU timing of the operator pair A*v + A^T*u ----------
// Runs the reference Matrix::matvec + matvec_transpose `iters` times; returns
// seconds per pair.
int ref_time_op_pair(const RefProblem* p, std::int64_t iters, double* sec_per_pair) {
  return guarded([&] {
    Matrix a = make_matrix(p);
    std::vector<double> v(static_cast<std::size_t>(a.cols()), 1.0), u(static_cast<std::size_t>(a.rows()));
    std::vector<double> g(static_cast<std::size_t>(a.cols()));
    for (Index j = 0; j < a.cols(); ++j) v[j] = 1.0 / (1.0 + static_cast<double>(j));
    auto t0 = std::chrono::steady_clock::now();
    for (std::int64_t it = 0; it < iters; ++it) {
      a.matvec(v, u);
      a.matvec_transpose(u, g);
      v[static_cast<std::size_t>(it % a.cols())] += 1e-300 * g[0];
    }
    *sec_per_pair = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() /
                    static_cast<double>(iters);
  });
}

// ---- BASELINE input generators (BASELINE.json "configs") -----
// The oracle's own restatement of the five seeded BASELINE inputs, built from
// the reference's primitives (Rng sub-streams rng.hpp:42-45, dense_matrix
// problems.hpp:105-127, thin_qr dense_factor.hpp:166-190, Matrix::matvec
// matrix.hpp:151-172).  The reference arm of bench.py generates its inputs here,
// so it never maps the product library; tests/test_oracle_cpu.py proves the
// bytes equal the product's generator (paper_2604_05065_b200 Problem).
// Streams (problem seed P = 20260415 + config unless given):
//   C1 dense_matrix(m, n, 10^(-6 i/(n-1)), incoherent, P); Rng(P, rhs): x*, noise
//   C2 Rng(P, problem, 0) column scales, (P, problem, 1) rows, (P, problem, 2)
//      empty-column fill; Rng(P, rhs): b
//   C3 Rng(P, problem): points; Rng(P, rhs): x*, noise
//   C4 Rng(P, user, 0/1): U, V Gaussians; Rng(P, problem, j): column j of G
//   C5 Rng(P, problem, 0) permutation, (P, problem, 1) scales,
//      (P, problem, 2 + blk) rows of 65536-row block blk; Rng(P, rhs): b
struct RefGen {
  Matrix a;
  std::vector<double> b;
};

}  // extern "C"

namespace {

template <class F>
void par_for(std::int64_t n, int threads, F f) {
  threads = std::max(1, threads);
  std::vector<std::thread> th;
  const std::int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const std::int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// CSC Matrix straight from arrays whose rows are strictly increasing within
// each column (what Matrix::sparse, matrix.hpp:68-94, would build from the
// same triplets, without sorting 1e8 of them; zero values are dropped there
// and cannot occur here: every value is a nonzero Gaussian times a power of ten).
Matrix csc_matrix(Index m, Index n, std::vector<Index> cptr, std::vector<Index> ridx,
                  std::vector<double> val) {
  for (Index j = 0; j < n; ++j)
    for (Index k = cptr[j] + 1; k < cptr[j + 1]; ++k)
      detail::require(ridx[k - 1] < ridx[k], ErrorKind::invalid_argument, "csc_matrix: unsorted column", j);
  for (double v : val) detail::require(v != 0.0, ErrorKind::invalid_argument, "csc_matrix: explicit zero");
  Matrix a;
  a.rows_ = m;
  a.cols_ = n;
  a.sparse_ = true;
  a.cptr_ = std::move(cptr);
  a.ridx_ = std::move(ridx);
  a.val_ = std::move(val);
  a.tbox_ = std::make_shared<Matrix::TransposeBox>();
  return a;
}

// CSC from per-row (sorted) column lists, rows visited in ascending order
Matrix csc_from_row_lists(Index m, Index n, const std::vector<std::vector<Index>>& rc,
                          const std::vector<std::vector<double>>& rv) {
  std::vector<Index> cptr(static_cast<std::size_t>(n) + 1, 0);
  for (Index i = 0; i < m; ++i)
    for (Index c : rc[i]) ++cptr[c + 1];
  for (Index j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
  std::vector<Index> ridx(static_cast<std::size_t>(cptr[n]));
  std::vector<double> val(ridx.size());
  std::vector<Index> next(cptr.begin(), cptr.end() - 1);
  for (Index i = 0; i < m; ++i)
    for (std::size_t q = 0; q < rc[i].size(); ++q) {
      Index at = next[rc[i][q]]++;
      ridx[at] = i;
      val[at] = rv[i][q];
    }
  return csc_matrix(m, n, std::move(cptr), std::move(ridx), std::move(val));
}

void gen_c1(RefGen& g, Index m, Index n, std::uint64_t P) {
  std::vector<double> sigma(static_cast<std::size_t>(n));
  for (Index j = 0; j < n; ++j)
    sigma[j] = std::pow(10.0, -6.0 * static_cast<double>(j) / static_cast<double>(n - 1));
  g.a = dense_matrix(m, n, sigma, Coherence::incoherent, P);
  Rng rr(P, RngStream::rhs);
  std::vector<double> xs(static_cast<std::size_t>(n));
  for (auto& x : xs) x = rr.gaussian();
  g.b.assign(static_cast<std::size_t>(m), 0.0);
  g.a.matvec(xs, g.b);
  for (Index i = 0; i < m; ++i) g.b[i] += 1e-4 * rr.gaussian();
}

void gen_c2(RefGen& g, Index m, Index n, std::uint64_t P) {
  const Index per_row = 10;
  const double decades = 4.0;
  detail::require(per_row <= n, ErrorKind::invalid_argument, "C2: more nonzeros per row than columns");
  std::vector<double> scale(static_cast<std::size_t>(n));
  Rng rs(P, RngStream::problem, 0);
  for (auto& s : scale) s = std::pow(10.0, -decades * rs.uniform());
  Rng rp(P, RngStream::problem, 1);
  std::vector<std::vector<Index>> rc(static_cast<std::size_t>(m));
  std::vector<std::vector<double>> rv(static_cast<std::size_t>(m));
  std::vector<char> seen(static_cast<std::size_t>(n), 0);
  std::vector<Index> count(static_cast<std::size_t>(n), 0);
  for (Index i = 0; i < m; ++i) {
    auto& c = rc[i];
    while (static_cast<Index>(c.size()) < per_row) {  // uniform distinct columns, redraw duplicates
      Index j = static_cast<Index>(rp.below(static_cast<std::uint64_t>(n)));
      if (seen[j]) continue;
      seen[j] = 1;
      c.push_back(j);
    }
    std::sort(c.begin(), c.end());
    for (Index j : c) seen[j] = 0;
    for (Index j : c) {
      rv[i].push_back(rp.gaussian() * scale[j]);
      ++count[j];
    }
  }
  Rng re(P, RngStream::problem, 2);  // one guaranteed entry per empty column
  for (Index j = 0; j < n; ++j) {
    if (count[j]) continue;
    Index i = static_cast<Index>(re.below(static_cast<std::uint64_t>(m)));
    auto it = std::lower_bound(rc[i].begin(), rc[i].end(), j);
    auto at = it - rc[i].begin();
    rc[i].insert(it, j);
    rv[i].insert(rv[i].begin() + at, re.gaussian() * scale[j]);
  }
  g.a = csc_from_row_lists(m, n, rc, rv);
  Rng rr(P, RngStream::rhs);
  g.b.resize(static_cast<std::size_t>(m));
  for (auto& x : g.b) x = rr.gaussian();
}

void gen_c3(RefGen& g, Index m, Index n, std::uint64_t P, int threads) {
  const Index d = 8;
  detail::require(n <= m, ErrorKind::invalid_argument, "C3: centers are the first n points");
  Rng rng(P, RngStream::problem);
  std::vector<double> pts(static_cast<std::size_t>(m * d));
  for (auto& x : pts) x = rng.gaussian();
  std::vector<double> val(static_cast<std::size_t>(m * n));
  const double two_l2 = 2.0 * 1.5 * 1.5;
  par_for(n, threads, [&](std::int64_t j0, std::int64_t j1) {
    for (Index j = j0; j < j1; ++j)
      for (Index i = 0; i < m; ++i) {
        double s = 0.0;  // ||p_i - c_j||^2, dimensions in index order
        for (Index k = 0; k < d; ++k) {
          double t = pts[i * d + k] - pts[j * d + k];
          s += t * t;
        }
        val[j * m + i] = std::exp(-s / two_l2);
      }
  });
  g.a = Matrix::dense(m, n, std::move(val));
  Rng rr(P, RngStream::rhs);
  std::vector<double> xs(static_cast<std::size_t>(n));
  for (auto& x : xs) x = rr.gaussian();
  g.b.assign(static_cast<std::size_t>(m), 0.0);
  // A x* in Matrix::matvec's order (column axpy, matrix.hpp:156-162); rows
  // are independent chains, so row blocks run in parallel with the same bits
  auto a = g.a.dense_data();
  par_for(m, threads, [&](std::int64_t i0, std::int64_t i1) {
    for (Index j = 0; j < n; ++j) {
      if (xs[j] == 0.0) continue;
      for (Index i = i0; i < i1; ++i) g.b[i] += xs[j] * a[j * m + i];
    }
  });
  for (Index i = 0; i < m; ++i) g.b[i] += 1e-3 * rr.gaussian();
}

void gen_c4(RefGen& g, Index m, Index n, std::uint64_t P, int threads) {
  const Index k = std::max<Index>(1, std::min<Index>(200, std::min(m, n) / 2));
  Rng ru(P, RngStream::user, 0), rv(P, RngStream::user, 1);
  Matrix u = thin_qr(detail::gaussian_dense(m, k, ru)).q;
  Matrix v = thin_qr(detail::gaussian_dense(n, k, rv)).q;
  std::vector<double> s = k == 1 ? std::vector<double>{100.0} : logspace(4.0, 2.0, k);
  auto ud = u.dense_data(), vd = v.dense_data();
  std::vector<double> val(static_cast<std::size_t>(m * n));
  const double isq = 1.0 / std::sqrt(static_cast<double>(m));
  par_for(n, threads, [&](std::int64_t j0, std::int64_t j1) {
    for (Index j = j0; j < j1; ++j) {
      Rng rg(P, RngStream::problem, static_cast<std::uint64_t>(j));
      double* col = val.data() + j * m;
      for (Index i = 0; i < m; ++i) col[i] = rg.gaussian() * isq;
      for (Index t = 0; t < k; ++t) {  // + U(:,t) s_t V(j,t), t ascending
        const double c = s[t] * vd[t * n + j];
        for (Index i = 0; i < m; ++i) col[i] += c * ud[t * m + i];
      }
    }
  });
  g.a = Matrix::dense(m, n, std::move(val));
  Rng rr(P, RngStream::rhs);
  g.b.resize(static_cast<std::size_t>(m));
  for (auto& x : g.b) x = rr.gaussian();
}

void gen_c5(RefGen& g, Index m, Index n, std::uint64_t P, int threads) {
  const Index per_row = std::min<Index>(16, n);
  const double zipf_s = 1.1, decades = 3.0;
  std::vector<Index> perm(static_cast<std::size_t>(n));  // Fisher-Yates shuffle of the column ids
  std::iota(perm.begin(), perm.end(), Index{0});
  Rng rperm(P, RngStream::problem, 0);
  for (Index i = n - 1; i >= 1; --i)
    std::swap(perm[i], perm[static_cast<Index>(rperm.below(static_cast<std::uint64_t>(i + 1)))]);
  std::vector<double> scale(static_cast<std::size_t>(n));
  Rng rs(P, RngStream::problem, 1);
  for (auto& s : scale) s = std::pow(10.0, -decades * rs.uniform());
  std::vector<double> cdf(static_cast<std::size_t>(n));  // Zipf(s) over ranks 1..n
  double acc = 0.0;
  for (Index z = 1; z <= n; ++z) cdf[z - 1] = (acc += std::pow(static_cast<double>(z), -zipf_s));
  for (auto& c : cdf) c /= acc;
  const Index blk_rows = 65536, nblk = (m + blk_rows - 1) / blk_rows;
  std::vector<std::vector<Index>> bc(static_cast<std::size_t>(nblk));
  std::vector<std::vector<double>> bv(static_cast<std::size_t>(nblk));
  par_for(nblk, threads, [&](std::int64_t b0, std::int64_t b1) {
    std::vector<char> seen(static_cast<std::size_t>(n), 0);
    std::vector<Index> row;
    for (Index blk = b0; blk < b1; ++blk) {
      Rng r(P, RngStream::problem, 2 + static_cast<std::uint64_t>(blk));
      for (Index i = blk * blk_rows; i < std::min(m, (blk + 1) * blk_rows); ++i) {
        row.clear();
        while (static_cast<Index>(row.size()) < per_row) {  // inverse CDF, redraw duplicates
          double u = r.uniform();
          Index z = std::min<Index>(n - 1, std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
          Index c = perm[z];
          if (seen[c]) continue;
          seen[c] = 1;
          row.push_back(c);
        }
        std::sort(row.begin(), row.end());
        for (Index c : row) {
          seen[c] = 0;
          bc[blk].push_back(c);
          bv[blk].push_back(r.gaussian() * scale[c]);
        }
      }
    }
  });
  std::vector<Index> cptr(static_cast<std::size_t>(n) + 1, 0);
  for (const auto& v : bc)
    for (Index c : v) ++cptr[c + 1];
  for (Index j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
  std::vector<Index> ridx(static_cast<std::size_t>(cptr[n]));
  std::vector<double> val(ridx.size());
  std::vector<Index> next(cptr.begin(), cptr.end() - 1);
  for (Index blk = 0; blk < nblk; ++blk) {
    for (std::size_t q = 0; q < bc[blk].size(); ++q) {
      Index at = next[bc[blk][q]]++;
      ridx[at] = blk * blk_rows + static_cast<Index>(q) / per_row;
      val[at] = bv[blk][q];
    }
    std::vector<Index>().swap(bc[blk]);
    std::vector<double>().swap(bv[blk]);
  }
  g.a = csc_matrix(m, n, std::move(cptr), std::move(ridx), std::move(val));
  Rng rr(P, RngStream::rhs);
  g.b.resize(static_cast<std::size_t>(m));
  for (auto& x : g.b) x = rr.gaussian();
}

}  // namespace

extern "C" {

// config 1..5; m, n = 0 -> the BASELINE shape; seed 0 -> 20260415 + config.
int ref_generate(std::int32_t config, std::int64_t m, std::int64_t n, std::uint64_t seed, std::int32_t threads,
                 RefGen** out) {
  return guarded([&] {
    static const Index dm[6] = {0, 4000, 200000, 100000, 50000, 8000000};
    static const Index dn[6] = {0, 500, 20000, 10000, 50000, 400000};
    detail::require(config >= 1 && config <= 5, ErrorKind::invalid_argument, "config must be 1..5");
    m = m > 0 ? m : dm[config];
    n = n > 0 ? n : dn[config];
    const std::uint64_t P = seed ? seed : 20260415ULL + static_cast<std::uint64_t>(config);
    auto g = std::make_unique<RefGen>();
    switch (config) {
      case 1: gen_c1(*g, m, n, P); break;
      case 2: gen_c2(*g, m, n, P); break;
      case 3: gen_c3(*g, m, n, P, threads); break;
      case 4: gen_c4(*g, m, n, P, threads); break;
      default: gen_c5(*g, m, n, P, threads); break;
    }
    *out = g.release();
  });
}

// Borrowed view of a generated input (valid until ref_gen_free).
int ref_gen_view(const RefGen* g, RefProblem* view, const double** b) {
  return guarded([&] {
    view->m = g->a.rows();
    view->n = g->a.cols();
    view->sparse = g->a.is_sparse() ? 1 : 0;
    view->dense = g->a.is_sparse() ? nullptr : g->a.dense_data().data();
    view->colptr = g->a.is_sparse() ? g->a.col_ptr().data() : nullptr;
    view->rowidx = g->a.is_sparse() ? g->a.row_idx().data() : nullptr;
    view->vals = g->a.is_sparse() ? g->a.values().data() : nullptr;
    *b = g->b.data();
  });
}

void ref_gen_free(RefGen* g) { delete g; }

// aplicur_solve / plain_lsqr_solve on a generated input without copying it
// into a second Matrix (C4 is 20 GB); consume != 0 moves A into the solve and
// leaves the handle's matrix empty.  b == nullptr uses the generated b.
int ref_solve_gen(RefGen* g, const double* b, const RefConfig* cfg, std::int32_t plain, std::int32_t consume,
                  RefOut* out) {
  return guarded([&] {
    ProblemInstance prob;
    prob.a = consume ? std::move(g->a) : g->a;
    if (b)
      prob.b.assign(b, b + prob.a.rows());
    else
      prob.b = g->b;
    prob.mu = cfg->mu;
    SolverConfig sc = make_config(cfg);
    auto t0 = std::chrono::steady_clock::now();
    SolveResult r = plain ? plain_lsqr_solve(prob, sc) : aplicur_solve(prob, sc);
    out->wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fill_out(r, out);
  });
}

// ---- Matrix Market (matrix_market.hpp:18-116) --------------------------------
int ref_mm_write(const RefProblem* p, const char* path) {
  return guarded([&] { write_matrix_market(make_matrix(p), std::string(path)); });
}

// two calls: sizes first (array pointers null), then the arrays (CSC or dense)
int ref_mm_read(const char* path, std::int64_t* m, std::int64_t* n, std::int32_t* sparse, std::int64_t* nnz,
                std::int64_t* colptr, std::int64_t* rowidx, double* vals, double* dense) {
  return guarded([&] {
    Matrix a = read_matrix_market(std::string(path));
    *m = a.rows();
    *n = a.cols();
    *sparse = a.is_sparse() ? 1 : 0;
    *nnz = a.nnz();
    if (a.is_sparse()) {
      if (colptr) std::copy(a.col_ptr().begin(), a.col_ptr().end(), colptr);
      if (rowidx) std::copy(a.row_idx().begin(), a.row_idx().end(), rowidx);
      if (vals) std::copy(a.values().begin(), a.values().end(), vals);
    } else if (dense) {
      std::copy(a.dense_data().begin(), a.dense_data().end(), dense);
    }
  });
}

}  // extern "C"
