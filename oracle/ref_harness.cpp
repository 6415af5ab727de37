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
