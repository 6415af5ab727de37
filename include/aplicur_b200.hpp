// aplicur_b200.hpp -- drop-in C++ front end for the B200 APLICUR hot path.
//
// Declares the reference's public solver API in namespace aplicur with the
// same names, fields and defaults (/root/reference/proj/include/aplicur/
// solver.hpp:29-120,162,396; lsqr.hpp:17-52; matrix.hpp:35-100; error.hpp;
// problems.hpp:251-256), implemented header-only over the C-ABI of
// libapc_b200.so (include/apc_b200.h).  A caller of aplicur_solve /
// plain_lsqr_solve switches by including this header instead of
// "aplicur/solver.hpp" and linking -lapc_b200; no source changes.
//
// The matrix is uploaded to the GPU on first use and cached with the Matrix
// (copies share the device image, like the reference's shared transpose box).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "apc_b200.h"

namespace aplicur {

using Index = std::int64_t;
using IndexList = std::vector<Index>;

enum class ErrorKind {  // error.hpp:10-20
  invalid_argument, dimension_mismatch, rank_deficient, singular, not_positive,
  no_convergence, numerical_breakdown, not_applicable, io,
};

class Error : public std::runtime_error {  // error.hpp:24-35
 public:
  Error(ErrorKind kind, const std::string& what, std::int64_t index = -1)
      : std::runtime_error(what), kind_(kind), index_(index) {}
  ErrorKind kind() const noexcept { return kind_; }
  std::int64_t index() const noexcept { return index_; }

 private:
  ErrorKind kind_;
  std::int64_t index_;
};

namespace b200 {
inline void check(int code) {
  if (code == APC_OK) return;
  std::int64_t idx = -1;
  const char* msg = apc_last_error(&idx);
  if (code >= 1 && code <= 9) throw Error(static_cast<ErrorKind>(code - 1), msg, idx);
  throw std::runtime_error(std::string("libapc_b200: ") + msg);
}

// one context per thread (device from APC_DEVICE, default 0)
inline apc_ctx* default_ctx() {
  struct Holder {
    apc_ctx* c = nullptr;
    ~Holder() { if (c) apc_ctx_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) {
    const char* d = std::getenv("APC_DEVICE");
    check(apc_ctx_create(d ? std::atoi(d) : 0, 1, 0, nullptr, &h.c));
  }
  return h.c;
}
}  // namespace b200

struct Triplet {
  Index row;
  Index col;
  double value;
};

/// Dense column-major or CSC (int64) matrix, immutable (matrix.hpp:35-100).
class Matrix {
 public:
  Matrix() = default;

  static Matrix dense(Index m, Index n, std::vector<double> colmajor) {
    if (m < 0 || n < 0) throw Error(ErrorKind::invalid_argument, "negative matrix shape");
    if (static_cast<Index>(colmajor.size()) != m * n)
      throw Error(ErrorKind::dimension_mismatch, "Matrix::dense: buffer size mismatch");
    Matrix a;
    a.rows_ = m;
    a.cols_ = n;
    a.val_ = std::move(colmajor);
    a.dev_ = std::make_shared<DeviceBox>();
    return a;
  }

  /// CSC from triplets; duplicates rejected, exact zeros dropped (matrix.hpp:66-94).
  static Matrix sparse(Index m, Index n, std::vector<Triplet> entries) {
    if (m < 0 || n < 0) throw Error(ErrorKind::invalid_argument, "negative matrix shape");
    for (const auto& t : entries)
      if (t.row < 0 || t.row >= m || t.col < 0 || t.col >= n)
        throw Error(ErrorKind::invalid_argument, "Matrix::sparse: entry out of range");
    std::sort(entries.begin(), entries.end(), [](const Triplet& x, const Triplet& y) {
      return std::tie(x.col, x.row) < std::tie(y.col, y.row);
    });
    Matrix a;
    a.rows_ = m;
    a.cols_ = n;
    a.sparse_ = true;
    a.cptr_.assign(static_cast<size_t>(n) + 1, 0);
    for (size_t k = 0; k < entries.size(); ++k) {
      if (k > 0 && entries[k].row == entries[k - 1].row && entries[k].col == entries[k - 1].col)
        throw Error(ErrorKind::invalid_argument, "Matrix::sparse: duplicate entry");
      if (entries[k].value == 0.0) continue;
      a.ridx_.push_back(entries[k].row);
      a.val_.push_back(entries[k].value);
      ++a.cptr_[static_cast<size_t>(entries[k].col) + 1];
    }
    for (Index j = 0; j < n; ++j) a.cptr_[j + 1] += a.cptr_[j];
    a.dev_ = std::make_shared<DeviceBox>();
    return a;
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  bool is_sparse() const { return sparse_; }
  Index nnz() const { return sparse_ ? static_cast<Index>(val_.size()) : rows_ * cols_; }
  double density() const {
    return rows_ * cols_ == 0 ? 0.0 : static_cast<double>(nnz()) / static_cast<double>(rows_ * cols_);
  }
  std::span<const double> dense_data() const { return val_; }
  std::span<const Index> col_ptr() const { return cptr_; }
  std::span<const Index> row_idx() const { return ridx_; }
  std::span<const double> values() const { return val_; }

  /// y = A x / y = A^T x, evaluated on the GPU (matrix.hpp:151-195)
  void matvec(std::span<const double> x, std::span<double> y) const { apply(x, y, false); }
  void matvec_transpose(std::span<const double> x, std::span<double> y) const { apply(x, y, true); }

  /// device image (uploaded once, shared by copies)
  apc_mat* device() const {
    std::call_once(dev_->flag, [this] {
      apc_ctx* ctx = b200::default_ctx();
      if (sparse_)
        b200::check(apc_mat_upload_csc(ctx, rows_, cols_, cptr_.data(), ridx_.data(), val_.data(), 0, rows_,
                                       &dev_->mat));
      else
        b200::check(apc_mat_upload_dense(ctx, rows_, cols_, val_.data(), 0, rows_, &dev_->mat));
    });
    return dev_->mat;
  }

 private:
  struct DeviceBox {
    std::once_flag flag;
    apc_mat* mat = nullptr;
    ~DeviceBox() { if (mat) apc_mat_free(mat); }
  };
  void apply(std::span<const double> x, std::span<double> y, bool t) const {
    if (static_cast<Index>(x.size()) != (t ? rows_ : cols_) || static_cast<Index>(y.size()) != (t ? cols_ : rows_))
      throw Error(ErrorKind::dimension_mismatch, t ? "matvec_transpose: shape mismatch" : "matvec: shape mismatch");
    b200::check(apc_op_apply_host(device(), 0.0, 0, t ? 1 : 0, x.data(), y.data()));
  }

  Index rows_ = 0, cols_ = 0;
  bool sparse_ = false;
  std::vector<double> val_;
  std::vector<Index> ridx_, cptr_;
  std::shared_ptr<DeviceBox> dev_;
};

struct ProblemMetadata {  // problems.hpp:242-248
  std::optional<std::vector<double>> x_star;
  double noise_norm = std::numeric_limits<double>::quiet_NaN();
  std::optional<double> opt_relres_unreg, opt_relres_reg, coherence;
};

struct ProblemInstance {  // problems.hpp:251-256
  Matrix a;
  std::vector<double> b;
  double mu = 0.0;
  ProblemMetadata meta;
};

enum class CoreFactorKind { qr, lu };
enum class PrecondVariant { svd, svd_free };
enum class StopReason { none, gradient_tol, dynamic_rate, dynamic_diff, iteration_cap, exact_zero_rhs };
enum class SolveStatus { converged, rank_exhausted, breakdown };

struct SolverConfig {  // solver.hpp:29-45 (+ sketch selection)
  Index block = 0;
  double eps_cur = -1.0;
  double eps_lsqr = 1e-10;
  double nu_prec = 10.0;
  double nu_lsqr = 100.0;
  double mu = 0.0;
  PrecondVariant variant = PrecondVariant::svd;
  Index sketch_xi = 8;
  Index probe_count = 10;
  Index lsqr_cap = 0;
  Index max_rank = 0;
  std::uint64_t seed = 0;
  CoreFactorKind core = CoreFactorKind::qr;
  Index trace_sample_stride = 1;
  Index outer_cap = 100000;
  bool gaussian_sketch = false;  // BASELINE C1/C3/C4 ask for a Gaussian embedding
};

struct LsqrTraceRow {  // lsqr.hpp:38-47
  int phase = 0;
  Index iter = 0;
  double phibar = 0.0, cvgrate = 0.0, cvgdiff = 0.0;
  std::uint64_t matvecs = 0;
  double wall_ms = 0.0;
  double true_relres = std::numeric_limits<double>::quiet_NaN();
};

struct LsqrTrace {
  std::vector<LsqrTraceRow> rows;
  StopReason reason = StopReason::none;
};

struct PhaseReport {  // solver.hpp:74-88
  int phase = 0;
  Index rank = 0;
  double rho = 0.0, sigma_hat = 0.0, mu = 0.0;
  Index lsqr_iters = 0;
  StopReason reason = StopReason::none;
  double t_augment_ms = 0.0, t_factor_ms = 0.0, t_precond_ms = 0.0, t_lsqr_ms = 0.0;
  double relres_at_end = 0.0;
  std::vector<double> precond_spectrum;
};

struct SolveResult {  // solver.hpp:101-112
  std::vector<double> x;
  std::vector<PhaseReport> phases;
  LsqrTrace trace;
  SolveStatus status = SolveStatus::converged;
  double final_rho = std::numeric_limits<double>::infinity();
  double final_relres = 0.0;
  std::uint64_t sketch_applications = 0;
  std::uint64_t system_matvecs = 0;
  IndexList row_indices, col_indices;
  std::vector<double> rho_history;
};

namespace b200 {
inline apc_solver_config to_c(const SolverConfig& c) {
  apc_solver_config k;
  apc_config_default(&k);
  k.block = c.block;
  k.eps_cur = c.eps_cur;
  k.eps_lsqr = c.eps_lsqr;
  k.nu_prec = c.nu_prec;
  k.nu_lsqr = c.nu_lsqr;
  k.mu = c.mu;
  k.variant = c.variant == PrecondVariant::svd ? 0 : 1;
  k.core = c.core == CoreFactorKind::qr ? 0 : 1;
  k.sketch_xi = c.sketch_xi;
  k.probe_count = c.probe_count;
  k.lsqr_cap = c.lsqr_cap;
  k.max_rank = c.max_rank;
  k.seed = c.seed;
  k.trace_sample_stride = c.trace_sample_stride;
  k.outer_cap = c.outer_cap;
  k.sketch_kind = c.gaussian_sketch ? 1 : 0;
  return k;
}

inline SolveResult run(const ProblemInstance& p, const SolverConfig& c, int plain, const apc_hooks* hooks = nullptr) {
  apc_solver_config k = to_c(c);
  if (static_cast<Index>(p.b.size()) != p.a.rows())
    throw Error(ErrorKind::dimension_mismatch, "aplicur_solve: rhs length mismatch");
  apc_result* r = nullptr;
  if (hooks) check(apc_solve_hooked(nullptr, p.a.device(), p.b.data(), &k, hooks, &r));
  else check(apc_solve(p.a.device(), p.b.data(), &k, plain, &r));
  std::unique_ptr<apc_result, int (*)(apc_result*)> guard(r, apc_result_free);
  int status = 0;
  std::int64_t nph = 0, ntr = 0, rank = 0, nrho = 0;
  SolveResult out;
  apc_result_summary(r, &status, &out.final_rho, &out.final_relres, &out.sketch_applications, &out.system_matvecs,
                     &nph, &ntr, &rank, &nrho);
  out.status = static_cast<SolveStatus>(status);
  out.x.resize(static_cast<size_t>(p.a.cols()));
  apc_result_x(r, out.x.data());
  out.row_indices.resize(static_cast<size_t>(rank));
  out.col_indices.resize(static_cast<size_t>(rank));
  apc_result_indices(r, out.row_indices.data(), out.col_indices.data());
  out.rho_history.resize(static_cast<size_t>(nrho));
  apc_result_rho_history(r, out.rho_history.data());
  std::vector<apc_phase_report> ph(static_cast<size_t>(nph));
  apc_result_phases(r, ph.data());
  for (size_t k = 0; k < ph.size(); ++k) {
    const apc_phase_report& q = ph[k];
    PhaseReport rep;
    std::int64_t ns = 0;
    apc_result_phase_spectrum(r, static_cast<std::int64_t>(k), nullptr, &ns);
    rep.precond_spectrum.resize(static_cast<size_t>(ns));
    apc_result_phase_spectrum(r, static_cast<std::int64_t>(k), rep.precond_spectrum.data(), &ns);
    rep.phase = q.phase;
    rep.rank = q.rank;
    rep.rho = q.rho;
    rep.sigma_hat = q.sigma_hat;
    rep.mu = q.mu;
    rep.lsqr_iters = q.lsqr_iters;
    rep.reason = static_cast<StopReason>(q.reason);
    rep.t_augment_ms = q.t_augment_ms;
    rep.t_factor_ms = q.t_factor_ms;
    rep.t_precond_ms = q.t_precond_ms;
    rep.t_lsqr_ms = q.t_lsqr_ms;
    rep.relres_at_end = q.relres_at_end;
    out.phases.push_back(std::move(rep));
  }
  std::vector<apc_trace_row> tr(static_cast<size_t>(ntr));
  apc_result_trace(r, tr.data());
  for (const auto& t : tr)
    out.trace.rows.push_back({t.phase, t.iter, t.phibar, t.cvgrate, t.cvgdiff, t.matvecs, t.wall_ms, t.true_relres});
  if (!out.phases.empty()) out.trace.reason = out.phases.back().reason;
  return out;
}
}  // namespace b200

/// Views handed to SolveHooks::on_rebuild.  The CUR state and the
/// preconditioner live on the device, so the hook sees their host-side
/// summary (CurState::row_indices/col_indices/rank/rho, cur.hpp:228-242;
/// Preconditioner::rank/target_level, SvdPreconditioner spectra,
/// preconditioner.hpp:19-56) instead of the objects themselves.
struct CurStateView {
  Index rank = 0;
  std::span<const Index> row_indices, col_indices;
  double rho = 0.0;
};
struct PreconditionerView {
  Index rank = 0;
  PrecondVariant variant = PrecondVariant::svd;
  double target_level = 0.0;
  double smallest_cur_sigma = 0.0;           // svd; svd-free: target_level
  std::span<const double> cur_spectrum;          // svd variant only
  std::span<const double> regularized_spectrum;  // svd variant only
};

/// Diagnostic observers (solver.hpp:114-120); they must not mutate solver state.
struct SolveHooks {
  // after a preconditioner rebuild, before its LSQR phase
  std::function<void(const CurStateView&, const PreconditionerView&, int phase)> on_rebuild;
  // at the end of each phase: (phase, x so far)
  std::function<void(int phase, std::span<const double> x)> on_phase_end;
};

namespace b200 {
struct HookBridge {
  const SolveHooks* hooks;
  std::exception_ptr error;
  static void rebuild(void* user, const apc_rebuild_info* ri) {
    auto* self = static_cast<HookBridge*>(user);
    if (self->error) return;
    try {
      CurStateView cv{ri->rank, {ri->rows, static_cast<size_t>(ri->rank)}, {ri->cols, static_cast<size_t>(ri->rank)},
                      ri->rho};
      PreconditionerView pv{ri->rank, static_cast<PrecondVariant>(ri->variant), ri->sigma_hat, ri->sigma_floor,
                            {ri->sigma_cur, static_cast<size_t>(ri->sigma_cur ? ri->n_sigma : 0)},
                            {ri->sigma_reg, static_cast<size_t>(ri->sigma_reg ? ri->n_sigma : 0)}};
      self->hooks->on_rebuild(cv, pv, ri->phase);
    } catch (...) {
      self->error = std::current_exception();
    }
  }
  static void phase_end(void* user, std::int32_t phase, const double* x, std::int64_t n) {
    auto* self = static_cast<HookBridge*>(user);
    if (self->error) return;
    try {
      self->hooks->on_phase_end(phase, std::span<const double>(x, static_cast<size_t>(n)));
    } catch (...) {
      self->error = std::current_exception();
    }
  }
};
}  // namespace b200

/// solver.hpp:162 -- adaptive CUR-preconditioned LSQR on the GPU.  A hook
/// that throws stops forwarding further callbacks; its exception is rethrown
/// after the solve returns.
inline SolveResult aplicur_solve(const ProblemInstance& problem, const SolverConfig& config,
                                 const SolveHooks* hooks = nullptr) {
  if (!hooks || (!hooks->on_rebuild && !hooks->on_phase_end)) return b200::run(problem, config, 0);
  b200::HookBridge bridge{hooks, nullptr};
  apc_hooks h{&bridge, hooks->on_rebuild ? &b200::HookBridge::rebuild : nullptr,
              hooks->on_phase_end ? &b200::HookBridge::phase_end : nullptr};
  SolveResult r = b200::run(problem, config, 0, &h);
  if (bridge.error) std::rethrow_exception(bridge.error);
  return r;
}

/// solver.hpp:396 -- unpreconditioned LSQR baseline on the GPU
inline SolveResult plain_lsqr_solve(const ProblemInstance& problem, const SolverConfig& config) {
  return b200::run(problem, config, 1);
}

// ---------------------------------------------------------------------------
// Formats around the path (host only): Matrix Market (matrix_market.hpp:18-116),
// trace CSV and solve report JSON (report_io.hpp:28-122), same names.
// ---------------------------------------------------------------------------
inline void write_matrix_market(const Matrix& a, const std::string& path) {
  if (a.is_sparse())
    b200::check(apc_mm_write_csc(path.c_str(), a.rows(), a.cols(), a.col_ptr().data(), a.row_idx().data(),
                                 a.values().data()));
  else
    b200::check(apc_mm_write_dense(path.c_str(), a.rows(), a.cols(), a.dense_data().data()));
}

inline Matrix read_matrix_market(const std::string& path) {
  apc_problem* h = nullptr;
  b200::check(apc_mm_read(path.c_str(), &h));
  std::unique_ptr<apc_problem, int (*)(apc_problem*)> guard(h, apc_problem_free);
  std::int64_t m = 0, n = 0, nnz = 0;
  int sparse = 0;
  apc_problem_info(h, &m, &n, &sparse, &nnz);
  if (!sparse) {
    const double* d = apc_problem_dense(h);
    return Matrix::dense(m, n, std::vector<double>(d, d + m * n));
  }
  const std::int64_t *cp = nullptr, *ri = nullptr;
  const double* va = nullptr;
  b200::check(apc_problem_csc(h, &cp, &ri, &va));
  std::vector<Triplet> t;
  t.reserve(static_cast<size_t>(nnz));
  for (Index j = 0; j < n; ++j)
    for (Index k = cp[j]; k < cp[j + 1]; ++k) t.push_back({ri[k], j, va[k]});
  return Matrix::sparse(m, n, std::move(t));
}

namespace b200 {
inline std::vector<apc_phase_report> to_c(std::span<const PhaseReport> phases) {
  std::vector<apc_phase_report> out;
  for (const auto& p : phases) {
    apc_phase_report q{};
    q.phase = p.phase;
    q.reason = static_cast<std::int32_t>(p.reason);
    q.rank = p.rank;
    q.rho = p.rho;
    q.sigma_hat = p.sigma_hat;
    q.mu = p.mu;
    q.lsqr_iters = p.lsqr_iters;
    q.t_augment_ms = p.t_augment_ms;
    q.t_factor_ms = p.t_factor_ms;
    q.t_precond_ms = p.t_precond_ms;
    q.t_lsqr_ms = p.t_lsqr_ms;
    q.relres_at_end = p.relres_at_end;
    out.push_back(q);
  }
  return out;
}
}  // namespace b200

/// report_io.hpp:28-47 (written to path.tmp, then renamed)
inline void trace_to_csv(const LsqrTrace& trace, const std::string& path, std::span<const PhaseReport> phases = {}) {
  std::vector<apc_trace_row> rows;
  for (const auto& r : trace.rows)
    rows.push_back({r.phase, 0, r.iter, r.phibar, r.cvgrate, r.cvgdiff, r.matvecs, r.wall_ms, r.true_relres});
  const auto ph = b200::to_c(phases);
  b200::check(apc_trace_csv_write(path.c_str(), rows.data(), static_cast<std::int64_t>(rows.size()), ph.data(),
                                  static_cast<std::int64_t>(ph.size()), static_cast<std::int32_t>(trace.reason)));
}

/// report_io.hpp:94-122: solve report JSON, atomic write
inline void write_solve_report(const SolverConfig& config, const SolveResult& r, const std::string& trace_path,
                               const std::string& path) {
  const apc_solver_config k = b200::to_c(config);
  const auto ph = b200::to_c(r.phases);
  std::vector<const double*> spec;
  std::vector<std::int64_t> nspec;
  for (const auto& p : r.phases) {
    spec.push_back(p.precond_spectrum.data());
    nspec.push_back(static_cast<std::int64_t>(p.precond_spectrum.size()));
  }
  b200::check(apc_report_json_write(path.c_str(), &k, static_cast<std::int32_t>(r.status), r.final_relres, r.final_rho,
                                    r.sketch_applications, r.system_matvecs, trace_path.c_str(),
                                    r.row_indices.data(), r.col_indices.data(),
                                    static_cast<std::int64_t>(r.row_indices.size()), r.rho_history.data(),
                                    static_cast<std::int64_t>(r.rho_history.size()), ph.data(),
                                    static_cast<std::int64_t>(ph.size()), spec.data(), nspec.data()));
}

}  // namespace aplicur
