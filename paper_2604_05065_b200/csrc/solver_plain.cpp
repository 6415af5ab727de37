// plain_lsqr_solve on the device (solver.hpp:396-448): unpreconditioned
// LSQR on [A; mu I] (or A), reported in the SolveResult shape.
#include <chrono>
#include <cmath>
#include <limits>

#include "solver.hpp"
#include "vec.hpp"

namespace apc {

apc_solver_config resolve_config(const apc_solver_config& in, i64 n) {
  apc_solver_config c = in;
  if (c.block <= 0)
    c.block = std::max<i64>(1, static_cast<i64>(std::llround(static_cast<double>(n) / 50.0)));
  c.block = std::min<i64>(c.block, n);
  if (c.eps_cur < 0.0) c.eps_cur = 30.0 * c.mu;
  require(c.mu >= 0.0, APC_INVALID_ARGUMENT, "SolverConfig: mu >= 0");
  require(c.nu_prec > 1.0, APC_INVALID_ARGUMENT, "SolverConfig: nu_prec > 1");
  require(c.nu_lsqr > 1.0, APC_INVALID_ARGUMENT, "SolverConfig: nu_lsqr > 1");
  require(c.eps_lsqr > 0.0, APC_INVALID_ARGUMENT, "SolverConfig: eps_lsqr > 0");
  require(c.sketch_xi >= 1 && c.probe_count >= 1, APC_INVALID_ARGUMENT,
          "SolverConfig: sketch parameters must be positive");
  return c;
}

double host_norm(const double* v, i64 n) {  // vec_norm (problems.hpp:258-262)
  double s = 0.0;
  for (i64 i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

apc_result* plain_solve(apc_mat& a, const double* b, const apc_solver_config& cfg_in) {
  using clock = std::chrono::steady_clock;
  auto t0 = clock::now();
  apc_solver_config cfg = resolve_config(cfg_in, a.n);
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  const double mu = cfg.mu;
  const i64 n = a.n, mloc = a.mloc();
  const double bnorm = host_norm(b, a.m);
  const i64 ulen = mloc + (mu > 0.0 ? n : 0);

  DBuf<double> d_b(std::max<i64>(1, mloc)), d_rhs(std::max<i64>(1, ulen)), d_x(std::max<i64>(1, n));
  if (mloc > 0)
    APC_CUDA(cudaMemcpyAsync(d_b.p, b + a.r0, sizeof(double) * mloc, cudaMemcpyHostToDevice, st));
  APC_CUDA(cudaMemsetAsync(d_rhs.p, 0, d_rhs.bytes(), st));
  if (mloc > 0)
    APC_CUDA(cudaMemcpyAsync(d_rhs.p, d_b.p, sizeof(double) * mloc, cudaMemcpyDeviceToDevice, st));

  StopCfg stop;
  stop.eps_lsqr = cfg.eps_lsqr;
  stop.nu_lsqr = std::numeric_limits<double>::infinity();  // StopConfig default
  stop.max_iters = cfg.lsqr_cap > 0 ? cfg.lsqr_cap : 4 * n;
  LsqrWork* w = lsqr_work_create(a, mu);
  PhaseOut po;
  try {
    SampleCfg samp;  // the observer of plain_lsqr_solve samples y itself (solver.hpp:418-427)
    samp.stride = cfg.trace_sample_stride;
    samp.b_local = d_b.p;
    samp.bnorm = bnorm;
    lsqr_phase(w, a, mu, nullptr, d_rhs.p, stop, 1, d_x.p, po, &samp);
  } catch (...) {
    lsqr_work_destroy(w);
    throw;
  }
  lsqr_work_destroy(w);

  auto* r = new apc_result();
  r->n = n;
  r->x.resize(static_cast<size_t>(n));
  copy_sync(st, r->x.data(), d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost);
  VecWork vw(a, mu);
  const double rr = bnorm > 0.0 ? std::sqrt(residual(a, vw, d_x.p, d_b.p, nullptr)) / bnorm : 0.0;
  for (size_t k = 0; k < po.rows.size(); ++k) {
    const auto& row = po.rows[k];
    const double tr = k < po.sampled.size() ? po.sampled[k] : std::numeric_limits<double>::quiet_NaN();
    r->trace.push_back(apc_trace_row{1, 0, row.iter, row.phibar, row.cvgrate, row.cvgdiff, row.matvecs,
                                     row.wall_ms, tr});
  }
  apc_phase_report rep{};
  rep.phase = 1;
  rep.reason = po.reason;
  rep.rank = 0;
  rep.mu = mu;
  rep.lsqr_iters = po.iters;
  rep.t_lsqr_ms = po.ms;
  rep.t_lsqr_device_ms = po.device_ms;
  rep.relres_at_end = rr;
  r->phases.push_back(rep);
  r->spectra.emplace_back();
  r->last_reason = po.reason;
  r->final_relres = rr;
  r->final_rho = std::numeric_limits<double>::infinity();
  r->system_matvecs = po.iters > 0 ? 1 + 2 * static_cast<std::uint64_t>(po.iters)
                                   : (po.reason == 5 ? 0 : 1);
  r->status = 0;
  r->lsqr_ms = po.ms;
  r->total_ms = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
  r->setup_ms = r->total_ms - r->lsqr_ms;
  return r;
}

}  // namespace apc
