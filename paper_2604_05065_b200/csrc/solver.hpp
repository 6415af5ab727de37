// Host orchestration of a solve (the drop-in for aplicur_solve /
// plain_lsqr_solve, /root/reference/proj/include/aplicur/solver.hpp:162-448).
#pragma once

#include <vector>

#include "apc_internal.hpp"
#include "lsqr.hpp"

struct apc_result {
  apc::i64 n = 0;
  std::vector<double> x;
  std::vector<apc_phase_report> phases;
  std::vector<std::vector<double>> spectra;  // PhaseReport::precond_spectrum per phase
  std::vector<apc_trace_row> trace;
  int status = 0;  // SolveStatus
  int last_reason = 0;
  double final_rho = 0.0, final_relres = 0.0;
  std::uint64_t sketch_applications = 0, system_matvecs = 0;
  std::vector<std::int64_t> rows, cols;
  std::vector<double> rho_history;
  double total_ms = 0.0, lsqr_ms = 0.0, setup_ms = 0.0;
};

namespace apc {

// SolverConfig::resolved / validate (solver.hpp:47-62)
apc_solver_config resolve_config(const apc_solver_config& in, i64 n);

apc_result* plain_solve(apc_mat& a, const double* b, const apc_solver_config& cfg);
apc_result* aplicur_solve(apc_mat& a, const double* b, const apc_solver_config& cfg,
                          const apc_hooks* hooks = nullptr);
apc_result* aplicur_solve_sharded(apc_mat& full, apc_mat& shard, const double* b, const apc_solver_config& cfg,
                                  const apc_hooks* hooks = nullptr);

}  // namespace apc
