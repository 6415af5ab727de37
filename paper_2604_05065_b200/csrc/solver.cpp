// aplicur_solve outer loop (placeholder until the CUR path lands).
#include "solver.hpp"

namespace apc {

apc_result* aplicur_solve(apc_mat& a, const double* b, const apc_solver_config& cfg) {
  (void)a; (void)b; (void)cfg;
  fail(APC_NOT_APPLICABLE, "aplicur_solve: CUR path not built yet");
}

}  // namespace apc
