// Drop-in check: reference-style caller code compiled against
// include/aplicur_b200.hpp + libapc_b200.so (no source changes beyond the
// include).  Prints a JSON summary for tests/test_gpu_dropin.py.
#include <cstdio>
#include <vector>

#include "aplicur_b200.hpp"

int main(int argc, char** argv) {
  using namespace aplicur;
  const int cfg = argc > 1 ? std::atoi(argv[1]) : 2;
  const Index m = argc > 2 ? std::atoll(argv[2]) : 4000, n = argc > 3 ? std::atoll(argv[3]) : 400;
  apc_problem* gp = nullptr;
  if (apc_problem_generate(cfg, m, n, 0, &gp) != APC_OK) return 2;
  int sparse = 0;
  std::int64_t mm, nn, nnz;
  apc_problem_info(gp, &mm, &nn, &sparse, &nnz);
  ProblemInstance p;
  if (sparse) {
    const std::int64_t *cp, *ri;
    const double* va;
    apc_problem_csc(gp, &cp, &ri, &va);
    std::vector<Triplet> t;
    for (Index j = 0; j < nn; ++j)
      for (Index k = cp[j]; k < cp[j + 1]; ++k) t.push_back({ri[k], j, va[k]});
    p.a = Matrix::sparse(mm, nn, std::move(t));
  } else {
    const double* d = apc_problem_dense(gp);
    p.a = Matrix::dense(mm, nn, std::vector<double>(d, d + mm * nn));
  }
  const double* b = apc_problem_b(gp);
  p.b.assign(b, b + mm);
  apc_problem_free(gp);

  SolverConfig c;
  c.mu = 1e-3;
  c.eps_lsqr = 1e-10;
  c.block = 8;
  c.seed = 3;
  c.max_rank = 40;
  c.trace_sample_stride = 0;
  SolveResult r = aplicur_solve(p, c);
  SolveResult q = plain_lsqr_solve(p, c);
  std::vector<double> y(static_cast<size_t>(mm));
  p.a.matvec(r.x, y);
  std::printf("{\"rank\": %zu, \"rows\": [", r.row_indices.size());
  for (size_t k = 0; k < r.row_indices.size(); ++k) std::printf("%s%lld", k ? ", " : "", (long long)r.row_indices[k]);
  std::printf("], \"cols\": [");
  for (size_t k = 0; k < r.col_indices.size(); ++k) std::printf("%s%lld", k ? ", " : "", (long long)r.col_indices[k]);
  Index it = 0;
  for (const auto& ph : r.phases) it += ph.lsqr_iters;
  std::printf("], \"iters\": %lld, \"final_relres\": %.17g, \"plain_iters\": %lld, \"status\": %d, \"ax0\": %.17g}\n",
              (long long)it, r.final_relres, (long long)q.phases[0].lsqr_iters, (int)r.status, y[0]);
  // SolveHooks (solver.hpp:114-120): observers see every rebuild and phase end
  int rebuilds = 0, phase_ends = 0, last_phase = 0, hook_ok = 1;
  std::vector<double> last_x;
  SolveHooks hooks;
  hooks.on_rebuild = [&](const CurStateView& cur, const PreconditionerView& pc, int phase) {
    ++rebuilds;
    if (cur.rank != pc.rank || pc.regularized_spectrum.size() != static_cast<size_t>(pc.rank)) hook_ok = 0;
    if (phase != last_phase + 1) hook_ok = 0;
  };
  hooks.on_phase_end = [&](int phase, std::span<const double> x) {
    ++phase_ends;
    last_phase = phase;
    last_x.assign(x.begin(), x.end());
  };
  SolveResult h = aplicur_solve(p, c, &hooks);
  const bool same = h.x == r.x && last_x == r.x && h.row_indices == r.row_indices;
  const size_t nspec = r.phases.back().precond_spectrum.size();
  std::printf("{\"hook_rebuilds\": %d, \"hook_phase_ends\": %d, \"phases\": %zu, \"hook_ok\": %d, \"same\": %d, "
              "\"spectrum\": %zu, \"last_rank\": %lld}\n",
              rebuilds, phase_ends, r.phases.size(), hook_ok, same ? 1 : 0, nspec, (long long)r.phases.back().rank);
  try {  // a throwing hook surfaces after the solve
    SolveHooks bad;
    bad.on_phase_end = [](int, std::span<const double>) { throw std::runtime_error("hook"); };
    aplicur_solve(p, c, &bad);
    return 4;
  } catch (const std::runtime_error& e) {
    if (std::string(e.what()) != "hook") return 5;
  }
  try {  // error mapping: shape errors arrive as aplicur::Error
    std::vector<double> bad(3);
    p.a.matvec(bad, y);
  } catch (const Error& e) {
    if (e.kind() != ErrorKind::dimension_mismatch) return 3;
  }
  return 0;
}
