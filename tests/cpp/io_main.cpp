// Host-only use of the drop-in header's formats (no GPU): Matrix Market
// round trip, trace CSV and solve report JSON written through the library.
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "aplicur_b200.hpp"

using namespace aplicur;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string dir = argv[1];
  Matrix a = Matrix::sparse(4, 3, {{2, 1, 7.0}, {0, 0, -2.0}, {1, 0, 0.1}, {0, 2, 1e-300}, {3, 2, 0.0}});
  write_matrix_market(a, dir + "/a.mtx");
  Matrix b = read_matrix_market(dir + "/a.mtx");
  if (b.rows() != 4 || b.cols() != 3 || b.nnz() != 4) return 3;
  for (Index k = 0; k < b.nnz(); ++k)
    if (b.values()[k] != a.values()[k] || b.row_idx()[k] != a.row_idx()[k]) return 4;
  Matrix d = Matrix::dense(2, 2, {1.0, 2.0, 3.0, 4.5});
  write_matrix_market(d, dir + "/d.mtx");
  if (read_matrix_market(dir + "/d.mtx").dense_data()[3] != 4.5) return 5;
  try {
    read_matrix_market(dir + "/missing.mtx");
    return 6;
  } catch (const Error& e) {
    if (e.kind() != ErrorKind::io) return 7;
  }
  LsqrTrace tr;
  tr.rows.push_back({1, 0, 1.0, 0.0, 0.0, 1, 0.0, std::numeric_limits<double>::quiet_NaN()});
  tr.rows.push_back({1, 1, 0.5, 0.69, 0.5, 3, 0.25, std::numeric_limits<double>::quiet_NaN()});
  tr.reason = StopReason::iteration_cap;
  trace_to_csv(tr, dir + "/t.csv");
  SolveResult r;
  r.status = SolveStatus::rank_exhausted;
  r.row_indices = {3, 1};
  r.col_indices = {0, 2};
  r.rho_history = {2.5};
  PhaseReport ph;
  ph.phase = 1;
  ph.reason = StopReason::iteration_cap;
  r.phases.push_back(ph);
  SolverConfig c;
  write_solve_report(c, r, "t.csv", dir + "/r.json");
  std::ifstream f(dir + "/t.csv");
  std::stringstream ss;
  ss << f.rdbuf();
  std::printf("%s", ss.str().c_str());
  return 0;
}
