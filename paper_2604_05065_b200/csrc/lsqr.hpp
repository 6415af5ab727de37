// Host interface of the device LSQR phase (lsqr.cu) and the device-resident
// right preconditioner.  Mirrors lsqr_solve / StopConfig / LsqrTraceRow
// (/root/reference/proj/include/aplicur/lsqr.hpp:17-207) and the
// Preconditioner apply contract (preconditioner.hpp:19-28).
#pragma once

#include <vector>

#include "apc_internal.hpp"

namespace apc {

struct TraceRowH {  // LsqrTraceRow (lsqr.hpp:38-47); layout == dev TraceRow
  double phibar, cvgrate, cvgdiff, wall_ms;
  long long iter;
  unsigned long long matvecs;
};

// Device form of a right preconditioner P^{-1} = I + B K B^T (explicit basis,
// B dense n x l) or I + R^T G R (implicit basis, R sparse l x n).  Both the
// SVD form (preconditioner.hpp:37-136; K = diag(sigma_hat/sigma_reg - 1),
// symmetric) and the SVD-free form (preconditioner.hpp:250-349; K = sigma_hat
// M^{-1} - I, transpose uses M^{-T}) reduce to this shape once the l x l
// middle operators are formed per rebuild.
struct PrecondDev {
  int kind = 0;  // 0 identity, 1 explicit, 2 implicit
  i64 n = 0, l = 0;
  DBuf<double> B;       // explicit basis, n x l column-major
  DBuf<double> Kf, Ka;  // l x l middle operators (P^{-1} / P^{-T}), stored row-major
  Csr R, RT;            // implicit basis rows (l x n) and their transpose (n x l)
  double sigma_hat = 1.0;
  double sigma_floor = 0.0;  // cvgdiff floor of the dynamic stop (solver.hpp:216-219)
};

struct StopCfg {  // StopConfig (lsqr.hpp:54-59)
  double eps_lsqr = 1e-10;
  double nu_lsqr = 0.0;  // <= 0 or inf: disabled
  double sigma_floor = 0.0;
  i64 max_iters = 0;
};

// True-residual sampling of the solver's observer (solver.hpp:222-236 and
// :418-427): at iterations j >= 1 with j % stride == 0 the phase records
// ||A_mu (x_base + P^{-1} y_j) - [b; 0]|| / bnorm (x_base null: y_j itself).
struct SampleCfg {
  i64 stride = 0;                  // 0: off
  const double* x_base = nullptr;  // device, n (the solver's x before this phase)
  const double* b_local = nullptr; // device, local rows of b
  double bnorm = 0.0;
};

struct PhaseOut {
  std::vector<double> sampled;  // per iteration (NaN where not sampled); empty when sampling is off
  i64 iters = 0;
  int reason = 0;
  bool breakdown = false;
  std::vector<TraceRowH> rows;
  double ms = 0.0;         // host wall time of the phase (init + loop + readback)
  double device_ms = 0.0;  // CUDA-event time of the iteration loop on the library stream
};

struct LsqrWork;  // device workspace, opaque
LsqrWork* lsqr_work_create(apc_mat& a, double mu);
void lsqr_work_destroy(LsqrWork* w);

// One LSQR call from y = 0 on the right-preconditioned system A_mu P^{-1}
// (operators.hpp:75-90) for rhs (device, local rows [+ n tail rows when
// mu > 0]); y_d (device, n) receives the solution.  Throws Status on breakdown.
// Sampling (samp non-null with stride > 0) runs the graph path: the sample's
// preconditioner apply and forward product are no-ops on other iterations.
void lsqr_phase(LsqrWork* w, apc_mat& a, double mu, const PrecondDev* p, const double* rhs_d,
                const StopCfg& stop, int phase, double* y_d, PhaseOut& out,
                const SampleCfg* samp = nullptr);

// out = P^{-1} x (transpose: P^{-T} x); device pointers, ctx stream.
void precond_apply(apc_ctx* ctx, PrecondDev& p, bool transpose, const double* x, double* out);

// allreduce(sum) of a device fp64 buffer over the ctx communicator (no-op at 1 rank)
void comm_allreduce(apc_ctx* ctx, double* buf, i64 count);
// broadcast(fp64) of a device buffer from `root` (the root-only setup of the
// row-sharded solve); no-op at 1 rank
void comm_bcast(apc_ctx* ctx, double* buf, i64 count, int root);
// allgather(fp64): recv (nranks x count, rank-major) = every rank's send;
// bit-exact on both backends (the sharded CUR's pivot candidates)
void comm_allgather(apc_ctx* ctx, const double* send, i64 count, double* recv);
// false when the collective cannot be captured in a CUDA graph (host-staged)
bool comm_graph_safe(const apc_ctx* ctx);
void comm_init(apc_ctx* ctx, const void* uid);
void comm_destroy(apc_ctx* ctx);

}  // namespace apc
