// aplicur_solve on the device: the adaptive outer loop of
// /root/reference/proj/include/aplicur/solver.hpp:162-392 (Alg. 5.3) driving
// the device CUR state (cur.cu), the per-rebuild preconditioner construction
// (precond.cpp) and device-resident warm-started LSQR phases (lsqr.cu).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <utility>
#include <vector>

#include "cur.hpp"
#include "precond.hpp"
#include "solver.hpp"
#include "vec.hpp"

namespace apc {

double host_norm(const double* v, i64 n);

namespace {

using clock_t_ = std::chrono::steady_clock;
double ms_since(clock_t_::time_point t0) {
  return std::chrono::duration<double, std::milli>(clock_t_::now() - t0).count();
}

// reprecondition_check (solver.hpp:68-72)
bool reprecondition_check(double d_cur, double rho, double eps_cur, double nu_prec) {
  if (rho <= eps_cur) return true;
  if (std::isinf(d_cur)) return true;
  return d_cur / (rho - eps_cur) >= nu_prec;
}

bool is_solver_error(const Status& s) { return s.code >= 1 && s.code <= 9; }

// ---- broadcasts of the root-only setup (comm_bcast: fp64; integers are
// carried as doubles, exact below 2^53)
void bcast_host(apc_ctx* ctx, Vec& v) {
  if (v.empty()) return;
  const i64 cnt = static_cast<i64>(v.size());
  DBuf<double> d(cnt);
  APC_CUDA(cudaMemcpyAsync(d.p, v.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice, ctx->stream));
  comm_bcast(ctx, d.p, cnt, 0);
  copy_sync(ctx->stream, v.data(), d.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost);
}

void bcast_scalar(apc_ctx* ctx, double& x) {
  Vec v{x};
  bcast_host(ctx, v);
  x = v[0];
}

void bcast_dbuf(apc_ctx* ctx, DBuf<double>& d, i64 cnt) {
  if (ctx->rank != 0) d.alloc(std::max<i64>(1, cnt));
  if (cnt > 0) comm_bcast(ctx, d.p, cnt, 0);
}

void bcast_ibuf(apc_ctx* ctx, DBuf<i32>& d, i64 cnt) {
  std::vector<i32> h(static_cast<size_t>(std::max<i64>(cnt, 0)));
  if (ctx->rank == 0 && cnt > 0) copy_sync(ctx->stream, h.data(), d.p, sizeof(i32) * cnt, cudaMemcpyDeviceToHost);
  Vec v(h.begin(), h.end());
  bcast_host(ctx, v);
  if (ctx->rank != 0) {
    d.alloc(std::max<i64>(1, cnt));
    for (i64 i = 0; i < cnt; ++i) h[i] = static_cast<i32>(v[i]);
    if (cnt > 0) APC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(i32) * cnt, cudaMemcpyHostToDevice, ctx->stream));
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
}

void bcast_csr(apc_ctx* ctx, Csr& c, i64 rows, i64 cols, i64 nnz) {
  c.rows = rows;
  c.cols = cols;
  c.nnz = nnz;
  bcast_ibuf(ctx, c.ptr, rows + 1);
  bcast_ibuf(ctx, c.idx, nnz);
  bcast_dbuf(ctx, c.val, nnz);
}

// one outer step: the decision, the phase report's setup timings and (when a
// phase runs) the device preconditioner and its spectra
void bcast_step(apc_ctx* ctx, int& action, bool& done, bool& final_phase, double& rho, apc_phase_report& rep,
                PrecondDev& P, PrecondInfo& info) {
  Vec h{static_cast<double>(action), done ? 1.0 : 0.0, final_phase ? 1.0 : 0.0, rho, rep.t_augment_ms,
        rep.t_factor_ms, rep.t_precond_ms, static_cast<double>(P.kind), static_cast<double>(P.n),
        static_cast<double>(P.l), static_cast<double>(P.R.nnz), static_cast<double>(P.B.n > 0 && P.kind == 1),
        P.sigma_hat, P.sigma_floor, info.sigma_hat, info.sigma_floor, static_cast<double>(info.sigma_cur.size()),
        static_cast<double>(info.sigma_reg.size())};
  bcast_host(ctx, h);
  action = static_cast<int>(h[0]);
  done = h[1] != 0.0;
  final_phase = h[2] != 0.0;
  rho = h[3];
  rep.t_augment_ms = h[4];
  rep.t_factor_ms = h[5];
  rep.t_precond_ms = h[6];
  if (action != 1) return;
  P.kind = static_cast<int>(h[7]);
  P.n = static_cast<i64>(h[8]);
  P.l = static_cast<i64>(h[9]);
  const i64 nnz = static_cast<i64>(h[10]), n = P.n, l = P.l;
  P.sigma_hat = h[12];
  P.sigma_floor = h[13];
  info.sigma_hat = h[14];
  info.sigma_floor = h[15];
  info.sigma_cur.resize(static_cast<size_t>(h[16]));
  info.sigma_reg.resize(static_cast<size_t>(h[17]));
  bcast_host(ctx, info.sigma_cur);
  bcast_host(ctx, info.sigma_reg);
  if (P.kind == 0) return;
  bcast_dbuf(ctx, P.Kf, l * l);
  bcast_dbuf(ctx, P.Ka, l * l);
  if (P.kind == 1) {
    bcast_dbuf(ctx, P.B, n * l);
  } else {
    bcast_csr(ctx, P.R, l, n, nnz);
    bcast_csr(ctx, P.RT, n, l, nnz);
  }
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
}

// the CUR outcome of the solve (indices, rho history, status)
void bcast_result(apc_ctx* ctx, apc_result& r) {
  Vec h{static_cast<double>(r.status), r.final_rho, static_cast<double>(r.sketch_applications),
        static_cast<double>(r.rows.size()), static_cast<double>(r.cols.size()),
        static_cast<double>(r.rho_history.size())};
  bcast_host(ctx, h);
  r.status = static_cast<int>(h[0]);
  r.final_rho = h[1];
  r.sketch_applications = static_cast<std::uint64_t>(h[2]);
  Vec rows(r.rows.begin(), r.rows.end()), cols(r.cols.begin(), r.cols.end());
  rows.resize(static_cast<size_t>(h[3]));
  cols.resize(static_cast<size_t>(h[4]));
  r.rho_history.resize(static_cast<size_t>(h[5]));
  bcast_host(ctx, rows);
  bcast_host(ctx, cols);
  bcast_host(ctx, r.rho_history);
  r.rows.assign(rows.begin(), rows.end());
  r.cols.assign(cols.begin(), cols.end());
}

}  // namespace

apc_result* aplicur_solve(apc_mat& a, const double* b, const apc_solver_config& cfg_in, const apc_hooks* hooks) {
  return aplicur_solve_sharded(a, a, b, cfg_in, hooks);
}

// `full`: the whole matrix (sketch + CUR selection, replicated on every rank);
// `a`: this rank's block of rows (LSQR operator, residuals; NCCL allreduce
// of the partial A^T u when the ctx has several ranks).
apc_result* aplicur_solve_sharded(apc_mat& full, apc_mat& a, const double* b, const apc_solver_config& cfg_in,
                                  const apc_hooks* hooks) {
  require(full.ctx == a.ctx && full.m == a.m && full.n == a.n, APC_INVALID_ARGUMENT,
          "aplicur_solve: full matrix and shard must describe the same A on the same context");
  require(&full == &a || (full.r0 == 0 && full.mloc() == full.m), APC_INVALID_ARGUMENT,
          "aplicur_solve: `full` must hold the whole matrix");
  auto t_start = clock_t_::now();
  const i64 n = a.n, m = a.m;
  apc_solver_config cfg = resolve_config(cfg_in, n);
  require(cfg.block <= n, APC_INVALID_ARGUMENT, "aplicur_solve: block > cols");
  const double mu = cfg.mu;
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  const double bnorm = host_norm(b, m);
  require(std::isfinite(bnorm), APC_INVALID_ARGUMENT, "aplicur_solve: non-finite right-hand side");
  // CUR target: A for the svd variant; the regularised stack [A; mu I] for the
  // svd-free variant whenever mu > 0 (solver.hpp:183-186)
  const bool target_augmented = cfg.variant == 1 && mu > 0.0;
  // Row-sharded solves (ctx->nranks > 1), two setups:
  //  * root-only (rank 0 passed the whole matrix as `full`): rank 0 runs the
  //    sketch, the CUR selection and every preconditioner build;
  //  * sharded (no rank holds the whole matrix): every rank runs the CUR state
  //    over its row block (DeviceCur distributed: carried sketch, local E^col,
  //    row LUPP over the shards, R rows from their owners), identical on all
  //    ranks; rank 0 builds the preconditioner (the Gram C^T C summed over the
  //    ranks).
  // Either way the other ranks receive each phase's decision and
  // preconditioner by broadcast, and the LSQR phases run on every rank over
  // the row partition.
  const bool multi = ctx->nranks > 1;
  const bool root = !multi || ctx->rank == 0;
  bool dist = false;
  if (multi) {
    double rootfull = (ctx->rank == 0 && &full != &a) ? 1.0 : 0.0;
    bcast_scalar(ctx, rootfull);
    dist = rootfull == 0.0;
  }
  const bool has_cur = root || dist;  // this rank holds a CUR state
  std::unique_ptr<ProfScope> ps_init(new ProfScope("cur_init"));
  std::unique_ptr<DeviceCur> curp;
  if (has_cur)
    curp.reset(new DeviceCur(dist ? a : full, cfg.block, cfg.seed, cfg.sketch_xi, cfg.probe_count, cfg.core,
                             cfg.sketch_kind, cfg.max_rank, target_augmented ? mu : 0.0, dist));
  ps_init.reset();
  i64 max_rank = has_cur ? std::min(curp->target_rows(), n) : n;
  if (cfg.max_rank > 0) max_rank = std::min(max_rank, cfg.max_rank);
  const double density = (m * n == 0) ? 0.0 : static_cast<double>(a.nnz_global) / static_cast<double>(m * n);
  const bool implicit_mode = a.sparse && density < 0.10;

  DevQrAcc qr_acc;
  qr_acc.ctx = ctx;
  Vec t_r_implicit;
  bool t_r_stale = false;
  auto* res = new apc_result();
  std::unique_ptr<apc_result> guard(res);
  res->n = n;
  const i64 mloc = a.mloc();
  const i64 ulen = mloc + (mu > 0.0 ? n : 0);
  DBuf<double> d_x(std::max<i64>(1, n)), d_y(std::max<i64>(1, n)), d_dx(std::max<i64>(1, n));
  DBuf<double> d_b(std::max<i64>(1, mloc)), d_rhs(std::max<i64>(1, ulen));
  APC_CUDA(cudaMemsetAsync(d_x.p, 0, d_x.bytes(), st));
  if (mloc > 0) APC_CUDA(cudaMemcpyAsync(d_b.p, b + a.r0, sizeof(double) * mloc, cudaMemcpyHostToDevice, st));
  VecWork vw(a, mu);
  LsqrWork* work = lsqr_work_create(a, mu);
  std::unique_ptr<LsqrWork, void (*)(LsqrWork*)> work_guard(work, lsqr_work_destroy);

  double d_cur = std::numeric_limits<double>::infinity();
  int phase = 0;
  bool done = false;
  std::uint64_t matvecs = 0;

  auto run_phase = [&](PrecondDev& P, bool final_phase, double rho_at_build, apc_phase_report& rep,
                       const PrecondInfo& info) {
    auto t0 = clock_t_::now();
    std::unique_ptr<ProfScope> ps_res(new ProfScope("residual"));
    residual(a, vw, d_x.p, d_b.p, d_rhs.p);  // rhs = b_aug - A_mu x (solver.hpp:207-210)
    ps_res.reset();
    matvecs += 1;
    StopCfg stop;
    stop.eps_lsqr = cfg.eps_lsqr;
    stop.nu_lsqr = final_phase ? std::numeric_limits<double>::infinity() : cfg.nu_lsqr;
    stop.max_iters = cfg.lsqr_cap > 0 ? cfg.lsqr_cap : 4 * n;
    stop.sigma_floor = info.sigma_floor;
    PhaseOut po;
    SampleCfg samp;  // the observer's true-residual samples (solver.hpp:222-236)
    samp.stride = cfg.trace_sample_stride;
    samp.x_base = d_x.p;
    samp.b_local = d_b.p;
    samp.bnorm = bnorm;
    lsqr_phase(work, a, mu, &P, d_rhs.p, stop, phase, d_y.p, po, &samp);
    matvecs += po.iters > 0 ? 1 + 2 * static_cast<std::uint64_t>(po.iters) : (po.reason == 5 ? 0 : 1);
    precond_apply(ctx, P, false, d_y.p, d_dx.p);  // x += P^{-1} y (solver.hpp:238-240)
    axpy(ctx, d_x.p, d_dx.p, n);
    for (size_t k = 0; k < po.rows.size(); ++k) {
      const auto& row = po.rows[k];
      const double tr = k < po.sampled.size() ? po.sampled[k] : std::numeric_limits<double>::quiet_NaN();
      res->trace.push_back(apc_trace_row{phase, 0, row.iter, row.phibar, row.cvgrate, row.cvgdiff, row.matvecs,
                                         row.wall_ms, tr});
    }
    res->last_reason = po.reason;
    rep.phase = phase;
    rep.mu = mu;
    rep.rho = rho_at_build;
    rep.sigma_hat = info.sigma_hat;
    rep.rank = P.kind == 0 ? 0 : P.l;
    rep.lsqr_iters = po.iters;
    rep.reason = po.reason;
    rep.t_lsqr_ms = ms_since(t0);
    rep.t_lsqr_device_ms = po.device_ms;
    res->lsqr_ms += po.ms;
    rep.relres_at_end = bnorm > 0.0 ? std::sqrt(residual(a, vw, d_x.p, d_b.p, nullptr)) / bnorm : 0.0;
    if (hooks && hooks->on_phase_end) {  // solver.hpp:261
      std::vector<double> xh(static_cast<size_t>(n));
      copy_sync(st, xh.data(), d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost);
      hooks->on_phase_end(hooks->user, phase, xh.data(), n);
    }
  };

  // one outer step's outcome, decided on rank 0 and broadcast
  enum { kSkip = 0, kRun = 1, kStop = 2 };
  for (i64 outer = 0; outer < cfg.outer_cap && !done; ++outer) {
    apc_phase_report rep{};
    bool final_phase = false;
    int action = kSkip;
    double rho = 0.0;
    PrecondDev P;
    PrecondInfo info;
    if (has_cur) {
      DeviceCur& cur = *curp;
      auto t_aug0 = clock_t_::now();
      bool grew = false;
      if (cur.rank() < max_rank) {
        AugmentResult out;
        {
          ProfScope ps("augment");
          out = cur.augment();
        }
        if (out.added > 0) {
          try {
            ProfScope ps("refresh");
            cur.refresh();
            grew = true;
          } catch (const Status& e) {
            if (e.code != APC_SINGULAR) throw;
            cur.rollback_last_augment();
            res->status = 1;
            final_phase = true;
            done = true;
          }
        } else {
          res->status = 1;
          final_phase = true;
          done = true;
        }
      } else {
        if (cur.rho() > cfg.eps_cur) res->status = 1;
        final_phase = true;
        done = true;
      }
      rep.t_augment_ms = ms_since(t_aug0);

      auto t_fac0 = clock_t_::now();
      std::unique_ptr<ProfScope> ps_fac(new ProfScope("factor"));
      if (grew) {
        const i64 l = cur.rank();
        if (!root) {
          // sharded setup, rank > 0: rank 0 alone builds the preconditioner
        } else if (implicit_mode) {
          // T_R with T_R^T T_R = R R^T (the reference maintains it with
          // CholGramAccumulator; the from-scratch gram_factor is the same
          // factor), computed when a preconditioner is next built
          t_r_stale = true;
        } else {
          const i64 added = cur.last_added();
          // rows of R are stored row-major on the device: added x n == column-major n x added
          try {
            qr_acc.append(n, added, cur.r_rows_dev(l - added));
          } catch (const Status& e) {
            if (!is_solver_error(e)) throw;
            qr_acc.clear();
            qr_acc.append(n, l, cur.r_rows_dev(0));  // full refactorisation
          }
        }
        if (cur.rank() >= max_rank) {
          final_phase = true;
          done = true;
          if (cur.rho() > cfg.eps_cur) res->status = 1;
        }
      }
      ps_fac.reset();
      rep.t_factor_ms = ms_since(t_fac0);

      rho = cur.rho();
      if (rho <= cfg.eps_cur) {
        final_phase = true;
        done = true;
        res->status = 0;
      }
      const bool trigger = final_phase || reprecondition_check(d_cur, rho, cfg.eps_cur, cfg.nu_prec);
      if (trigger && cur.rank() > 0) {
        if (!res->phases.empty() && res->phases.back().rank == cur.rank()) {
          action = kStop;  // duplicate rank
        } else if (!root) {
          (void)cur.c_gram();  // rank 0's Gram is a sum over every rank's rows (collective)
          action = kRun;
        } else {
          if (implicit_mode && t_r_stale) {
            ProfScope ps("factor");
            auto t_f0 = clock_t_::now();
            std::vector<i64> rp, ri;
            Vec rv;
            cur.rt_csc(rp, ri, rv);
            t_r_implicit = gram_factor_rows_dev(ctx, n, cur.rank(), cur.r_rowmajor_dev(), rp, ri, rv);
            t_r_stale = false;
            rep.t_factor_ms += ms_since(t_f0);
          }
          auto t_pre0 = clock_t_::now();
          try {
            BuildInputs in;
            in.ctx = ctx;
            in.variant = cfg.variant;
            in.implicit = implicit_mode;
            in.m = cur.target_rows();
            in.n = n;
            in.l = cur.rank();
            in.mu = mu;
            in.target_level = rho;
            in.core_solve_rm = [&cur](const Vec& bb, i64 nc) { return cur.core_solve_rm(bb, nc); };  // U T_R^T
            if (cfg.variant == 1) in.block = &cur.intersection();  // svd-free: A(I, J)
            in.t_r = implicit_mode ? &t_r_implicit : &qr_acc.t;
            in.q_dev = qr_acc.q.p;
            in.gram = cur.c_gram();  // collective in the sharded setup
            in.c_dense = [&cur, &full]() -> Vec {  // only for the QR fallback of gram_factor
              if (!full.sparse) return cur.c_dense();
              std::vector<i64> cp, ci;
              Vec cv;
              cur.c_csc(cp, ci, cv);
              const i64 mt = cur.target_rows(), l = cur.rank();
              Vec dd(static_cast<size_t>(mt * l), 0.0);
              for (i64 j = 0; j < l; ++j)
                for (i64 q = cp[j]; q < cp[j + 1]; ++q) dd[j * mt + ci[q]] = cv[q];
              return dd;
            };
            ProfScope ps("precond");
            if (implicit_mode) cur.rt_csc(in.r_ptr, in.r_idx, in.r_val);
            build_precond(in, P, info);
            action = kRun;
          } catch (const Status& e) {
            if (!is_solver_error(e)) throw;
            res->status = 2;
            action = kStop;
          }
          rep.t_precond_ms = ms_since(t_pre0);
          if (action == kRun && hooks && hooks->on_rebuild) {  // solver.hpp:367
            const bool svd = cfg.variant == 0;
            const i64 ns = svd ? static_cast<i64>(std::min(info.sigma_cur.size(), info.sigma_reg.size())) : 0;
            apc_rebuild_info ri{phase + 1, cfg.variant, cur.rank(), cur.rows().data(), cur.cols().data(), rho,
                                info.sigma_hat, info.sigma_floor, ns ? info.sigma_cur.data() : nullptr,
                                ns ? info.sigma_reg.data() : nullptr, ns};
            hooks->on_rebuild(hooks->user, &ri);
          }
        }
      }
    }
    if (multi) bcast_step(ctx, action, done, final_phase, rho, rep, P, info);
    if (action == kStop) break;
    if (action == kRun) {
      ++phase;
      run_phase(P, final_phase, rho, rep, info);
      if (std::isfinite(rho)) d_cur = rho - cfg.eps_cur;
      res->phases.push_back(rep);
      res->spectra.push_back(cfg.variant == 0 ? info.sigma_reg : Vec{});  // solver.hpp:258-260
    }
  }

  if (res->phases.empty()) {  // identity-preconditioned phase (solver.hpp:376-383)
    ++phase;
    apc_phase_report rep{};
    PrecondDev ident;
    ident.n = n;
    PrecondInfo info;
    double rho0 = root ? curp->rho() : 0.0;
    if (multi) bcast_scalar(ctx, rho0);
    run_phase(ident, true, rho0, rep, info);
    res->phases.push_back(rep);
    res->spectra.emplace_back();
  }

  res->x.resize(static_cast<size_t>(n));
  copy_sync(st, res->x.data(), d_x.p, sizeof(double) * n, cudaMemcpyDeviceToHost);
  if (root) {
    res->final_rho = curp->rho();
    res->sketch_applications = curp->sketch_applications();
    res->rows.assign(curp->rows().begin(), curp->rows().end());
    res->cols.assign(curp->cols().begin(), curp->cols().end());
    res->rho_history = curp->rho_history();
  }
  if (multi) bcast_result(ctx, *res);
  res->final_relres = bnorm > 0.0 ? std::sqrt(residual(a, vw, d_x.p, d_b.p, nullptr)) / bnorm : 0.0;
  res->system_matvecs = matvecs;
  res->total_ms = ms_since(t_start);
  res->setup_ms = res->total_ms - res->lsqr_ms;
  SetupProf::add("lsqr_phases(total)", res->lsqr_ms);
  SetupProf::dump_and_reset("aplicur_solve setup profile");
  guard.release();
  return res;
}

}  // namespace apc
