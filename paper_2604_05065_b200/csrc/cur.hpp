// Device-side incremental CUR (the single-sketch IterativeCUR state,
// /root/reference/proj/include/aplicur/cur.hpp:200-371).
//
// Everything that decides indices runs in exact-order kernels (per-element
// summation chains in the reference's order, no FMA): the sketch Y = S A,
// E^row = Y - Y(:,J) U R, E^col = A(:,J+) - C U R(:,J+), the LUPP pivot order
// and the rho probes.  Only the l x l intersection factor (CoreFactor) and the
// small U R(:,J+) solve run on the host with the restated reference routines
// (host_dense.hpp), so I, J and rho_history are bit-identical to the reference.
#pragma once

#include <future>
#include <vector>

#include "apc_internal.hpp"
#include "host_dense.hpp"
#include "host_rng.hpp"

namespace apc {

struct LuppOut {
  std::vector<i64> order;
  std::vector<double> mags;
};

// Pivot order of partial-pivoting elimination on a column-major rows x cols
// device matrix (destroyed), lu_partial_pivot semantics (dense_factor.hpp:119-157).
LuppOut device_lupp(apc_ctx* ctx, double* w, i64 rows, i64 cols, i64 max_pivots);
// The same order over a row-sharded matrix: this rank holds rows
// [row0, row0 + rows) of rows_global; collective over the ctx ranks.
LuppOut device_lupp_dist(apc_ctx* ctx, double* w, i64 rows, i64 row0, i64 rows_global, i64 cols, i64 max_pivots);

struct AugmentResult {
  i64 added = 0;
  bool exhausted = false;
};

class DeviceCur {
 public:
  // target = A (aug_mu == 0: the svd variant, or svd-free with mu == 0), or the
  // stacked [A; aug_mu I] (svd-free with mu > 0, CurTarget(aug), cur.hpp:21-47)
  //
  // distributed: the sharded setup.  `a` is this rank's row
  // block and every rank of the ctx constructs the state (collective calls):
  // Y = sum_p S_p A_p as one running sum carried from rank to rank in row
  // order, E^col on the local rows, the row LUPP over the shards with one
  // candidate allgather per pivot, R = A(I, :) broadcast by the owners of the
  // new rows.  Every rank then holds the same Y, E^row, R, factor, I, J and rho
  // (bit-identical to one rank's); no rank needs the whole matrix.
  DeviceCur(apc_mat& a, i64 block, std::uint64_t seed, i64 xi, i64 probes, int core_kind,
            int sketch_kind, i64 max_rank, double aug_mu = 0.0, bool distributed = false);
  bool distributed() const { return dist_; }
  i64 target_rows() const { return mt_; }
  double embedding_ms() const { return embed_ms_; }
  double sketch_ms() const { return sketch_ms_; }
  bool augmented() const { return amu_ > 0.0; }
  ~DeviceCur();

  i64 rank() const { return static_cast<i64>(I_.size()); }
  const std::vector<i64>& rows() const { return I_; }
  const std::vector<i64>& cols() const { return J_; }
  double rho() const { return rho_; }
  const std::vector<double>& rho_history() const { return rho_hist_; }
  i64 last_added() const { return last_added_; }
  i64 sketch_rows() const { return s_; }
  i64 n() const { return n_; }
  // host copies of the factor and of A(I, J) (the svd-free preconditioner
  // builders use them), downloaded on first use after each refresh
  const CoreFactorH& core() const;
  const Vec& intersection() const;  // l x l column-major
  // U B for the ncols columns of a host row-major l x ncols block, on the
  // device (the svd form's U T_R^T, preconditioner.hpp:158-192); row-major out
  Vec core_solve_rm(const Vec& rhs_rm, i64 ncols) const;
  std::uint64_t sketch_applications() const { return 1; }

  AugmentResult augment();   // cur.hpp:248-294
  void refresh();            // cur.hpp:298-315 (throws Status(APC_SINGULAR) on a singular core)
  void rollback_last_augment();

  // host copies used by the preconditioner builders
  Vec r_dense_rows(i64 first, i64 count) const;  // rows I[first..first+count) of A, row-major count x n
  Vec c_dense() const;                           // dense target_rows x l, column-major (dense A only)
  Vec c_gram() const;                            // C^T C (l x l), computed on the device
  const double* r_rows_dev(i64 first) const { return Rrm_.p + first * n_; }  // row-major rows of R
  // sparse C / R on the host (CSC of C = A(:,J), CSC of R^T = A(I,:)^T)
  void c_csc(std::vector<i64>& ptr, std::vector<i64>& idx, Vec& val) const;
  void rt_csc(std::vector<i64>& ptr, std::vector<i64>& idx, Vec& val) const;

  // device views for tests / builders
  const double* y_dev() const { return Y_.p; }
  const double* eres_dev() const { return E_.p; }
  const double* r_rowmajor_dev() const { return Rrm_.p; }

 private:
  void compute_rho();
  std::vector<double> draw_probes();  // the next probes_ x n Gaussians of probe_rng_
  void upload_core();

  apc_mat& a_;
  apc_ctx* ctx_;
  i64 m_, n_, s_, block_size_, probes_, max_rank_;
  i64 mt_ = 0;       // target rows: m, or m + n for the augmented stack
  double amu_ = 0.0; // mu of the augmented target (0: plain A)
  double embed_ms_ = 0.0, sketch_ms_ = 0.0;
  int core_kind_;
  double ztol_ = -1.0;
  std::future<double> ztol_future_;  // the host's exact sequential ||Y||_F^2 (joined on first use)
  cudaEvent_t ev_sketch_ = nullptr;
  double ztol() {
    if (ztol_ < 0.0) ztol_ = ztol_future_.get();
    return ztol_;
  }
  double rho_;
  i64 last_added_ = 0;
  std::vector<i64> I_, J_;
  std::vector<double> rho_hist_;
  HostRng probe_rng_;
  // the probe set of the next compute_rho, drawn on a host thread while the
  // device works (the stream is consumed strictly in order, one set at a time)
  std::future<std::vector<double>> next_probes_;
  void build_core_device(i64 l);  // CoreFactor::build on the device (exact order)
  void launch_core_solve(const double* rhs_rm, double* out_rm, i64 ncols) const;
  mutable CoreFactorH core_;
  mutable Vec block_;
  mutable bool host_core_stale_ = false;
  i64 core_l_ = 0;
  DBuf<double> block_d_;      // A(I, J) l x l col-major
  DBuf<double> Y_, E_;        // s x n column-major
  DBuf<double> Rrm_;          // R = A(I,:) row-major, capacity max_rank x n
  DBuf<double> H_;            // U R row-major l x n
  DBuf<double> core_a_, core_h_;  // factor payload (l x l)
  DBuf<double> core_at_;          // the factor transposed (row-major), for the warp-per-column solve
  Vec core_at_host_;              // its host staging copy (alive until the async upload completes)
  DBuf<long long> core_perm_;
  DBuf<double> work_;         // generic scratch
  DBuf<int> rowsel_, colsel_;  // flags (rows in I, cols in J); rows: local rows when distributed
  // sharded setup
  bool dist_ = false;
  i64 row0_ = 0, mloc_ = 0;     // this rank's rows [row0_, row0_ + mloc_)
  std::vector<i64> bounds_;     // every rank's first row, then m
  i64 rvalid_ = 0;              // rows of Rrm_ already gathered (I[0..rvalid_))
  i64 rowsel_len() const { return dist_ ? mloc_ : mt_; }
  void set_row_flags(const std::vector<i64>& rows, int value);
  void gather_r_rows_dist(i64 first);
};

}  // namespace apc
