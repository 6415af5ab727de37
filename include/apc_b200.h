/*
 * apc_b200.h -- C-ABI of the B200-native APLICUR hot path (libapc_b200.so).
 *
 * Plain C types only (pointers, sizes, int status codes); no torch or CUDA
 * types cross this boundary.  Every entry point returns 0 (APC_OK) or an
 * APC_* status; codes 1..9 are aplicur::ErrorKind + 1
 * (/root/reference/proj/include/aplicur/error.hpp:10-20) so a C++ shim can
 * rethrow aplicur::Error(kind, msg, index) unchanged.
 *
 * Each entry point cites the reference interface it replaces.  The reference
 * is header-only C++ (no FFI of its own); the "binding" a maintainer adds is
 * include/aplicur_b200.hpp (same namespace/types as the reference) or a ctypes
 * stub -- see INTEGRATION.md.
 */
#ifndef APC_B200_H
#define APC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APC_ABI_VERSION 1

enum apc_status {
  APC_OK = 0,
  APC_INVALID_ARGUMENT = 1,    /* ErrorKind::invalid_argument */
  APC_DIMENSION_MISMATCH = 2,  /* ErrorKind::dimension_mismatch */
  APC_RANK_DEFICIENT = 3,      /* ErrorKind::rank_deficient */
  APC_SINGULAR = 4,            /* ErrorKind::singular */
  APC_NOT_POSITIVE = 5,        /* ErrorKind::not_positive */
  APC_NO_CONVERGENCE = 6,      /* ErrorKind::no_convergence */
  APC_NUMERICAL_BREAKDOWN = 7, /* ErrorKind::numerical_breakdown */
  APC_NOT_APPLICABLE = 8,      /* ErrorKind::not_applicable */
  APC_IO = 9,                  /* ErrorKind::io */
  APC_CUDA_ERROR = 20,         /* CUDA runtime failure */
  APC_NCCL_ERROR = 21,         /* NCCL failure */
  APC_NO_DEVICE = 22           /* no CUDA device: there is no CPU fallback */
};

typedef struct apc_ctx apc_ctx;         /* one per GPU / rank: stream, scratch, comm */
typedef struct apc_mat apc_mat;         /* device-resident A (dense col-major or CSR+CSR^T) */
typedef struct apc_result apc_result;   /* SolveResult (solver.hpp:101-112) */
typedef struct apc_problem apc_problem; /* host-side synthetic problem (BASELINE configs) */

/* ---- library / context --------------------------------------------------- */
int apc_abi_version(void);
/* last error message of the calling thread (for calls without a ctx) */
const char* apc_last_error(int64_t* index);
int apc_device_count(int* count);
/* nccl_unique_id: 128 bytes from apc_nccl_unique_id() on rank 0 (NULL if nranks==1) */
int apc_ctx_create(int device, int nranks, int rank, const void* nccl_unique_id, apc_ctx** out);
/* Host-staged collectives instead of NCCL: every allreduce of the row-sharded
 * solve copies the device buffer to pinned host memory and calls
 * fn(buf, count, user), which must replace buf by the elementwise sum over all
 * ranks, added in rank order (so every rank holds the same bits), and return 0.
 * Lets several ranks share one GPU or use any host transport; the LSQR phase
 * then runs eagerly (one host round trip per iteration). */
typedef int (*apc_host_allreduce_fn)(double* buf, int64_t count, void* user);
int apc_ctx_create_host_comm(int device, int nranks, int rank, apc_host_allreduce_fn fn, void* user,
                             apc_ctx** out);
int apc_ctx_destroy(apc_ctx* ctx);
int apc_nccl_unique_id(void* out128);
void* apc_ctx_stream(apc_ctx* ctx);              /* cudaStream_t all library work runs on */
uint64_t apc_ctx_launches(apc_ctx* ctx);         /* kernels launched by this library so far */
int apc_ctx_sync(apc_ctx* ctx);

/* ---- matrices (replaces aplicur::Matrix storage, matrix.hpp:35-268) ------ */
/* Host buffers are borrowed for the call only.  Rows [r0, r1) are kept on the
 * device (block-row shard); pass r0 = 0, r1 = m for the whole matrix. */
int apc_mat_upload_dense(apc_ctx* ctx, int64_t m, int64_t n, const double* colmajor,
                         int64_t r0, int64_t r1, apc_mat** out);
/* CSC with int64 indices, rows strictly increasing per column (the reference
 * layout, matrix.hpp:66-94).  Device keeps CSR(A) and CSR(A^T) with int32 indices. */
int apc_mat_upload_csc(apc_ctx* ctx, int64_t m, int64_t n, const int64_t* colptr,
                       const int64_t* rowidx, const double* val, int64_t r0, int64_t r1,
                       apc_mat** out);
int apc_mat_free(apc_mat* a);
int apc_mat_info(const apc_mat* a, int64_t* m, int64_t* n, int64_t* nnz, int* sparse,
                 int64_t* r0, int64_t* r1);

/* ---- operator products (Matrix::matvec / matvec_transpose, matrix.hpp:151-195;
 *      AugmentedOperator::matvec / matvec_transpose, matrix.hpp:377-392) ------
 * augmented == 0: y = A x (len m) / y = A^T x (len n).
 * augmented != 0: y = [A x; mu x] (len m+n) / y = A^T x[0:m] + mu x[m:m+n] (len n).
 * *_dev take device pointers and run on the ctx stream (asynchronous);
 * *_host copy host buffers in and out (synchronous).  Sharded matrices use
 * local row blocks (the transpose product is then a partial sum). */
int apc_op_apply_dev(apc_mat* a, double mu, int augmented, int transpose, const double* x_dev,
                     double* y_dev);
int apc_op_apply_host(apc_mat* a, double mu, int augmented, int transpose, const double* x,
                      double* y);
/* The operator pair of one LSQR iteration (lsqr.hpp:139-150 calls matvec and
 * matvec_transpose back to back): y = A x (len local m), g[0:n] = A^T y and
 * g[n] = ||y||^2, device pointers, ctx stream.  A dense A of 64 MB or more
 * goes through the fused kernel that reads A from HBM once (a panel of rows
 * stays in shared memory between the two products); everything else runs the
 * two products one after the other.  *fused (may be NULL) reports which. */
int apc_op_pair_dev(apc_mat* a, const double* x_dev, double* y_dev, double* g_dev, int* fused);

/* The dense kernels of the preconditioner construction, on device pointers
 * (column-major; hand-written DMMA GEMM with a fixed-order split over k, and
 * a blocked TRSM): C = alpha op(A) op(B) + beta C, and B <- B T^{-1} (T upper).
 * They replace the QrAccumulator / basis products of preconditioner.hpp:435-476,
 * 171-193 (the reference's own loops there are plain matmul / tri-solves). */
int apc_dgemm(apc_ctx* ctx, int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
              const double* A_dev, int64_t lda, const double* B_dev, int64_t ldb, double beta, double* C_dev,
              int64_t ldc);
int apc_dtrsm_right_upper(apc_ctx* ctx, int64_t m, int64_t n, const double* T_dev, int64_t ldt, double* B_dev,
                          int64_t ldb);
/* The l x l algebra of every rebuild (dense_small.cu): in-place upper
 * Cholesky of a column-major k x k matrix (chol_upper, dense_factor.hpp:229-244;
 * lower part zeroed), *bad = -1 or the first column with a non-positive pivot
 * (the caller's APC_NOT_POSITIVE); and X <- T^{-1} X or T^{-T} X for a
 * row-major k x ncols X and upper column-major T (tri_solve on every column,
 * dense_factor.hpp:406-424; APC_SINGULAR on a zero diagonal). */
int apc_dpotrf_upper(apc_ctx* ctx, int64_t k, double* A_dev, int64_t* bad);
int apc_dtrsm_rows(apc_ctx* ctx, int64_t k, const double* T_dev, double* X_dev, int64_t ncols, int transpose);

/* ---- row partitioning for multi-GPU -------------------- */
/* bounds[0..nranks]: contiguous row blocks balanced by nnz when row_nnz is
 * given (prefix-sum split), else by row count. Host-only. */
int apc_partition_rows(int64_t m, const int64_t* row_nnz, int nranks, int64_t* bounds);

/* ---- seeded randomness (rng.hpp:12-78), host-side, bit-identical -------- */
/* kind: 0 next_u64 (uint64 out), 1 uniform, 2 gaussian, 3 below(bound) (uint64 out), 4 sign.
 * stream < 0: Rng(seed); else Rng(seed, RngStream(stream), index). */
int apc_rng_fill(uint64_t seed, int stream, uint64_t index, int kind, uint64_t bound,
                 int64_t count, void* out);
uint64_t apc_mix64(uint64_t x);
/* the same stream generated on the device: kind-0 draws (next_u64) of
 * Rng(seed) (stream < 0) or Rng(seed, stream, index), count of them into the
 * host buffer out.  Used by the sketch embedding; exposed for tests. */
int apc_rng_fill_device(apc_ctx* ctx, uint64_t seed, int stream, uint64_t index, int64_t count, uint64_t* out);

/* ---- single-sketch incremental CUR (CurState, cur.hpp:200-371) ----------
 * Exact-order device kernels: Y, E^row, the LUPP pivot order and rho are
 * bit-identical to the reference.  sketch_kind 0 = SparseSignEmbedding
 * (CurState::init, cur.hpp:209-226), 1 = GaussianEmbedding (sketch.hpp:173-197),
 * 2 = GaussianEmbedding applied on the FP64 tensor cores (DMMA, opt-in: Y is not
 * bit-identical, the indices are checked against the exact path in the tests). */
typedef struct apc_cur apc_cur;
int apc_cur_create(apc_mat* a, int64_t block, uint64_t seed, int64_t xi, int64_t probe_count,
                   int core_kind, int sketch_kind, apc_cur** out);
int apc_cur_free(apc_cur* c);
/* CurState::augment: added = 0 and exhausted = 1 when no admissible pivot remains */
int apc_cur_augment(apc_cur* c, int64_t* added, int* exhausted);
/* CurState::refresh: returns APC_SINGULAR on a numerically singular intersection */
int apc_cur_refresh(apc_cur* c);
int apc_cur_rollback_last_augment(apc_cur* c);
int apc_cur_state(const apc_cur* c, int64_t* rank, double* rho, int64_t* sketch_rows, int64_t* n_rho);
int apc_cur_indices(const apc_cur* c, int64_t* rows, int64_t* cols);
int apc_cur_rho_history(const apc_cur* c, double* rho);
/* time of the one-time sketch: host embedding generation (seeded RNG) and the
 * device sketch kernels (CUDA events on the library stream), ms */
int apc_cur_timing(const apc_cur* c, double* embedding_host_ms, double* sketch_device_ms);
/* sketch_matrix() / sketch_residual(): s x n column-major, host copies */
int apc_cur_sketch(const apc_cur* c, double* y);
int apc_cur_residual(const apc_cur* c, double* e);

/* lu_partial_pivot (dense_factor.hpp:119-157) on a host column-major matrix,
 * run on the device; order/mags sized min(rows, cols, max_pivots). */
int apc_lupp(apc_ctx* ctx, const double* w, int64_t rows, int64_t cols, int64_t max_pivots,
             int64_t* order, double* mags, int64_t* steps);

/* ---- synthetic BASELINE inputs (host) ---------------------------------- */
/* config 1..5 = BASELINE.json configs[0..4]; m, n = 0 -> the BASELINE shape;
 * seed = 0 -> 20260415 + config.  Dense problems are column-major; sparse ones
 * are CSC with int64 indices (the reference Matrix layout). */
int apc_problem_generate(int config, int64_t m, int64_t n, uint64_t seed, apc_problem** out);
int apc_problem_info(const apc_problem* p, int64_t* m, int64_t* n, int* sparse, int64_t* nnz);
const double* apc_problem_dense(const apc_problem* p);
int apc_problem_csc(const apc_problem* p, const int64_t** colptr, const int64_t** rowidx,
                    const double** vals);
const double* apc_problem_b(const apc_problem* p);
int apc_problem_free(apc_problem* p);

/* ---- solver (aplicur_solve / plain_lsqr_solve, solver.hpp:162-448) ------ */
/* Mirrors SolverConfig (solver.hpp:29-45) field for field, plus sketch_kind. */
typedef struct apc_solver_config {
  int64_t block;               /* 0: max(1, llround(n / 50)) */
  double eps_cur;              /* < 0: 30 * mu */
  double eps_lsqr;             /* 1e-10 */
  double nu_prec;              /* 10 */
  double nu_lsqr;              /* 100 */
  double mu;                   /* scale of the [A; mu I] block */
  int32_t variant;             /* 0 svd, 1 svd_free */
  int32_t core;                /* 0 qr, 1 lu (CoreFactorKind) */
  int64_t sketch_xi;           /* 8 */
  int64_t probe_count;         /* 10 */
  int64_t lsqr_cap;            /* 0: 4 n per phase */
  int64_t max_rank;            /* 0: min of target dimensions */
  uint64_t seed;               /* 0 */
  int64_t trace_sample_stride; /* 1; true-residual sample every k-th iteration, 0 off (bench: 0) */
  int64_t outer_cap;           /* 100000 */
  int32_t sketch_kind;         /* 0 sparse sign (reference), 1 Gaussian (BASELINE C1/C3/C4),
                                  2 Gaussian on the FP64 tensor cores (DMMA; opt-in, Y not bit-exact) */
  int32_t reserved;
} apc_solver_config;

typedef struct apc_phase_report { /* PhaseReport, solver.hpp:74-88 */
  int32_t phase;
  int32_t reason;  /* StopReason: 0 none 1 gradient-tol 2 dynamic-rate 3 dynamic-diff 4 iteration-cap 5 exact-zero-rhs */
  int64_t rank;
  double rho, sigma_hat, mu;
  int64_t lsqr_iters;
  double t_augment_ms, t_factor_ms, t_precond_ms, t_lsqr_ms;
  double relres_at_end;
  double t_lsqr_device_ms; /* device time of the iteration loop (CUDA events on the library stream) */
} apc_phase_report;

typedef struct apc_trace_row { /* LsqrTraceRow, lsqr.hpp:38-47 */
  int32_t phase;
  int32_t pad;
  int64_t iter;
  double phibar, cvgrate, cvgdiff;
  uint64_t matvecs;
  double wall_ms, true_relres;
} apc_trace_row;

int apc_config_default(apc_solver_config* cfg);
/* b: full right-hand side (length m, host).  plain != 0 runs plain_lsqr_solve. */
int apc_solve(apc_mat* a, const double* b, const apc_solver_config* cfg, int plain,
              apc_result** out);
/* Row-partitioned solve: `shard` holds this rank's rows
 * [r0, r1) on a ctx created with nranks > 1 (contiguous blocks in rank order
 * for the sharded setup).  Two setups:
 *  - rank 0 passes `full`, the whole matrix: the sketch, the CUR selection
 *    and every preconditioner build run there and are broadcast (decision,
 *    preconditioner, indices); the other ranks' `full` is not used;
 *  - `full` NULL on rank 0 (sharded setup): no rank holds the whole matrix.
 *    The sketch is one running sum carried from rank to rank in row order,
 *    E^col stays on the row blocks, the row pivots come from one candidate
 *    allgather per pivot, R's rows are broadcast by their owners; I, J and
 *    rho are bit-identical to one rank's.  Rank 0 builds the preconditioner
 *    (C^T C summed over the ranks) and broadcasts it.  Not for the svd-free
 *    variant with mu > 0 (its [A; mu I] target): APC_NOT_APPLICABLE.
 * `full` may be NULL everywhere for plain != 0.  Every rank passes the full
 * b; per LSQR iteration the ranks exchange one allreduce of n + 1 doubles
 * ([A_p^T u_p | ||u_p||^2]). */
int apc_solve_sharded(apc_mat* full, apc_mat* shard, const double* b, const apc_solver_config* cfg,
                      int plain, apc_result** out);
/* SolveHooks (solver.hpp:114-120): diagnostic observers, called on the host
 * thread of the solve.  on_rebuild runs after each preconditioner build and
 * before its LSQR phase (solver.hpp:367) with a view of the CUR state and the
 * preconditioner (pointers valid during the call only); on_phase_end runs at
 * the end of every phase with x so far (solver.hpp:261), copied to the host. */
typedef struct apc_rebuild_info {
  int32_t phase;
  int32_t variant;          /* 0 svd, 1 svd-free */
  int64_t rank;             /* l = |I| = |J| */
  const int64_t* rows;      /* I */
  const int64_t* cols;      /* J */
  double rho;               /* CUR error estimate the preconditioner was built at */
  double sigma_hat;         /* Preconditioner::target_level() */
  double sigma_floor;       /* smallest_cur_sigma() (svd) / target_level() (svd-free) */
  const double* sigma_cur;  /* svd variant: CUR singular values (n_sigma), else NULL */
  const double* sigma_reg;  /* svd variant: regularized_spectrum() (n_sigma), else NULL */
  int64_t n_sigma;
} apc_rebuild_info;
typedef void (*apc_rebuild_fn)(void* user, const apc_rebuild_info* info);
typedef void (*apc_phase_end_fn)(void* user, int32_t phase, const double* x, int64_t n);
typedef struct apc_hooks {
  void* user;
  apc_rebuild_fn on_rebuild;     /* may be NULL */
  apc_phase_end_fn on_phase_end; /* may be NULL */
} apc_hooks;
/* aplicur_solve(problem, cfg, &hooks) (solver.hpp:162-163).  full: NULL for a
 * single-rank solve, else as in apc_solve_sharded.  hooks may be NULL. */
int apc_solve_hooked(apc_mat* full, apc_mat* a, const double* b, const apc_solver_config* cfg,
                     const apc_hooks* hooks, apc_result** out);
int apc_result_free(apc_result* r);
/* status: SolveStatus 0 converged, 1 rank-exhausted, 2 breakdown */
int apc_result_summary(const apc_result* r, int* status, double* final_rho, double* final_relres,
                       uint64_t* sketch_applications, uint64_t* system_matvecs, int64_t* n_phases,
                       int64_t* n_trace, int64_t* rank, int64_t* n_rho);
int apc_result_x(const apc_result* r, double* x);
int apc_result_indices(const apc_result* r, int64_t* row_indices, int64_t* col_indices);
int apc_result_rho_history(const apc_result* r, double* rho);
int apc_result_phases(const apc_result* r, apc_phase_report* phases);
/* PhaseReport::precond_spectrum of phase k (solver.hpp:87,258-260; svd
 * variant only, else empty): *n receives its length, out (may be NULL) the values */
int apc_result_phase_spectrum(const apc_result* r, int64_t k, double* out, int64_t* n);
int apc_result_trace(const apc_result* r, apc_trace_row* rows);
/* wall-clock split of the last solve: setup (sketch + CUR + builds) and LSQR, ms */
int apc_result_timing(const apc_result* r, double* total_ms, double* lsqr_ms, double* setup_ms);

/* ---- formats around the path (host only, no GPU needed) ----------------- */
/* Matrix Market, matrix_market.hpp:18-46 (write: coordinate for CSC, array for
 * dense column-major; %.17g values, bit-exact on read-back) and :48-116 (read:
 * general real/integer coordinate or array; entries sorted by (col,row),
 * duplicates -> APC_INVALID_ARGUMENT, explicit zeros dropped, malformed ->
 * APC_IO).  The read result is a host apc_problem (b = zeros(m)); use
 * apc_problem_info / _csc / _dense and apc_mat_upload_* as for generated inputs. */
int apc_mm_write_csc(const char* path, int64_t m, int64_t n, const int64_t* colptr, const int64_t* rowidx,
                     const double* vals);
int apc_mm_write_dense(const char* path, int64_t m, int64_t n, const double* a_colmajor);
int apc_mm_read(const char* path, apc_problem** out);
/* trace CSV, report_io.hpp:28-47: "phase,iter,phibar,relres,matvecs,wall_ms,reason",
 * reason on the last row of each phase (that phase's report, else trace_reason);
 * written to path.tmp then renamed (report_io.hpp:112-122) */
int apc_trace_csv_write(const char* path, const apc_trace_row* rows, int64_t n_rows, const apc_phase_report* phases,
                        int64_t n_phases, int32_t trace_reason);
/* solve report JSON, report_io.hpp:49-110 (config, status, residuals, counters,
 * trace path, CUR indices + rho history, phase reports); non-finite -> null */
int apc_report_json_write(const char* path, const apc_solver_config* cfg, int32_t status, double final_relres,
                          double final_rho, uint64_t sketch_applications, uint64_t system_matvecs,
                          const char* trace_path, const int64_t* row_indices, const int64_t* col_indices,
                          int64_t rank, const double* rho_history, int64_t n_rho, const apc_phase_report* phases,
                          int64_t n_phases, const double* const* spectra, const int64_t* n_spectra);
/* spectra / n_spectra: per phase precond_spectrum (both may be NULL: none) */

#ifdef __cplusplus
}
#endif

#endif /* APC_B200_H */
