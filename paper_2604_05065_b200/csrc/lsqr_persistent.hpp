// Persistent cooperative LSQR phase (lsqr_persistent.cu).
#pragma once

#include "dev_common.cuh"
#include "lsqr.hpp"

namespace apc {

struct PersistentBuffers {
  double *u, *v, *vr, *w, *y, *z, *h, *s, *t, *part;  // vr: raw v (n)
  LsqrState* st;
  TraceRow* trace;
  int blocks_per_sm;
  unsigned long long* prof;  // optional: 64 x 8 stage timestamps (7 used)
};

// sparse A, one rank, no split transpose rows, identity or implicit basis
bool persistent_eligible(const apc_mat& a, const PrecondDev* p, const apc_ctx* ctx);
// runs every remaining iteration of an initialised phase (state in b.st)
void lsqr_persistent_run(apc_mat& a, double mu, const PrecondDev* p, const PersistentBuffers& b);
int persistent_max_grid(apc_ctx* ctx);
int csr_group_size(double avg_row_nnz);
inline int csr_group_size_p(double avg) { return csr_group_size(avg); }

}  // namespace apc
