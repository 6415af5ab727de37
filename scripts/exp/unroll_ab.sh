# n-space gather loops unrolled (default build) vs the plain loops (-DAPC_NO_GATHER_UNROLL):
# C5 rank-500 phase us/iteration, and the fused/unfused n-space bit-identity check
TAG=unroll timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -2
APC_LIB_PATH=_variants/libapc_nounroll.so TAG=plain timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -2
