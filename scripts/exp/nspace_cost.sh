# where the C5 iteration's non-pair time goes: unfused n-space (default), the
# fused cooperative n-space kernel, the fused kernel as a no-op (pair + launch
# only), and the operator pair alone
TAG=default timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -1
APC_NSPACE=1 TAG=nspace timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -1
APC_NSPACE=1 APC_NSPACE_NOOP=1 TAG=noop timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -1
timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1
