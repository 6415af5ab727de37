# iterations per pass of the conditional WHILE body (C5 rank-500 phase us/iteration)
for u in 1 2 4; do APC_WHILE_UNROLL=$u TAG=unroll$u timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -1; done
APC_NSPACE=1 APC_NSPACE_NOOP=1 APC_WHILE_UNROLL=4 TAG=noop4 timeout 300 python scripts/exp/c5_iter.py 2000 2>&1 | tail -1
