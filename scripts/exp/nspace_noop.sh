APC_NSPACE=1 APC_NSPACE_NOOP=1 TAG=noop timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1
APC_NSPACE=1 TAG=ns1 timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1
timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1
