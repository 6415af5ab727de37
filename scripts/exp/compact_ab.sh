timeout 200 python scripts/exp/adj_check.py 5 2>&1 | tail -2
for c in 1 0; do APC_TAIL_COMPACT=$c timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1 | sed "s/^/compact=$c /"; done
