for v in 1 0; do APC_U_PREFETCH=$v timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1 | sed "s/^/upref=$v /"; done
