for sb in 1 2 4 8; do for ec in 16384 65536; do APC_TAIL_SB=$sb APC_TAIL_ECAP=$ec timeout 120 python scripts/exp/adj_parts.py 2>&1 | tail -1 | sed "s/^/sb=$sb ec=$ec /"; done; done
