for hm in 1 1.5 2 3; do
  APC_SETUP_PROF=1 APC_HEAD_MIN=$hm timeout 200 python scripts/exp/adj_parts.py 2>&1 | grep -E "head adjoint|mask" | sed "s/^/hm=$hm /"
done
