# head block rows (wave fit) and tail group cap sweep on C5
for hr in auto 8192 6757; do for ec in 16384 16900 12800; do
  if [ $hr = auto ]; then H=""; else H=$hr; fi
  APC_SETUP_PROF=1 APC_HEAD_BLOCK_ROWS=$H APC_TAIL_ECAP=$ec timeout 120 python scripts/exp/adj_parts.py 2>&1 | grep -E "head adjoint|mask" | sed "s/^/hr=$hr ec=$ec /"
done; done
