# one-launch head+tail adjoint vs two launches (C5)
timeout 200 python scripts/exp/adj_check.py 5 2>&1 | tail -2
for d in 1 0; do for ec in 16384 16900; do
  APC_SEG_DUAL=$d APC_TAIL_ECAP=$ec timeout 120 python scripts/exp/adj_parts.py 2>&1 | grep mask | sed "s/^/dual=$d ec=$ec /"
done; done
