# A/B of adjoint kernel variants on C5: correctness (componentwise bound, rerun
# bit-identity) and the live adjoint / pair time per variant
for v in default tminb1 nopf2; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  echo "== $v"
  APC_LIB_PATH=$L timeout 200 python scripts/exp/adj_check.py 5 2>&1 | tail -2
  APC_LIB_PATH=$L timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1
done
