for v in default pf2; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  APC_LIB_PATH=$L timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1 | sed "s/^/$v /"
done
