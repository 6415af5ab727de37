for v in minb6 minb7 minb8; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  APC_LIB_PATH=$L TAG=$v timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1
  APC_LIB_PATH=$L timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1
done
