timeout 200 python scripts/exp/adj_check.py 5 2>&1 | tail -2
for v in default ring6 noring; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  APC_LIB_PATH=$L timeout 200 python scripts/exp/adj_parts.py 2>&1 | tail -1 | sed "s/^/$v /"
done
