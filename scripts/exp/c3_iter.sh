for v in default vol default vol; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  APC_LIB_PATH=$L timeout 300 python scripts/prof_cfg.py 3 300 1 2>&1 | tail -1 | sed "s/^/$v C3 /"
done
for v in default vol; do
  if [ $v = default ]; then L=""; else L="$PWD/_variants/libapc_$v.so"; fi
  APC_LIB_PATH=$L timeout 300 python scripts/prof_cfg.py 4 100 1 2>&1 | tail -1 | sed "s/^/$v C4 /"
done
