# dense sparse-sign sketch variants (C3 block 100, C4 block 250): device sketch ms
for v in old c4 c4r512 c8r512 c4r1024 default; do
  if [ $v = default ]; then L=""; else L="APC_LIB_PATH=_variants/libapc_$v.so"; fi
  echo "== $v C3 $(env $L timeout 300 python scripts/sketch_time.py 3 100 2>&1 | tail -1)"
  echo "== $v C4 $(env $L timeout 600 python scripts/sketch_time.py 4 250 2>&1 | tail -1)"
done
