for v in nx4b10 nx6b10 nx7b7 nx3b10 nx7b5; do
  echo "== $v" >> gpurun_out/dp_variants.log
  APC_LIB_PATH=$PWD/_variants/libapc_$v.so timeout 200 python scripts/pair_bench.py c3 >> gpurun_out/dp_variants.log 2>&1
done
for v in nx4b10 nx7b7 nx3b10; do
  echo "== $v" >> gpurun_out/dp_variants.log
  APC_LIB_PATH=$PWD/_variants/libapc_$v.so timeout 300 python scripts/pair_bench.py c4 >> gpurun_out/dp_variants.log 2>&1
done
