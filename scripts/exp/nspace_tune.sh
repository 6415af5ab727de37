for v in 0 1; do APC_NSPACE=$v timeout 300 python scripts/exp/nspace_plain.py > gpurun_out/nsp$v.txt 2>&1; done
for c in 1 2 3 4; do APC_NSPACE_CTAS_PER_SM=$c TAG=cps$c timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1; done
APC_NSPACE=0 TAG=old timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lsqr_nspace_kernel -s 20 -c 1 -o gpurun_out/nspace python scripts/prof_c5.py 40 > gpurun_out/nspace_ncu.log 2>&1
