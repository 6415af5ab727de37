# kernel durations of the C5 LSQR iteration (eager launches, ncu launch list, warm L2):
# unfused n-space, fused cooperative n-space, fused as a no-op
K='regex:lsqr_|pc_|hot_sell|seg_adj|tail_scatter|head_combine'
for v in unfused fused noop; do
  case $v in unfused) E="";; fused) E="APC_NSPACE=1";; noop) E="APC_NSPACE=1 APC_NSPACE_NOOP=1";; esac
  env $E APC_LSQR_MODE=eager timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" \
    --launch-skip 200 --launch-count 300 --csv --log-file gpurun_out/nsncu_$v.csv python scripts/prof_c5.py 60 > /dev/null 2>&1
  echo "== $v"; python scripts/launch_summary.py gpurun_out/nsncu_$v.csv 20
done
