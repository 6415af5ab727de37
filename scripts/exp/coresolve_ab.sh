for v in 0 1; do
  if [ $v = 1 ]; then export APC_CORE_SOLVE_WARP=1; fi
  APC_SETUP_PROF=1 timeout 300 python scripts/prof_cfg.py 5 5 2 2>&1 | tail -2 | sed "s/^/warp=$v /"
  APC_SETUP_PROF=1 timeout 300 python scripts/prof_cfg.py 3 5 2 2>&1 | tail -2 | sed "s/^/warp=$v /"
done
