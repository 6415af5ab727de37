timeout 300 python scripts/prof_cfg.py 3 300 1 2>&1 | tail -1 | sed "s/^/C3 /"
timeout 300 python scripts/prof_cfg.py 4 100 1 2>&1 | tail -1 | sed "s/^/C4 /"
timeout 300 python scripts/prof_cfg.py 1 0 2 2>&1 | tail -1 | sed "s/^/C1 /"
timeout 300 python scripts/opbench.py 3 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_solver.py tests/test_gpu_lsqr.py tests/test_gpu_baseline.py tests/test_gpu_baseline_capped.py -m gpu -q -x 2>&1 | tail -2
