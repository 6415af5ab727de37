for v in 1 0; do APC_EXPAND_TOUCHED=$v TAG=touched$v timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_baseline_capped.py tests/test_gpu_hot.py tests/test_gpu_sampling.py tests/test_gpu_multirank.py -m gpu -q -x 2>&1 | tail -3
