for v in 0 1; do APC_NSPACE=$v timeout 300 python scripts/exp/nspace_check.py 5 300 gpurun_out/ns$v.npz 2>&1 | tail -1; done
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/ns0.npz"), np.load("gpurun_out/ns1.npz")
for k in ("x", "phibar", "xp", "phibar_p"):
    print(k, "bit-identical" if np.array_equal(a[k], b[k]) else f"max rel diff {np.max(np.abs(a[k]-b[k])/np.maximum(np.abs(a[k]),1e-300)):.3e}")
PY
for c in 2 4; do APC_NSPACE=1 APC_NSPACE_CTAS_PER_SM=$c TAG=ns1cps$c timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1; done
APC_NSPACE=0 TAG=ns0 timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1
