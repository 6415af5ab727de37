for v in 0 1 0 1; do APC_PDL=$v TAG=pdl$v timeout 300 python scripts/exp/c5_iter.py 1000 2>&1 | tail -1; done
for v in 0 1; do APC_PDL=$v timeout 300 python scripts/exp/nspace_check.py 5 200 gpurun_out/pdl$v.npz 2>&1 | tail -1; done
python -c "
import numpy as np
a,b=np.load('gpurun_out/pdl0.npz'),np.load('gpurun_out/pdl1.npz')
print({k: bool(np.array_equal(a[k],b[k])) for k in ('x','phibar','xp','phibar_p')})"
for v in 0 1; do APC_PDL=$v timeout 300 python scripts/prof_cfg.py 3 300 1 2>&1 | tail -1 | sed "s/^/pdl=$v C3 /"; done
