"""Wall time of the device LUPP (cooperative kernel) through the C-ABI, C1-like shapes."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2604_05065_b200 as apc  # noqa: E402

ctx = apc.Context(0)
for rows, cols in ((4000, 20), (4000, 100), (100000, 100), (8000000, 250)):
    W = np.random.default_rng(0).standard_normal((rows, cols))
    apc.lu_partial_pivot(ctx, W, cols)
    t0 = time.perf_counter()
    reps = 20 if rows < 1e6 else 2
    for _ in range(reps):
        apc.lu_partial_pivot(ctx, W, cols)
    print(f"lupp {rows}x{cols}: {1e3 * (time.perf_counter() - t0) / reps:.2f} ms per call (incl. upload)", flush=True)
