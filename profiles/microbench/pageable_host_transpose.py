import os, sys, time, subprocess
sys.path.insert(0, ".")
import numpy as np
import paper_2005_10427_b200 as qb
rng = np.random.default_rng(1)
n = 30_000_000
dims = [12092, 9184, 28818]
c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
c = c[np.lexsort(c.T[::-1])]
v = rng.random(n)
ws = qb.Workspace(0)
for tgt in ([1, 0, 2], [2, 1, 0]):
    ts = []
    for _ in range(4):
        t = qb.CooTensor(dims, c.ravel().copy(), v.copy())
        t0 = time.perf_counter(); qb.transpose_inplace(t, tgt, ws=ws); ts.append(time.perf_counter() - t0)
    print(os.environ.get("QD_NO_STAGE", "stage"), tgt, "min ms", round(min(ts) * 1e3, 1), "Mnnz/s", round(n / min(ts) / 1e6, 1))
