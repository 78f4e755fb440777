"""Synchronous transpose_inplace on PAGEABLE host buffers (the C++ drop-in's
std::vector signature, transpose.hpp:59-61): 30M c2-shaped rows, one target
per call, min of 4 calls.  Every H2D/D2H byte is inside the timed call (the
library stages through its pinned chunk ring with a pooled parallel memcpy).
QD_NO_STAGE=1: the driver's own pageable copies; QD_COPY_THREADS=k: copy
threads."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_2005_10427_b200 as qd  # noqa: E402

rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
dims = [12092, 9184, 28818]
c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
c = c[np.lexsort(c.T[::-1])]
v = rng.random(n)
ws = qd.Workspace(0)
for tgt in ([1, 0, 2], [2, 1, 0]):
    ts = []
    for _ in range(4):
        t = qd.CooTensor(dims, c.ravel().copy(), v.copy())
        t0 = time.perf_counter()
        qd.transpose_inplace(t, tgt, ws=ws)
        ts.append(time.perf_counter() - t0)
    print(os.environ.get("QD_NO_STAGE", "staged"), "threads", os.environ.get("QD_COPY_THREADS", "auto"),
          tgt, "min ms", round(min(ts) * 1e3, 1), "Mnnz/s", round(n / min(ts) / 1e6, 1), flush=True)
