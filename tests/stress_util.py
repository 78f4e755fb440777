"""Randomised GPU-vs-oracle stress (shared by tests/test_parity_gpu.py).
Run as a subprocess with QD_POISON set so every fresh workspace buffer is
filled with garbage: a kernel that reads scratch it never wrote shows up as
a mismatch instead of passing on zero-filled memory."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, ".."))
sys.path.insert(0, os.path.join(HERE, "..", "oracle"))


def run(seed: int, trials: int) -> int:
    import paper_2005_10427_b200 as qd
    from pyoracle import Oracle
    orc = Oracle()
    ws = qd.Workspace(0)
    strategies = {"quesadilla": qd.SortStrategy.quesadilla(), "radix": qd.SortStrategy.full_radix(),
                  "comparison": qd.SortStrategy.comparison_sort()}
    rng = np.random.default_rng(seed)
    extents = [33_554_467, 3_000_017, 1_000_003, 40_000, 5000, 700, 60, 3, 1, 2, 1 << 20]
    bad = 0
    for trial in range(trials):
        r = int(rng.integers(1, 7))
        dims = [int(rng.choice(extents)) for _ in range(r)]
        n = int(rng.choice([0, 1, 2, 100, 5000, 60_000, 400_000]))
        cols = []
        for d in dims:
            if rng.random() < 0.5:  # few distinct values: long runs, run-level sorts
                k = int(rng.integers(1, 80))
                cols.append(rng.integers(0, d, k)[rng.integers(0, k, n)])
            else:
                cols.append(rng.integers(0, d, n, dtype=np.int64))
        c = np.stack(cols, 1).astype(np.uint32) if n else np.zeros((0, r), np.uint32)
        if n:
            c = c[np.lexsort(c.T[::-1])]
        t = qd.CooTensor(dims, c.ravel(), rng.random(n))
        target = [int(x) for x in rng.permutation(r)]
        name = ["quesadilla", "radix", "topk", "comparison", "quesadilla"][trial % 5]
        k = int(rng.integers(1, r + 1))
        s = qd.SortStrategy.top_k(k) if name == "topk" else strategies[name]
        out = qd.transpose(t, target, s, ws=ws)
        ec, ev, _ = orc.transpose(t.dims, t.coords, t.values, target, name, k)
        if not (np.array_equal(out.coords, ec) and
                np.array_equal(out.values.view(np.uint64), ev.view(np.uint64))):
            bad += 1
            print("MISMATCH", trial, dims, n, target, name, k, flush=True)
    return bad


if __name__ == "__main__":
    sys.exit(1 if run(int(sys.argv[1]), int(sys.argv[2])) else 0)
