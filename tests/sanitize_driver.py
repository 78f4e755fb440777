"""Driven under compute-sanitizer by tests/test_sanitizer_gpu.py: small
c2/c4/c5-shaped transposes through the C ABI (host buffers, no torch in the
process), every kernel path once — chunked digit passes (plain and packed
rows), bucketed groups with small runs (k_local2) and large runs, the
run-level sort, rank 5, verify_input, an out-of-range error, the device
sortedness check — each checked against the C oracle.  Single-group plans on
these small tensors take k_small (the latency-regime cooperative kernel)
unless QD_SMALL=0, which the tests set for a second run."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2005_10427_b200 as qd  # noqa: E402
from pyoracle import Oracle  # noqa: E402


def zipf(rng, dims, n, s):
    cols = []
    for d in dims:
        p = 1.0 / np.arange(1, d + 1) ** s
        cols.append(rng.choice(d, n, p=p / p.sum()))
    c = np.unique(np.stack(cols, 1).astype(np.uint32), axis=0)
    return c, rng.random(len(c))


def main():
    scale = int(os.environ.get("QD_SAN_ROWS", "6000"))
    orc = Oracle()
    ws = qd.Workspace(0)
    rng = np.random.default_rng(5)
    cases = [
        ([300, 200, 900], 1.1, [[0, 2, 1], [1, 0, 2], [2, 1, 0]]),        # c2-like
        ([80, 60, 50, 40, 900], 1.0, [[4, 3, 2, 1, 0], [0, 1, 4, 2, 3]]),  # c4-like, rank 5
        ([20, 5000, 5000], 1.05, [[0, 2, 1], [1, 0, 2]]),                  # c5-like: big + small runs
    ]
    for dims, s, targets in cases:
        c, v = zipf(rng, dims, scale, s)
        t = qd.CooTensor(dims, c.ravel(), v)
        for tgt in targets:
            out = qd.transpose(t, tgt, qd.SortStrategy.quesadilla(),
                               qd.TransposeOptions(verify_input=True), ws)
            ec, ev, _ = orc.transpose(dims, t.coords, t.values, tgt)
            assert np.array_equal(out.coords, ec) and np.array_equal(
                out.values.view(np.uint64), ev.view(np.uint64)), (dims, tgt)
    # an out-of-range coordinate: the error path, tensor untouched
    c, v = zipf(rng, [30, 40, 50], scale, 1.0)
    c[len(c) // 2, 1] = 40
    bad = qd.CooTensor([30, 40, 50], c.ravel(), v)
    try:
        qd.transpose(bad, [1, 0, 2], ws=ws)
        raise SystemExit("expected OutOfRange")
    except qd.OutOfRange:
        pass
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
