"""Host-buffer transposes copy pageable buffers through the pinned chunk ring
(staged_h2d / staged_d2h, tns.cu) and pinned buffers directly
(engine.cu run_groups_host).  Both must give the oracle's rows, including the
bucket boundaries, across several 32 MB chunks."""
import numpy as np
import pytest

from pyoracle import Oracle


def _tensor(n, seed):
    rng = np.random.default_rng(seed)
    dims = [300, 2000, 4000]
    c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
    c = c[np.lexsort(c.T[::-1])]
    return dims, c.ravel(), rng.random(n)


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [False, True])
def test_host_transpose_pageable_and_pinned(pinned):
    import torch
    import paper_2005_10427_b200 as qb
    n = 9_000_000  # 108 MB of coordinates: four ring chunks
    dims, c, v = _tensor(n, 4)
    if pinned:
        tc = torch.empty(len(c), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        tv = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        tc[:] = c
        tv[:] = v
        t = qb.CooTensor(dims, tc, tv)
        assert t.coords.ctypes.data == tc.ctypes.data  # no copy: really pinned
    else:
        t = qb.CooTensor(dims, c.copy(), v.copy())
    bounds = []
    qb.transpose_inplace(t, [2, 0, 1], qb.SortStrategy.quesadilla(), None,
                         qb.TransposeOptions(boundaries=bounds))
    rc, rv, _ = Oracle().transpose(dims, c, v, [2, 0, 1])
    assert np.array_equal(t.coords, rc)
    assert np.array_equal(t.values.view(np.uint64), rv.view(np.uint64))
    col = rc.reshape(-1, 3)[:, 2]
    starts = np.flatnonzero(np.r_[True, col[1:] != col[:-1]])
    assert bounds == list(starts) + [n]
