"""Sliced host-buffer calls (engine.cu run_groups_host / run_slices):
when every pass of a call keeps a common prefix mode (Alg. 2 only,
sort.cpp:80-134), qd_transpose_inplace on host buffers (pinned: direct copies;
pageable: staged by a feeder thread) cuts the tensor where that mode changes
and pipelines the slices' input copies, passes and output copies.  The rows
must be the oracle's, bit for bit, however the tensor is cut; an error must leave the caller's rows untouched and be the
whole-tensor call's error."""
import os

import numpy as np
import pytest

from pyoracle import Oracle


def _pinned_tensor(qb, dims, c, v, pinned=True):
    import torch
    if not pinned:  # pageable buffers: staged through the pinned chunk ring by a feeder thread
        return qb.CooTensor(dims, c.copy(), v.copy())
    tc = torch.empty(len(c), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    tv = torch.empty(len(v), dtype=torch.float64, pin_memory=True).numpy()
    tc[:] = c
    tv[:] = v
    t = qb.CooTensor(dims, tc, tv)
    assert t.coords.ctypes.data == tc.ctypes.data
    return t


def _rows(n, dims, seed, head=0.0):
    rng = np.random.default_rng(seed)
    c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
    if head:  # a giant leading-mode run (the Zipf head of config 5)
        c[: int(n * head), 0] = 0
    c = c[np.lexsort(c.T[::-1])]
    return c.ravel(), rng.random(n)


@pytest.fixture
def slice_rows():
    old = os.environ.get("QD_SLICE_ROWS")
    os.environ["QD_SLICE_PAGEABLE"] = "1"  # pageable buffers are sliced on request only

    def set_(v):
        os.environ["QD_SLICE_ROWS"] = str(v)
    yield set_
    os.environ.pop("QD_SLICE_PAGEABLE", None)
    if old is None:
        os.environ.pop("QD_SLICE_ROWS", None)
    else:
        os.environ["QD_SLICE_ROWS"] = old


@pytest.mark.gpu
@pytest.mark.parametrize("dims,target,head", [
    ([300, 2000, 4000], [0, 2, 1], 0.0),
    ([300, 2000, 4000], [0, 2, 1], 0.4),
    ([40, 50, 60, 70], [0, 3, 1, 2], 0.0),
    ([40, 50, 60, 70], [0, 1, 3, 2], 0.1),
    ([7, 9, 50, 60, 70], [0, 1, 4, 2, 3], 0.0),
])
@pytest.mark.parametrize("pinned", [True, False])
def test_sliced_matches_oracle(slice_rows, dims, target, head, pinned):
    import paper_2005_10427_b200 as qb
    n = 400_000
    c, v = _rows(n, dims, 11, head)
    ws = qb.Workspace(0)
    rc, rv, _ = Oracle().transpose(dims, c, v, target)
    for rows in (30_000, 7_001, 150_000):
        slice_rows(rows)
        t = _pinned_tensor(qb, dims, c, v, pinned)
        qb.transpose_inplace(t, target, qb.SortStrategy.quesadilla(), ws)
        assert ws.slices() > 1, "the call was not sliced"
        assert np.array_equal(t.coords, rc)
        assert np.array_equal(t.values.view(np.uint64), rv.view(np.uint64))
    # never slice: the same rows
    slice_rows(0)
    t = _pinned_tensor(qb, dims, c, v)
    qb.transpose_inplace(t, target, qb.SortStrategy.quesadilla(), ws)
    assert ws.slices() == 1
    assert np.array_equal(t.coords, rc)


@pytest.mark.gpu
def test_not_sliced_when_the_leading_mode_moves(slice_rows):
    import paper_2005_10427_b200 as qb
    dims = [300, 2000, 4000]
    c, v = _rows(200_000, dims, 5)
    ws = qb.Workspace(0)
    slice_rows(10_000)
    for target in ([1, 0, 2], [2, 1, 0]):
        t = _pinned_tensor(qb, dims, c, v)
        qb.transpose_inplace(t, target, qb.SortStrategy.quesadilla(), ws)
        assert ws.slices() == 1
        rc, rv, _ = Oracle().transpose(dims, c, v, target)
        assert np.array_equal(t.coords, rc)
        assert np.array_equal(t.values.view(np.uint64), rv.view(np.uint64))


@pytest.mark.gpu
def test_sliced_unordered_rows(slice_rows):
    """Rows that are NOT ordered by the leading mode: a cut at any change of
    the mode is still a boundary of Alg. 2's runs (maximal runs of equal
    prefix in the current order), so slices give the whole call's rows."""
    import paper_2005_10427_b200 as qb
    dims = [50, 2000, 4000]
    rng = np.random.default_rng(3)
    n = 300_000
    c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32)
    c[:, 0] = np.repeat(rng.integers(0, dims[0], n // 100), 100)  # unordered runs of 100 rows
    c = c.ravel()
    v = rng.random(n)
    ws = qb.Workspace(0)
    rc, rv, _ = Oracle().transpose(dims, c, v, [0, 2, 1])
    slice_rows(20_000)
    t = _pinned_tensor(qb, dims, c, v)
    qb.transpose_inplace(t, [0, 2, 1], qb.SortStrategy.quesadilla(), ws)
    assert ws.slices() > 1
    assert np.array_equal(t.coords, rc)
    assert np.array_equal(t.values.view(np.uint64), rv.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("pinned", [True, False])
def test_sliced_error_leaves_rows_untouched(slice_rows, pinned):
    import paper_2005_10427_b200 as qb
    dims = [300, 2000, 4000]
    n = 300_000
    c, v = _rows(n, dims, 9)
    bad = c.copy().reshape(-1, 3)
    bad_row = n - 5000  # in the last slice: earlier slices were already copied out
    bad[bad_row, 2] = dims[2] + 7
    bad = bad.ravel()
    ws = qb.Workspace(0)
    errs = []
    for rows in (0, 25_000):
        slice_rows(rows)
        t = _pinned_tensor(qb, dims, bad, v, pinned)
        with pytest.raises(qb.OutOfRange) as ei:
            qb.transpose_inplace(t, [0, 2, 1], qb.SortStrategy.quesadilla(), ws)
        assert np.array_equal(t.coords, bad), "rows changed by a failed call"
        assert np.array_equal(t.values.view(np.uint64), v.view(np.uint64))
        errs.append(str(ei.value))
    assert ws.slices() > 1
    assert errs[0] == errs[1] and str(bad_row) in errs[0]
    # the workspace is usable afterwards
    t = _pinned_tensor(qb, dims, c, v)
    qb.transpose_inplace(t, [0, 2, 1], qb.SortStrategy.quesadilla(), ws)
    rc, _, _ = Oracle().transpose(dims, c, v, [0, 2, 1])
    assert np.array_equal(t.coords, rc)
