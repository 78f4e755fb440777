"""Multi-process host logic of the sharded transpose (paper_2005_10427_b200/
shard.py) with world_size 2 over gloo on the CPU: splitters, stable partition,
all_to_all exchange, source-rank-order concatenation, sigma1-aligned
communication-free slices.  The per-rank local transpose is the C oracle here
(the GPU backend is exercised by tests/test_parity_gpu.py on one GPU); the
concatenated rank outputs must equal the oracle transpose of the global
tensor bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_10427_b200 import shard
from pyoracle import Oracle


class CpuBackend:
    """Test stand-in for shard.GpuBackend (numpy + the C oracle)."""

    def __init__(self):
        self.orc = Oracle()

    def zeros_like_rows(self, n, rank):
        return shard.LocalRows(torch.empty(n * rank, dtype=torch.int32),
                               torch.empty(n, dtype=torch.float64))

    def slice_info(self, rows, rank):
        c = rows.coords.numpy().view(np.uint32).reshape(-1, rank)
        return (0, 0, 0) if len(c) == 0 else (len(c), int(c[0, 0]), int(c[-1, 0]))

    def mode_hist(self, rows, rank, mode, dim):
        c = rows.coords.numpy().view(np.uint32).reshape(-1, rank)
        return torch.from_numpy(np.bincount(c[:, mode], minlength=dim).astype(np.int64))

    def partition(self, rows, rank, mode, lookup, parts):
        c = rows.coords.numpy().view(np.uint32).reshape(-1, rank)
        part = lookup[c[:, mode]]
        order = np.argsort(part, kind="stable")
        counts = np.bincount(part, minlength=parts).tolist()
        out = shard.LocalRows(torch.from_numpy(np.ascontiguousarray(c[order]).view(np.int32).ravel()),
                              torch.from_numpy(rows.values.numpy()[order].copy()))
        return out, counts

    def transpose(self, rows, dims, target):
        c, v, _ = self.orc.transpose(dims, rows.coords.numpy().view(np.uint32), rows.values.numpy(),
                                     target)
        return shard.LocalRows(torch.from_numpy(c.view(np.int32)), torch.from_numpy(v))

    # QD_EXCHANGE=p2p: the peer writes are emulated over gloo (each sender
    # ships its part with the row offset shard.p2p_layout gave it, and the
    # receiver stores it there), so the offset arithmetic is what is tested
    def symmetric_rows(self, cap, rank, dist):
        return shard.SymRows(torch.zeros(cap * rank, dtype=torch.int32),
                             torch.zeros(cap, dtype=torch.float64), [], [], cap)

    def partition_to_peers(self, rows, rank, mode, lookup, parts, buf, offs):
        part_rows, counts = self.partition(rows, rank, mode, lookup, parts)
        send = torch.tensor(list(counts) + list(offs), dtype=torch.int64)
        got = torch.empty(2 * parts, dtype=torch.int64)
        dist.all_to_all_single(got, send.view(2, parts).t().contiguous().view(-1))
        rc = got.view(parts, 2)[:, 0].tolist()  # rows from each source
        ro = got.view(parts, 2)[:, 1].tolist()  # where each source said they go
        out_c = torch.empty(sum(rc) * rank, dtype=torch.int32)
        out_v = torch.empty(sum(rc), dtype=torch.float64)
        dist.all_to_all_single(out_c, part_rows.coords, [c * rank for c in rc],
                               [c * rank for c in counts])
        dist.all_to_all_single(out_v, part_rows.values, rc, list(counts))
        k = 0
        for src in range(parts):
            n, o = rc[src], ro[src]
            buf.coords[o * rank:(o + n) * rank] = out_c[k * rank:(k + n) * rank]
            buf.values[o:o + n] = out_v[k:k + n]
            k += n
        return counts

    def to_numpy_i64(self, h):
        return h.numpy()

    def synchronize(self):
        pass

    def from_numpy_i64(self, a):
        return torch.from_numpy(np.asarray(a, np.int64))


def global_tensor(seed, dims, n, skew):
    rng = np.random.default_rng(seed)
    cols = []
    for d in dims:
        if skew:
            p = 1.0 / np.arange(1, d + 1) ** 1.3
            cols.append(rng.choice(d, n, p=p / p.sum()))
        else:
            cols.append(rng.integers(0, d, n))
    c = np.unique(np.stack(cols, 1).astype(np.uint32), axis=0)  # unique + simply sorted
    return c, rng.random(len(c))


def worker(rank, world, port, cases, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = CpuBackend()
    out = []
    for dims, seed, skew, target in cases:
        c, v = global_tensor(seed, dims, 4000, skew)
        r = len(dims)
        if target[0] == 0 and seed != 8:  # seed 8: even slices that split a mode-0 run
            b = shard.aligned_bounds(c[:, 0], world)
        else:
            b = [len(c) * p // world for p in range(world)] + [len(c)]
        lo, hi = b[rank], b[rank + 1]
        rows = shard.LocalRows(torch.from_numpy(np.ascontiguousarray(c[lo:hi]).view(np.int32).ravel()),
                               torch.from_numpy(v[lo:hi].copy()))
        st = {}
        res, exchanged = shard.sharded_transpose(dist, be, rows, dims, target, stats=st)
        assert st["rows_out"] == res.nnz()
        assert exchanged or st["sent_bytes"] == 0
        out.append((res.coords.numpy().copy(), res.values.numpy().copy(), exchanged))
    results[rank] = out
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    ([30, 40, 50], 1, False, [1, 0, 2]),
    ([30, 40, 50], 2, True, [1, 0, 2]),
    ([30, 40, 50], 3, True, [2, 1, 0]),
    ([30, 40, 50], 4, True, [0, 2, 1]),
    ([12, 9, 7, 11], 5, False, [3, 1, 0, 2]),
    ([12, 9, 7, 11], 6, True, [0, 3, 1, 2]),
    ([3, 200, 200], 7, True, [2, 0, 1]),
    ([3, 200, 200], 8, True, [0, 2, 1]),  # unaligned slices: exchange fallback
]


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_sharded_transpose_world2_gloo(exchange, monkeypatch):
    monkeypatch.setenv("QD_EXCHANGE", exchange)  # inherited by the forked ranks
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.start_processes(worker, args=(world, free_port(), CASES, results), nprocs=world,
                       join=True, start_method="fork")
    orc = Oracle()
    for k, (dims, seed, skew, target) in enumerate(CASES):
        c, v = global_tensor(seed, dims, 4000, skew)
        ec, ev, _ = orc.transpose(dims, c.ravel(), v, target)
        got_c = np.concatenate([results[r][k][0].view(np.uint32) for r in range(world)])
        got_v = np.concatenate([results[r][k][1] for r in range(world)])
        assert np.array_equal(got_c, ec), (dims, target)
        assert np.array_equal(got_v.view(np.uint64), ev.view(np.uint64))
        # an exchange exactly when sigma1 != 0 or a mode-0 run straddles the slices
        assert results[0][k][2] == (target[0] != 0 or seed == 8)


def test_splitters_balance_and_monotone():
    h = np.array([100, 1, 1, 50, 0, 0, 30, 30, 30], np.int64)
    for parts in (1, 2, 3, 4):
        lk = shard.splitters(h, parts)
        assert (np.diff(lk.astype(int)) >= 0).all() and lk.max() < parts
    lk = shard.splitters(np.array([5] * 8), 4)
    assert lk.tolist() == [0, 0, 1, 1, 2, 2, 3, 3]


def test_p2p_layout_offsets():
    C = np.array([[5, 0, 2],
                  [1, 4, 0],
                  [3, 3, 3]])
    assert shard.p2p_layout(C, 0) == ([0, 0, 0], 9, 9)
    assert shard.p2p_layout(C, 1) == ([5, 0, 2], 7, 9)
    assert shard.p2p_layout(C, 2) == ([6, 4, 2], 5, 9)


def test_aligned_bounds_never_split_runs():
    m0 = np.array([0, 0, 0, 1, 1, 2, 2, 2, 2, 3])
    for parts in (2, 3, 4):
        b = shard.aligned_bounds(m0, parts)
        assert b[0] == 0 and b[-1] == len(m0)
        for x in b[1:-1]:
            assert x == len(m0) or m0[x] != m0[x - 1]
