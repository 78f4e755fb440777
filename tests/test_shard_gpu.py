"""The sharded transpose in the C++ library (qd_sharded_transpose_device,
csrc/shard.cu): world sizes 2-4 and 8 with the emulated transport (ranks as host
threads on one GPU: device copies + host barriers, no kernel waits on another
rank's), and world size 1 over real NCCL.  Output slices concatenated in rank
order must equal the oracle's transpose of the global tensor bit for bit
(SURVEY §8c's sharded oracle, parallel.cpp:113-154's region semantics)."""
import threading

import numpy as np
import pytest

import paper_2005_10427_b200 as qd
from pyoracle import Oracle

pytestmark = pytest.mark.gpu
ORC = Oracle()


def zipf_tensor(rng, dims, n, s=1.1):
    cols = []
    for d in dims:
        p = 1.0 / np.arange(1, d + 1) ** s
        cols.append(rng.choice(d, n, p=p / p.sum()))
    c = np.unique(np.stack(cols, 1).astype(np.uint32), axis=0)  # unique, simply sorted
    return c, rng.random(len(c))


def aligned_bounds(mode0, parts):
    n = len(mode0)
    b = [0]
    for p in range(1, parts):
        j = n * p // parts
        while 0 < j < n and mode0[j] == mode0[j - 1]:
            j += 1
        b.append(max(j, b[-1]))
    return b + [n]


def run_emulated(world, c, v, dims, target, bounds, strategy=None, capacity=None):
    import torch
    hub = qd.Hub(world)
    outs, errs, stats = [None] * world, [], [None] * world
    r = len(dims)

    def run(rank):
        ws = qd.Workspace(0)
        comm = qd.Comm(hub=hub, rank=rank, ws=ws)
        try:
            lo, hi = bounds[rank], bounds[rank + 1]
            ci = torch.from_numpy(np.ascontiguousarray(c[lo:hi]).view(np.int32).ravel()).cuda()
            vi = torch.from_numpy(v[lo:hi].copy()).cuda()
            cap = capacity if capacity is not None else len(v)
            co = torch.empty(max(cap, 1) * r, dtype=torch.int32, device="cuda")
            vo = torch.empty(max(cap, 1), dtype=torch.float64, device="cuda")
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                n, s = qd.sharded_transpose_device(
                    comm, r, dims, hi - lo, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                    vo.data_ptr(), cap, target, strategy or qd.SortStrategy.quesadilla(), ws,
                    st.cuda_stream)
            st.synchronize()
            outs[rank] = (co[:n * r].cpu().numpy().view(np.uint32), vo[:n].cpu().numpy())
            stats[rank] = s
        except Exception as e:  # surfaced below
            errs.append(e)
        finally:
            comm.close()
            ws.close()

    th = [threading.Thread(target=run, args=(k,)) for k in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    hub.close()
    return outs, stats, errs


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_cpp_emulated(world):
    rng = np.random.default_rng(200 + world)
    dims = [60, 700, 900]
    c, v = zipf_tensor(rng, dims, 300_000)
    for target in ([1, 0, 2], [2, 1, 0], [1, 2, 0], [0, 2, 1], [2, 0, 1], [0, 1, 2]):
        for aligned in (True, False):
            if aligned:
                b = aligned_bounds(c[:, 0], world)
            else:  # even row slices: mode-0 runs straddle ranks
                b = [len(c) * p // world for p in range(world)] + [len(c)]
            outs, stats, errs = run_emulated(world, c, v, dims, target, b)
            assert not errs, errs
            ec, ev, _ = ORC.transpose(dims, c.ravel(), v, target)
            got_c = np.concatenate([o[0] for o in outs])
            got_v = np.concatenate([o[1] for o in outs])
            assert np.array_equal(got_c, ec), (world, target, aligned)
            assert np.array_equal(got_v.view(np.uint64), ev.view(np.uint64))
            exchanged = [s["exchanged"] for s in stats]
            if target == [0, 1, 2]:
                assert not any(exchanged)  # identity: no exchange, no passes
            elif target[0] == 0 and aligned:
                assert not any(exchanged), (target, exchanged)  # communication-free
            else:
                # straddling mode-0 runs, or a leading mode other than 0: one exchange
                assert target[0] != 0 or not aligned
                assert all(exchanged), (target, exchanged)
                assert sum(s["rows_out"] for s in stats) == len(v)
                if target[0] != 0:  # balanced sigma1 ranges
                    assert max(s["rows_out"] for s in stats) < 0.8 * len(v)
                sent = sum(s["bytes_sent"] for s in stats)
                assert sent == sum(s["bytes_received"] for s in stats) > 0


def test_sharded_cpp_empty_ranks_and_strategies():
    rng = np.random.default_rng(7)
    dims = [40, 300, 500]
    c, v = zipf_tensor(rng, dims, 50_000)
    n = len(v)
    # rank 1 holds nothing; rank 2 holds everything else
    b = [0, n // 3, n // 3, n]
    for strat in (qd.SortStrategy.full_radix(), qd.SortStrategy.top_k(1)):
        for target in ([2, 0, 1], [0, 2, 1]):
            outs, stats, errs = run_emulated(3, c, v, dims, target, b, strategy=strat)
            assert not errs, errs
            name = "radix" if strat.kind == "radix" else "topk"
            ec, ev, _ = ORC.transpose(dims, c.ravel(), v, target, name, strat.k)
            assert np.array_equal(np.concatenate([o[0] for o in outs]), ec)
            assert np.array_equal(np.concatenate([o[1] for o in outs]).view(np.uint64),
                                  ev.view(np.uint64))


def test_sharded_cpp_capacity_error_is_collective():
    """A rank whose output slice does not fit fails, and every other rank
    fails too instead of waiting forever in the exchange."""
    rng = np.random.default_rng(8)
    dims = [30, 200, 300]
    c, v = zipf_tensor(rng, dims, 20_000)
    b = [0, len(v) // 2, len(v)]
    outs, stats, errs = run_emulated(2, c, v, dims, [2, 1, 0], b, capacity=10)
    assert len(errs) == 2 and all(isinstance(e, qd.InvalidArgument) for e in errs)


def test_sharded_cpp_nccl_world1():
    """The real NCCL transport (ncclCommInitRank, one rank on this GPU)."""
    import torch
    rng = np.random.default_rng(9)
    dims = [50, 400, 600]
    c, v = zipf_tensor(rng, dims, 100_000)
    ws = qd.Workspace(0)
    comm = qd.Comm(nranks=1, rank=0, device=0, unique_id=qd.comm_unique_id())
    try:
        ci = torch.from_numpy(np.ascontiguousarray(c).view(np.int32).ravel()).cuda()
        vi = torch.from_numpy(v.copy()).cuda()
        co, vo = torch.empty_like(ci), torch.empty_like(vi)
        for target in ([1, 0, 2], [0, 2, 1], [2, 1, 0]):
            n, s = qd.sharded_transpose_device(comm, 3, dims, len(v), ci.data_ptr(), vi.data_ptr(),
                                               co.data_ptr(), vo.data_ptr(), len(v), target,
                                               ws=ws, stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            ec, ev, _ = ORC.transpose(dims, c.ravel(), v, target)
            assert n == len(v) and not s["exchanged"]
            assert np.array_equal(co.cpu().numpy().view(np.uint32), ec)
            assert np.array_equal(vo.cpu().numpy().view(np.uint64), ev.view(np.uint64))
    finally:
        comm.close()
        ws.close()


def test_sharded_cpp_emulated_config5_shape():
    """Config 5's shape and distribution (dimensions / 100, Zipf(1.05)) at
    ~40 M unique rows over two emulated ranks, so each rank's slice is above the
    latency-mode size and runs the general kernels (segmented passes, small-run
    sorts, the exchange's partition pass): (1,0,2) with one exchange, (0,2,1)
    communication-free on mode-0-aligned slices; concatenated rank outputs
    against the oracle's transpose of the global tensor."""
    import torch
    rng = np.random.default_rng(205)
    dims = [48212, 17742, 18051]
    n0 = 60_000_000
    cols = []
    for d in dims:
        cdf = np.cumsum(1.0 / np.arange(1, d + 1) ** 1.05)
        cols.append(np.searchsorted(cdf / cdf[-1], rng.random(n0), side="right").clip(max=d - 1))
    c = np.unique(np.stack(cols, 1).astype(np.uint32), axis=0)
    v = rng.random(len(c))
    n = len(v)
    assert n > (1 << 25)
    j = int(np.searchsorted(c[:, 0], c[n // 2 - 1, 0], side="right"))  # no mode-0 run split
    bounds = [0, j, n]
    for target in ([1, 0, 2], [0, 2, 1]):
        outs, stats, errs = run_emulated(2, c, v, dims, target, bounds)
        assert not errs, errs
        ec, ev, _ = ORC.transpose(dims, c.ravel(), v, target)
        got_c = np.concatenate([o[0] for o in outs])
        got_v = np.concatenate([o[1] for o in outs])
        assert np.array_equal(got_c, ec), target
        assert np.array_equal(got_v.view(np.uint64), ev.view(np.uint64)), target
        assert all(s["exchanged"] for s in stats) == (target[0] != 0)
        torch.cuda.empty_cache()
