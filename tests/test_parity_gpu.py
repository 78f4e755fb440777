"""GPU parity: the CUDA path through the C ABI versus the oracle, bit for bit
(coords by value, values by raw f64 bits).  Mirrors the reference's own test
strategy (proj/tests/test_sort.cpp, test_parallel.cpp, acceptance.cpp)."""
import itertools
import os

import numpy as np
import pytest

import paper_2005_10427_b200 as qd
from golden_util import cases, golden
from pyoracle import Oracle, OracleError, Reference, reference_available

pytestmark = pytest.mark.gpu

ORC = Oracle()
STRATS = {"quesadilla": qd.SortStrategy.quesadilla(), "radix": qd.SortStrategy.full_radix(),
          "comparison": qd.SortStrategy.comparison_sort()}


@pytest.fixture(scope="module")
def ws():
    w = qd.Workspace(0)
    yield w
    w.close()


def same(out: qd.CooTensor, c, v):
    return np.array_equal(out.coords, c) and np.array_equal(out.values.view(np.uint64),
                                                            np.asarray(v).view(np.uint64))


def strategy(name, k):
    return qd.SortStrategy.top_k(k) if name == "topk" else STRATS[name]


def rand_tensor(rng, dims, nnz, sort=True, distinct=False):
    c = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.uint32)
    if distinct:
        c = np.unique(c, axis=0)
    if sort:
        c = c[np.lexsort(c.T[::-1])]
    v = rng.random(len(c))
    return qd.CooTensor(dims, c.ravel(), v)


# --- the reference's worked example -----------------------------------------

def test_golden_example(ws):
    g = golden()["golden"]
    t = qd.CooTensor(g["dims"], g["input_coords"], g["input_values"])
    log = []
    out = qd.transpose(t, g["target"], qd.SortStrategy.quesadilla(),
                       qd.TransposeOptions(verify_input=True, pass_log=log), ws)
    assert out.coords.tolist() == g["output_coords"]
    assert out.values.tolist() == g["output_values"]
    assert log == [qd.PlanStep(2, 3)]


def test_golden_step1_and_bucketed_call(ws):
    g = golden()["golden"]
    t = qd.CooTensor(g["dims"], g["input_coords"], g["input_values"])
    s = t.copy()
    qd.partial_sort(s, [], 3, ws)
    assert s.coords.tolist() == g["step1_mode3_coords"]
    assert s.values.tolist() == g["step1_mode3_values"]
    b = t.copy()
    qd.partial_sort(b, [0, 1], 3, ws)
    assert b.coords.tolist() == g["output_coords"]
    assert qd.is_sorted_under(b, g["target"])


# --- committed reference cases (all strategies) --------------------------------

@pytest.mark.parametrize("case", cases(), ids=lambda c: f"case{c['i']}")
def test_reference_cases(case, ws):
    t = qd.CooTensor(case["dims"], case["c_in"], case["v_in"])
    log = []
    out = qd.transpose(t, case["target"], strategy(case["strategy"], case["k"]),
                       qd.TransposeOptions(pass_log=log), ws)
    assert same(out, case["c_out"], case["v_out"])
    assert [[s.prefix_len, s.mode] for s in log] == case["pass_log"]


# --- randomised equivalence with the oracle ----------------------------------

def test_every_strategy_random(ws):
    rng = np.random.default_rng(1234)
    n_cases = 0
    for r in range(1, 6):
        for i in range(6):
            dims = [int(x) for x in rng.integers(1, 12 if i % 2 else 3000, r)]
            t = rand_tensor(rng, dims, int(rng.integers(0, 6000)))
            target = [int(x) for x in rng.permutation(r)]
            for name, k in [("quesadilla", 0), ("radix", 0), ("comparison", 0),
                            ("topk", 1), ("topk", r)]:
                out = qd.transpose(t, target, strategy(name, k), None, ws)
                c, v, _ = ORC.transpose(dims, t.coords, t.values, target, name, k)
                assert same(out, c, v), (dims, target, name, k)
                n_cases += 1
    assert n_cases >= 150


def test_all_targets_rank4_pass_log(ws):
    rng = np.random.default_rng(99)
    t = rand_tensor(rng, [7, 5, 6, 4], 300)
    for target in itertools.permutations(range(4)):
        log = []
        out = qd.transpose(t, list(target), qd.SortStrategy.quesadilla(),
                           qd.TransposeOptions(pass_log=log), ws)
        c, v, olog = ORC.transpose(t.dims, t.coords, t.values, list(target))
        assert same(out, c, v)
        assert [(s.prefix_len, s.mode) for s in log] == olog


@pytest.mark.parametrize("seed", range(4))
def test_partial_sort_any_prefix_any_order(ws, seed):
    # Alg. 2 semantics on arbitrary (even unsorted) inputs: buckets are maximal runs.
    rng = np.random.default_rng(seed)
    for _ in range(10):
        r = int(rng.integers(2, 6))
        dims = [int(x) for x in rng.integers(1, 40, r)]
        t = rand_tensor(rng, dims, int(rng.integers(1, 20000)), sort=bool(rng.integers(0, 2)))
        perm = [int(x) for x in rng.permutation(r)]
        mode = perm[-1]
        prefix = perm[: int(rng.integers(0, r))]
        s = t.copy()
        qd.partial_sort(s, prefix, mode, ws)
        c, v = ORC.partial_sort(dims, t.coords, t.values, prefix, mode)
        assert same(s, c, v), (dims, prefix, mode)


# --- shapes that exercise every kernel path -----------------------------------

@pytest.mark.parametrize("shape", [
    # (dims, nnz, target): large single run (uniform tiles), multi-digit keys
    ([50, 4000, 70000], 300_000, [2, 1, 0]),
    ([50, 4000, 70000], 300_000, [1, 0, 2]),
    # huge buckets (few prefix values) -> look-back across many tiles per run
    ([3, 5000, 900], 400_000, [0, 2, 1]),
    # tiny buckets -> local CTA sorts
    ([20000, 40, 9000], 200_000, [0, 2, 1]),
    # mixture of large and small buckets (skewed)
    ("zipf", 400_000, [0, 2, 1]),
    # rank 5, multi-step bucketed plan
    ([30, 20, 40, 25, 900], 250_000, [0, 1, 4, 2, 3]),
    ([30, 20, 40, 25, 900], 250_000, [4, 3, 2, 1, 0]),
    # 1-bit and extent-1 modes
    ([1, 2, 1, 3000], 50_000, [3, 1, 0, 2]),
])
def test_kernel_paths(ws, shape):
    dims, nnz, target = shape
    rng = np.random.default_rng(7)
    if dims == "zipf":
        from paper_2005_10427_b200 import synth
        cfg = synth.CONFIGS["c2"]
        c, v = synth.generate(cfg, nnz, seed=11)
        t = qd.CooTensor(cfg.dims, c, v)
        dims = cfg.dims
    else:
        t = rand_tensor(rng, dims, nnz)
    for name in ("quesadilla", "radix"):
        out = qd.transpose(t, target, STRATS[name], None, ws)
        c, v, _ = ORC.transpose(dims, t.coords, t.values, target, name)
        assert same(out, c, v), (dims, target, name)


# --- edge cases the reference tests ------------------------------------------

def test_rank1_and_extent1(ws):
    t = qd.CooTensor([3], [2, 0, 1], [1.0, 2.0, 3.0])
    s = t.copy()
    qd.partial_sort(s, [], 0, ws)
    assert s.coords.tolist() == [0, 1, 2] and s.values.tolist() == [2.0, 3.0, 1.0]
    u = qd.CooTensor([1, 3], [0, 2, 0, 0, 0, 1], [1.0, 2.0, 3.0])
    s = u.copy()
    qd.partial_sort(s, [], 0, ws)
    assert s == u  # every key 0: stable, order kept
    e = qd.CooTensor([1, 3], [0, 0, 0, 1, 0, 2], [1.0, 2.0, 3.0])
    for target in ([0, 1], [1, 0]):
        assert qd.transpose(e, target, ws=ws) == qd.comparison_transpose(e, target, ws=ws)


def test_empty_tensor(ws):
    t = qd.CooTensor([4, 4], np.zeros(0, np.uint32), np.zeros(0))
    qd.partial_sort(t, [], 1, ws)
    qd.partial_sort(t, [0], 1, ws)
    out = qd.transpose(t, [1, 0], ws=ws)
    assert out.nnz() == 0


def test_identity_is_zero_pass_noop(ws):
    rng = np.random.default_rng(21)
    t = rand_tensor(rng, [8, 8, 8], 300)
    log = []
    out = qd.transpose(t, [0, 1, 2], qd.SortStrategy.quesadilla(),
                       qd.TransposeOptions(pass_log=log), ws)
    assert out == t and log == []


def test_argument_errors(ws):
    t = qd.CooTensor([2, 2], [0, 1], [1.0])
    with pytest.raises(qd.InvalidArgument):
        qd.partial_sort(t, [1], 1, ws)
    with pytest.raises(qd.InvalidArgument):
        qd.partial_sort(t, [], 2, ws)
    with pytest.raises(qd.InvalidArgument):
        qd.topk_transpose(t, [1, 0], 0, ws=ws)
    with pytest.raises(qd.InvalidArgument):
        qd.topk_transpose(t, [1, 0], 3, ws=ws)
    with pytest.raises(qd.InvalidArgument):
        qd.transpose(t, [1, 0], qd.SortStrategy.quesadilla(),
                     qd.TransposeOptions(parallel=qd.ParallelConfig(0)), ws)


def test_out_of_range_detected_and_tensor_untouched(ws):
    t = qd.CooTensor([4, 4], [0, 1, 1, 0], [1.0, 2.0])
    t.coords[1] = 9
    before = t.copy()
    with pytest.raises(qd.OutOfRange) as e:
        qd.partial_sort(t, [], 1, ws)
    assert t == before and e.value.mode == 1 and e.value.row == 0
    # a mode the plan never sorts is never checked (as in the reference)
    u = qd.CooTensor([4, 4], [9, 1, 9, 3], [1.0, 2.0])
    with pytest.raises(OracleError):
        ORC.partial_sort(u.dims, u.coords, u.values, [], 0)
    out = qd.transpose(u, [0, 1], ws=ws)  # identity: zero passes
    assert out == u
    # larger tensor, bad coordinate deep inside a large run
    rng = np.random.default_rng(3)
    big = rand_tensor(rng, [5, 3000, 3000], 200_000)
    big.coords[3 * 150_000 + 2] = 3000
    with pytest.raises(qd.OutOfRange):
        qd.transpose(big, [2, 1, 0], ws=ws)
    with pytest.raises(qd.OutOfRange):
        qd.transpose(big, [0, 2, 1], ws=ws)


def test_verify_input(ws):
    t = qd.CooTensor([3, 3], [2, 0, 0, 1], [1.0, 2.0])
    with pytest.raises(qd.InvalidArgument):
        qd.transpose(t, [1, 0], qd.SortStrategy.quesadilla(),
                     qd.TransposeOptions(verify_input=True), ws)


def test_stability_with_duplicates(ws):
    # test_sort.cpp:259-278: identical coordinates keep their value order
    t = qd.CooTensor([3, 3, 3], [0, 1, 2, 1, 2, 0, 1, 2, 0, 2, 0, 1], [10, 20, 30, 40])
    for target in itertools.permutations(range(3)):
        for s in (qd.SortStrategy.quesadilla(), qd.SortStrategy.full_radix(),
                  qd.SortStrategy.top_k(1), qd.SortStrategy.top_k(2)):
            out = qd.transpose(t, list(target), s, None, ws)
            j = list(out.values).index(20.0)
            assert out.values[j + 1] == 30.0
    # duplicate-heavy tensor (test_parallel.cpp:347-362)
    rng = np.random.default_rng(5)
    d = rand_tensor(rng, [2, 2, 3], 20_000)
    for target in itertools.permutations(range(3)):
        out = qd.transpose(d, list(target), ws=ws)
        c, v, _ = ORC.transpose(d.dims, d.coords, d.values, list(target), "comparison")
        assert same(out, c, v)


def test_determinism(ws):
    rng = np.random.default_rng(8)
    t = rand_tensor(rng, [100, 3000, 500], 500_000)
    a = qd.transpose(t, [2, 0, 1], ws=ws)
    for _ in range(3):
        assert qd.transpose(t, [2, 0, 1], ws=ws) == a


# --- against the reference library itself ------------------------------------

@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_config1_against_reference(ws):
    ref = Reference()
    c, v = ref.generate([1000, 1000, 1000], 1_000_000, 1, distinct=True)
    t = qd.CooTensor([1000, 1000, 1000], c, v)
    bounds = []
    log = []
    out = qd.transpose(t, [2, 1, 0], qd.SortStrategy.quesadilla(),
                       qd.TransposeOptions(pass_log=log, boundaries=bounds), ws)
    rc, rv, rlog = ref.transpose(t.dims, c, v, [2, 1, 0], workers=4)
    assert same(out, rc, rv)
    assert [(s.prefix_len, s.mode) for s in log] == rlog == [(0, 1), (0, 2)]
    starts = ref.bucket_starts(t.dims, rc, rv, [2])
    assert bounds == list(starts) + [t.nnz()]


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg_name,n", [("c2", 2_000_000), ("c3", 1_000_000), ("c4", None)])
def test_configs_scaled_against_reference(ws, cfg_name, n):
    from paper_2005_10427_b200 import synth
    cfg = synth.CONFIGS[cfg_name]
    c, v = synth.generate(cfg, n)
    t = qd.CooTensor(cfg.dims, c, v)
    ref = Reference()
    for target in cfg.targets:
        out = qd.transpose(t, target, qd.SortStrategy.quesadilla(), None, ws)
        rc, rv, _ = ref.transpose(cfg.dims, c, v, target, workers=8)
        assert same(out, rc, rv), (cfg_name, target)


# --- device API -------------------------------------------------------------------

def test_device_api_with_torch(ws):
    import torch
    rng = np.random.default_rng(4)
    t = rand_tensor(rng, [64, 2000, 5000], 300_000)
    ci = torch.from_numpy(t.coords.view(np.int32)).cuda()
    vi = torch.from_numpy(t.values).cuda()
    co = torch.empty_like(ci)
    vo = torch.empty_like(vi)
    b = torch.empty(t.nnz() + 1, dtype=torch.int64, device="cuda")
    nb = qd.transpose_device_boundaries(3, t.dims, t.nnz(), ci.data_ptr(), vi.data_ptr(),
                                        co.data_ptr(), vo.data_ptr(), [1, 0, 2], b.data_ptr(),
                                        ws=ws, stream=torch.cuda.current_stream().cuda_stream)
    c, v, _ = ORC.transpose(t.dims, t.coords, t.values, [1, 0, 2])
    assert np.array_equal(co.cpu().numpy().view(np.uint32), c)
    assert np.array_equal(vo.cpu().numpy().view(np.uint64), v.view(np.uint64))
    starts = ORC.bucket_starts(3, c, [1])
    assert b[:nb].cpu().numpy().tolist() == list(starts) + [t.nnz()]
    assert qd.is_sorted_device(3, t.nnz(), co.data_ptr(), [1, 0, 2], ws=ws)
    assert not qd.is_sorted_device(3, t.nnz(), co.data_ptr(), [0, 1, 2], ws=ws)


@pytest.mark.parametrize("shift", [0, 1, 2, 3])
def test_device_api_unaligned_buffers(ws, shift):
    """Rank-4 rows take 16-byte shared loads / global stores in k_scatter when
    the staged tile and the output are 16-byte aligned; device buffers that
    start 4, 8 or 12 bytes off (any caller pointer; values 8 bytes off) must
    take the word path and give the same bytes.  Packed, AoS, implicit-prefix,
    run-move, k_local (small runs) and rank-5 paths."""
    import torch
    rng = np.random.default_rng(40 + shift)
    for dims, target, env in (([40, 3000, 900, 70], [3, 2, 1, 0], {}),          # packed rows
                              ([3000, 2 ** 20, 2 ** 22, 1500], [3, 2, 1, 0], {}),  # AoS
                              ([3000, 2 ** 20, 2 ** 22, 1500], [0, 3, 1, 2], {}),
                              ([300, 40, 2 ** 22, 1500], [1, 0, 2, 3],        # run move
                               {"QD_RUN_SORT": "1", "QD_RUN_SORT_MIN_ROWS": "1"}),
                              ([20000, 300, 5000], [0, 2, 1], {}),              # k_local
                              ([700, 900, 300, 20, 50], [4, 3, 2, 1, 0], {})):  # rank 5
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        t = rand_tensor(rng, dims, 200_000)
        n, R = t.nnz(), len(dims)
        cbuf = torch.zeros(n * R + 8, dtype=torch.int32, device="cuda")
        obuf = torch.zeros(n * R + 8, dtype=torch.int32, device="cuda")
        ci = cbuf[shift:shift + n * R]
        ci.copy_(torch.from_numpy(t.coords.view(np.int32)))
        co = obuf[(4 - shift) % 4:(4 - shift) % 4 + n * R]
        # values 8 bytes off a 16-byte line on odd shifts
        vbuf = torch.zeros(n + 2, dtype=torch.float64, device="cuda")
        vi = vbuf[shift & 1:(shift & 1) + n]
        vi.copy_(torch.from_numpy(t.values))
        vobuf = torch.zeros(n + 2, dtype=torch.float64, device="cuda")
        vo = vobuf[1 - (shift & 1):1 - (shift & 1) + n]
        qd.transpose_device(R, dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                            vo.data_ptr(), target, qd.SortStrategy.quesadilla(), ws,
                            torch.cuda.current_stream().cuda_stream)
        for k, x in old.items():
            if x is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = x
        c, v, _ = ORC.transpose(dims, t.coords, t.values, target)
        assert np.array_equal(co.cpu().numpy().view(np.uint32), c), (dims, target, shift)
        assert np.array_equal(vo.cpu().numpy().view(np.uint64), v.view(np.uint64))


def test_two_workspaces_on_two_threads():
    """Distinct workspaces may be used concurrently from different host threads
    (the reference forbids only sharing one Workspace, sort.hpp:12-13): no
    library-global state may leak between the calls."""
    import threading
    rng = np.random.default_rng(77)
    jobs = [(rand_tensor(rng, [300, 2000, 900], 400_000), [2, 1, 0]),
            (rand_tensor(rng, [50, 7000, 40, 30], 300_000), [0, 3, 1, 2])]
    want = [ORC.transpose(t.dims, t.coords, t.values, tg) for t, tg in jobs]
    errors = []

    def run(k):
        try:
            w = qd.Workspace(0)
            t, tg = jobs[k]
            for _ in range(4):
                out = qd.transpose(t, tg, qd.SortStrategy.quesadilla(), None, w)
                if not same(out, want[k][0], want[k][1]):
                    errors.append(f"job {k}: output differs")
            w.close()
        except Exception as e:  # noqa: BLE001
            errors.append(f"job {k}: {e!r}")

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


# --- multi-GPU building blocks on one GPU ---------------------------------------

def test_partition_rows_and_mode_hist(ws):
    import torch
    from paper_2005_10427_b200 import shard
    rng = np.random.default_rng(12)
    t = rand_tensor(rng, [50, 700, 90], 300_000)
    be = shard.GpuBackend(0, ws)
    rows = shard.LocalRows(torch.from_numpy(t.coords.view(np.int32)).cuda(),
                           torch.from_numpy(t.values).cuda())
    h = be.to_numpy_i64(be.mode_hist(rows, 3, 1, 700))
    c = t.coords.reshape(-1, 3)
    assert np.array_equal(h, np.bincount(c[:, 1], minlength=700))
    for parts in (1, 2, 5, 8):
        lk = shard.splitters(h, parts)
        out, counts = be.partition(rows, 3, 1, lk, parts)
        part = lk[c[:, 1]]
        order = np.argsort(part, kind="stable")  # stable partition = reference order inside parts
        assert counts == np.bincount(part, minlength=parts).tolist()
        assert np.array_equal(out.coords.cpu().numpy().view(np.uint32).reshape(-1, 3), c[order])
        assert np.array_equal(out.values.cpu().numpy(), t.values[order])


def test_sharded_single_rank_is_plain_transpose(ws):
    import torch
    import torch.distributed as dist
    from paper_2005_10427_b200 import shard
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=0, world_size=1)
    rng = np.random.default_rng(13)
    t = rand_tensor(rng, [40, 300, 500], 100_000)
    be = shard.GpuBackend(0, ws)
    rows = shard.LocalRows(torch.from_numpy(t.coords.view(np.int32)).cuda(),
                           torch.from_numpy(t.values).cuda())
    for target in ([1, 0, 2], [0, 2, 1]):
        out, _ = shard.sharded_transpose(dist, be, rows, t.dims.tolist(), target)
        c, v, _ = ORC.transpose(t.dims, t.coords, t.values, target)
        assert np.array_equal(out.coords.cpu().numpy().view(np.uint32), c)


def test_unchecked_mode_out_of_range_is_moved_not_truncated(ws):
    # Mode 0 is never a key of the (2,1,0) plan, so the reference never
    # range-checks it (sort.cpp:26-30 only checks the sorted mode) and just
    # moves the value 9 along; the packed intermediate cannot hold it, so the
    # library must detect that and redo the call unpacked.
    rng = np.random.default_rng(17)
    t = rand_tensor(rng, [4, 3000, 3000], 100_000)
    t.coords[3 * 5000] = 9
    c, v, _ = ORC.transpose(t.dims, t.coords, t.values, [2, 1, 0])
    out = qd.transpose(t, [2, 1, 0], ws=ws)
    assert same(out, c, v)


@pytest.mark.parametrize("target", [[1, 0, 2], [2, 1, 0], [1, 2, 0], [0, 2, 1], [2, 0, 1]])
@pytest.mark.parametrize("skew", [False, True])
def test_run_level_sort_chains(ws, target, skew):
    # long runs of equal (i0, i1) make the run-level sort (and the MSD/LSD
    # chains that start with it) kick in; forced on at this size via env
    os.environ["QD_RUN_SORT_MIN_ROWS"] = "1"
    os.environ["QD_RUN_SORT"] = "1"
    try:
        rng = np.random.default_rng(31 + skew)
        if skew:
            from paper_2005_10427_b200 import synth
            cfg = synth.Config("t", [60, 80, 20000], 400_000, ["zipf"] * 3, s=1.3, seed=5)
            c, v = synth.generate(cfg)
            t = qd.CooTensor(cfg.dims, c, v)
        else:
            t = rand_tensor(rng, [20, 50, 20000], 300_000)
        out = qd.transpose(t, target, ws=ws)
        c, v, _ = ORC.transpose(t.dims, t.coords, t.values, target)
        assert same(out, c, v)
        # an out-of-range mode-1 coordinate: found through the run records
        # when mode 1 is sorted by the plan, moved untouched otherwise
        bad = t.copy()
        bad.coords[3 * 1000 + 1] = 50 if not skew else 80
        sorted_modes = {s.mode for s in qd.quesadilla_plan(target).steps}
        if 1 in sorted_modes:
            with pytest.raises(qd.OutOfRange):
                qd.transpose(bad, target, ws=ws)
        else:
            c, v, _ = ORC.transpose(bad.dims, bad.coords, bad.values, target)
            assert same(qd.transpose(bad, target, ws=ws), c, v)
    finally:
        del os.environ["QD_RUN_SORT_MIN_ROWS"]
        del os.environ["QD_RUN_SORT"]


# --- asynchronous host-buffer calls (qd_transpose_inplace_async) ------------

def test_async_pipeline_matches_oracle(ws):
    """A pipeline of async calls (one tensor copy per target, as the CLI bench
    loop does) gives every call the oracle's output once synchronized."""
    rng = np.random.default_rng(11)
    base = rand_tensor(rng, [300, 200, 500], 400_000, distinct=True)
    targets = [[0, 2, 1], [1, 0, 2], [1, 2, 0], [2, 0, 1], [2, 1, 0]]
    copies = [base.copy() for _ in targets]
    logs = [[] for _ in targets]
    for t, tgt, lg in zip(copies, targets, logs):
        qd.transpose_inplace_async(t, tgt, qd.SortStrategy.quesadilla(), ws,
                                   qd.TransposeOptions(pass_log=lg))
    ws.synchronize()
    for t, tgt, lg in zip(copies, targets, logs):
        c, v, steps = ORC.transpose(base.dims, base.coords, base.values, tgt)
        assert same(t, c, v), tgt
        assert [(s.prefix_len, s.mode) for s in lg] == [tuple(x) for x in steps]


def test_async_chained_on_same_buffers(ws):
    """Chained in-place async calls on ONE tensor: the second call's input copy
    must wait for the first call's output copy."""
    rng = np.random.default_rng(12)
    base = rand_tensor(rng, [60, 70, 80], 150_000)
    t = base.copy()
    qd.transpose_inplace_async(t, [0, 2, 1], qd.SortStrategy.quesadilla(), ws)
    # (0,2,1)-sorted data is not simply sorted; a full radix re-sort to (2,1,0)
    # is valid on any order and must see the first call's output
    qd.transpose_inplace_async(t, [2, 1, 0], qd.SortStrategy.full_radix(), ws)
    ws.synchronize()
    c1, v1, _ = ORC.transpose(base.dims, base.coords, base.values, [0, 2, 1])
    c2, v2, _ = ORC.transpose(base.dims, c1, v1, [2, 1, 0], "radix")
    assert same(t, c2, v2)


@pytest.mark.parametrize("ntensors", [2, 3])
def test_async_interleaved_buffers(ws, ntensors):
    """Tensors transposed alternately in place, A, B, A, B, ... (or A, B, C,
    A, ...: with two device slots A's previous call is then not even the
    latest call of any slot): every call on A must read the bytes the previous
    call on A wrote back (only the immediately previous call was
    checked).  Full radix re-sorts are valid on any input order."""
    rng = np.random.default_rng(14 + ntensors)
    shapes = [[50, 3000, 40], [70, 60, 2000], [900, 30, 30]][:ntensors]
    base = [rand_tensor(rng, d, 400_000 + 50_000 * i) for i, d in enumerate(shapes)]
    work = [t.copy() for t in base]
    seq = [[2, 1, 0], [1, 0, 2], [0, 2, 1], [2, 0, 1], [1, 2, 0], [0, 1, 2]]
    for tgt in seq:
        for i, t in enumerate(work):
            qd.transpose_inplace_async(t, tgt if i % 2 == 0 else tgt[::-1],
                                       qd.SortStrategy.full_radix(), ws)
    ws.synchronize()
    for i, (b, t) in enumerate(zip(base, work)):
        c, v = b.coords, b.values
        for tgt in seq:
            c, v, _ = ORC.transpose(b.dims, c, v, tgt if i % 2 == 0 else tgt[::-1], "radix")
        assert same(t, c, v), i


def test_async_errors_leave_tensor_untouched(ws):
    rng = np.random.default_rng(13)
    big = rand_tensor(rng, [5, 300, 300], 50_000)
    big.coords[3 * 20_000 + 2] = 300
    before = big.copy()
    ok = rand_tensor(rng, [5, 300, 300], 50_000)
    ok_before = ok.copy()
    # device errors of queued calls surface at synchronize (the first one);
    # the failing call's tensor is untouched, the other calls complete
    qd.transpose_inplace_async(big, [2, 1, 0], qd.SortStrategy.quesadilla(), ws)
    qd.transpose_inplace_async(ok, [2, 1, 0], qd.SortStrategy.quesadilla(), ws)
    with pytest.raises(qd.OutOfRange):
        ws.synchronize()
    assert big == before
    c, v, _ = ORC.transpose(ok_before.dims, ok_before.coords, ok_before.values, [2, 1, 0])
    assert same(ok, c, v)
    ws.synchronize()  # the error was reported once
    with pytest.raises(qd.InvalidArgument):
        qd.transpose_inplace_async(before, [2, 1, 0], qd.SortStrategy.quesadilla(), ws,
                                   qd.TransposeOptions(boundaries=[]))
    empty = qd.CooTensor([3, 3], np.zeros(0, np.uint32), np.zeros(0))
    qd.transpose_inplace_async(empty, [1, 0], qd.SortStrategy.quesadilla(), ws)
    ws.synchronize()
    assert empty.nnz() == 0


# --- the sharded (multi-GPU) path with the GPU backend, W ranks emulated ----
# as host threads of one process on one GPU.  Collectives are host-side
# (barrier + tensor copies); no kernel ever waits on another rank's kernel.

class _Hub:
    def __init__(self, world):
        import threading
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = {}


class _ThreadDist:
    """The torch.distributed calls shard.py makes, over threads."""

    def __init__(self, hub, rank):
        self.hub, self.rank, self.calls = hub, rank, 0

    def get_world_size(self):
        return self.hub.world

    def get_rank(self):
        return self.rank

    def _post(self, value):
        key = self.calls
        self.calls += 1
        self.hub.slots[(key, self.rank)] = value
        self.hub.barrier.wait()
        return key

    def all_reduce(self, t):
        import torch
        key = self._post(t.clone())
        total = torch.stack([self.hub.slots[(key, r)] for r in range(self.hub.world)]).sum(0)
        self.hub.barrier.wait()
        t.copy_(total)

    def barrier(self):
        self.hub.barrier.wait()

    class group:  # noqa: N801 (torch.distributed's attribute name)
        WORLD = None

    def symmetric_empty(self, nbytes, device):
        """Emulated symmetric memory: every rank's buffer lives on the one GPU,
        so the other ranks' base addresses are directly writable."""
        import torch
        raw = torch.empty(nbytes, dtype=torch.uint8, device=device)
        key = self._post(raw)
        ptrs = [self.hub.slots[(key, r)].data_ptr() for r in range(self.hub.world)]
        self.hub.barrier.wait()
        return raw, ptrs

    def all_to_all_single(self, out, inp, output_split_sizes=None, input_split_sizes=None):
        import torch
        w = self.hub.world
        sizes = input_split_sizes or [inp.numel() // w] * w
        parts = list(torch.split(inp, list(sizes)))
        key = self._post(parts)
        got = [self.hub.slots[(key, src)][self.rank] for src in range(w)]
        if output_split_sizes is not None:
            assert [g.numel() for g in got] == list(output_split_sizes)
        if got:
            out.copy_(torch.cat(got))
        self.hub.barrier.wait()


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_gpu_backend_emulated_ranks(world, exchange, monkeypatch):
    """exchange='p2p': the partition kernel writes every part straight into
    its destination rank's receive buffer (qd_partition_rows_to_peers_device);
    the emulated ranks' buffers share the one GPU, so the peer addresses are
    real device addresses and no kernel waits on another."""
    monkeypatch.setenv("QD_EXCHANGE", exchange)
    import threading
    import torch
    from paper_2005_10427_b200 import shard
    rng = np.random.default_rng(100 + world)
    dims = [60, 700, 900]
    cols = []
    for d in dims:
        p = 1.0 / np.arange(1, d + 1) ** 1.1
        cols.append(rng.choice(d, 300_000, p=p / p.sum()))
    c = np.unique(np.stack(cols, 1).astype(np.uint32), axis=0)  # unique, simply sorted
    v = rng.random(len(c))
    for target in ([1, 0, 2], [2, 1, 0], [1, 2, 0], [0, 2, 1], [2, 0, 1]):
        if target[0] == 0:
            b = shard.aligned_bounds(c[:, 0], world)
        else:
            b = [len(c) * p // world for p in range(world)] + [len(c)]
        hub = _Hub(world)
        outs, errs = [None] * world, []

        def run(rank):
            try:
                be = shard.GpuBackend(0)
                lo, hi = b[rank], b[rank + 1]
                rows = shard.LocalRows(
                    torch.from_numpy(np.ascontiguousarray(c[lo:hi]).view(np.int32).ravel()).cuda(),
                    torch.from_numpy(v[lo:hi].copy()).cuda())
                res, exchanged = shard.sharded_transpose(_ThreadDist(hub, rank), be, rows, dims,
                                                         target)
                outs[rank] = (res.coords.cpu().numpy().view(np.uint32), res.values.cpu().numpy(),
                              exchanged)
            except Exception as e:  # surfaced below
                errs.append(e)
                hub.barrier.abort()

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        ec, ev, _ = ORC.transpose(dims, c.ravel(), v, target)
        got_c = np.concatenate([o[0] for o in outs])
        got_v = np.concatenate([o[1] for o in outs])
        assert np.array_equal(got_c, ec), (world, target)
        assert np.array_equal(got_v.view(np.uint64), ev.view(np.uint64))
        assert all(o[2] == (target[0] != 0) for o in outs)
        # the exchange balanced the sigma1 ranges (no rank got everything)
        if target[0] != 0:
            assert max(len(o[1]) for o in outs) < 0.8 * len(v)


# --- sort_rows_by (sort.cpp:203-235), canonicalisation, relabel_target ------

def test_sort_rows_by_matches_oracle(ws):
    rng = np.random.default_rng(31)
    for trial in range(25):
        r = int(rng.integers(1, 6))
        dims = [int(x) for x in rng.integers(1, 3000, r)]
        n = int(rng.choice([0, 1, 2, 50, 5000, 120_000]))
        t = rand_tensor(rng, dims, n, sort=bool(trial % 2))
        keys = [int(x) for x in rng.integers(0, r, int(rng.integers(0, 2 * r + 1)))]
        b = int(rng.integers(0, n + 1)) if trial % 3 else 0
        e = int(rng.integers(b, n + 1)) if trial % 3 else n
        got = t.copy()
        qd.sort_rows_by(got, b, e, keys, ws)
        c, v = ORC.sort_rows_by(r, t.coords, t.values, b, e, keys)
        assert same(got, c, v), (dims, n, keys, b, e)


def test_sort_rows_by_device_and_errors(ws):
    import torch
    rng = np.random.default_rng(32)
    t = rand_tensor(rng, [50, 60, 70], 200_000, sort=False)
    ci = torch.from_numpy(t.coords.view(np.int32)).cuda()
    vi = torch.from_numpy(t.values).cuda()
    co, vo = torch.empty_like(ci), torch.empty_like(vi)
    for keys, b, e in (([2, 0], 1000, 150_000), ([0, 1, 2], 0, 200_000), ([], 5, 10)):
        qd.sort_rows_by_device(3, t.dims, t.nnz(), ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                               vo.data_ptr(), b, e, keys, ws)
        c, v = ORC.sort_rows_by(3, t.coords, t.values, b, e, keys)
        assert np.array_equal(co.cpu().numpy().view(np.uint32), c)
        assert np.array_equal(vo.cpu().numpy().view(np.uint64), v.view(np.uint64))
    # coordinates beyond dims are sorted, not rejected (a comparison sort)
    u = qd.CooTensor([4, 4], [9, 1, 2, 3, 7, 0], [1.0, 2.0, 3.0])
    qd.sort_rows_by(u, 0, 3, [0], ws)
    assert u.coords.tolist() == [2, 3, 7, 0, 9, 1]
    with pytest.raises(qd.InvalidArgument):
        qd.sort_rows_by(u, 0, 3, [2], ws)
    with pytest.raises(qd.InvalidArgument):
        qd.sort_rows_by(u, 2, 4, [0], ws)


def test_canonicalize_then_transpose(ws):
    """read_tns's canonicalisation: any row order -> simple order, then the
    Quesadilla transpose (the reference's read_tns + transpose path)."""
    rng = np.random.default_rng(33)
    t = rand_tensor(rng, [200, 300, 400], 300_000, sort=True, distinct=True)
    perm = rng.permutation(t.nnz())
    shuffled = qd.CooTensor(t.dims, t.coords.reshape(-1, 3)[perm].ravel(), t.values[perm])
    qd.canonicalize(shuffled, ws)
    assert shuffled == t
    out = qd.transpose(shuffled, [2, 0, 1], ws=ws)
    c, v, _ = ORC.transpose(t.dims, t.coords, t.values, [2, 0, 1])
    assert same(out, c, v)


def test_relabel_target_matches_oracle():
    for r in (1, 2, 3, 4):
        for s in itertools.permutations(range(r)):
            for t in itertools.permutations(range(r)):
                assert qd.relabel_target(list(s), list(t)).modes() == ORC.relabel_target(list(s), list(t))
    with pytest.raises(qd.InvalidArgument):
        qd.relabel_target([0, 1], [0, 1, 2])


def test_async_then_sync_calls_on_one_workspace(ws):
    """A synchronous call on a workspace with queued async calls waits for
    the worker first; results of both are correct."""
    rng = np.random.default_rng(14)
    a = rand_tensor(rng, [80, 90, 100], 300_000)
    b = rand_tensor(rng, [80, 90, 100], 300_000)
    a0, b0 = a.copy(), b.copy()
    qd.transpose_inplace_async(a, [1, 2, 0], qd.SortStrategy.quesadilla(), ws)
    out = qd.transpose(b, [2, 0, 1], ws=ws)
    ws.synchronize()
    ca, va, _ = ORC.transpose(a0.dims, a0.coords, a0.values, [1, 2, 0])
    cb, vb, _ = ORC.transpose(b0.dims, b0.coords, b0.values, [2, 0, 1])
    assert same(a, ca, va) and same(out, cb, vb)


# --- extreme shapes ----------------------------------------------------------

def _np_transpose(dims, coords, values, target):
    """Stable sort of simply sorted rows by the target key (numpy lexsort)."""
    r = len(dims)
    c = np.asarray(coords, np.uint32).reshape(-1, r)
    order = np.lexsort(tuple(c[:, m] for m in reversed(list(target))))  # stable
    return c[order].ravel(), np.asarray(values)[order]


def test_full_width_dimensions(ws):
    """Modes of extent up to 2^32 - 1 (32-bit keys, > 64 packed bits: AoS
    intermediates, no local sort); the reference's count arrays would need
    16 GB here, so numpy's stable lexsort is the check."""
    rng = np.random.default_rng(41)
    dims = [2**32 - 1, 5, 2**31 + 7]
    n = 400_000
    c = np.stack([rng.integers(0, d, n, dtype=np.uint64) for d in dims], 1).astype(np.uint32)
    c[: n // 2, 0] = c[0, 0]  # one huge mode-0 run as well
    c = c[np.lexsort(c.T[::-1])]
    v = rng.random(n)
    t = qd.CooTensor(dims, c.ravel(), v)
    for target in ([2, 0, 1], [1, 2, 0], [0, 2, 1], [2, 1, 0]):
        out = qd.transpose(t, target, ws=ws)
        ec, ev = _np_transpose(dims, t.coords, t.values, target)
        assert same(out, ec, ev), target


def test_high_rank_against_oracle(ws):
    rng = np.random.default_rng(42)
    for r in (9, 12, 16):
        dims = [int(x) for x in rng.integers(2, 5, r)]
        t = rand_tensor(rng, dims, 30_000)
        for _ in range(3):
            target = [int(x) for x in rng.permutation(r)]
            log = []
            out = qd.transpose(t, target, qd.SortStrategy.quesadilla(),
                               qd.TransposeOptions(pass_log=log), ws)
            c, v, steps = ORC.transpose(t.dims, t.coords, t.values, target)
            assert same(out, c, v), (r, target)
            assert [(s.prefix_len, s.mode) for s in log] == [tuple(x) for x in steps]


def _np_csf(c, r, order):
    """CSF levels from numpy (rows sorted under `order`)."""
    c = c.reshape(-1, r)
    pos, crd, prev_starts = [], [], None
    n = len(c)
    for k in range(r):
        key = c[:, list(order[: k + 1])]
        head = np.ones(n, bool)
        if n > 1:
            head[1:] = (key[1:] != key[:-1]).any(1)
        starts = np.flatnonzero(head)
        crd.append(c[starts, order[k]])
        if k == 0:
            pos.append(np.array([0, len(starts)]))
        else:
            pos.append(np.searchsorted(starts, np.append(prev_starts, n)))
        prev_starts = starts
    return pos, crd


def test_csf_levels_after_transpose(ws):
    import torch
    rng = np.random.default_rng(51)
    for dims, n, target in (([30, 40, 50], 50_000, [2, 0, 1]), ([7, 9, 11, 13], 20_000, [3, 1, 0, 2]),
                            ([5, 5], 0, [1, 0]), ([4, 4, 4], 200, [0, 1, 2])):
        t = rand_tensor(rng, dims, n)
        out = qd.transpose(t, target, ws=ws)
        dc = torch.from_numpy(out.coords.view(np.int32)).cuda()
        pos, crd = qd.csf_device(dc, len(dims), target, ws)
        epos, ecrd = _np_csf(out.coords, len(dims), target)
        for k in range(len(dims)):
            assert np.array_equal(pos[k].cpu().numpy(), epos[k]), (dims, k)
            assert np.array_equal(crd[k].cpu().numpy().view(np.uint32), ecrd[k]), (dims, k)


def test_mixed_radix_packing(ws):
    """Coordinates whose bit widths exceed 64 (23+21+21 = 65, config 5's
    shape) but whose non-key modes fit as one mixed-radix number: packed
    16-byte rows with a mixed-radix high part; unchecked out-of-range
    non-key coordinates fall back to unpacked rows."""
    rng = np.random.default_rng(61)
    dims = [4821207, 1774269, 1805187]
    t = rand_tensor(rng, dims, 300_000)
    for target in ([1, 0, 2], [0, 2, 1], [2, 0, 1], [1, 2, 0]):
        out = qd.transpose(t, target, ws=ws)
        c, v, _ = ORC.transpose(t.dims, t.coords, t.values, target)
        assert same(out, c, v), target
    # mode 0 is never a key of (1,0,2): a coordinate beyond its dimension is
    # moved untouched (not range-checked), so the pack must not wrap it
    u = t.copy()
    u.coords[3 * 1000] = dims[0] + 12345
    out = qd.transpose(u, [1, 0, 2], ws=ws)
    c, v = _np_transpose(dims, u.coords, u.values, [1, 0, 2])
    assert same(out, c, v)


def test_implicit_prefix_packing(ws):
    """config 3's shape, target (0,3,1,2): the plan sorts mode 3 inside mode-0
    runs; 11 key bits + modes 1, 2 pack into 64 bits only when mode 0 (the
    run prefix) is left out of the row and restored from the run."""
    rng = np.random.default_rng(71)
    dims = [532924, 17262471, 2480308, 1443]
    n = 300_000
    c = np.stack([rng.integers(0, 12, n) * 40000 + rng.integers(0, 3, n),  # few long mode-0 runs
                  rng.integers(0, dims[1], n), rng.integers(0, dims[2], n),
                  rng.integers(0, dims[3], n)], 1).astype(np.uint32)
    c = np.unique(c, axis=0)
    t = qd.CooTensor(dims, c.ravel(), rng.random(len(c)))
    for target in ([0, 3, 1, 2], [0, 3, 2, 1], [0, 1, 3, 2]):
        out = qd.transpose(t, target, ws=ws)
        ec, ev, _ = ORC.transpose(t.dims, t.coords, t.values, target)
        assert same(out, ec, ev), target


def test_randomised_stress_against_oracle(ws):
    """Random shapes across the engine's layout choices (bit-field, mixed-
    radix and implicit-prefix packing, AoS rows, run-level sort, local
    sorts) and strategies, against the C oracle."""
    rng = np.random.default_rng(2027)
    big = [33_554_467, 3_000_017, 1_000_003, 40_000, 5000, 700, 60, 3]
    for trial in range(40):
        r = int(rng.integers(2, 6))
        dims = [int(rng.choice(big)) for _ in range(r)]
        n = int(rng.choice([1000, 30_000, 150_000]))
        cols = []
        for d in dims:
            if rng.random() < 0.5:
                k = int(rng.integers(1, 50))  # few distinct values -> long runs
                vals = rng.integers(0, d, k)
                cols.append(vals[rng.integers(0, k, n)])
            else:
                cols.append(rng.integers(0, d, n, dtype=np.int64))
        c = np.stack(cols, 1).astype(np.uint32)
        c = c[np.lexsort(c.T[::-1])]
        t = qd.CooTensor(dims, c.ravel(), rng.random(n))
        target = [int(x) for x in rng.permutation(r)]
        name = ["quesadilla", "radix", "topk", "comparison"][trial % 4]
        k = int(rng.integers(1, r + 1))
        out = qd.transpose(t, target, strategy(name, k), ws=ws)
        ec, ev, _ = ORC.transpose(t.dims, t.coords, t.values, target, name, k)
        assert same(out, ec, ev), (trial, dims, n, target, name, k)


def test_stress_with_poisoned_scratch():
    """The randomised stress in a fresh process whose workspace buffers start
    as garbage (QD_POISON): no kernel may depend on zero-filled scratch."""
    import subprocess
    import sys as _sys
    env = dict(os.environ, QD_POISON="255")
    r = subprocess.run([_sys.executable, os.path.join(os.path.dirname(__file__), "stress_util.py"),
                        "8", "60"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


# --- latency mode: no host syncs inside the call, CUDA graph replays ---------

def test_latency_mode_graph_replays(ws):
    """Small tensors run without host round trips and, from the second call
    of a shape on the same buffers, as a replayed CUDA graph: new bytes in
    the same buffers, alternating shapes and targets, a bucketed plan with
    small and large runs, and a buffer that grows in between (invalidating
    the captured graphs) must all still match the oracle."""
    import torch
    rng = np.random.default_rng(77)
    shapes = [([40, 300, 500], 120_000, [2, 1, 0]),
              ([40, 300, 500], 120_000, [0, 2, 1]),
              ([15, 12, 9, 3000, 700], 90_000, [4, 3, 2, 1, 0]),
              ([15, 12, 9, 3000, 700], 90_000, [0, 1, 4, 2, 3])]
    bufs = {}
    for rep in range(4):
        for k, (dims, n, target) in enumerate(shapes):
            t = rand_tensor(rng, dims, n)
            r = len(dims)
            nn = t.nnz()
            if k not in bufs:
                cap = n + 10
                bufs[k] = [torch.empty(cap * r, dtype=torch.int32, device="cuda"),
                           torch.empty(cap, dtype=torch.float64, device="cuda"),
                           torch.empty(cap * r, dtype=torch.int32, device="cuda"),
                           torch.empty(cap, dtype=torch.float64, device="cuda")]
            ci, vi, co, vo = bufs[k]
            ci[:nn * r].copy_(torch.from_numpy(t.coords.view(np.int32)))
            vi[:nn].copy_(torch.from_numpy(t.values))
            qd.transpose_device(r, dims, nn, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                                vo.data_ptr(), target, qd.SortStrategy.quesadilla(), ws,
                                torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            c, v, _ = ORC.transpose(dims, t.coords, t.values, target)
            assert np.array_equal(co[:nn * r].cpu().numpy().view(np.uint32), c), (rep, k)
            assert np.array_equal(vo[:nn].cpu().numpy().view(np.uint64), v.view(np.uint64))
        if rep == 1:  # a bigger call grows workspace buffers: graphs recaptured
            big = rand_tensor(rng, [200, 300, 900], 2_000_000)
            out = qd.transpose(big, [1, 2, 0], ws=ws)
            c, v, _ = ORC.transpose(big.dims, big.coords, big.values, [1, 2, 0])
            assert np.array_equal(out.coords, c)


def test_latency_mode_out_of_range_on_replay(ws):
    """An out-of-range coordinate found by a replayed graph raises
    OutOfRange with the reference's first (row, mode)."""
    import torch
    rng = np.random.default_rng(78)
    dims = [30, 40, 50]
    t = rand_tensor(rng, dims, 50_000)
    n, r = t.nnz(), 3
    ci = torch.from_numpy(t.coords.view(np.int32).copy()).cuda()
    vi = torch.from_numpy(t.values.copy()).cuda()
    co, vo = torch.empty_like(ci), torch.empty_like(vi)
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(3):  # eager, capture, replay
        qd.transpose_device(r, dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(), vo.data_ptr(),
                            [1, 0, 2], qd.SortStrategy.quesadilla(), ws, sp)
    bad = t.coords.copy().reshape(-1, 3)
    bad[n // 3, 1] = 40
    ci.copy_(torch.from_numpy(bad.ravel().view(np.int32)))
    with pytest.raises(qd.OutOfRange) as e:
        qd.transpose_device(r, dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                            vo.data_ptr(), [1, 0, 2], qd.SortStrategy.quesadilla(), ws, sp)
    assert e.value.row == n // 3 and e.value.mode == 1


def test_small_engine_preconditions(ws):
    """k_small (one cooperative kernel for a single-group plan on <= 2^22
    rows) sorts by the composite (prefix, key): valid only when the rows are
    ordered by the group prefix and every composite coordinate is in range.
    On a created stream (graphs on), eager / captured / replayed calls on the
    same buffers must match the oracle for valid input, for input NOT ordered
    by the prefix and for an out-of-range PREFIX coordinate (both redone on the
    general path, reference semantics: no error), raise OutOfRange for a key
    coordinate, and a composite wider than 64 bits takes the general path."""
    import torch
    rng = np.random.default_rng(91)
    st = torch.cuda.Stream()
    sp = st.cuda_stream

    def run(dims, coords, values, target, bufs):
        n, r = len(values), len(dims)
        ci, vi, co, vo = bufs
        ci[:n * r].copy_(torch.from_numpy(coords.view(np.int32)))
        vi[:n].copy_(torch.from_numpy(values))
        torch.cuda.synchronize()
        qd.transpose_device(r, dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(), vo.data_ptr(),
                            target, qd.SortStrategy.quesadilla(), ws, sp)
        st.synchronize()
        return (co[:n * r].cpu().numpy().view(np.uint32).copy(),
                vo[:n].cpu().numpy().view(np.uint64).copy())

    for dims, target in (([40, 300, 500], [0, 2, 1]), ([40, 300, 500], [2, 1, 0]),
                         ([15, 12, 9, 3000, 700], [0, 1, 4, 2, 3])):
        n, r = 60_000, len(dims)
        t = rand_tensor(rng, dims, n)
        bufs = [torch.empty(n * r, dtype=torch.int32, device="cuda"),
                torch.empty(n, dtype=torch.float64, device="cuda"),
                torch.empty(n * r, dtype=torch.int32, device="cuda"),
                torch.empty(n, dtype=torch.float64, device="cuda")]
        c0, v0, _ = ORC.transpose(dims, t.coords, t.values, target)
        for _ in range(3):  # eager, capture, replay
            c, v = run(dims, t.coords, t.values, target, bufs)
            assert np.array_equal(c, c0) and np.array_equal(v, v0.view(np.uint64)), target
        # rows not ordered by the prefix (a shuffled block): general-path redo
        bad = t.coords.reshape(-1, r).copy()
        perm = np.arange(n)
        perm[1000:3000] = rng.permutation(perm[1000:3000])
        bad = bad[perm]
        badv = t.values[perm]
        c1, v1, _ = ORC.transpose(dims, bad.ravel(), badv, target)
        c, v = run(dims, bad.ravel(), badv, target, bufs)
        assert np.array_equal(c, c1) and np.array_equal(v, v1.view(np.uint64)), ("unsorted", target)
        if target[0] == 0:
            # an out-of-range coordinate in the prefix mode (never range-checked)
            oor = t.coords.reshape(-1, r).copy()
            oor[-1, 0] = dims[0] + 3
            c2, v2, _ = ORC.transpose(dims, oor.ravel(), t.values, target)
            c, v = run(dims, oor.ravel(), t.values, target, bufs)
            assert np.array_equal(c, c2) and np.array_equal(v, v2.view(np.uint64)), ("prefix", target)
            # the same in a LARGE run and too wide for its packed field: k_small's
            # redo takes the general path, whose packed attempt is redone unpacked
            # (that second redo must not go back to k_small)
            big = t.coords.reshape(-1, r).copy()
            big[-5000:, 0] = 4 * dims[0] + 3
            c3, v3, _ = ORC.transpose(dims, big.ravel(), t.values, target)
            c, v = run(dims, big.ravel(), t.values, target, bufs)
            assert np.array_equal(c, c3) and np.array_equal(v, v3.view(np.uint64)), ("wide prefix", target)
        # a key coordinate out of range: the reference's out_of_range
        key_mode = {(0, 2, 1): 2, (2, 1, 0): 2, (0, 1, 4, 2, 3): 4}[tuple(target)]
        kb = t.coords.reshape(-1, r).copy()
        kb[n // 2, key_mode] = dims[key_mode]
        with pytest.raises(qd.OutOfRange):
            run(dims, kb.ravel(), t.values, target, bufs)
        c, v = run(dims, t.coords, t.values, target, bufs)  # and valid again
        assert np.array_equal(c, c0) and np.array_equal(v, v0.view(np.uint64))
    # a composite key wider than 64 bits: the general path
    dims = [1 << 22] * 4
    t = rand_tensor(rng, dims, 40_000)
    out = qd.transpose(t, [3, 2, 1, 0], ws=ws)
    c, v, _ = ORC.transpose(dims, t.coords, t.values, [3, 2, 1, 0])
    assert same(out, c, v)


def test_large_bucketed_group_prefix_order(ws):
    """A bucketed group above the latency-mode size (chunked passes for the
    large runs, k_local3 for the small ones) on rows ordered by the prefix,
    and on rows whose prefix order is broken inside runs (a row of a large
    and of a small run takes another mode-0 value): the output equals the
    reference's maximal-run semantics (oracle) in both cases."""
    rng = np.random.default_rng(93)
    dims = [40000, 3000, 5000]
    n = (1 << 24) + 4099  # above the latency-mode size, where sampling applies
    t = rand_tensor(rng, dims, n)
    c0, v0, _ = ORC.transpose(dims, t.coords, t.values, [0, 2, 1])
    out = qd.transpose(t, [0, 2, 1], ws=ws)
    assert same(out, c0, v0)
    # break the prefix order inside windows (a row in the middle of a run of
    # a large and of a small run takes another mode-0 value)
    bad = t.coords.reshape(-1, 3).copy()
    for p in (123_457, n // 2 + 17, n - 1000):
        bad[p, 0] = (bad[p, 0] + 7) % dims[0]
    tb = qd.CooTensor(dims, bad.ravel(), t.values)
    c1, v1, _ = ORC.transpose(dims, tb.coords, tb.values, [0, 2, 1])
    out = qd.transpose(tb, [0, 2, 1], ws=ws)
    assert same(out, c1, v1)


# --- run discovery fused with the first digit pass (k_heads_quad) -------------

@pytest.mark.parametrize("dims,target", [([50, 700, 3000], [0, 2, 1]), ([30, 40, 900, 70], [0, 3, 1, 2]),
                                         ([30, 40, 900, 70], [0, 2, 1, 3])])
def test_fused_run_discovery_sizes(ws, dims, target):
    """Bucketed groups of rank-3/4 tensors with one prefix mode take
    k_heads_quad (four rows per thread; head words from eight lanes' nibbles;
    the first digit as a byte per row; range and pack checks): row counts
    around the quad / word / CTA boundaries, a giant run beside tiny ones, the
    reference's out_of_range (first bad row), and device rows that are NOT
    16-byte aligned (the per-row kernel) must all give the oracle's rows."""
    import torch
    rng = np.random.default_rng(123)
    r = len(dims)
    for n in (1, 2, 3, 5, 31, 33, 127, 129, 4095, 4097, 8191, 20_001, 131_075):
        t = rand_tensor(rng, dims, n)
        co = t.coords.reshape(-1, r).copy()
        co[: n // 2, 0] = 0  # one long run (large), then short ones
        co = co[np.lexsort(co.T[::-1])]
        t = qd.CooTensor(dims, co.ravel(), t.values)
        out = qd.transpose(t, target, ws=ws)
        c, v, _ = ORC.transpose(dims, t.coords, t.values, target)
        assert same(out, c, v), (n, target)
    # a key coordinate out of range in two rows: the first one is reported
    n = 50_000
    t = rand_tensor(rng, dims, n)
    co = t.coords.reshape(-1, r).copy()
    km = target[1]  # the mode the plan sorts (the others are never range-checked)
    co[40_001, km] = dims[km]
    co[17_003, km] = dims[km] + 5
    with pytest.raises(qd.OutOfRange) as ei:
        qd.transpose(qd.CooTensor(dims, co.ravel(), t.values), target, ws=ws)
    with pytest.raises(OracleError):
        ORC.transpose(dims, co.ravel(), t.values, target)
    assert ei.value.row == 17_003 and ei.value.mode == km
    # misaligned device rows: a view starting at row 1 of a device buffer
    t = rand_tensor(rng, dims, 30_001)
    ci = torch.from_numpy(t.coords.view(np.int32)).cuda()
    vi = torch.from_numpy(t.values).cuda()
    co_ = torch.empty_like(ci)
    vo_ = torch.empty_like(vi)
    m = 30_000
    qd.transpose_device(r, dims, m, ci.data_ptr() + 4 * r, vi.data_ptr() + 8, co_.data_ptr() + 4 * r,
                        vo_.data_ptr() + 8, target, qd.SortStrategy.quesadilla(), ws, 0)
    torch.cuda.synchronize()
    c, v, _ = ORC.transpose(dims, t.coords[r:], t.values[1:], target)
    assert np.array_equal(co_[r:].cpu().numpy().view(np.uint32), c)
    assert np.array_equal(vo_[1:].cpu().numpy().view(np.uint64), v.view(np.uint64))
