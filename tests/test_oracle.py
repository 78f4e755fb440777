"""Pins the C oracle (oracle/oracle.c) before anything is checked against it:
against the reference's own golden vectors (tests/golden/, generated from the
unmodified reference library) and, where oracle/_ref is built, bit-for-bit
against the reference on fresh random cases.  CPU only."""
import itertools

import numpy as np
import pytest

from golden_util import cases, golden
from pyoracle import Oracle, OracleError, Reference, reference_available

ORC = Oracle()


def test_golden_worked_example():
    g = golden()["golden"]
    c, v, log = ORC.transpose(g["dims"], g["input_coords"], g["input_values"],
                              g["target"], verify_input=True)
    assert c.tolist() == g["output_coords"]
    assert v.tolist() == g["output_values"]
    assert [list(s) for s in log] == g["pass_log"] == [[2, 3]]


def test_golden_step1_permutation():
    # test_sort.cpp:93-105 — non-bucketed sort on mode 3
    g = golden()["golden"]
    c, v = ORC.partial_sort(g["dims"], g["input_coords"], g["input_values"], [], 3)
    assert c.tolist() == g["step1_mode3_coords"]
    assert v.tolist() == g["step1_mode3_values"]
    cin = np.array(g["input_coords"], np.uint32).reshape(-1, 4)
    assert (c.reshape(-1, 4) == cin[g["step1_perm0"]]).all()


def test_planner_matches_reference_plans():
    g = golden()
    for key, steps in g["plans"].items():
        t = [int(x) for x in key.split(",")]
        assert [list(s) for s in ORC.plan(t)] == steps, key
    for key, steps in g["prefix_plans"].items():
        t, k = key.split("@")
        assert [list(s) for s in ORC.plan([int(x) for x in t.split(",")], int(k))] == steps


def test_pass_histograms():
    g = golden()["pass_histograms"]
    for r in range(2, 7):
        hist = {}
        for t in itertools.permutations(range(r)):
            n = len(ORC.plan(list(t)))
            hist[str(n)] = hist.get(str(n), 0) + 1
        assert hist == g[str(r)], r


def test_plans_are_bruteforce_optimal():
    g = golden()["bruteforce"]
    for key, (total, bucketed) in g.items():
        p = ORC.plan([int(x) for x in key.split(",")])
        assert len(p) == total
        assert sum(1 for l, _ in p if l > 0) == bucketed


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"case{c['i']}")
def test_reference_cases(case):
    r = len(case["dims"])
    c, v, log = ORC.transpose(case["dims"], case["c_in"], case["v_in"], case["target"],
                              case["strategy"], case["k"])
    assert np.array_equal(c, case["c_out"])
    assert np.array_equal(v.view(np.uint64), case["v_out"].view(np.uint64))
    assert [list(s) for s in log] == case["pass_log"]
    assert ORC.is_sorted(r, c, case["target"]) or len(v) == 0


def test_errors():
    # sort.cpp:153-166 argument checks, sort.cpp:26-30 corrupt coordinate
    with pytest.raises(OracleError) as e:
        ORC.partial_sort([2, 2], [0, 1], [1.0], [1], 1)
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        ORC.partial_sort([4, 4], [0, 9, 1, 0], [1.0, 2.0], [], 1)
    assert e.value.code == 2
    with pytest.raises(OracleError) as e:  # verify_input on unsorted input
        ORC.transpose([3, 3], [2, 0, 0, 1], [1.0, 2.0], [1, 0], verify_input=True)
    assert e.value.code == 1


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_equals_reference_random():
    ref = Reference()
    rng = np.random.Generator(np.random.Philox(7))
    for i in range(40):
        r = int(rng.integers(1, 6))
        dims = [int(x) for x in rng.integers(1, 40, size=r)]
        nnz = int(rng.integers(0, 3000))
        c, v = ref.generate(dims, nnz, int(rng.integers(0, 2**62)))
        t = [int(x) for x in rng.permutation(r)]
        for strat, k in [("quesadilla", 0), ("radix", 0), ("topk", 1)]:
            a = ORC.transpose(dims, c, v, t, strat, k)
            b = ref.transpose(dims, c, v, t, strat, k, workers=1 + i % 4)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert a[2] == b[2]
        # bucketed primitive with an arbitrary prefix, unsorted input allowed
        if r >= 2:
            mode = t[-1]
            pre = [m for m in t[:-1]][: int(rng.integers(0, r))]
            a = ORC.partial_sort(dims, c, v, pre, mode)
            b = ref.partial_sort(dims, c, v, pre, mode)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert np.array_equal(ORC.bucket_starts(r, a[0], pre[:1] or [mode]),
                                  ref.bucket_starts(dims, b[0], b[1], pre[:1] or [mode]))


def test_sort_rows_by_and_relabel_match_reference():
    """The restatement's sort_rows_by / relabel_target equal the reference's."""
    import itertools
    from pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    ref, orc = Reference(), Oracle()
    rng = np.random.default_rng(21)
    for trial in range(20):
        r = int(rng.integers(1, 5))
        dims = [int(x) for x in rng.integers(1, 9, r)]
        n = int(rng.integers(0, 300))
        c = np.stack([rng.integers(0, d, n) for d in dims], 1).astype(np.uint32).ravel()
        v = rng.random(n)
        keys = [int(x) for x in rng.integers(0, r, int(rng.integers(0, 2 * r + 1)))]
        b = int(rng.integers(0, n + 1)); e = int(rng.integers(b, n + 1))
        rc, rv = ref.sort_rows_by(dims, c, v, b, e, keys)
        oc, ov = orc.sort_rows_by(r, c, v, b, e, keys)
        assert np.array_equal(rc, oc) and np.array_equal(rv.view(np.uint64), ov.view(np.uint64))
    for r in (1, 2, 3, 4):
        for s in itertools.permutations(range(r)):
            for t in itertools.permutations(range(r)):
                assert ref.relabel_target(list(s), list(t)) == orc.relabel_target(list(s), list(t))
