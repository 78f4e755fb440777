"""CPU-only checks of the product library: it loads, exports every symbol the
C ABI header declares, and its host planner equals the reference planner
(golden fixtures + the C oracle) for every ordering up to rank 6."""
import itertools
import os
import re

import pytest

import paper_2005_10427_b200 as qd
from golden_util import golden
from pyoracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORC = Oracle()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "quesadilla_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(qd_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    L = qd.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert L.qd_abi_version() == 1


def test_shared_object_is_sm100a():
    # the cubin inside the .so is built for sm_100a only
    out = os.popen(f"cuobjdump --list-elf {qd.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_planner_all_orderings_vs_oracle():
    for r in range(1, 7):
        for t in itertools.permutations(range(r)):
            mine = [(s.prefix_len, s.mode) for s in qd.quesadilla_plan(list(t)).steps]
            assert mine == ORC.plan(list(t)), t
            for k in range(1, r + 1):
                mine = [(s.prefix_len, s.mode) for s in qd.prefix_plan(list(t), k).steps]
                assert mine == ORC.plan(list(t), k), (t, k)


def test_planner_golden_plans_and_histograms():
    g = golden()
    for key, steps in g["plans"].items():
        t = [int(x) for x in key.split(",")]
        assert [[s.prefix_len, s.mode] for s in qd.quesadilla_plan(t).steps] == steps
    for r in range(2, 7):
        hist = {}
        for t in itertools.permutations(range(r)):
            n = len(qd.quesadilla_plan(list(t)).steps)
            hist[str(n)] = hist.get(str(n), 0) + 1
        assert hist == g["pass_histograms"][str(r)]


def test_plans_land_on_target_and_are_optimal():
    g = golden()["bruteforce"]
    for r in range(2, 6):
        simple = qd.Ordering.simple(r)
        for t in itertools.permutations(range(r)):
            plan = qd.quesadilla_plan(list(t))
            assert qd.simulate_plan(plan) == qd.Ordering(t)
            cost = qd.plan_cost(plan)
            total, bucketed = g[",".join(map(str, t))]
            assert cost.total_passes == total == qd.required_sort_count(simple, t)
            assert cost.bucketed_passes == bucketed
            for i in range(1, len(plan.steps)):
                assert plan.steps[i].prefix_len >= plan.steps[i - 1].prefix_len


def test_strategy_pass_cost_and_names():
    t = [3, 2, 1, 0]
    assert qd.strategy_pass_cost(qd.SortStrategy.quesadilla(), t) == qd.PlanCost(3, 0)
    assert qd.strategy_pass_cost(qd.SortStrategy.full_radix(), t) == qd.PlanCost(4, 0)
    assert qd.strategy_pass_cost(qd.SortStrategy.comparison_sort(), t) == qd.PlanCost(0, 0)
    assert qd.strategy_pass_cost(qd.SortStrategy.top_k(1), t) == qd.PlanCost(1, 0)
    assert qd.parse_strategy("splatt") == qd.SortStrategy.top_k(1)
    assert qd.parse_strategy("top3").name() == "top3"
    assert qd.parse_strategy("qsort") == qd.SortStrategy.comparison_sort()
    for bad in ("bogus", "top0"):
        with pytest.raises(qd.InvalidArgument):
            qd.parse_strategy(bad)


def test_ordering_errors_and_transitions():
    with pytest.raises(qd.InvalidArgument):
        qd.quesadilla_plan([0, 0, 1])
    with pytest.raises(qd.InvalidArgument):
        qd.prefix_plan([0, 1, 2, 3], 5)
    with pytest.raises(qd.InvalidArgument):
        qd.prefix_plan([0, 1, 2, 3], 0)
    with pytest.raises(qd.InvalidArgument):
        qd.apply_transition([0, 1, 2], qd.PlanStep(2, 1))
    assert qd.apply_transition([0, 1, 2, 3], qd.PlanStep(1, 3)) == qd.Ordering([0, 3, 1, 2])
    assert qd.parse_ordering("2134") == qd.Ordering([1, 0, 2, 3])
    assert qd.format_ordering(qd.Ordering([1, 0, 2, 3])) == "2134"
    assert qd.required_sort_count([0, 2, 1], [2, 0, 1]) == 1


def test_no_cpu_fallback_without_device():
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("a GPU is visible")
    with pytest.raises(qd.DeviceError):
        qd.Workspace(0)


HOST_PARITY = os.path.join(ROOT, "oracle", "_ref", "host_parity")


@pytest.mark.skipif(not os.path.exists(HOST_PARITY), reason="oracle/_ref/host_parity not built")
def test_cpp_host_utilities_match_reference():
    """The C++ drop-in's parse_ordering / format_ordering / parse_strategy and
    Ordering checks against the reference library's own, including the
    std::from_chars edge cases (overflow, sign, spaces, empty tokens) and the
    exact exception messages (tests/cpp/host_parity.cpp)."""
    import subprocess
    r = subprocess.run([HOST_PARITY], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("PASS")


@pytest.mark.parametrize("text,outcome", [
    ("4294967297,2", "bad ordering element '4294967297'"),
    ("99999999999999999999,1", "bad ordering element '99999999999999999999'"),
    ("4294967295,1", "ordering contains mode 4294967294 outside 0..1"),
    ("+1,2", "bad ordering element '+1'"),
    (" 1,2", "bad ordering element ' 1'"),
    ("1,", "bad ordering element ''"),
    ("0,1", "bad ordering element '0'"),
    ("²,1", "bad ordering element '²'"),
    ("1,1", "ordering repeats mode 0"),
    ("3,1", "ordering contains mode 2 outside 0..1"),
    ("01,2", [0, 1]),
    ("2,1,3", [1, 0, 2]),
])
def test_python_parse_ordering_matches_reference(text, outcome):
    """Python mirror of parse_ordering (ordering.cpp:68-99): from_chars
    semantics and the reference's messages (same cases as host_parity.cpp)."""
    if isinstance(outcome, list):
        assert qd.parse_ordering(text).modes() == outcome
    else:
        with pytest.raises(qd.InvalidArgument) as e:
            qd.parse_ordering(text)
        assert str(e.value) == outcome


def test_python_parse_strategy_overflow():
    assert qd.parse_strategy("top4294967295").k == 4294967295
    for bad in ("top4294967296", "top+2", "top 2", "top0", "top²"):
        with pytest.raises(qd.InvalidArgument):
            qd.parse_strategy(bad)
