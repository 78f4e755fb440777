"""TEST INFRASTRUCTURE ONLY — regenerates tests/golden/ from the unmodified
reference library (oracle/_ref/libqref.so, built by ``make -C oracle``).

Run in the build container (where /root/reference exists):
    python oracle/make_golden.py

Fixtures written:
  tests/golden/golden.json   — the reference tests' worked example
      (proj/tests/test_util.hpp:37-70, test_sort.cpp:93-113), its step-1
      permutation, the planner's explicit plans (test_planner.cpp:39-49),
      prefix plans (136-142), pass histograms (125-134) and the plans of every
      BASELINE target (SURVEY.md §8 plan table), each as the reference emits it.
  tests/golden/cases.npz     — randomised small tensors (reference ``generate``,
      io.cpp:154-204) with targets, strategies and the reference's outputs,
      the same style as acceptance.cpp:128-184 (oracle equivalence) and
      test_sort.cpp:247-278 (duplicates / stability).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from pyoracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def digits(v):
    # test_util.hpp:39-46: 4-digit numbers, 1-based digits stored 0-based.
    return [v // 1000 % 10 - 1, v // 100 % 10 - 1, v // 10 % 10 - 1, v % 10 - 1]


def main():
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    gin = [1218, 1224, 1274, 1421, 1437, 1456, 1472, 3216, 3283, 3286]
    gout = [1224, 1274, 1218, 1421, 1472, 1456, 1437, 3283, 3216, 3286]
    dims = [9, 9, 9, 9]
    cin = np.array([digits(v) for v in gin], np.uint32).ravel()
    vin = np.arange(1, 11, dtype=np.float64)
    # Reference outputs on the worked example.
    c_step, v_step = ref.partial_sort(dims, cin, vin, [], 3)
    c_bkt, v_bkt = ref.partial_sort(dims, cin, vin, [0, 1], 3)
    c_q, v_q, log_q = ref.transpose(dims, cin, vin, [0, 1, 3, 2], verify_input=True)
    expect_out = np.array([digits(v) for v in gout], np.uint32).ravel()
    assert (c_bkt == expect_out).all() and (c_q == expect_out).all()
    assert list(v_q) == [2, 3, 1, 4, 7, 6, 5, 9, 8, 10]
    g = {
        "source": "reference library oracle/_ref/libqref.so (proj/src/*.cpp)",
        "golden": {
            "dims": dims,
            "input_coords": cin.tolist(),
            "input_values": vin.tolist(),
            "target": [0, 1, 3, 2],
            "output_coords": c_q.tolist(),
            "output_values": v_q.tolist(),
            "pass_log": log_q,
            "step1_mode3_coords": c_step.tolist(),
            "step1_mode3_values": v_step.tolist(),
            # 1-based perm (4,7,9,2,3,6,8,10,5,1), test_sort.cpp:97
            "step1_perm0": [3, 6, 8, 1, 2, 5, 7, 9, 4, 0],
        },
        "plans": {},
        "prefix_plans": {},
        "pass_histograms": {},
        "bruteforce": {},
    }
    targets = [[3, 0, 1, 2], [1, 3, 0, 2], [3, 2, 1, 0], [0, 1, 3, 2], [0, 1, 2, 3], [0],
               [2, 1, 0], [0, 2, 1], [1, 0, 2], [1, 2, 0], [2, 0, 1],
               [3, 2, 1, 0], [1, 0, 2, 3], [0, 3, 1, 2],
               [4, 3, 2, 1, 0], [0, 1, 4, 2, 3]]
    for t in targets:
        g["plans"][",".join(map(str, t))] = ref.plan(t)
    for t, k in [([3, 2, 1, 0], 1), ([0, 1, 2, 3], 2), ([2, 3, 0, 1], 1), ([2, 3, 0, 1], 3)]:
        g["prefix_plans"][",".join(map(str, t)) + f"@{k}"] = ref.plan(t, k)
    for r in range(2, 7):
        g["pass_histograms"][str(r)] = ref.pass_histogram(r)
    import itertools
    for r in range(2, 6):
        for t in itertools.permutations(range(r)):
            g["bruteforce"][",".join(map(str, t))] = list(ref.min_plan_bruteforce(list(t)))
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)

    # Randomised cases (small, committed).
    rng = np.random.Generator(np.random.Philox(20260809))
    arrays = {}
    meta = []
    strategies = [("quesadilla", 0), ("radix", 0), ("topk", 1), ("topk", 2),
                  ("comparison", 0)]
    for i in range(60):
        r = int(rng.integers(1, 6))
        dims_i = [int(x) for x in rng.integers(1, 17, size=r)]
        nnz = int(rng.integers(0, 1500))
        distinct = bool(rng.integers(0, 2))
        cells = int(np.prod(dims_i))
        if distinct and nnz > cells:
            nnz = cells
        seed = int(rng.integers(0, 2**62))
        c, v = ref.generate(dims_i, nnz, seed, distinct)
        target = [int(x) for x in rng.permutation(r)]
        name, k = strategies[i % len(strategies)]
        if name == "topk":
            k = min(k, r)
        co, vo, log = ref.transpose(dims_i, c, v, target, name, k)
        arrays[f"c{i}_in"] = c
        arrays[f"v{i}_in"] = v
        arrays[f"c{i}_out"] = co
        arrays[f"v{i}_out"] = vo
        meta.append({"i": i, "dims": dims_i, "target": target, "strategy": name,
                     "k": k, "seed": seed, "distinct": distinct, "pass_log": log})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(OUT, "cases.npz"), **arrays)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
