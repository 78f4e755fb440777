#!/usr/bin/env python
"""Profiling driver: generate a BASELINE config's input on the device, run
every target once untimed (workspace growth, graph capture), then run each
target once more between cudaProfilerStart/Stop, so that
`ncu --profile-from-start off` sees exactly one transposition per target and
none of the generator's sorts.

  python profiles/r2/prof_targets.py --config c5 --nnz 200000000
  ncu --profile-from-start off --set full ... python profiles/r2/prof_targets.py ...
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_10427_b200 as qd  # noqa: E402
from paper_2005_10427_b200 import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--nnz", type=int, default=None)
    p.add_argument("--targets", default=None, help="e.g. 102,021 (default: the config's)")
    p.add_argument("--reps", type=int, default=1)
    a = p.parse_args()
    cfg = synth.CONFIGS[a.config]
    targets = cfg.targets
    if a.targets:
        targets = [tuple(int(ch) for ch in t) for t in a.targets.split(",")]
    ci, vi = bench.make_input(cfg, a.nnz, "cuda")
    n, r = vi.numel(), len(cfg.dims)
    co, vo = torch.empty_like(ci), torch.empty_like(vi)
    ws = qd.Workspace(0)
    st = torch.cuda.Stream(0)
    torch.cuda.set_stream(st)
    strat = qd.SortStrategy.quesadilla()

    def one(t):
        qd.transpose_device(r, cfg.dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                            vo.data_ptr(), t, strat, ws, st.cuda_stream)

    for _ in range(3):
        for t in targets:
            one(t)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.reps):
        for t in targets:
            one(t)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"profiled {a.config} n={n} targets={targets} launches={ws.launches()}")


if __name__ == "__main__":
    main()
