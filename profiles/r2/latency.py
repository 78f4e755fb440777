#!/usr/bin/env python
"""Latency of one synchronous device-resident transpose call for the small
configs (c1, c4): the Python wrapper (qd.transpose_device), the raw C-ABI call
through ctypes with prebuilt arguments (what a C/C++ caller pays, plus ~1 us of
ctypes), and the device time alone (CUDA events around the call, which waits
for its own completion).  Median over --reps calls after warm-up.

  python profiles/r2/latency.py --config c1
"""
import argparse
import ctypes as C
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2005_10427_b200 as qd  # noqa: E402
from paper_2005_10427_b200 import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--reps", type=int, default=200)
    a = p.parse_args()
    cfg = synth.CONFIGS[a.config]
    ci, vi = bench.make_input(cfg, None, "cuda")
    n, r = vi.numel(), len(cfg.dims)
    co, vo = torch.empty_like(ci), torch.empty_like(vi)
    ws = qd.Workspace(0)
    st = torch.cuda.Stream(0)
    torch.cuda.set_stream(st)
    lib = qd.lib()
    dims = (C.c_uint32 * r)(*cfg.dims)
    opts = qd.OptionsC()
    opts.workers = 1
    out = {}
    for t in cfg.targets:
        tgt = (C.c_uint32 * r)(*t)
        kind = qd.KINDS[qd.SortStrategy.quesadilla().kind]
        args = (r, dims, n, C.c_void_p(ci.data_ptr()), C.c_void_p(vi.data_ptr()),
                C.c_void_p(co.data_ptr()), C.c_void_p(vo.data_ptr()), tgt, kind, 0,
                C.byref(opts), ws.handle, C.c_void_p(st.cuda_stream))

        def wrapper():
            qd.transpose_device(r, cfg.dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                                vo.data_ptr(), t, qd.SortStrategy.quesadilla(), ws, st.cuda_stream)

        def raw():
            rc = lib.qd_transpose_device(*args)
            assert rc == 0, rc

        for f in (wrapper, raw):
            for _ in range(5):
                f()
        res = {}
        for name, f in (("python_wrapper_us", wrapper), ("c_abi_us", raw)):
            xs = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                f()
                xs.append((time.perf_counter() - t0) * 1e6)
            res[name] = round(statistics.median(xs), 1)
        ev = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            raw()
            e1.record(st)
            torch.cuda.synchronize()
            ev.append(e0.elapsed_time(e1) * 1e3)
        res["events_around_call_us"] = round(statistics.median(ev), 1)
        out["".join(map(str, t))] = res
    print({"config": a.config, "nnz": n, "per_target": out})


if __name__ == "__main__":
    main()
