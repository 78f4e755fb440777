#!/usr/bin/env python
"""bench.py — Quesadilla COO transposition on B200 (BASELINE.json metric:
nonzeros transposed/sec (Mnnz/s) and achieved HBM GB/s vs roofline, on
1/2/4/8 B200).

Workload (default --config c5 = BASELINE.json configs[4], the configuration
the 1/2/4/8-GPU metric is quoted on; it fits one B200): 4821207 x 1774269 x
1805187 with 1,741,809,018 unique Zipf(1.05) nonzeros (seeded synthetic
stand-in, paper_2005_10427_b200/synth.generate_device), input sorted in
(0,1,2).  One STEP = transposing it to both of the config's targets, (1,0,2)
(one exchange when sharded) and (0,2,1) (bucketed; communication-free when
sharded), each through the full Quesadilla plan on the GPU: 2 x 1.74 G
nonzeros per step.  `--config c1..c4` run the other configurations (per-target
diagnostics).

  value : whole-job Mnnz/s, inputs resident in HBM (34.8 GB, far above the
          126 MB L2: no flush needed), CUDA events around exactly K steps
  e2e   : the same metric through the reference-facing host call
          (qd_transpose_inplace on host buffers = transpose_inplace's
          signature, transpose.hpp:59-61): every H2D byte, the device passes
          and every D2H byte inside the timed region, one call per target
          (the library pipelines a target that keeps the leading mode,
          (0,2,1), slice by slice: e2e.per_target reports the slice count)
  roofline : the dominant kernel class, algorithmic bytes / its event-timed
          duration (recorded by the library on its launch stream) vs the
          measured HBM copy peak (MEASURED_PEAKS.json); model_roofline = the
          SURVEY §8(d) B_total byte model per target
  cpu_baseline : the reference library itself (oracle/_ref: the unmodified
          reference sources) on this host's cores, on a bounded sample of the
          same tensor (contiguous row windows, which stay simply sorted):
          parallel (std::thread workers = all cores) and serial (workers = 1)

--impl reference times the reference's own CPU implementation (oracle/_ref,
std::thread workers = all host cores) on the same bytes: each step
transposes one contiguous window of the tensor (2^27 rows, the window moving
each step) to both targets; one full-size run per target is added when host
RAM allows.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c5")
    p.add_argument("--nnz", type=int, default=None, help="override nnz (testing only)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--ref-window", type=int, default=1 << 27,
                   help="rows per reference-arm step (a contiguous window)")
    p.add_argument("--no-ref-full", action="store_true",
                   help="reference arm: skip the one full-size run per target")
    return p.parse_args()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock, max clock and throttle reasons sampled every ~5 ms through NVML
    on a background thread while the timed region runs (nvidia-smi's query
    loop as the fallback when NVML is unavailable)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines = []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            h = None
            try:
                import torch
                pr = torch.cuda.get_device_properties(device)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                h = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = N.nvmlDeviceGetHandleByIndex(device)
            self.nvml, self.h = N, h
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    def __enter__(self):
        if self.nvml is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        N, h = self.nvml, self.h
        bits = [("hw_slowdown", N.nvmlClocksEventReasonHwSlowdown),
                ("hw_thermal_slowdown", N.nvmlClocksEventReasonHwThermalSlowdown),
                ("sw_thermal_slowdown", N.nvmlClocksEventReasonSwThermalSlowdown),
                ("sw_power_cap", N.nvmlClocksEventReasonSwPowerCap)]
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if rs & b else "Not Active" for _, b in bits]
                self.lines.append(", ".join([str(self.device), str(sm), str(self.max_mhz), "0",
                                             hex(rs)] + flags))
            except Exception:
                pass
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}




def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic():
    """dram bytes per row moved by k_scatter, from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def host_info():
    """nproc, lscpu model name and host RAM."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    ram = None
    try:
        import psutil
        ram = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gib": ram}


def avail_ram():
    try:
        import psutil
        return psutil.virtual_memory().available
    except Exception:
        return 0


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_input(cfg, nnz, device="cuda"):
    """Device-resident seeded input (int32 coords [N*r], f64 values [N])."""
    from paper_2005_10427_b200 import synth
    n = cfg.nnz if nnz is None else nnz
    if n > 200_000_000 and all(k in ("zipf", "uniform") for k in cfg.dist):
        return synth.generate_device(cfg, n, device=device)
    return synth.generate_torch(cfg, n, device=device)


def row_checksum_device(ci, vi, r):
    """Order-independent checksum of the (coords, value bits) row multiset,
    computed on the device in chunks (two wrapping int64 sums of mixed
    words): equal for a permutation of the rows, different (w.h.p.) when a
    row is dropped, duplicated or altered."""
    import torch
    n = vi.numel()
    c = ci.view(n, r)
    s1 = torch.zeros((), dtype=torch.int64, device=vi.device)
    s2 = torch.zeros((), dtype=torch.int64, device=vi.device)
    k1 = [0x1F3D5B79A3C4E1, 0x2E4C6A8F1B3D5, 0x3A5C7E9B2D4F6, 0x4B6D8FA3C5E71, 0x5C7E9A1B3D5F8]
    for a in range(0, n, 1 << 27):
        b = min(n, a + (1 << 27))
        x = vi[a:b].view(torch.int64).clone()
        for m in range(r):
            x = x * 0x5851F42D4C957F2D + (c[a:b, m].to(torch.int64) + 1) * k1[m % 5]
            x = x ^ (x >> 29)
        s1 += x.sum()
        s2 += (x * x + (x >> 17)).sum()
    return (int(s1.item()), int(s2.item()))


def survey_bytes(dims, target, n):
    """SURVEY.md §8(d) algorithmic byte model B_total for one transpose."""
    import paper_2005_10427_b200 as qd
    r = len(dims)
    steps = qd.quesadilla_plan(target).steps
    if not steps:
        return 0
    used = set()
    for st in steps:
        used.add(st.mode)
        used.update(target[: st.prefix_len])
    b = n * (4 * r + 4 * len(used))
    for i, st in enumerate(steps):
        l = st.prefix_len
        b += n * (4 + 4 + 4 * (i > 0) + (4 * l + 8 if l > 0 else 0)) + 8 * (dims[st.mode] + 1)
    b += n * (4 + 2 * (4 * r + 8)) + 4 * (dims[target[0]] + 1)
    return b


def tname(t):
    return "(" + ",".join(map(str, t)) + ")"


def workload_config(cfg, n, world=1):
    return {"workload": f"{cfg.name}: {'x'.join(map(str, cfg.dims))}, {n} unique nnz "
                        f"({cfg.dist[0]} s={cfg.s}), targets "
                        + " ".join(tname(t) for t in cfg.targets),
            "nnz": n, "rank": len(cfg.dims), "targets_per_step": len(cfg.targets),
            "parallelism": f"shard{world}" if world > 1 else "single-gpu",
            "l2": "inputs (>= 1.5 GB) larger than the 126 MB L2; no flush needed"}


# ---------------------------------------------------------------------------
# the reference's CPU implementation (oracle/_ref): test infrastructure used
# only as the timed baseline
# ---------------------------------------------------------------------------
def ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference, reference_available
    if not reference_available():
        return None
    return Reference()


def ref_windows(n, rows):
    """Row windows [a, b) of `rows` rows each (the last one clipped)."""
    rows = max(1, min(rows, n))
    return [(a, min(n, a + rows)) for a in range(0, n, rows)]


def ref_time_window(ref, dims, hc, hv, a, b, targets, workers, ctx_cache):
    """Reference transpose_inplace of rows [a, b) (a contiguous window of a
    simply sorted tensor is simply sorted) to every target; returns the
    summed seconds of the transpose calls (the pristine restore is untimed)."""
    r = len(dims)
    rows = b - a
    key = rows
    if ctx_cache.get("rows") != key:
        if ctx_cache.get("ctx"):
            ref.lib.qref_ctx_destroy(ctx_cache["ctx"])
        ctx_cache["ctx"] = ref.lib.qref_ctx_create(r, np.asarray(dims, np.uint32), rows,
                                                   hc[a * r:b * r], hv[a:b])
        ctx_cache["rows"] = key
    ctx = ctx_cache["ctx"]
    tot = 0.0
    for t in targets:
        ref.lib.qref_ctx_reset(ctx, hc[a * r:b * r], hv[a:b])
        ta = np.asarray(t, np.uint32)
        t0 = time.perf_counter()
        s = ref.lib.qref_ctx_transpose(ctx, ta, workers)
        tot += time.perf_counter() - t0
        if s:
            raise RuntimeError(ref.lib.qref_last_error().decode())
    return tot


def ref_sample(ref, cfg, hc, hv, rows, workers, reps, start=0):
    """`reps` steps over consecutive windows of `rows` rows (cycling);
    returns (Mnnz/s, seconds, nnz processed)."""
    n = len(hv)
    wins = ref_windows(n, rows)
    cache = {}
    secs = units = 0
    for k in range(reps):
        a, b = wins[(start + k) % len(wins)]
        secs += ref_time_window(ref, cfg.dims, hc, hv, a, b, cfg.targets, workers, cache)
        units += (b - a) * len(cfg.targets)
    if cache.get("ctx"):
        ref.lib.qref_ctx_destroy(cache["ctx"])
    return units / secs / 1e6, secs, units


def host_input(cfg, nnz):
    """The workload's bytes on the host (generated on the device when one is
    present, so both arms see identical bytes)."""
    try:
        import torch
        dev = torch.cuda.is_available()
    except Exception:
        dev = False
    if dev:
        ci, vi = make_input(cfg, nnz, "cuda")
        hc = ci.cpu().numpy().view(np.uint32)
        hv = vi.cpu().numpy()
        del ci, vi
        torch.cuda.empty_cache()
        return hc, hv
    from paper_2005_10427_b200 import synth
    c, v = synth.generate(cfg, nnz)
    return c.view(np.uint32), v


def run_reference(args, cfg, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    the unmodified reference sources compiled in place) on this host."""
    if rank != 0:
        return
    ref = ref_lib()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqref.so not built"}))
        return
    hc, hv = host_input(cfg, args.nnz)
    n = len(hv)
    workers = os.cpu_count() or 1
    rows = min(n, args.ref_window)
    nwin = len(ref_windows(n, rows))
    ref_sample(ref, cfg, hc, hv, rows, workers, args.warmup, start=nwin // 2)
    v, secs, units = ref_sample(ref, cfg, hc, hv, rows, workers, args.steps)
    # serial path (workers = 1, sort.cpp) on a smaller window
    srows = max(1, min(n, rows // 16))
    sv, ssecs, sunits = ref_sample(ref, cfg, hc, hv, srows, 1, 2)
    full = None
    # one full-size run per target when the host can hold the tensor, the
    # reference's working copy, its Workspace and the pristine bytes
    need = n * (4 * len(cfg.dims) + 8) * 3 + n * 12 + (1 << 30)
    if rows < n and not args.no_ref_full:
        if avail_ram() > need:
            cache = {}
            per = {}
            for t in cfg.targets:
                s = ref_time_window(ref, cfg.dims, hc, hv, 0, n, [t], workers, cache)
                per[tname(t)] = {"s": round(s, 3), "Mnnz_s": round(n / s / 1e6, 2)}
            ref.lib.qref_ctx_destroy(cache["ctx"])
            tot = sum(x["s"] for x in per.values())
            full = {"Mnnz_s": round(n * len(cfg.targets) / tot / 1e6, 3), "per_target": per,
                    "workers": workers, "reps": 1}
        else:
            full = {"value": None,
                    "reason": f"not run (RAM: {avail_ram() / 2**30:.0f} GiB available, "
                              f"{need / 2**30:.0f} GiB needed)"}
    elif rows >= n:
        full = {"note": "the sample windows are the whole tensor"}
    hi = host_info()
    sample = (f"{args.steps} steps, each one contiguous window of {rows} rows of the "
              f"{n}-row tensor (windows advance each step; {nwin} windows) transposed to "
              f"{len(cfg.targets)} targets by the reference transpose_inplace (Quesadilla, "
              f"std::thread workers = {workers}); pristine restore untimed")
    print(json.dumps({
        "impl": "reference", "metric": "nonzeros transposed/sec (Mnnz/s)", "value": round(v, 3),
        "unit": "Mnnz/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 coords + f64 values",
        "data": "synthetic (same seeded bytes as the GPU arm)",
        "config": workload_config(cfg, n),
        "cpu_baseline": {"value": round(v, 3), "unit": "Mnnz/s", "cores": workers,
                         "kind": "reference", "sample": sample,
                         "parallel": {"value": round(v, 3), "workers": workers,
                                      "rows_per_step": rows},
                         "serial": {"value": round(sv, 3), "workers": 1,
                                    "sample": f"2 windows of {srows} rows x {len(cfg.targets)} "
                                              "targets (sort.cpp serial path)"},
                         "full_size": full, **hi},
        "e2e": {"value": round(v, 3), "unit": "Mnnz/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def cpu_baseline(cfg, hc, hv):
    """Reference library (oracle/_ref) on this host, bounded samples of the
    same tensor: parallel (all cores) and serial (workers = 1)."""
    try:
        ref = ref_lib()
    except Exception:
        ref = None
    if ref is None:
        return None
    n = len(hv)
    workers = os.cpu_count() or 1
    # windows from the middle of the tensor, as the reference arm takes them
    # (the first rows of a Zipf tensor are one giant mode-0 run, on which the
    # reference's bucketed parallel sort has a single worker)
    prow = min(n, 1 << 26)
    pv, _, _ = ref_sample(ref, cfg, hc, hv, prow, workers, 2,
                          start=len(ref_windows(n, prow)) // 2)
    srow = min(n, 1 << 22)
    sv, _, _ = ref_sample(ref, cfg, hc, hv, srow, 1, 2, start=len(ref_windows(n, srow)) // 2)
    return {"value": round(pv, 3), "unit": "Mnnz/s", "cores": workers, "kind": "reference",
            "sample": f"2 contiguous windows of {prow} rows from the middle of the same tensor x "
                      f"{len(cfg.targets)} targets, reference transpose_inplace (Quesadilla, "
                      f"std::thread workers = {workers})",
            "parallel": {"value": round(pv, 3), "workers": workers, "rows": prow},
            "serial": {"value": round(sv, 3), "workers": 1, "rows": srow,
                       "sample": "2 windows from the middle, sort.cpp serial path"},
            **host_info()}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    args = parse_args()
    from paper_2005_10427_b200 import synth
    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, cfg, rank)

    import torch
    import paper_2005_10427_b200 as qd
    torch.cuda.set_device(local)
    if world > 1 or os.environ.get("QD_FORCE_SHARDED"):
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2005_10427_b200 import shard
        return shard.bench_sharded(args, cfg, dist, rank, world, local)

    t_gen = time.perf_counter()
    ci, vi = make_input(cfg, args.nnz, "cuda")
    t_gen = time.perf_counter() - t_gen
    n = vi.numel()
    r = len(cfg.dims)
    co = torch.empty_like(ci)
    vo = torch.empty_like(vi)
    ws = qd.Workspace(local)
    # a created (non-default) stream: the library captures latency-mode calls
    # (tensors up to 2^24 rows) into CUDA graphs, which the legacy default
    # stream cannot do
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    strat = qd.SortStrategy.quesadilla()

    def one(t):
        qd.transpose_device(r, cfg.dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                            vo.data_ptr(), t, strat, ws, sp)

    def step():
        for t in cfg.targets:
            one(t)

    for _ in range(args.warmup):
        step()
    # the output of every target: sorted under it, and the same row multiset
    checks = {}
    if not os.environ.get("QD_SCATTER_DBG"):  # experiment switch: stores skipped
        h_in = row_checksum_device(ci, vi, r)
        for t in cfg.targets:
            one(t)
            ok_sorted = qd.is_sorted_device(r, n, co.data_ptr(), t, ws, sp)
            ok_rows = row_checksum_device(co, vo, r) == h_in
            assert ok_sorted and ok_rows, (t, ok_sorted, ok_rows)
            checks[tname(t)] = "sorted under target; row-multiset checksum equal"

    # timed region 1 (value): exactly K steps, library profiling off
    l0 = ws.launches()
    torch.cuda.synchronize()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        marks[0].record(stream)
        for k in range(args.steps):
            step()
            marks[k + 1].record(stream)
        torch.cuda.synchronize()
    ms = marks[0].elapsed_time(marks[-1])
    per_step = sorted(marks[k].elapsed_time(marks[k + 1]) for k in range(args.steps))
    launches = ws.launches() - l0
    units = n * len(cfg.targets) * args.steps
    value = units / (ms / 1e3) / 1e6

    # timed region 2 (roofline): the same K steps with the library's CUDA
    # events around every kernel on its launch stream (per-class durations)
    ws.profile(True)
    ws.profile_reset()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    ms_prof = p0.elapsed_time(p1)
    prof = ws.profile_stats()
    ws.profile(False)

    top = max(("scatter", "local", "hist"), key=lambda k: prof[k]["ms"])
    p = prof[top]
    peak, peak_kind = peaks()
    achieved = (p["bytes"] / p["launches"]) / (p["ms"] / p["launches"] / 1e3) / 1e9 if p["ms"] else 0
    tr = ncu_traffic()
    traffic = None
    if tr and tr.get("kernel_class") == top and p["launches"]:
        rows_per_launch = p["bytes"] / p["launches"] / (2 * (4 * r + 8))
        traffic = round(tr["dram_bytes_per_row"] * rows_per_launch)
    step_ms = ms_prof / args.steps
    share = {k: round(v["ms"] / args.steps / step_ms, 4) for k, v in prof.items()}

    # per-target device time (min of 3) and the SURVEY §8(d) byte-model
    # roofline fraction of each
    per_target = {}
    model_bytes = 0
    for t in cfg.targets:
        tms = []
        for _ in range(3):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            one(t)
            a1.record(stream)
            torch.cuda.synchronize()
            tms.append(a0.elapsed_time(a1))
        tm = min(tms)
        mb = survey_bytes(cfg.dims, t, n)
        model_bytes += mb
        lb = n * (2 * (4 * r + 8) + 4 * len(qd.quesadilla_plan(t).steps))
        per_target["".join(str(x) for x in t)] = {
            "ms": round(tm, 4), "Mnnz_s": round(n / tm / 1e3, 1),
            "model_GB": round(mb / 1e9, 3),
            "model_frac": round(mb / (tm / 1e3) / 1e9 / peak, 4),
            "model_frac_nominal_8TBs": round(mb / (tm / 1e3) / 1e9 / 8000.0, 4),
            "lowerbound_frac": round(lb / (tm / 1e3) / 1e9 / peak, 4)}

    # host copy of the input (pinned) for e2e and the CPU baseline
    need_host = n * (4 * r + 8) * 2
    e2e = None
    hc0 = hv0 = None
    if not (args.no_e2e and args.no_cpu_baseline):
        pc = torch.empty(ci.shape, dtype=torch.int32, pin_memory=True)
        pv = torch.empty(vi.shape, dtype=torch.float64, pin_memory=True)
        pc.copy_(ci)
        pv.copy_(vi)
        hc0, hv0 = pc.numpy().view(np.uint32), pv.numpy()
    # the device-resident tensors are released: the host-buffer call stages
    # its own device copies (34.8 GB in + 34.8 GB out at c5)
    del ci, vi, co, vo
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    if not args.no_e2e and avail_ram() > need_host // 2:
        e2e = run_e2e(args, cfg, qd, ws, hc0, hv0, r, n)

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, hc0, hv0)

    out = {
        "metric": "nonzeros transposed/sec (Mnnz/s)", "value": round(value, 3), "unit": "Mnnz/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "ms_per_step_min": round(per_step[0], 4),
        "ms_per_step_median": round(per_step[len(per_step) // 2], 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 coords + f64 values (moved, not computed)",
        "data": f"synthetic (seeded {cfg.dist[0]} stand-in; FROSTT files unavailable offline; "
                f"generated on the device in {t_gen:.1f} s)",
        "config": workload_config(cfg, n),
        "checks": checks,
        "roofline": {"bound": "hbm", "kernel": {"scatter": "k_scatter", "local": "k_local",
                                                "hist": "k_chunk_hist"}[top],
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "launches": p["launches"],
                     "bytes_per_launch": round(p["bytes"] / max(1, p["launches"])),
                     "avg_launch_us": round(p["ms"] / max(1, p["launches"]) * 1e3, 2),
                     "step_share": share,
                     "timing": "second timed region of the same K steps with the library's "
                               "per-kernel CUDA events (ms_per_step there: %.4f)" % step_ms},
        "model_roofline": {"note": "SURVEY.md §8(d) B_total byte model per step over the "
                                   "targets; per target: min of 3 event-timed calls",
                           "bytes_per_step": model_bytes,
                           "achieved_GBs": round(model_bytes / (ms / args.steps / 1e3) / 1e9, 1),
                           "frac": round(model_bytes / (ms / args.steps / 1e3) / 1e9 / peak, 4),
                           "frac_nominal_8TBs": round(
                               model_bytes / (ms / args.steps / 1e3) / 1e9 / 8000.0, 4),
                           "per_target": per_target},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))


def run_e2e(args, cfg, qd, ws, hc0, hv0, r, n):
    """End to end through the reference-facing host call: qd_transpose_inplace
    on pinned host buffers (transpose_inplace's signature; synchronous), one
    call per target per step, the tensor's bytes refreshed from the pristine
    copy before every call (untimed: the call is in place).  Host wall clock
    around each call: H2D + device passes + D2H."""
    import torch
    k_e2e = max(1, min(args.steps, 2 if n > 500_000_000 else 5))
    wc = torch.empty(hc0.shape, dtype=torch.int32, pin_memory=True)
    wv = torch.empty(hv0.shape, dtype=torch.float64, pin_memory=True)
    hc, hv = wc.numpy().view(np.uint32), wv.numpy()
    tens = qd.CooTensor(cfg.dims, hc, hv)  # wraps the pinned buffers
    strat = qd.SortStrategy.quesadilla()
    secs = 0.0
    per_t = {tname(t): {"ms": 0.0, "slices": 1} for t in cfg.targets}
    step_ms = []  # each timed step's total (the host link of a shared box is noisy)
    for it in range(1 + k_e2e):  # one untimed warm-up step (workspace growth)
        if it:
            step_ms.append(0.0)
        for t in cfg.targets:
            wc.copy_(torch.from_numpy(hc0.view(np.int32)))
            wv.copy_(torch.from_numpy(hv0))
            t0 = time.perf_counter()
            qd.transpose_inplace(tens, t, strat, ws)
            dt = time.perf_counter() - t0
            if it:
                secs += dt
                step_ms[-1] += dt * 1e3
                per_t[tname(t)]["ms"] += dt * 1e3 / k_e2e
                # > 1: the call kept the leading mode, so the library cut the tensor
                # where it changes and pipelined H2D / passes / D2H per slice
                per_t[tname(t)]["slices"] = ws.slices()
    for v in per_t.values():
        v["ms"] = round(v["ms"], 2)
    last = hc.reshape(-1, r)
    m = min(len(last), 1 << 21)
    for a in (0, len(last) - m):  # spot check: host output sorted under the last target
        blk = last[a:a + m]
        key = np.lexsort(tuple(blk[:, j] for j in reversed(cfg.targets[-1])))
        assert np.array_equal(key, np.arange(len(key))), "e2e output not sorted"
    del tens, wc, wv
    # the same call on PAGEABLE host buffers (the C++ drop-in's std::vector):
    # one step, staged through the library's pinned chunk ring
    pageable = None
    if avail_ram() > n * (4 * r + 8) * 2:
        pc_ = np.empty(hc0.shape, np.uint32)
        pv_ = np.empty(hv0.shape, np.float64)
        ptens = qd.CooTensor(cfg.dims, pc_, pv_)
        psecs = 0.0
        for t in cfg.targets:
            np.copyto(pc_, hc0)
            np.copyto(pv_, hv0)
            t0 = time.perf_counter()
            qd.transpose_inplace(ptens, t, strat, ws)
            psecs += time.perf_counter() - t0
        pageable = {"value": round(n * len(cfg.targets) / psecs / 1e6, 3),
                    "ms_per_step": round(psecs * 1e3, 2), "steps": 1,
                    "api": "qd_transpose_inplace (pageable host buffers) x targets"}
        del ptens, pc_, pv_
    per = n * (4 * r + 8) * len(cfg.targets)
    return {"value": round(n * len(cfg.targets) * k_e2e / secs / 1e6, 3), "unit": "Mnnz/s",
            "h2d_bytes_per_step": per, "d2h_bytes_per_step": per, "steps": k_e2e,
            "ms_per_step": round(secs / k_e2e * 1e3, 2),
            "timing": "host wall clock around each synchronous call (every H2D/D2H byte "
                      "inside), summed over the step's targets",
            "api": "qd_transpose_inplace (pinned host buffers) x targets",
            "per_target": per_t,
            "steps_ms": [round(x, 1) for x in step_ms],
            "pageable": pageable}


if __name__ == "__main__":
    main()
