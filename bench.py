#!/usr/bin/env python
"""bench.py — Quesadilla COO transposition on B200 (BASELINE.json metric:
nonzeros transposed/sec (Mnnz/s) and achieved HBM GB/s vs roofline).

Workload (BASELINE.json configs[1], the metric's headline config): the
nell-2-shaped 3-order tensor 12092x9184x28818 with 76,879,419 unique Zipf(1.1)
nonzeros (seeded synthetic stand-in, paper_2005_10427_b200/synth.py), input
sorted in (0,1,2).  One STEP = transposing it to all 5 non-identity target
orderings (each through the full Quesadilla plan on the GPU), so one step
moves 5 x 76.9M nonzeros.

  value : whole-job Mnnz/s, inputs resident in HBM, device-timed (CUDA events
          around exactly K steps, max over ranks)
  e2e   : the same metric through the host C-ABI entry (qd_transpose_inplace_async
          + qd_workspace_synchronize on pinned host buffers, one call per target,
          K steps enqueued back to back): every H2D + GPU pass + D2H inside the
          timed region; the per-step synchronised figure is reported beside it
  roofline : dominant kernel class, algorithmic bytes / its event-timed
          duration (recorded by the library on its launch stream) vs the
          measured HBM copy peak (MEASURED_PEAKS.json)
  cpu_baseline : the reference library itself (oracle/_ref, compiled from the
          reference sources) on this host's cores, one full step

--impl reference times the reference's own CPU implementation (oracle/_ref,
std::thread workers = all host cores) on the same workload and prints the same
JSON line with "impl": "reference".
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
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c2")
    p.add_argument("--nnz", type=int, default=None, help="override nnz (testing only)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
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
    """dram bytes per row moved by k_onesweep from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_input(cfg, nnz, device):
    from paper_2005_10427_b200 import synth
    if device is not None:
        return synth.generate_torch(cfg, nnz, device=device)
    c, v = synth.generate(cfg, nnz)
    return c.view(np.int32), v


def reference_step(ref, ctx, hc, hv, targets, workers):
    """Reference transpose_inplace for every target; returns seconds (sum)."""
    import ctypes as C
    tot = 0.0
    for t in targets:
        ref.lib.qref_ctx_reset(ctx, hc, hv)
        ta = np.asarray(t, np.uint32)
        t0 = time.perf_counter()
        s = ref.lib.qref_ctx_transpose(ctx, ta, workers)
        tot += time.perf_counter() - t0
        if s:
            raise RuntimeError(ref.lib.qref_last_error().decode())
    return tot


def run_reference(args, cfg, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference, reference_available
    import ctypes as C
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqref.so not built"}))
        return
    try:
        import torch
        dev = "cuda" if torch.cuda.is_available() else None
    except Exception:
        dev = None
    ci, vi = make_input(cfg, args.nnz, dev)
    hc = np.ascontiguousarray(ci.cpu().numpy() if dev else ci).view(np.uint32)
    hv = np.ascontiguousarray(vi.cpu().numpy() if dev else vi)
    del ci, vi
    n = len(hv)
    ref = Reference()
    workers = os.cpu_count() or 1
    dims = np.asarray(cfg.dims, np.uint32)
    ctx = ref.lib.qref_ctx_create(len(dims), dims, n, hc, hv)
    for _ in range(args.warmup):
        reference_step(ref, ctx, hc, hv, cfg.targets, workers)
    secs = sum(reference_step(ref, ctx, hc, hv, cfg.targets, workers) for _ in range(args.steps))
    ref.lib.qref_ctx_destroy(ctx)
    units = n * len(cfg.targets) * args.steps
    v = units / secs / 1e6
    print(json.dumps({
        "impl": "reference", "metric": "nonzeros transposed/sec (Mnnz/s)", "value": round(v, 3),
        "unit": "Mnnz/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64", "data": "synthetic",
        "config": workload_config(cfg, n),
        "cpu_baseline": {"value": round(v, 3), "unit": "Mnnz/s", "cores": workers,
                         "kind": "reference",
                         "sample": f"full workload: {len(cfg.targets)} targets x {n} nnz per step, "
                                   "reference transpose_inplace (Quesadilla, std::thread workers)"},
        "e2e": {"value": round(v, 3), "unit": "Mnnz/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


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


def workload_config(cfg, n, world=1):
    return {"workload": f"{cfg.name}: {'x'.join(map(str, cfg.dims))}, {n} unique nnz "
                        f"({cfg.dist[0]} s={cfg.s}), targets "
                        + " ".join("(" + ",".join(map(str, t)) + ")" for t in cfg.targets),
            "nnz": n, "rank": len(cfg.dims), "targets_per_step": len(cfg.targets),
            "parallelism": f"shard{world}" if world > 1 else "single-gpu",
            "l2": "inputs (>= 1.5 GB) larger than the 126 MB L2; no flush needed"}


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
    dist = None
    if world > 1 or os.environ.get("QD_FORCE_SHARDED"):
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2005_10427_b200 import shard
        return shard.bench_sharded(args, cfg, dist, rank, world, local)

    ci, vi = make_input(cfg, args.nnz, "cuda")
    n = vi.numel()
    r = len(cfg.dims)
    co = torch.empty_like(ci)
    vo = torch.empty_like(vi)
    ws = qd.Workspace(local)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step():
        for t in cfg.targets:
            qd.transpose_device(r, cfg.dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                                vo.data_ptr(), t, qd.SortStrategy.quesadilla(), ws, sp)

    for _ in range(args.warmup):
        step()
    # sanity: the last target's output is sorted under it (device check)
    if not os.environ.get("QD_SCATTER_DBG"):  # experiment switch: stores skipped
        assert qd.is_sorted_device(r, n, co.data_ptr(), cfg.targets[-1], ws, sp)

    # timed region 1 (value): exactly K steps, library profiling off
    l0 = ws.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        e0.record(stream)
        marks[0].record(stream)
        for k in range(args.steps):
            step()
            marks[k + 1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    per_step = sorted(marks[k].elapsed_time(marks[k + 1]) for k in range(args.steps))
    launches = ws.launches() - l0
    units = n * len(cfg.targets) * args.steps
    value = units / (ms / 1e3) / 1e6

    # timed region 2 (roofline): the same K steps with the library's CUDA
    # events around every kernel on its launch stream (per-class durations);
    # the events add ~6 % to the step, so they stay out of region 1
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

    # roofline of the dominant kernel class
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

    # per-target device time (one extra untimed-for-value round) and the
    # SURVEY §8(d) byte-model roofline fraction of each
    per_target = {}
    model_bytes = 0
    for t in cfg.targets:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        qd.transpose_device(r, cfg.dims, n, ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                            vo.data_ptr(), t, qd.SortStrategy.quesadilla(), ws, sp)
        a1.record(stream)
        torch.cuda.synchronize()
        tms = a0.elapsed_time(a1)
        mb = survey_bytes(cfg.dims, t, n)
        model_bytes += mb
        per_target["".join(str(x) for x in t)] = {
            "ms": round(tms, 4), "Mnnz_s": round(n / tms / 1e3, 1),
            "model_GB": round(mb / 1e9, 3),
            "model_frac": round(mb / (tms / 1e3) / 1e9 / peaks()[0], 4)}

    # end to end through the host C-ABI entry, pinned host buffers: every
    # step transposes a fresh host copy of the input to each target with
    # qd_transpose_inplace_async (one call per target, as the reference CLI's
    # bench loop makes) and waits for the last output copy; the input copy of
    # call i+1 overlaps the output copy of call i (full-duplex PCIe).  Wall
    # clock around the whole step: H2D + device work + D2H of all targets.
    e2e = None
    if not args.no_e2e:
        # K steps, each step = one async call per target on its own pinned
        # host copy of the input (25 buffer pairs for K = 5: the in-place API
        # overwrites its input, so every call of the timed region needs fresh
        # host bytes).  The K steps are enqueued back to back and waited for
        # once: consecutive steps overlap their copies like consecutive
        # targets do (a stream of tensors through the API).  The per-step
        # synchronised figure (wait after every step) is reported beside it.
        hc0 = ci.cpu().numpy().view(np.uint32)
        hv0 = vi.cpu().numpy()
        # K = 5 steps (fewer when the host lacks the RAM for 5 x targets
        # pinned input copies, leaving half of it free)
        step_bytes = n * (4 * r + 8) * len(cfg.targets)
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 0
        k_e2e = max(1, min(args.steps, 5, int(avail // 2 // max(1, step_bytes))))
        pins = [(torch.empty(hc0.shape, dtype=torch.int32).pin_memory(),
                 torch.empty(hv0.shape, dtype=torch.float64).pin_memory())
                for _ in range(k_e2e * len(cfg.targets))]
        bufs = [(pc.numpy().view(np.uint32), pv.numpy()) for pc, pv in pins]

        def fill(bs):
            tens = []
            for hc, hv in bs:
                np.copyto(hc, hc0)
                np.copyto(hv, hv0)
                tens.append(qd.CooTensor(cfg.dims, hc, hv))  # wraps the pinned buffers
            return tens

        nt = len(cfg.targets)
        sync_s = 0.0
        warm = 2  # both async device slots grow during warm-up
        for it in range(warm + k_e2e):
            tens = fill(bufs[:nt])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for tn, t in zip(tens, cfg.targets):
                qd.transpose_inplace_async(tn, t, qd.SortStrategy.quesadilla(), ws)
            ws.synchronize()
            if it >= warm:
                sync_s += time.perf_counter() - t0
        tens = fill(bufs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j, tn in enumerate(tens):
            qd.transpose_inplace_async(tn, cfg.targets[j % nt], qd.SortStrategy.quesadilla(), ws)
        ws.synchronize()
        pipe_s = time.perf_counter() - t0
        # spot check: the last call's host output is sorted under its target
        last = tens[-1].coords.reshape(-1, r)[:200_000]
        key = np.lexsort(tuple(last[:, m] for m in reversed(cfg.targets[-1])))
        assert np.array_equal(key, np.arange(len(key))), "e2e output not sorted"
        e2e = {"value": round(n * nt * k_e2e / pipe_s / 1e6, 3),
               "unit": "Mnnz/s", "h2d_bytes_per_step": n * (4 * r + 8) * nt,
               "d2h_bytes_per_step": n * (4 * r + 8) * nt,
               "steps": k_e2e, "ms_per_step": round(pipe_s / k_e2e * 1e3, 2),
               "timing": "host wall clock around K steps enqueued back to back "
                         "(every H2D/D2H byte inside), one wait at the end",
               "step_synchronized": {"value": round(n * nt * k_e2e / sync_s / 1e6, 3),
                                     "ms_per_step": round(sync_s / k_e2e * 1e3, 2),
                                     "timing": "wait after every step"},
               "api": "qd_transpose_inplace_async x targets + qd_workspace_synchronize "
                      "(host buffers, pinned)"}
        del pins, bufs, tens

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, ci, vi)

    out = {
        "metric": "nonzeros transposed/sec (Mnnz/s)", "value": round(value, 3), "unit": "Mnnz/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4),
        "ms_per_step_min": round(per_step[0], 4),
        "ms_per_step_median": round(per_step[len(per_step) // 2], 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32 coords + f64 values (moved, not computed)",
        "data": "synthetic (seeded Zipf stand-in for nell-2; FROSTT files unavailable offline)",
        "config": workload_config(cfg, n),
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
        "model_roofline": {"note": "SURVEY.md §8(d) B_total byte model per step over the 5 targets",
                           "bytes_per_step": model_bytes,
                           "achieved_GBs": round(model_bytes / (ms / args.steps / 1e3) / 1e9, 1),
                           "frac": round(model_bytes / (ms / args.steps / 1e3) / 1e9 / peaks()[0], 4),
                           "per_target": per_target},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))


def cpu_baseline(cfg, ci, vi):
    """Reference library (oracle/_ref) on this host: one full step, all cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        from pyoracle import Reference, reference_available
    except Exception:
        return None
    if not reference_available():
        return None
    ref = Reference()
    hc = ci.cpu().numpy().view(np.uint32).copy()
    hv = vi.cpu().numpy().copy()
    n = len(hv)
    dims = np.asarray(cfg.dims, np.uint32)
    workers = os.cpu_count() or 1
    ctx = ref.lib.qref_ctx_create(len(dims), dims, n, hc, hv)
    best = min(reference_step(ref, ctx, hc, hv, cfg.targets, workers) for _ in range(2))
    ref.lib.qref_ctx_destroy(ctx)
    return {"value": round(n * len(cfg.targets) / best / 1e6, 3), "unit": "Mnnz/s",
            "cores": workers, "kind": "reference",
            "sample": f"one full step ({len(cfg.targets)} targets x {n} nnz), min of 2 reps, "
                      "reference transpose_inplace Quesadilla with std::thread workers"}


if __name__ == "__main__":
    main()
