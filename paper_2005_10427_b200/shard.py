"""Multi-GPU transpose: one process per GPU, sharded by the range of the
output's leading mode sigma1.

Every rank holds a contiguous slice of the input rows (the global input is
sorted in the simple order, slices in rank order).  The output of rank g is
the slice of the global output whose sigma1 values fall in rank g's range, so
the concatenation of the rank outputs in rank order is exactly the reference
transpose of the global tensor:

* sigma1 == 0 (the plan's first step is bucketed, e.g. (0,2,1)): the slices
  are already sigma1-aligned when no mode-0 run straddles two ranks
  (``aligned_bounds`` produces such slices) — every rank transposes its own
  rows, no communication (the GPU lift of parallel.cpp:125-139).
* otherwise (e.g. (1,0,2)): one exchange.  Global histogram of sigma1
  (all_reduce of each rank's ``qd_mode_histogram_device``), splitters that
  balance rows at sigma1-value boundaries, a stable device partition of the
  local rows into destination parts (``qd_partition_rows_device``), one
  all_to_all over NCCL/NVLink, and the received parts concatenated in SOURCE
  RANK order — a subsequence of the simply sorted input, hence still simply
  sorted — then the full local Quesadilla plan.
  ``QD_EXCHANGE=p2p`` fuses the partition with the exchange instead: the
  (rank x part) row counts are all-reduced (a world x world matrix), every
  rank's receive buffer lives in symmetric memory (NVLink peer mappings), and
  ``qd_partition_rows_to_peers_device`` writes each part straight into its
  destination rank's buffer at this rank's source-order offset — the same
  bytes as the all_to_all path, with no local partitioned copy and no NCCL
  send/recv (``p2p_layout`` is the offset arithmetic).

The local work goes through a backend: ``GpuBackend`` (the CUDA library) in
the product; tests substitute a CPU backend to check the host logic with
world_size 2 over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


def splitters(hist: np.ndarray, parts: int) -> np.ndarray:
    """Cut sigma1 values 0..dim-1 into `parts` contiguous value ranges with
    balanced row counts; returns part id per sigma1 value (uint32[dim])."""
    hist = np.asarray(hist, np.int64)
    dim = len(hist)
    total = int(hist.sum())
    cum = np.cumsum(hist)
    lookup = np.zeros(dim, np.uint32)
    if total == 0 or parts == 1:
        return lookup
    # value v goes to part floor(rows strictly before v's end * parts / total)
    # using the midpoint of v's rows so an indivisible head value lands once
    mid = cum - hist / 2.0
    lookup[:] = np.minimum(parts - 1, np.floor(mid * parts / total)).astype(np.uint32)
    # monotone by construction (cum is non-decreasing)
    return lookup


def aligned_bounds(mode0: np.ndarray, parts: int) -> List[int]:
    """Row bounds of `parts` contiguous slices of a simply sorted tensor with
    no mode-0 run split across slices (parallel.cpp:125-139)."""
    n = len(mode0)
    b = [0]
    for p in range(1, parts):
        j = n * p // parts
        while 0 < j < n and mode0[j] == mode0[j - 1]:
            j += 1
        b.append(max(j, b[-1]))
    b.append(n)
    return b


@dataclass
class LocalRows:
    """A rank's rows: coords (int32/uint32, n*rank) and values (f64, n) on the
    backend's device."""
    coords: object
    values: object

    def nnz(self) -> int:
        return int(self.values.shape[0])


@dataclass
class SymRows:
    """A rank's symmetric receive buffer: local coords/values views and every
    rank's coords/values base address (valid in this process)."""
    coords: object
    values: object
    peer_c: List[int]
    peer_v: List[int]
    cap: int
    raw: object = None


class GpuBackend:
    """Local work on this rank's GPU through the C ABI."""

    def __init__(self, device: int, ws=None):
        import torch

        import paper_2005_10427_b200 as qd
        self.qd, self.torch = qd, torch
        self.device = torch.device("cuda", device)
        self.ws = ws or qd.Workspace(device)

    def stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def zeros_like_rows(self, n, rank):
        t = self.torch
        return LocalRows(t.empty(n * rank, dtype=t.int32, device=self.device),
                         t.empty(n, dtype=t.float64, device=self.device))

    def mode_hist(self, rows: LocalRows, rank: int, mode: int, dim: int):
        t = self.torch
        h = t.zeros(dim, dtype=t.int64, device=self.device)
        if rows.nnz():
            self.qd.mode_histogram_device(rank, rows.nnz(), rows.coords.data_ptr(), mode, dim,
                                          h.data_ptr(), self.ws, self.stream())
        return h

    def partition(self, rows: LocalRows, rank: int, mode: int, lookup: np.ndarray, parts: int):
        t = self.torch
        out = self.zeros_like_rows(rows.nnz(), rank)
        lk = t.from_numpy(np.ascontiguousarray(lookup).view(np.int32)).to(self.device)
        counts = self.qd.partition_rows_device(rank, rows.nnz(), rows.coords.data_ptr(),
                                               rows.values.data_ptr(), mode, len(lookup),
                                               lk.data_ptr(), parts, out.coords.data_ptr(),
                                               out.values.data_ptr(), self.ws, self.stream())
        return out, counts

    def transpose(self, rows: LocalRows, dims, target) -> LocalRows:
        out = self.zeros_like_rows(rows.nnz(), len(dims))
        if rows.nnz():
            self.qd.transpose_device(len(dims), dims, rows.nnz(), rows.coords.data_ptr(),
                                     rows.values.data_ptr(), out.coords.data_ptr(),
                                     out.values.data_ptr(), target,
                                     self.qd.SortStrategy.quesadilla(), self.ws, self.stream())
        return out

    def symmetric_rows(self, cap: int, rank: int, dist):
        """This rank's receive buffer for `cap` rows and every rank's buffer
        address in this process: torch symmetric memory (NVLink peer
        mappings) on a multi-GPU box, or the test hub's emulation
        (``dist.symmetric_empty``) when ranks are emulated on one GPU.
        Grow-only and cached (cap is the same on every rank)."""
        t = self.torch
        if getattr(self, "_sym", None) is None or self._sym.cap < cap:
            cap2 = max(cap, int((self._sym.cap if getattr(self, "_sym", None) else 0) * 1.25), 1)
            voff = ((cap2 * rank * 4 + 255) // 256) * 256
            nbytes = voff + cap2 * 8
            if hasattr(dist, "symmetric_empty"):
                raw, ptrs = dist.symmetric_empty(nbytes, self.device)
            else:
                import torch.distributed._symmetric_memory as symm_mem
                raw = symm_mem.empty(nbytes, dtype=t.uint8, device=self.device)
                hdl = symm_mem.rendezvous(raw, dist.group.WORLD.group_name)
                ptrs = [int(p) for p in hdl.buffer_ptrs]
            self._sym = SymRows(raw[:cap2 * rank * 4].view(t.int32),
                                raw[voff:voff + cap2 * 8].view(t.float64),
                                list(ptrs), [p + voff for p in ptrs], cap2, raw)
        return self._sym

    def partition_to_peers(self, rows: LocalRows, rank: int, mode: int, lookup: np.ndarray,
                           parts: int, buf, offs):
        t = self.torch
        lk = t.from_numpy(np.ascontiguousarray(lookup).view(np.int32)).to(self.device)
        return self.qd.partition_rows_to_peers_device(
            rank, rows.nnz(), rows.coords.data_ptr(), rows.values.data_ptr(), mode, len(lookup),
            lk.data_ptr(), parts, buf.peer_c, buf.peer_v, offs, self.ws, self.stream())

    def to_numpy_i64(self, h):
        return h.cpu().numpy()

    def synchronize(self):
        self.torch.cuda.synchronize(self.device)

    def from_numpy_i64(self, a):
        return self.torch.from_numpy(np.asarray(a, np.int64)).to(self.device)


def p2p_layout(C: np.ndarray, me: int):
    """C[s, p] = rows source rank s sends to destination p.  Returns the row
    offset of this rank's part p inside destination p's receive buffer (all
    lower source ranks first: source-rank order), this rank's receive count
    and the symmetric buffer capacity (the largest receive count)."""
    C = np.asarray(C, np.int64)
    offs = C[:me, :].sum(0) if me else np.zeros(C.shape[1], np.int64)
    return [int(x) for x in offs], int(C[:, me].sum()), int(C.sum(0).max())


def exchange_p2p(dist, be, rows: LocalRows, rank_modes: int, mode: int, lookup: np.ndarray,
                 local_counts: Sequence[int]) -> LocalRows:
    """Partition fused with the exchange: part p of this rank's rows is
    written by the partition kernel directly into rank p's receive buffer."""
    world, me = dist.get_world_size(), dist.get_rank()
    M = np.zeros((world, world), np.int64)
    M[me] = np.asarray(local_counts, np.int64)
    t = be.from_numpy_i64(M.ravel())
    dist.all_reduce(t)
    C = be.to_numpy_i64(t).reshape(world, world)
    offs, recv, cap = p2p_layout(C, me)
    # every receiver has finished reading its buffer from the previous call
    be.synchronize()
    dist.barrier()
    buf = be.symmetric_rows(cap, rank_modes, dist)
    counts = be.partition_to_peers(rows, rank_modes, mode, lookup, world, buf, offs)
    assert list(counts) == list(M[me]), (counts, M[me])
    # every sender's writes have landed before this rank reads its buffer
    be.synchronize()
    dist.barrier()
    return LocalRows(buf.coords[:recv * rank_modes], buf.values[:recv])


def exchange(dist, be, rows: LocalRows, counts: Sequence[int], rank_modes: int) -> LocalRows:
    """all_to_all of the partitioned rows; part p of every rank goes to rank p
    and the received parts are concatenated in source-rank order."""
    world = dist.get_world_size()
    send = be.from_numpy_i64(np.asarray(counts, np.int64))
    recv = be.from_numpy_i64(np.zeros(world, np.int64))
    dist.all_to_all_single(recv, send)
    rc = [int(x) for x in be.to_numpy_i64(recv)]
    out = be.zeros_like_rows(sum(rc), rank_modes)
    dist.all_to_all_single(out.coords, rows.coords, [c * rank_modes for c in rc],
                           [int(c) * rank_modes for c in counts])
    dist.all_to_all_single(out.values, rows.values, rc, [int(c) for c in counts])
    return out


def exchange_mode() -> str:
    """QD_EXCHANGE: 'nccl' (default: partition + all_to_all) or 'p2p' (the
    partition writes into peer receive buffers)."""
    import os
    m = os.environ.get("QD_EXCHANGE", "nccl").lower()
    if m not in ("nccl", "p2p"):
        raise ValueError(f"QD_EXCHANGE must be nccl or p2p, not {m!r}")
    return m


def sharded_transpose(dist, be, rows: LocalRows, dims: Sequence[int], target: Sequence[int],
                      stats: dict = None):
    """Transpose the global tensor whose rank-ordered slices are `rows`;
    returns this rank's slice of the global output (and whether an exchange
    was needed).  For target[0] == 0 the input slices must be mode-0 aligned
    (see aligned_bounds).  `stats` (optional) receives the exchange's bytes
    sent to other ranks and its host-synchronised duration (SURVEY §8e's
    NVLink reporting)."""
    r = len(dims)
    target = [int(x) for x in target]
    world = dist.get_world_size()
    if world == 1 or target[0] == 0:
        out = be.transpose(rows, dims, target)
        if stats is not None:
            stats.update(sent_bytes=0, exchange_s=0.0, rows_out=out.nnz())
        return out, False
    s1 = target[0]
    h = be.mode_hist(rows, r, s1, dims[s1])
    p2p = exchange_mode() == "p2p"
    h_local = be.to_numpy_i64(h).copy() if p2p else None
    dist.all_reduce(h)
    lookup = splitters(be.to_numpy_i64(h), world)
    if stats is not None:
        import time
        be.synchronize()
        t0 = time.perf_counter()
    if p2p:
        local_counts = np.bincount(lookup, weights=h_local, minlength=world).astype(np.int64)
        recv = exchange_p2p(dist, be, rows, r, s1, lookup, local_counts)
        counts = local_counts
    else:
        parts, counts = be.partition(rows, r, s1, lookup, world)
        recv = exchange(dist, be, parts, counts, r)
    if stats is not None:
        be.synchronize()
        me = dist.get_rank()
        stats.update(sent_bytes=sum(int(c) for p, c in enumerate(counts) if p != me) * (4 * r + 8),
                     exchange_s=time.perf_counter() - t0)
    out = be.transpose(recv, dims, target)
    if stats is not None:
        stats["rows_out"] = out.nnz()
    return out, True


def bench_sharded(args, cfg, dist, rank, world, local):
    """bench.py --gpus N: weak scaling.  Each rank generates its own
    c2-shaped slice with mode-0 values offset by rank, so the global tensor
    (dims[0] * N) x dims[1] x dims[2] is the rank-ordered concatenation, simply
    sorted; every step transposes it to all 5 targets (the (0,2,1) target
    without communication, the others with one all_to_all)."""
    import json
    import time

    import torch

    from paper_2005_10427_b200 import synth
    torch.cuda.set_device(local)
    ci, vi = synth.generate_torch(cfg, args.nnz, seed=cfg.seed + 1000 * rank, device="cuda")
    r = len(cfg.dims)
    dims = list(cfg.dims)
    ci = ci.view(-1, r)
    ci[:, 0] += rank * dims[0]
    ci = ci.reshape(-1).contiguous()
    gdims = [dims[0] * world] + dims[1:]
    be = GpuBackend(local)
    rows = LocalRows(ci, vi)
    n_local = vi.numel()

    def step():
        for t in cfg.targets:
            sharded_transpose(dist, be, rows, gdims, t)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    import bench as B  # the driver-side helpers (clock sampler, peaks)
    l0 = be.ws.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with B.ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    launches = be.ws.launches() - l0
    # roofline: a second region with the library's per-kernel events
    be.ws.profile(True)
    be.ws.profile_reset()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = be.ws.profile_stats()
    be.ws.profile(False)
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total = torch.tensor([n_local], device="cuda", dtype=torch.int64)
    dist.all_reduce(total)

    # SURVEY §8e reporting: one instrumented step (exchange bytes and time,
    # output balance), separate from the timed regions
    ex_bytes = ex_s = 0.0
    imbalance = []
    for t in cfg.targets:
        st = {}
        sharded_transpose(dist, be, rows, gdims, t, stats=st)
        vals = torch.tensor([st["sent_bytes"], st["exchange_s"], st["rows_out"], st["rows_out"]],
                            device="cuda", dtype=torch.float64)
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm)
        ex_bytes += sm[0].item()
        ex_s += mx[1].item()
        imbalance.append(round(mx[2].item() / max(1.0, sm[3].item() / world), 4))

    # end to end: every rank copies its slice in from pinned host memory,
    # runs the sharded transpose and copies its output slice back
    hc = torch.empty(ci.shape, dtype=ci.dtype).pin_memory()
    hv = torch.empty(vi.shape, dtype=vi.dtype).pin_memory()
    hc.copy_(ci)
    hv.copy_(vi)
    dc, dv = torch.empty_like(ci), torch.empty_like(vi)
    # output slices may be larger than the input slice after the exchange
    cap = 2 * n_local + 1024
    oc = torch.empty(cap * r, dtype=ci.dtype).pin_memory()
    ov = torch.empty(cap, dtype=vi.dtype).pin_memory()
    torch.cuda.synchronize()
    dist.barrier()
    k_e2e = max(1, min(args.steps, 3))
    # input copies on s_in into two device slots, output copies on s_out: the
    # output copy of target i overlaps the input copy of target i+1
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    slots = [(dc, dv), (torch.empty_like(ci), torch.empty_like(vi))]
    h2d = d2h = 0
    keep = []
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    k = 0
    for _ in range(k_e2e):
        for t in cfg.targets:
            sc, sv = slots[k % 2]
            k += 1
            with torch.cuda.stream(s_in):
                sc.copy_(hc, non_blocking=True)
                sv.copy_(hv, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_in)
            out, _ = sharded_transpose(dist, be, LocalRows(sc, sv), gdims, t)
            n_out = out.values.numel()
            if n_out > ov.numel():
                oc = torch.empty(n_out * r, dtype=ci.dtype).pin_memory()
                ov = torch.empty(n_out, dtype=vi.dtype).pin_memory()
            s_out.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_out):
                oc[:n_out * r].copy_(out.coords, non_blocking=True)
                ov[:n_out].copy_(out.values, non_blocking=True)
            keep.append(out)
            h2d += sc.numel() * 4 + sv.numel() * 8
            d2h += n_out * (4 * r + 8)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    del keep
    e2e_ms = torch.tensor([wall * 1e3], device="cuda")
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        units = int(total.item()) * len(cfg.targets) * args.steps
        v = units / (ms.item() / 1e3) / 1e6
        top = max(("scatter", "local", "hist"), key=lambda k: prof[k]["ms"])
        p = prof[top]
        peak, peak_kind = B.peaks()
        achieved = (p["bytes"] / p["launches"]) / (p["ms"] / p["launches"] / 1e3) / 1e9 \
            if p["ms"] and p["launches"] else 0.0
        e2e_units = int(total.item()) * len(cfg.targets) * k_e2e
        print(json.dumps({
            "metric": "nonzeros transposed/sec (Mnnz/s)", "value": round(v, 3), "unit": "Mnnz/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms.item() / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "u32 coords + f64 values (moved, not computed)",
            "data": "synthetic (seeded Zipf, per-rank slices of one global tensor)",
            "config": {"workload": f"c2 x {world}: {gdims[0]}x{gdims[1]}x{gdims[2]}, "
                                   f"{int(total.item())} nnz, 5 targets",
                       "parallelism": f"shard{world} (sigma1 ranges; all_to_all over NCCL)",
                       "l2": "inputs larger than L2; no flush needed"},
            "roofline": {"bound": "hbm", "kernel": {"scatter": "k_scatter", "local": "k_local",
                                                    "hist": "k_chunk_hist"}[top],
                         "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "rank": 0},
            "e2e": {"value": round(e2e_units / (e2e_ms.item() / 1e3) / 1e6, 3), "unit": "Mnnz/s",
                    "h2d_bytes_per_step": h2d // k_e2e, "d2h_bytes_per_step": d2h // k_e2e,
                    "note": "rank 0's bytes; every rank moves its own slice; host wall clock, "
                            "max over ranks; output copy of target i overlaps input copy of i+1"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "exchange": {"note": "one instrumented step: all_to_all bytes to other ranks summed "
                                 "over ranks and targets; time = max over ranks per target, host-"
                                 "synchronised around the exchange",
                         "bytes_sent_total": int(ex_bytes), "exchange_ms": round(ex_s * 1e3, 3),
                         "nvlink_GBs_per_rank": (round(ex_bytes / world / ex_s / 1e9, 1)
                                                 if ex_s > 0 else None),
                         "nvlink_frac": (round(ex_bytes / world / ex_s / 1e9 / 900.0, 4)
                                         if ex_s > 0 else None),
                         "imbalance_max_over_mean": dict(zip(
                             ["".join(str(x) for x in t) for t in cfg.targets], imbalance))},
        }))
    dist.destroy_process_group()
