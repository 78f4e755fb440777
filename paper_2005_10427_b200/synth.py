"""Seeded synthetic COO tensors standing in for the paper's FROSTT inputs
(the datasets are not available offline; BASELINE.json configs 2-5 give the
shapes and value distributions, SURVEY.md §8(d) the generator rules).

* Coordinates are drawn per mode (Zipf(s) over ranks 1..n -> index rank-1,
  uniform, or clustered Gaussian), from numpy's counter-based Philox
  generator keyed by the seed.
* The unique set is the first N distinct coordinate rows in draw order (the
  reference generate()'s Distinct semantics, io.cpp:187-196), topped up with
  more draws when duplicates leave it short.
* Values are U[0,1) (or lognormal(0,1) for the clustered config), drawn per
  accepted row; rows are then sorted into the simple order (0, 1, ..., r-1).

This is harness code (inputs for tests and bench.py), not the measured path.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np


@dataclass
class Config:
    name: str
    dims: List[int]
    nnz: int
    dist: List[str]           # per mode: "zipf", "uniform", "cluster"
    s: float = 1.0            # Zipf exponent
    values: str = "uniform"   # or "lognormal"
    seed: int = 0
    targets: List[List[int]] = field(default_factory=list)
    clusters: int = 0
    sigma: float = 0.0


CONFIGS = {
    "c1": Config("c1", [1000, 1000, 1000], 1_000_000, ["uniform"] * 3, seed=1,
                 targets=[[2, 1, 0]]),
    "c2": Config("c2", [12092, 9184, 28818], 76_879_419, ["zipf"] * 3, s=1.1, seed=2,
                 targets=[[0, 2, 1], [1, 0, 2], [1, 2, 0], [2, 0, 1], [2, 1, 0]]),
    "c3": Config("c3", [532924, 17262471, 2480308, 1443], 140_126_220,
                 ["zipf", "zipf", "zipf", "uniform"], s=1.2, seed=3,
                 targets=[[3, 2, 1, 0], [1, 0, 2, 3], [0, 3, 1, 2]]),
    "c4": Config("c4", [1605, 4198, 1631, 4209, 868131], 1_698_825, ["cluster"] * 5,
                 values="lognormal", seed=4, targets=[[4, 3, 2, 1, 0], [0, 1, 4, 2, 3]],
                 clusters=10_000, sigma=0.02),
    "c5": Config("c5", [4821207, 1774269, 1805187], 1_741_809_018, ["zipf"] * 3, s=1.05,
                 seed=5, targets=[[1, 0, 2], [0, 2, 1]]),
}


def _zipf_cdf(n: int, s: float) -> np.ndarray:
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    c /= c[-1]
    return c


def _bits(d: int) -> int:
    return max(1, int(d - 1).bit_length())


def _draw(cfg: Config, rng: np.random.Generator, m: int, cdfs, centres) -> np.ndarray:
    r = len(cfg.dims)
    out = np.empty((m, r), np.uint32)
    if "cluster" in cfg.dist:
        pick = rng.integers(0, cfg.clusters, m)
    for j, (d, kind) in enumerate(zip(cfg.dims, cfg.dist)):
        if kind == "zipf":
            out[:, j] = np.minimum(np.searchsorted(cdfs[j], rng.random(m), side="right"), d - 1)
        elif kind == "uniform":
            out[:, j] = rng.integers(0, d, m)
        elif kind == "cluster":
            x = centres[pick, j] + rng.normal(0.0, cfg.sigma * d, m)
            out[:, j] = np.clip(np.rint(x), 0, d - 1).astype(np.uint32)
        else:
            raise ValueError(kind)
    return out


def _pack(rows: np.ndarray, dims: Sequence[int]) -> np.ndarray:
    """Lexicographic key (mode 0 most significant); needs sum of bits <= 64."""
    key = np.zeros(len(rows), np.uint64)
    for j, d in enumerate(dims):
        key = (key << np.uint64(_bits(d))) | rows[:, j].astype(np.uint64)
    return key


def generate(cfg: Config, nnz: Optional[int] = None, seed: Optional[int] = None):
    """Returns (coords uint32[N*r], values f64[N]) simply sorted, N unique rows."""
    n = cfg.nnz if nnz is None else int(nnz)
    seed = cfg.seed if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    r = len(cfg.dims)
    cdfs = [(_zipf_cdf(d, cfg.s) if k == "zipf" else None) for d, k in zip(cfg.dims, cfg.dist)]
    centres = None
    if "cluster" in cfg.dist:
        centres = np.stack([rng.uniform(0, d, cfg.clusters) for d in cfg.dims], 1)
    packable = sum(_bits(d) for d in cfg.dims) <= 64
    drawn = []
    total = 0
    m = int(n * 1.25) + 1024
    while True:
        drawn.append(_draw(cfg, rng, m, cdfs, centres))
        total += m
        rows = np.concatenate(drawn) if len(drawn) > 1 else drawn[0]
        if packable:
            _, first = np.unique(_pack(rows, cfg.dims), return_index=True)
        else:
            v = np.ascontiguousarray(rows).view(np.dtype((np.void, 4 * r))).ravel()
            _, first = np.unique(v, return_index=True)
        if len(first) >= n:
            break
        deficit = n - len(first)
        m = int(deficit * max(2.0, total / max(1, len(first)))) + 1024
    chosen = np.sort(first)[:n]            # draw indices of the first n distinct rows
    sel = rows[chosen]
    if cfg.values == "lognormal":
        values = np.exp(rng.normal(0.0, 1.0, n))
    else:
        values = rng.random(n)
    if packable:
        perm = np.argsort(_pack(sel, cfg.dims), kind="stable")
    else:
        perm = np.lexsort(sel.T[::-1])
    sel, values = sel[perm], values[perm]
    return np.ascontiguousarray(sel).reshape(-1), values


def generate_torch(cfg: Config, nnz: Optional[int] = None, seed: Optional[int] = None,
                   device: str = "cuda"):
    """Same rules as generate(), drawn with torch's Philox generator on `device`
    (fast for the 77M-1.7B row configs).  Returns (coords int32 [N*r],
    values float64 [N]) as device tensors.  The stream differs from the numpy
    one, so tests feed the SAME generated bytes to both implementations."""
    import torch

    n = cfg.nnz if nnz is None else int(nnz)
    seed = cfg.seed if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    r = len(cfg.dims)
    cdfs = [torch.from_numpy(_zipf_cdf(d, cfg.s)).to(device) if k == "zipf" else None
            for d, k in zip(cfg.dims, cfg.dist)]
    centres = None
    if "cluster" in cfg.dist:
        centres = torch.stack([torch.rand(cfg.clusters, generator=g, device=device,
                                          dtype=torch.float64) * d for d in cfg.dims], 1)
    prod = 1
    for d in cfg.dims:
        prod *= d
    mixed = prod < 2**63

    def draw(m):
        out = torch.empty((m, r), dtype=torch.int64, device=device)
        if centres is not None:
            pick = torch.randint(0, cfg.clusters, (m,), generator=g, device=device)
        for j, (d, kind) in enumerate(zip(cfg.dims, cfg.dist)):
            if kind == "zipf":
                u = torch.rand(m, generator=g, device=device, dtype=torch.float64)
                out[:, j] = torch.searchsorted(cdfs[j], u, right=True).clamp_(max=d - 1)
            elif kind == "uniform":
                out[:, j] = torch.randint(0, d, (m,), generator=g, device=device)
            else:
                x = centres[pick, j] + torch.randn(m, generator=g, device=device,
                                                   dtype=torch.float64) * (cfg.sigma * d)
                out[:, j] = torch.round(x).clamp_(0, d - 1).to(torch.int64)
        return out

    def lex_order(rows):
        """Stable permutation sorting rows lexicographically (mode 0 first)."""
        if mixed:
            key = torch.zeros(len(rows), dtype=torch.int64, device=device)
            for j, d in enumerate(cfg.dims):
                key = key * d + rows[:, j]
            return torch.sort(key, stable=True).indices, key
        perm = torch.arange(len(rows), device=device)
        for j in reversed(range(r)):
            perm = perm[torch.sort(rows[perm, j], stable=True).indices]
        return perm, None

    rows = draw(int(n * 1.3) + 1024)
    while True:
        perm, key = lex_order(rows)
        s = rows[perm]
        if key is not None:
            ks = key[perm]
            head = torch.ones(len(ks), dtype=torch.bool, device=device)
            head[1:] = ks[1:] != ks[:-1]
        else:
            head = torch.ones(len(s), dtype=torch.bool, device=device)
            head[1:] = (s[1:] != s[:-1]).any(1)
        first = perm[head]          # draw index of each distinct row (stable sort)
        if len(first) >= n:
            break
        rows = torch.cat([rows, draw(int((n - len(first)) * 2) + 1024)])
    chosen = torch.sort(first).values[:n]
    sel = rows[chosen]
    if cfg.values == "lognormal":
        values = torch.randn(n, generator=g, device=device, dtype=torch.float64).exp_()
    else:
        values = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    perm, _ = lex_order(sel)
    sel, values = sel[perm], values[perm]
    return sel.to(torch.int32).reshape(-1).contiguous(), values.contiguous()


def generate_device(cfg: Config, nnz: Optional[int] = None, seed: Optional[int] = None,
                    device: str = "cuda", parts: int = 3, ws=None):
    """Fast seeded generator for the billion-row configs (config 5: 1.74B
    unique Zipf(1.05) rows in ~3 s on one B200), device-resident throughout.

    * ~1.5 N coordinate rows are drawn per mode from torch's Philox generator
      (Zipf by inverse CDF, as generate_torch);
    * the draws are canonicalised (simple order) and deduplicated in `parts`
      ranges of mode 0 (cut at sampled quantiles, so each range's sort fits
      beside the draws), each with the library's stable device sort
      (``sort_rows_by_device``, the engine's segmented sort — the same one the
      .tns reader canonicalises with); the ranges concatenate in order;
    * exactly N of the unique rows are kept by a seeded uniform subset (a
      subsequence of a sorted list stays sorted) and values U[0,1) are drawn
      per kept row.

    The unique set differs from generate()'s first-N-distinct-in-draw-order
    rule (a uniform N-subset of the distinct draws instead); both are seeded
    and deterministic, and every consumer (bench arms, tests) uses the same
    bytes.  Only "zipf"/"uniform" modes and uniform values are supported.
    Returns (coords int32 [N*r], values float64 [N]) on `device`."""
    import torch

    import paper_2005_10427_b200 as qd

    if any(k not in ("zipf", "uniform") for k in cfg.dist) or cfg.values != "uniform":
        raise ValueError("generate_device supports zipf/uniform modes with U[0,1) values")
    n = cfg.nnz if nnz is None else int(nnz)
    seed = cfg.seed if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    r = len(cfg.dims)
    m = int(n * 1.5) + 1024
    raw = torch.empty((m, r), dtype=torch.int32, device=device)
    step = 1 << 28
    for j, (d, kind) in enumerate(zip(cfg.dims, cfg.dist)):
        cdf = torch.from_numpy(_zipf_cdf(d, cfg.s)).to(device) if kind == "zipf" else None
        for a in range(0, m, step):
            b = min(m, a + step)
            if kind == "zipf":
                u = torch.rand(b - a, generator=g, device=device, dtype=torch.float64)
                raw[a:b, j] = torch.searchsorted(cdf, u, right=True).clamp_(max=d - 1).to(torch.int32)
                del u
            else:
                raw[a:b, j] = torch.randint(0, d, (b - a,), generator=g, device=device,
                                            dtype=torch.int32)
        del cdf
    smp = raw[: 1 << 24, 0].double().sort().values
    cuts = [0] + [int(smp[k * len(smp) // parts].item()) + 1 for k in range(1, parts)] + [2**31 - 1]
    del smp
    own_ws = ws is None
    ws = ws or qd.Workspace(torch.device(device).index or 0)
    sp = torch.cuda.current_stream().cuda_stream
    uniq = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        if hi <= lo:
            continue
        sel = (raw[:, 0] >= lo) & (raw[:, 0] < hi)
        part = raw[sel].reshape(-1).contiguous()
        del sel
        k = part.numel() // r
        if k == 0:
            continue
        dummy = torch.zeros(k, dtype=torch.float64, device=device)
        po = torch.empty_like(part)
        pv = torch.empty_like(dummy)
        qd.sort_rows_by_device(r, cfg.dims, k, part.data_ptr(), dummy.data_ptr(), po.data_ptr(),
                               pv.data_ptr(), 0, k, list(range(r)), ws, sp)
        torch.cuda.synchronize()
        del part, dummy, pv
        s = po.view(k, r)
        head = torch.ones(k, dtype=torch.bool, device=device)
        head[1:] = (s[1:] != s[:-1]).any(1)
        uniq.append(s[head])
        del s, po, head
        torch.cuda.empty_cache()
    del raw
    if own_ws:
        ws.close()
    torch.cuda.empty_cache()
    u = sum(x.shape[0] for x in uniq)
    if u < n:
        raise RuntimeError(f"generate_device: only {u} unique rows drawn for {n}")
    # a seeded uniform N-subset in order (torch.randperm stalls at this size)
    keep = torch.rand(u, generator=g, device=device, dtype=torch.float64).argsort()[:n].sort().values
    ci = torch.cat(uniq)[keep].reshape(-1).contiguous()
    del uniq, keep
    vi = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return ci, vi
