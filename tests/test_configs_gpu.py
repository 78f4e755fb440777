"""BASELINE.json configurations at their full sizes on the GPU, against the
reference library itself (oracle/_ref, std::thread workers) on the same bytes,
plus size-independent properties where the full reference run is too large
(config 5: sortedness, row-multiset checksum, and the sharded oracle of
SURVEY.md §8c — the output slice with sigma1 in a value range equals the
reference transpose of the input rows with sigma1 in that range)."""
import os

import numpy as np
import pytest

import paper_2005_10427_b200 as qd
from paper_2005_10427_b200 import synth
from pyoracle import Reference, reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]

WORKERS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def ws():
    w = qd.Workspace(0)
    yield w
    w.close()


def device_transpose(ws, dims, ci, vi, target):
    import torch
    co, vo = torch.empty_like(ci), torch.empty_like(vi)
    qd.transpose_device(len(dims), dims, vi.numel(), ci.data_ptr(), vi.data_ptr(), co.data_ptr(),
                        vo.data_ptr(), target, qd.SortStrategy.quesadilla(), ws,
                        torch.cuda.current_stream().cuda_stream)
    return co, vo


def row_hash(c: np.ndarray, v: np.ndarray, r: int) -> int:
    """Order-independent checksum of the (coords, value bits) row multiset."""
    x = v.view(np.uint64).copy()
    cc = c.reshape(-1, r).astype(np.uint64)
    for m in range(r):
        x ^= (cc[:, m] + np.uint64(0x9E3779B97F4A7C15 * (m + 1) & 0xFFFFFFFFFFFFFFFF)) * \
            np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(29))) * np.uint64(0x94D049BB133111EB)
    return int(np.bitwise_xor.reduce(x)) ^ int(x.sum(dtype=np.uint64))


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_full_size_vs_reference(ws, name):
    cfg = synth.CONFIGS[name]
    ci, vi = synth.generate_torch(cfg)
    hc = ci.cpu().numpy().view(np.uint32)
    hv = vi.cpu().numpy()
    ref = Reference()
    for target in cfg.targets:
        co, vo = device_transpose(ws, cfg.dims, ci, vi, target)
        rc, rv, _ = ref.transpose(cfg.dims, hc, hv, target, workers=WORKERS)
        assert np.array_equal(co.cpu().numpy().view(np.uint32), rc), (name, target)
        assert np.array_equal(vo.cpu().numpy().view(np.uint64), rv.view(np.uint64)), (name, target)
        del co, vo


def test_config5_properties_and_sharded_oracle(ws):
    """Config 5's shape and distribution (Zipf 1.05 over 4821207x1774269x1805187)
    at 200M nonzeros: device sortedness + multiset checksum of the whole output,
    and bit-exact slices against the reference via the sharded oracle."""
    import torch
    cfg = synth.CONFIGS["c5"]
    n = 200_000_000
    ci, vi = synth.generate_torch(cfg, n)
    r = 3
    hc = ci.cpu().numpy().view(np.uint32)
    hv = vi.cpu().numpy()
    h_in = row_hash(hc, hv, r)
    ref = Reference()
    for target in cfg.targets:
        co, vo = device_transpose(ws, cfg.dims, ci, vi, target)
        assert qd.is_sorted_device(r, n, co.data_ptr(), target, ws)
        oc = co.cpu().numpy().view(np.uint32)
        ov = vo.cpu().numpy()
        assert row_hash(oc, ov, r) == h_in
        s1 = target[0]
        key = hc.reshape(-1, r)[:, s1]
        okey = oc.reshape(-1, r)[:, s1]
        for lo, hi in [(0, 1), (1, 40), (5000, 2_000_000)]:
            sel = (key >= lo) & (key < hi)
            rc, rv, _ = ref.transpose(cfg.dims, hc.reshape(-1, r)[sel].ravel(), hv[sel], target,
                                      workers=WORKERS)
            osel = (okey >= lo) & (okey < hi)
            assert np.array_equal(oc.reshape(-1, r)[osel].ravel(), rc), (target, lo, hi)
            assert np.array_equal(ov[osel].view(np.uint64), rv.view(np.uint64))
        del co, vo
    del ci, vi
    torch.cuda.empty_cache()


def test_config5_full_size():
    """BASELINE config 5 at FULL size on one B200 (1,741,809,018 unique
    Zipf(1.05) rows, the bench workload): for both targets the whole output
    is sorted under the target (device check) and holds the input's row
    multiset (device checksum); bit-exact slices against the reference
    library through the sharded oracle: the sigma1 = 0 slice
    (the Zipf head) and one seeded interior sigma1 range."""
    import torch
    sys_path_bench()
    import bench
    cfg = synth.CONFIGS["c5"]
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 150 * 2**30:
        pytest.skip(f"needs ~150 GiB of free device memory ({free / 2**30:.0f} GiB free)")
    w = qd.Workspace(0)
    ci, vi = synth.generate_device(cfg, ws=w)
    n, r = vi.numel(), 3
    assert n == cfg.nnz
    h_in = bench.row_checksum_device(ci, vi, r)
    ref = Reference()
    rng = np.random.default_rng(2026)
    cin = ci.view(n, r)
    try:
        for target in cfg.targets:
            co, vo = device_transpose(w, cfg.dims, ci, vi, target)
            assert qd.is_sorted_device(r, n, co.data_ptr(), target, w)
            assert bench.row_checksum_device(co, vo, r) == h_in, target
            s1 = target[0]
            ocol = co.view(n, r)[:, s1].contiguous()
            lo = int(rng.integers(1000, cfg.dims[s1] // 4))
            for a, b in [(0, 1), (lo, lo + 2000)]:
                sel = (cin[:, s1] >= a) & (cin[:, s1] < b)
                hc = cin[sel].cpu().numpy().view(np.uint32).ravel()
                hv = vi[sel].cpu().numpy()
                del sel
                rc, rv, _ = ref.transpose(cfg.dims, hc, hv, target, workers=WORKERS)
                # the output slice is contiguous: the output is sorted by sigma1
                bnd = torch.tensor([a, b], dtype=torch.int32, device=ocol.device)
                s, e = [int(x) for x in torch.searchsorted(ocol, bnd).cpu()]
                assert e - s == len(hv) > 0, (target, a, b)
                oc = co.view(n, r)[s:e].cpu().numpy().view(np.uint32).ravel()
                ov = vo[s:e].cpu().numpy()
                assert np.array_equal(oc, rc), (target, a, b)
                assert np.array_equal(ov.view(np.uint64), rv.view(np.uint64)), (target, a, b)
                del hc, hv, rc, rv, oc, ov
            del co, vo, ocol
            torch.cuda.empty_cache()
    finally:
        del ci, vi, cin
        w.close()
        torch.cuda.empty_cache()


def sys_path_bench():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
