"""Alternating whole-tensor ((1,0,2)) and sliced ((0,2,1)) host-buffer calls on config 5 (pinned
buffers): wall clock per call; QD_HOST_DBG=1 prints the phases.  python profiles/r2/e2e_alternate.py"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2005_10427_b200 as qd
from paper_2005_10427_b200 import synth
cfg = synth.CONFIGS["c5"]
ci, vi = synth.generate_device(cfg, cfg.nnz, device="cuda")
n = vi.numel()
pc = torch.empty(ci.shape, dtype=torch.int32, pin_memory=True); pv = torch.empty(vi.shape, dtype=torch.float64, pin_memory=True)
wc = torch.empty(ci.shape, dtype=torch.int32, pin_memory=True); wv = torch.empty(vi.shape, dtype=torch.float64, pin_memory=True)
pc.copy_(ci); pv.copy_(vi); del ci, vi; torch.cuda.empty_cache()
ws = qd.Workspace(0)
tens = qd.CooTensor(cfg.dims, wc.numpy().view(np.uint32), wv.numpy())
for t in ("102","102","021","102","021","102","102","021","021","102"):
    wc.copy_(pc); wv.copy_(pv)
    t0 = time.perf_counter()
    qd.transpose_inplace(tens, [int(ch) for ch in t], qd.SortStrategy.quesadilla(), ws)
    print(t, round((time.perf_counter()-t0)*1e3,1), "ms", ws.slices(), flush=True)
