"""The sliced host-buffer call on config 5's (0,2,1) (and the whole-tensor
call with QD_SLICE_ROWS=0 beside it): wall clock per call and, with
QD_HOST_DBG=1, the per-slice timeline.  python profiles/r2/e2e_sliced.py [reps]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2005_10427_b200 as qd  # noqa: E402
from paper_2005_10427_b200 import synth  # noqa: E402

cfg = synth.CONFIGS["c5"]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(os.environ.get("NNZ", cfg.nnz))
ci, vi = synth.generate_device(cfg, n, device="cuda")
n = vi.numel()
pc = torch.empty(ci.shape, dtype=torch.int32, pin_memory=True)
pv = torch.empty(vi.shape, dtype=torch.float64, pin_memory=True)
wc = torch.empty(ci.shape, dtype=torch.int32, pin_memory=True)
wv = torch.empty(vi.shape, dtype=torch.float64, pin_memory=True)
pc.copy_(ci)
pv.copy_(vi)
del ci, vi
torch.cuda.empty_cache()
ws = qd.Workspace(0)
tens = qd.CooTensor(cfg.dims, wc.numpy().view(np.uint32), wv.numpy())
PAGEABLE = os.environ.get("PAGEABLE")
if PAGEABLE:
    wc, wv = torch.empty(wc.shape, dtype=torch.int32), torch.empty(wv.shape, dtype=torch.float64)
    tens = qd.CooTensor(cfg.dims, wc.numpy().view(np.uint32), wv.numpy())
for env in ((None, "0", None) if os.environ.get("FIRST_SLICED") else ("0", None, "0", None)):
    if env is None:
        os.environ.pop("QD_SLICE_ROWS", None)
    else:
        os.environ["QD_SLICE_ROWS"] = env
    for it in range(reps):
        wc.copy_(pc)
        wv.copy_(pv)
        t0 = time.perf_counter()
        qd.transpose_inplace(tens, [int(ch) for ch in os.environ.get("TARGET", "021")], qd.SortStrategy.quesadilla(), ws)
        dt = time.perf_counter() - t0
        print(f"QD_SLICE_ROWS={env}: {ws.slices()} slices, {dt * 1e3:.1f} ms, "
              f"{n / dt / 1e6:.1f} Mnnz/s", flush=True)
