#!/usr/bin/env python
"""A/B driver for experiment switches: runs bench.py (no e2e / cpu baseline)
once per (config, env assignment) and prints value + per-target ms.

  python profiles/r2/ab.py c5,c2 "QD_RANK_MODE=0" "QD_RANK_MODE=1" ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
configs = sys.argv[1].split(",")
variants = sys.argv[2:] or [""]
extra = os.environ.get("AB_ARGS", "--steps 10 --warmup 3").split()
for cfg in configs:
    for var in variants:
        env = dict(os.environ)
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg,
                            "--no-cpu-baseline", "--no-e2e"] + extra, env=env,
                           capture_output=True, text=True)
        line = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if r.returncode or not line:
            print(cfg, var or "-", "FAILED", r.stderr[-800:], flush=True)
            continue
        d = json.loads(line[-1])
        pt = d["model_roofline"]["per_target"]
        sh = d["roofline"]["step_share"]
        print(f"{cfg} {var or '-':28s} {d['value']:10.1f} Mnnz/s {d['ms_per_step']:8.3f} ms/step "
              f"k_scatter frac {d['roofline']['frac']:.3f} model {d['model_roofline']['frac']:.3f} | "
              + " ".join(f"{k}:{v['ms']:.3f}" for k, v in pt.items())
              + " | " + " ".join(f"{k}:{v:.2f}" for k, v in sh.items()), flush=True)
