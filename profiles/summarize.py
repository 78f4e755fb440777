"""Summarise the raw outputs of profiles/refresh.sh (in gpurun_out/) into the
tracked round files under profiles/:

  r<N>_bench_line.json      the bench.py JSON line (value, roofline, e2e, ...)
  r<N>_reference_arm.json   bench.py --impl reference
  r<N>_launches.csv         ncu launch list (gpu__time_duration.sum per launch)
  r<N>_launches_summary.txt per-step time by kernel (cold-cache, serialised)
  r<N>_ncu_full_summary.txt ncu --set full metrics + top stall reasons per launch
  ncu_traffic.json          DRAM bytes per row of k_scatter (bench.py's traffic)

usage: python profiles/summarize.py [round]   (default 1)
"""
import csv
import collections
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "1"
pre = os.path.join(OUT, f"r{rnd}_")

# the bench run under ncu: 3 warm-up steps, 1 timed step, 1 profiled step and
# one per-target pass = 6 steps of launches
STEPS_UNDER_NCU = 6
C2_ROWS = 76_879_419


def last_json(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith("{")]
    return json.loads(lines[-1])


bench = last_json(os.path.join(RAW, "prof_bench.log"))
with open(pre + "bench_line.json", "w") as f:
    f.write(json.dumps(bench) + "\n")
ref = last_json(os.path.join(RAW, "prof_reference.log"))
with open(pre + "reference_arm.json", "w") as f:
    f.write(json.dumps(ref) + "\n")

# launch list
shutil.copy(os.path.join(RAW, "prof_launches.csv"), pre + "launches.csv")
with open(pre + "launches.csv") as f:
    rows = list(csv.reader(l for l in f if l.startswith('"')))
h, rows = rows[0], rows[1:]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows:
    name = r[ki].split("(")[0]
    if "k_" not in name:
        continue  # torch's input generation
    us = float(r[mi].replace(",", "")) * scale[r[ui]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(v[1] for v in agg.values())
with open(pre + "launches_summary.txt", "w") as f:
    f.write(f"# per step (totals / {STEPS_UNDER_NCU}); ncu --metrics gpu__time_duration.sum "
            "--clock-control none, bench.py c2 --steps 1 --warmup 3: serialised cold-cache "
            "launch durations (compare shares, not absolutes)\n")
    for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{name:40s} launches={n / STEPS_UNDER_NCU:6.1f} "
                f"time={us / STEPS_UNDER_NCU:10.1f}us share={100 * us / tot:5.1f}%\n")
    f.write(f"total {tot / STEPS_UNDER_NCU:.1f} us per step\n")

# ncu --set full
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
raw = subprocess.run(["ncu", "-i", os.path.join(RAW, "prof_full.ncu-rep"), "--page", "raw", "--csv"],
                     check=True, capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rd[0], rd[1], rd[2:]
col = {n: i for i, n in enumerate(hdr)}
stall_cols = [n for n in hdr if n.startswith("smsp__average_warp_latency_issue_stalled_")
              and n.endswith(".ratio")] or \
             [n for n in hdr if n.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not n.endswith("_not_issued")]
traffic = collections.defaultdict(list)
with open(pre + "ncu_full_summary.txt", "w") as f:
    f.write("# ncu --set full --clock-control none --import-source on, bench.py c2 "
            "(--steps 1 --warmup 3), first 20 launches of k_scatter|k_chunk_hist|k_local|k_heads "
            "(cold cache, serialised: compare shares, not absolutes)\n")
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0]
        f.write(f"{name} id {r[col['ID']]}\n")
        for m in METRICS:
            if m in col:
                f.write(f"    {m:60s} {r[col[m]]} {units[col[m]]}\n")
        st = {}
        for n in stall_cols:
            try:
                st[n] = float(r[col[n]].replace(",", ""))
            except ValueError:
                pass
        tot_st = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        short = {k.split("stalled_")[1].split(".")[0]: round(100 * v / tot_st, 1) for k, v in top}
        f.write(f"    stalls: {short}\n")
        if "k_scatter" in name:
            gb = lambda m: float(r[col[m]].replace(",", "")) * (1e9 if units[col[m]] == "Gbyte" else
                                                              1e6 if units[col[m]] == "Mbyte" else 1)
            traffic[name].append((gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")) / C2_ROWS)
per_variant = {k: round(sum(v) / len(v), 2) for k, v in traffic.items()}
allv = [x for v in traffic.values() for x in v]
with open(os.path.join(OUT, "ncu_traffic.json"), "w") as f:
    json.dump({"kernel_class": "scatter", "kernel": "k_scatter",
               "dram_bytes_per_row": round(sum(allv) / len(allv), 2),
               "per_variant": per_variant,
               "algorithmic_bytes_per_row": {"AoS->PK": 37, "PK->PK": 34, "PK->AoS": 37,
                                             "model (bench achieved)": 40},
               "source": f"profiles/r{rnd}_ncu_full_summary.txt (ncu --set full --clock-control "
                         "none, c2 bench, dram__bytes_read.sum + dram__bytes_write.sum per launch / "
                         "rows)"}, f, indent=1)
print(open(pre + "launches_summary.txt").read())
print(json.dumps(per_variant))
