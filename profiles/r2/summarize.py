#!/usr/bin/env python
"""Summarise profiles/r2/refresh.sh's raw outputs (gpurun_out/r2_*) into the
tracked round-2 files:

  profiles/r2/bench_line.json        bench.py (c5, the driver's workload)
  profiles/r2/reference_arm.json     bench.py --impl reference
  profiles/r2/other_configs.txt      bench.py --config c2/c3/c4/c1 (per target) + c1/c4 call latency
  profiles/r2/launches_c5.csv        ncu launch list, one transposition per c5 target (full size)
  profiles/r2/launches_summary.txt   per-target time by kernel from that list (cold, serialised)
  profiles/r2/ncu_full_summary.txt   ncu --set full metrics per launch (c5 shape, 200M rows)
  profiles/ncu_traffic.json          k_scatter DRAM bytes per row (bench.py's roofline.traffic)
  profiles/r2/e2e_sliced.txt         sliced vs whole host-buffer call on c5 (0,2,1), per-slice timeline
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
RAW = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles", "r2")


def last_json(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    b = last_json(os.path.join(RAW, "r2_bench.log"))
    with open(os.path.join(OUT, "bench_line.json"), "w") as f:
        f.write(json.dumps(b) + "\n")
    ref = last_json(os.path.join(RAW, "r2_reference.log"))
    if ref:
        with open(os.path.join(OUT, "reference_arm.json"), "w") as f:
            f.write(json.dumps(ref) + "\n")
    with open(os.path.join(OUT, "other_configs.txt"), "w") as f:
        f.write("# bench.py --config cN --no-cpu-baseline --no-e2e (same build): value, ms/step, "
                "per target (ms, SURVEY 8(d) model fraction)\n")
        for c in ("c2", "c3", "c4", "c1"):
            d = last_json(os.path.join(RAW, f"r2_bench_{c}.log"))
            if not d:
                continue
            pt = d["model_roofline"]["per_target"]
            f.write(f"{c} {d['value']:.1f} Mnnz/s {d['ms_per_step']:.4f} ms/step | " +
                    " ".join(f"{k}: {v['ms']:.4f} ms / {v['model_frac']:.3f}" for k, v in pt.items()) + "\n")
        for c in ("c1", "c4"):
            p = os.path.join(RAW, f"r2_latency_{c}.log")
            if os.path.exists(p):
                f.write(f"latency {c}: " + open(p).read().strip().splitlines()[-1] + "\n")
    p = os.path.join(RAW, "r2_e2e_sliced.log")
    if os.path.exists(p):
        lines = open(p).read().splitlines()
        last = max(i for i, l in enumerate(lines) if l.startswith("  slice  0:"))
        keep = [l for l in lines if l.startswith("QD_SLICE_ROWS")] + ["# per-slice timeline of the last sliced call "
                "(ms from the first input copy; CUDA events)"] + [l for l in lines[last:] if l.startswith("  slice")]
        with open(os.path.join(OUT, "e2e_sliced.txt"), "w") as f:
            f.write("# profiles/r2/e2e_sliced.py: qd_transpose_inplace on pinned host buffers, c5 (0,2,1) at full size; "
                    "QD_SLICE_ROWS=0 = the whole-tensor call\n" + "\n".join(keep) + "\n")
    # launch list
    shutil.copy(os.path.join(RAW, "r2_launches_c5.csv"), os.path.join(OUT, "launches_c5.csv"))
    with open(os.path.join(OUT, "launches_c5.csv")) as f:
        rows = list(csv.reader(l for l in f if l.startswith('"')))
    h, rows = rows[0], rows[1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    seq = [(r[ki].split("(")[0], float(r[mi].replace(",", "")) * scale[r[ui]]) for r in rows]
    # the two targets: (1,0,2) first (no run discovery), (0,2,1) starts at its k_heads / k_heads_quad
    split = next(i for i, (k, _) in enumerate(seq) if "k_heads" in k)
    with open(os.path.join(OUT, "launches_summary.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, profiles/r2/prof_targets.py "
                "--config c5: one transposition per target at full size (cold cache, serialised)\n")
        for name, part in (("(1,0,2)", seq[:split]), ("(0,2,1)", seq[split:])):
            tot = sum(u for _, u in part)
            agg = collections.OrderedDict()
            for k, u in part:
                a = agg.setdefault(k, [0, 0.0])
                a[0] += 1
                a[1] += u
            f.write(f"{name}: {tot / 1e3:.2f} ms in {len(part)} launches\n")
            for k, (nl, u) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"    {u / 1e3:9.3f} ms {100 * u / tot:5.1f} %  x{nl:<3d} {k}\n")
    # full-set summary
    rep = os.path.join(RAW, "r2_full_c5.ncu-rep")
    mets = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hh, units, data = r[0], r[1], r[2:]
    n = 200_000_000
    traffic = collections.OrderedDict()
    with open(os.path.join(OUT, "ncu_full_summary.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none --import-source on, profiles/r2/prof_targets.py "
                "--config c5 --nnz 200000000 (both targets; cold cache, serialised: compare shares, "
                "not absolutes). Per-row figures divide by 200M rows.\n")
        tgt = "(1,0,2)"
        for row in data:
            d = dict(zip(hh, row))
            name = d["Kernel Name"].split("(")[0]
            if "k_heads" in name:
                tgt = "(0,2,1)"  # its run discovery opens the second target
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            un = units[hh.index("dram__bytes_read.sum")]
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(un, 1)
            inst = float(d["smsp__inst_executed.sum"].replace(",", ""))
            f.write(f"{d['ID']:>3} {name}   [target {tgt}]\n")
            for m in mets:
                f.write(f"      {m:60s} {d[m]} {units[hh.index(m)]}\n")
            f.write(f"      per row of the tensor: dram bytes {(rd + wr) * mul / n:.2f}, thread "
                    f"instructions {inst * 32 / n:.1f}" + (" ((0,2,1): only its large-run rows pass "
                    "here)" if tgt == "(0,2,1)" else "") + "\n")
            if name.startswith("void k_scatter") and tgt == "(1,0,2)":  # every row
                traffic.setdefault(name, []).append((rd + wr) * mul / n)
    if traffic:
        allv = [v for vs in traffic.values() for v in vs]
        t = {"kernel_class": "scatter", "kernel": "k_scatter",
             "dram_bytes_per_row": round(sum(allv) / len(allv), 2),
             "per_variant": {k: round(sum(v) / len(v), 2) for k, v in traffic.items()},
             "algorithmic_bytes_per_row": {"AoS->PK": 37, "PK->PK": 34, "PK->AoS": 37,
                                           "model (bench achieved)": 40},
             "source": "profiles/r2/ncu_full_summary.txt (ncu --set full --clock-control none, c5 "
                       "shape at 200M rows, target (1,0,2) whose passes move every row; "
                       "dram__bytes_read.sum + dram__bytes_write.sum per launch / rows)"}
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
            json.dump(t, f, indent=1)
    print("summarised into", OUT)


if __name__ == "__main__":
    main()
