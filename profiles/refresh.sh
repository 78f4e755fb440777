#!/bin/bash
# Round profile refresh, run on the GPU box from the repo root:
#   gpurun -- profiles/refresh.sh
# Writes raw outputs to gpurun_out/ (summarised into profiles/ by
# profiles/summarize.py here).  Each ncu pass only after the same command
# exited 0 without ncu; numbers printed under ncu are never bench values.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/prof_bench.log 2>&1 || exit 1
python bench.py --impl reference > gpurun_out/prof_reference.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_scatter|k_chunk_hist|k_local|k_heads" -c 20 -f -o gpurun_out/prof_full \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_ncu_full.log 2>&1
tail -1 gpurun_out/prof_bench.log
tail -1 gpurun_out/prof_reference.log
ls -la gpurun_out/prof_*
