#!/bin/bash
# Round-2 profile refresh, run on the GPU box from the repo root:
#   gpurun -- profiles/r2/refresh.sh
# Raw outputs go to gpurun_out/r2_*; profiles/r2/summarize.py turns them
# into the tracked files under profiles/r2/.  Every ncu pass runs only after
# the same command exited 0 without ncu; numbers printed under ncu are never
# bench values.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r2_bench.log 2>&1 || exit 1
python bench.py --impl reference > gpurun_out/r2_reference.log 2>&1
for c in c2 c3 c4 c1; do
  python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_$c.log 2>&1
done
python profiles/r2/latency.py --config c1 > gpurun_out/r2_latency_c1.log 2>&1
python profiles/r2/latency.py --config c4 > gpurun_out/r2_latency_c4.log 2>&1
# the sliced host-buffer call on c5 (0,2,1) with its per-slice timeline, whole-tensor call beside it
QD_HOST_DBG=1 python profiles/r2/e2e_sliced.py 2 > gpurun_out/r2_e2e_sliced.log 2>&1
# launch list of one transposition per target of the bench workload (c5, full size)
python profiles/r2/prof_targets.py --config c5 > /dev/null 2>&1 || exit 1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches_c5.csv python profiles/r2/prof_targets.py --config c5 \
    > gpurun_out/r2_ncu_launch.log 2>&1
# full sections of the hot kernels, both c5 targets on 200M rows of the same
# distribution (kernel replay saves and restores every buffer it writes)
python profiles/r2/prof_targets.py --config c5 --nnz 200000000 > /dev/null 2>&1 || exit 1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_scatter|k_chunk_hist|k_local3|k_heads" -f -o gpurun_out/r2_full_c5 \
    python profiles/r2/prof_targets.py --config c5 --nnz 200000000 > gpurun_out/r2_ncu_full.log 2>&1
ls -la gpurun_out/r2_*
