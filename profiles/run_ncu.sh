#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU).
#  1) launch list: every kernel's device time (cold-cache, serialised)
#  2) one --set full capture of the paged-decode kernel (full + SWA layer)
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_decode|reshape_and_cache|build_tables" -c 200 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:paged_decode -s 4 -c 2 -o $OUT/prof_decode \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu_full_bench.log 2>&1
echo "full capture rc=$?"
