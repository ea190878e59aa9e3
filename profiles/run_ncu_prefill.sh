#!/bin/bash
# ncu evidence for the tcgen05 prefill kernel (run under gpurun, 1 GPU):
# launch list of one bench_prefill configuration and one --set full capture.
set -u
OUT=${1:-gpurun_out/prefill}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|reshape_and_cache" -c 40 --csv \
    --log-file $OUT/launches.csv python profiles/bench_prefill.py > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:prefill_tc5 -c 1 -o $OUT/prof_prefill_tc5 \
    python profiles/bench_prefill.py > $OUT/ncu_full.log 2>&1
echo "full capture rc=$?"
