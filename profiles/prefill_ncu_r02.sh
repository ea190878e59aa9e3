#!/bin/bash
# --set full captures of the prefill kernel on B=4 x 2048-token chunks at 8k (full
# layer): D=256 without and with Gemma's softcap, D=128.
set -u
OUT=${1:-gpurun_out/prefill_ncu}
mkdir -p $OUT
for v in "d256 (16,8,256) 0.0" "d256cap (16,8,256) 50.0" "d128 (32,8,128) 0.0"; do
  set -- $v
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc5 -c 1 -o $OUT/prof_$1 \
      python -c "import sys; sys.path.insert(0,'profiles'); import bench_prefill; bench_prefill.run(4, 8192, 2048, iters=1, heads=$2, softcap=$3)" \
      > $OUT/$1.log 2>&1
  echo "$1 rc=$?"
done
