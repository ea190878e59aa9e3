#!/bin/bash
# Per-kernel DRAM evidence for every kernel on the path (run under gpurun, 1 GPU):
# device time + DRAM bytes read/written per launch, for each BASELINE config's
# decode loop (eager launches so every kernel is its own ncu result) and the
# chunked-prefill bench.  Summarise with: python profiles/summarize_ncu.py --dram <tag> (writes profiles/<tag>_kernels_dram.md; the round-2 table is r02_all_kernels_dram.md)
set -u
OUT=${1:-gpurun_out/kernels}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
K='regex:paged_|reshape_and_cache|build_tables|slot_mapping|token_rows|apply_deltas'
run() {  # name, command...
  local name=$1; shift
  timeout 900 ncu --metrics $M --clock-control none -k "$K" -c ${NCU_COUNT:-400} --csv --log-file $OUT/$name.csv "$@" \
      > $OUT/$name.log 2>&1
  echo "$name rc=$?"
}
run gemma   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph
run jamba   python bench.py --workload jamba-style --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph
run vision  python bench.py --workload llama-3.2-11b-vision --ctx 2048 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph
run jamba_fused python bench.py --workload jamba-style --mamba-mode fused-step --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph
run prefixmix python bench.py --workload prefix-mix --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph
NCU_COUNT=60 run prefill python profiles/bench_prefill.py
NCU_COUNT=200 run tokenrows python -m pytest -q -m gpu tests/test_gpu_vision_spec.py
