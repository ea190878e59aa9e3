#!/bin/bash
# One GPU call that refreshes every committed number (run under gpurun, 1 GPU):
# bench lines for configs 2-5 (+ the G=4 shard of config 2, the fused-step
# Jamba variant) and the reference arm, the prefill / delta-upload micro-
# benches, the two-rank launcher rehearsal, the ncu launch list + --set full
# capture of the headline decode kernel, and the per-kernel DRAM table.
set -u
OUT=${1:-gpurun_out/ev}
mkdir -p $OUT/wl
b() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py "$@" > $OUT/wl/$name.json 2> $OUT/wl/$name.err
  echo "$name rc=$? $(tail -c 300 $OUT/wl/$name.json | head -c 0)"
}
b wl_gemma
b wl_gemma_g4 --batch-per-gpu 64 --steps 10 --warmup 3 --no-cpu-baseline
b wl_jamba --workload jamba-style --steps 10 --warmup 3
b wl_jamba_fused --workload jamba-style --mamba-mode fused-step --steps 10 --warmup 3 --no-cpu-baseline
b wl_vision --workload llama-3.2-11b-vision --ctx 2048 --steps 10 --warmup 3
b wl_prefix --workload prefix-mix --steps 10 --warmup 3
b wl_ref --impl reference --steps 2 --warmup 1
JENGA_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --batch-per-gpu 8 --steps 5 --warmup 3 --no-cpu-baseline \
    > $OUT/wl/wl_2rank.json 2> $OUT/wl/wl_2rank.err
echo "2rank rc=$?"
timeout 400 python profiles/bench_prefill.py --d128 --softcap > $OUT/prefill.jsonl 2> $OUT/prefill.err
timeout 300 python profiles/bench_delta_upload.py > $OUT/delta_upload.jsonl 2> $OUT/delta_upload.err
bash profiles/run_ncu.sh $OUT/ncu
bash profiles/run_ncu_kernels.sh $OUT/kernels
echo done
