#!/bin/bash
# One GPU call that refreshes every committed number (run under gpurun, 1 GPU):
# bench lines for configs 2-4 and the reference arm, the prefill / copy
# micro-benches, the ncu launch list + --set full capture of the headline
# decode kernel, and the per-kernel DRAM table of every kernel on the path.
set -u
OUT=${1:-gpurun_out/ev}
mkdir -p $OUT/wl
timeout 400 python bench.py > $OUT/wl/wl_gemma.json 2> $OUT/wl/wl_gemma.err
timeout 300 python bench.py --workload jamba-style --steps 10 --warmup 3 > $OUT/wl/wl_jamba.json 2> $OUT/wl/wl_jamba.err
timeout 300 python bench.py --workload llama-3.2-11b-vision --ctx 2048 --steps 10 --warmup 3 > $OUT/wl/wl_vision.json 2> $OUT/wl/wl_vision.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/wl/wl_ref.json 2> $OUT/wl/wl_ref.err
timeout 400 python profiles/bench_prefill.py --d128 > $OUT/prefill.jsonl 2> $OUT/prefill.err
timeout 120 python profiles/bench_copy.py > $OUT/copy.jsonl 2> $OUT/copy.err
bash profiles/run_ncu.sh $OUT/ncu
bash profiles/run_ncu_kernels.sh $OUT/kernels
echo done
