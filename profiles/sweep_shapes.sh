#!/bin/bash
# Headline decode across batch x context at ~constant KV footprint (Gemma-2-9B
# geometry, 42 layers): one bench line each (no e2e / CPU legs).
OUT=${1:-gpurun_out/shapes}
mkdir -p $OUT
for bc in ${SHAPES:-"8 32768" "16 16384" "32 8192" "64 4096" "128 2048" "256 1024"}; do
  set -- $bc
  timeout 400 python bench.py --batch-per-gpu $1 --ctx $2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    > $OUT/b$1_c$2.json 2> $OUT/b$1_c$2.err
  tail -1 $OUT/b$1_c$2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'batch': $1, 'ctx': $2, 'GBps': d['value'], 'frac': round(d['value']/6463, 4), 'decode_GBps': d['roofline']['achieved'], 'tok_s': d['tokens_per_s'], 'ms_per_step': d['ms_per_step']}))" >> $OUT/shapes.jsonl
done
cat $OUT/shapes.jsonl
