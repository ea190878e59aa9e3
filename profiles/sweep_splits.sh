#!/bin/bash
# Decode split policy sweep (DESIGN §3 "Split count"): the bench step of the
# Gemma shard, Llama-3.2-Vision and Jamba-style workloads under compile-time
# variants of the split policy (paper_2503_18292_b200/build.py --variant).
#   bytes: byte-sized splits (32 tiles at D=256, 96 at D=128)
#   cN:    wave-aware splits with N tiles of per-CTA overhead (product: c32);
#   other names: residency variants (CTAs per SM x ring bytes), see DESIGN.md §3
out=${1:-gpurun_out/r02_sweep_splits.jsonl}
variants=${2:-"product bytes c2 c8 c16 c32 c64"}
workloads=${3:-"gemma2-9b|llama-3.2-11b-vision --ctx 2048|jamba-style|prefix-mix"}
: > $out
IFS='|' read -ra specs <<< "$workloads"
for spec in "${specs[@]}"; do
  set -- $spec
  wl=$1; shift
  extra="$*"
  for v in $variants; do
    if [ $v = product ]; then lib=paper_2503_18292_b200/libjenga_b200.so; else lib=paper_2503_18292_b200/variants/libjenga_b200_$v.so; fi
    line=$(JENGA_B200_LIB=$lib timeout 400 python bench.py --workload $wl $extra --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1)
    python - "$wl" "$v" "$line" >> $out <<'PY'
import json, sys
wl, v, line = sys.argv[1:4]
try:
    d = json.loads(line)
    print(json.dumps({"workload": wl, "policy": v, "value": d["value"], "ms_per_step": d["ms_per_step"],
                      "roofline_achieved": d["roofline"]["achieved"], "frac": d["roofline"]["frac"],
                      "verified": d.get("verified")}))
except Exception as e:
    print(json.dumps({"workload": wl, "policy": v, "error": str(e), "line": line[:300]}))
PY
  done
done
cat $out
