mkdir -p gpurun_out/e2e2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/e2e2/gemma_nograph.json 2>/dev/null
for io in none in-only out-only overlap; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-io $io > gpurun_out/e2e2/gemma_$io.json 2>/dev/null
done
