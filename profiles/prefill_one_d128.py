"""One bench_prefill configuration on Llama / Jamba heads (D=128) for ncu captures."""
import sys
sys.path.insert(0, "profiles")
import bench_prefill
bench_prefill.run(4, 8192, 2048, iters=2, heads=(32, 8, 128))
