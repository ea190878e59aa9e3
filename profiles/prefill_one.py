"""One bench_prefill configuration (B=4, 8k ctx, 2048-token chunks) for ncu captures."""
import sys
sys.path.insert(0, "profiles")
import bench_prefill
bench_prefill.run(4, 8192, 2048, iters=2)
