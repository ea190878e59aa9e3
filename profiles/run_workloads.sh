set -x
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wl_gemma.json 2> gpurun_out/wl_gemma.err
timeout 300 python bench.py --workload jamba-style --steps 10 --warmup 3 > gpurun_out/wl_jamba.json 2> gpurun_out/wl_jamba.err
timeout 300 python bench.py --workload llama-3.2-11b-vision --ctx 2048 --steps 10 --warmup 3 > gpurun_out/wl_vision.json 2> gpurun_out/wl_vision.err
JENGA_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --batch-per-gpu 8 > gpurun_out/wl_2rank.json 2> gpurun_out/wl_2rank.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/wl_ref.json 2> gpurun_out/wl_ref.err
