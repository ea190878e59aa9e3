set -u
for v in product pp32; do
  if [ $v = product ]; then lib=paper_2503_18292_b200/libjenga_b200.so; else lib=paper_2503_18292_b200/variants/libjenga_b200_$v.so; fi
  echo "== $v"
  JENGA_B200_LIB=$lib timeout 300 python -c "
import sys; sys.path.insert(0,'profiles'); import bench_prefill
bench_prefill.run(4, 8192, 2048, heads=(32,8,128)); bench_prefill.run(16, 4096, 512, heads=(32,8,128))" 2>&1 | tail -2
done
JENGA_B200_LIB=paper_2503_18292_b200/variants/libjenga_b200_pp32.so timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x -k "128" 2>&1 | tail -2
