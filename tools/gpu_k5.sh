# K5 (tcgen05 stream vs mma.sync): tests, then warm timing for the three configs
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "reduce" 2>&1 | tail -3
for c in llama2-7b llama3-8b llama2-13b; do
  CFG=$c timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
done
CFG=llama2-7b COLLM_K5_TC=0 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
