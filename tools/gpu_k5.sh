for c in llama2-13b llama3-8b llama2-7b; do
  echo "== $c"; CFG=$c LAYERS=2 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  COLLM_LIB=$PWD/tools/_ab/libcollm_old.so CFG=$c LAYERS=2 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1 | sed 's/^/OLD /'
done
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_kernels.py -q -x -k "reduce or baseline" 2>&1 | tail -2
