for c in llama2-7b llama3-8b llama2-13b; do
  CFG=$c timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  CFG=$c COLLM_DEBUG_K5_NO_MMA=1 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  for ts in 1 2 4; do echo "ts=$ts"; CFG=$c COLLM_K5_TSPLIT=$ts timeout 300 python tools/reduce_bench.py 2>&1 | tail -1; done
done
