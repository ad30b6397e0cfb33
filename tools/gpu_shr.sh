for c in llama2-7b llama3-8b llama2-13b; do
  for tc in 0 64 148; do echo "$c"; CFG=$c TC=$tc timeout 300 python tools/shrink_bench.py 2>&1 | tail -1; done
done
