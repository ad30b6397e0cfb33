timeout 600 python -m pytest tests/test_gpu_many_adapters.py -q -x 2>&1 | tail -3
for r in 16 64; do timeout 300 python tools/many_adapter_bench.py $r 2>&1 | tail -1; done
