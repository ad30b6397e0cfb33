timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -k "flash or attention" 2>&1 | tail -2
timeout 300 python tools/flash_bench.py 2>&1 | tail -3
