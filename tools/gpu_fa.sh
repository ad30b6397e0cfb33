timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x -k "flash or attention" 2>&1 | tail -25
timeout 300 python tools/flash_bench.py 2>&1 | tail -4
COLLM_FA_TC=0 timeout 300 python tools/flash_bench.py 2>&1 | tail -4
