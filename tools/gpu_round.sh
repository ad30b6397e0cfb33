# K5 tests + the parity / stack suites that run K5, then the three bench configs
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_baseline_parity.py -q -x 2>&1 | tail -5
bash tools/r02_configs.sh
