timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x -k "flash or attention" 2>&1 | tail -1
for d in 0 1 2 3; do echo "debug=$d"; COLLM_DEBUG_FB=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flash_bwd" -c 2 --csv python tools/flash_bench.py llama2-13b 2>/dev/null | grep -E "flash" | awk -F'","' '{print $5, $NF}'; done
timeout 300 python tools/flash_bench.py 2>&1 | tail -3
