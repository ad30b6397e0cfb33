timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k shrink_tc 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -x -k partition 2>&1 | tail -2
TC=16 timeout 120 python tools/shrink_bench.py 2>&1 | tail -1
for w in 16 0; do echo "== RANK_SMS=$w"; COLLM_RANK_SMS=$w timeout 300 python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -2; done
