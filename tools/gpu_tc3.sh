TC=16 timeout 120 python tools/shrink_bench.py 2>&1 | tail -1
TC=8 timeout 120 python tools/shrink_bench.py 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k shrink_tc 2>&1 | tail -2
for w in 8 16 0; do echo "== RANK_SMS=$w"; COLLM_RANK_SMS=$w timeout 300 python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -2; done
