mkdir -p gpurun_out/tc
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "shrink" -x > gpurun_out/tc/k.txt 2>&1; echo "kernels rc=$?"; tail -15 gpurun_out/tc/k.txt
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -q -x > gpurun_out/tc/p.txt 2>&1; echo "parity rc=$?"; tail -15 gpurun_out/tc/p.txt
for w in 8 16; do echo "== RANK_SMS=$w"; COLLM_RANK_SMS=$w timeout 300 python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -2; done
echo "== RANK_SMS=0"; timeout 300 python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -2
