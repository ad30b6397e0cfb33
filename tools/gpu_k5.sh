# K5 (tcgen05 stream vs mma.sync): tests, then warm timing for the three configs
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "reduce" 2>&1 | tail -15
for c in llama2-7b llama3-8b llama2-13b; do
  CFG=$c timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  CFG=$c COLLM_K5_TC=0 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
done
if [ "${FULL:-0}" = 1 ]; then
  timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stack.py tests/test_gpu_baseline_parity.py -q -x 2>&1 | tail -5
fi
if [ "${NCU:-0}" = 1 ]; then
  mkdir -p gpurun_out/k5
  for c in llama3-8b llama2-7b; do
    CFG=$c LAYERS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:lora_reduce_tc -s 3 -c 1 \
      -o gpurun_out/k5/k5tc_$c -f python tools/reduce_bench.py > gpurun_out/k5/ncu_$c.log 2>&1
    ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page details > gpurun_out/k5/details_$c.txt 2>&1
    ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page raw --csv > gpurun_out/k5/raw_$c.csv 2>&1
    ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page source --csv > gpurun_out/k5/source_$c.csv 2>&1
    rm -f gpurun_out/k5/k5tc_$c.ncu-rep
  done
fi
