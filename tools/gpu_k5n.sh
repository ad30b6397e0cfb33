mkdir -p gpurun_out/k5
c=llama2-7b
CFG=$c LAYERS=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:lora_reduce_tc -s 3 -c 1 \
  -o gpurun_out/k5/k5tc_$c -f python tools/reduce_bench.py > gpurun_out/k5/ncu_$c.log 2>&1
ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page details > gpurun_out/k5/details_$c.txt 2>&1
ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page raw --csv > gpurun_out/k5/raw_$c.csv 2>&1
ncu -i gpurun_out/k5/k5tc_$c.ncu-rep --page source --csv > gpurun_out/k5/source_$c.csv 2>&1
rm -f gpurun_out/k5/k5tc_$c.ncu-rep
