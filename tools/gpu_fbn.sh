mkdir -p gpurun_out/fb
for k in flash_bwd_dq_tc flash_bwd_dkdv_tc; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/fb/$k -f python tools/flash_bench.py llama2-13b > gpurun_out/fb/ncu_$k.log 2>&1
ncu -i gpurun_out/fb/$k.ncu-rep --page details > gpurun_out/fb/details_$k.txt 2>&1
ncu -i gpurun_out/fb/$k.ncu-rep --page source --csv > gpurun_out/fb/source_$k.csv 2>&1
rm -f gpurun_out/fb/$k.ncu-rep
done
