mkdir -p gpurun_out/k1
for o in "fwd qkv" "dH o"; do
  t=$(echo $o | tr ' ' '_')
  ONLY="$o" timeout 600 ncu --set full --import-source on --clock-control none -k regex:lora_shrink -s 5 -c 1 \
    -o gpurun_out/k1/k1_$t -f python tools/shrink_bench.py > gpurun_out/k1/ncu_$t.log 2>&1
  ncu -i gpurun_out/k1/k1_$t.ncu-rep --page details > gpurun_out/k1/details_$t.txt 2>&1
  ncu -i gpurun_out/k1/k1_$t.ncu-rep --page source --csv > gpurun_out/k1/source_$t.csv 2>&1
  rm -f gpurun_out/k1/k1_$t.ncu-rep
done
