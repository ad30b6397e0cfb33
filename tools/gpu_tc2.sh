mkdir -p gpurun_out/tc
for w in 0 8 16 32 74 148; do TC=$w timeout 120 python tools/shrink_bench.py 2>&1 | tail -1; done
TC=16 ONLY="fwd qkv" timeout 300 ncu --set full --import-source on -k regex:lora_shrink_tc -c 1 -s 3 -o gpurun_out/tc/shrink_tc_qkv -f python tools/shrink_bench.py > gpurun_out/tc/ncu.log 2>&1; echo ncu rc=$?
