#!/bin/bash
# Round-2 evidence for the kernels added this round (under gpurun, 1 GPU): one `ncu --set full`
# capture each of K9 fwd / dK-dV / dQ (7B and 13B batch shapes), K1' on a 16-SM partition (7B fwd
# q|k|v), the per-row expand (256 distinct adapters, r=16) and the 64-wide K5 tile (one 13B layer),
# plus the 7B step's launch list WITH attention (duration, DRAM bytes, tc-pipe).
OUT=gpurun_out/r02b; mkdir -p $OUT
F="--set full --import-source on --clock-control none"
timeout 600 ncu $F -k regex:flash -c 4 -o $OUT/flash_7b -f python tools/flash_bench.py llama2-7b > $OUT/flash_7b.log 2>&1; echo "flash 7b rc=$?"
timeout 900 ncu $F -k regex:flash -c 4 -o $OUT/flash_13b -f python tools/flash_bench.py llama2-13b > $OUT/flash_13b.log 2>&1; echo "flash 13b rc=$?"
TC=16 ONLY="fwd qkv" timeout 600 ncu $F -k regex:lora_shrink_tc -s 3 -c 1 -o $OUT/shrink_tc_qkv -f python tools/shrink_bench.py > $OUT/shrink_tc.log 2>&1; echo "shrink_tc rc=$?"
timeout 600 ncu $F -k regex:expand_rows -c 1 -o $OUT/expand_rows -f python tools/many_adapter_bench.py 16 > $OUT/expand_rows.log 2>&1; echo "expand rc=$?"
CFG=llama2-13b LAYERS=1 timeout 900 ncu $F -k regex:lora_reduce -c 1 -o $OUT/reduce_13b -f python tools/reduce_bench.py > $OUT/reduce_13b.log 2>&1; echo "reduce rc=$?"
for k in flash_fwd flash_bwd_dkdv flash_bwd_dq; do
  python tools/ncu_hotspots.py $OUT/flash_13b.ncu-rep $k > $OUT/flash_13b_hotspots_$k.txt 2>&1
done
for r in flash_7b flash_13b shrink_tc_qkv expand_rows reduce_13b; do
  python tools/ncu_summary.py $OUT/$r.ncu-rep > $OUT/$r.summary.txt 2>&1
  ncu -i $OUT/$r.ncu-rep --page raw --csv > $OUT/$r.raw.csv 2>/dev/null
  rm -f $OUT/$r.ncu-rep   # gpurun copies back <= 64 MiB: keep the text
done
ls -la $OUT
