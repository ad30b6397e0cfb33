#!/bin/bash
# Round-2 final evidence (under gpurun, 1 GPU): launch lists of one step of each BASELINE config
# (the K5 / K1' / K9 tcgen05 kernels in), and --set full captures of the new kernels.
OUT=gpurun_out/r02c_prof; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed
for CFG in llama2-7b llama3-8b llama2-13b; do
  read N NG NS NR < <(python tools/profile_step.py --config $CFG --count 2>/dev/null | tail -1)
  echo "$CFG launches/step=$N gemm=$NG shrink=$NS reduce=$NR"
  timeout 900 ncu --metrics $M --clock-control none -k regex:"gemm_lora|lora_|expand_" -s $N -c $N --csv \
      --log-file $OUT/launches_$CFG.csv python tools/profile_step.py --config $CFG 2>&1 | tail -1
done
full() {  # name, kernel regex, skip, command...
  n=$1; k=$2; s=$3; shift 3
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -o $OUT/$n -f "$@" > $OUT/$n.log 2>&1
  python tools/ncu_summary.py $OUT/$n.ncu-rep > $OUT/full_$n.txt 2>&1
  ncu -i $OUT/$n.ncu-rep --page raw --csv > $OUT/raw_$n.csv 2>&1
  python - $OUT/raw_$n.csv >> $OUT/full_$n.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, v = rows[0], rows[2]
for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sector_hit_rate.pct", "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]:
    if w in h:
        i = h.index(w)
        print(f"    {w:60s} {v[i]} {rows[1][i]}")
PY
  rm -f $OUT/$n.ncu-rep $OUT/raw_$n.csv
}
CFG=llama2-7b full reduce_tc_7b lora_reduce_tc 3 python tools/reduce_bench.py
CFG=llama2-13b LAYERS=2 full reduce_tc_13b lora_reduce_tc 3 python tools/reduce_bench.py
CFG=llama3-8b TC=148 ONLY="fwd qkv" full shrink_tc_8b_fwd_qkv lora_shrink_tc 5 python tools/shrink_bench.py
full flash_fwd_tc_13b flash_fwd_tc 3 python tools/flash_bench.py llama2-13b
full flash_bwd_dkdv_tc_13b flash_bwd_dkdv_tc 1 python tools/flash_bench.py llama2-13b
full flash_bwd_dq_tc_13b flash_bwd_dq_tc 1 python tools/flash_bench.py llama2-13b
ls -la $OUT
