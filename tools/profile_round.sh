#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU): launch list of one step, per-launch DRAM bytes +
# tensor-pipe activity for the whole step, and --set full captures of the key kernels.
# usage: bash tools/profile_round.sh r01 [config]
TAG=${1:-r01}; CFG=${2:-llama2-7b}; OUT=gpurun_out/$TAG; mkdir -p $OUT
# launches per step (and per kind) from one eager step
read N NG NS NR < <(python tools/profile_step.py --config $CFG --count 2>/dev/null | tail -1)
echo "launches/step=$N gemm=$NG shrink=$NS reduce=$NR"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_lora|lora_|expand_" \
    -s $N -c $N --csv --log-file $OUT/launches_$CFG.csv python tools/profile_step.py --config $CFG 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"gemm_lora|lora_|expand_" -s $N -c $N --csv --log-file $OUT/metrics_$CFG.csv \
    python tools/profile_step.py --config $CFG 2>&1 | tail -1
# full sets: first forward GEMM (q|k|v of layer 0) and its shrink, first dX GEMM (down of the top
# layer), first K5 reduction of the step
ncu --set full --clock-control none --import-source on -k regex:"gemm_lora" -s $NG -c 1 -o $OUT/full_gemm_fwd_qkv python tools/profile_step.py --config $CFG 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"gemm_lora" -s $((NG + NG / 2)) -c 1 -o $OUT/full_gemm_dx_down python tools/profile_step.py --config $CFG 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"lora_shrink" -s $NS -c 1 -o $OUT/full_shrink_fwd_qkv python tools/profile_step.py --config $CFG 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"lora_reduce" -s $NR -c 1 -o $OUT/full_reduce_layer python tools/profile_step.py --config $CFG 2>&1 | tail -1
# a split-2 dX GEMM in 4-CTA clusters (o of the top layer: the third dX GEMM of the backward) and
# the LM-head cross-entropy kernel (K7) at the 7B head shape
ncu --set full --clock-control none --import-source on -k regex:"gemm_lora" -s $((NG + NG / 2 + 2)) -c 1 -o $OUT/full_gemm_dx_o_split2 python tools/profile_step.py --config $CFG 2>&1 | tail -1
ncu --set full --clock-control none --import-source on -k regex:"cross_entropy" -s 3 -c 1 -o $OUT/full_ce_head python tools/ce_bench.py 512 32000 2>&1 | tail -1
