#!/bin/bash
# Round-2 evidence (under gpurun, 1 GPU):
#  1. which ncu counter reads the tcgen05 tensor pipe: candidates on cuBLAS / ours at 8192^3 and
#     two 7B step shapes (timing printed by the same script, unprofiled run first)
#  2. ours vs cuBLAS per GEMM shape of the 7B / 8B / 13B steps
#  3. launch lists of one step of each config (duration, DRAM bytes, tensor-pipe counter)
OUT=gpurun_out/r02; mkdir -p $OUT
python tools/tensor_pipe_check.py > $OUT/tensor_pipe_timing.txt 2>&1
for m in sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed \
         sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
         sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed \
         sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum \
         sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed \
         sm__inst_executed_pipe_tc.sum \
         sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
         TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed; do
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,$m --clock-control none \
    -k regex:"gemm|nvjet|cutlass|sm100|xmma" --csv --log-file $OUT/tp_$m.csv \
    python tools/tensor_pipe_check.py --once > /dev/null 2>&1 || echo "metric $m failed"
done
timeout 1200 python tools/gemm_table.py > $OUT/gemm_table.md 2> $OUT/gemm_table.err
for CFG in llama2-7b llama3-8b llama2-13b; do
  read N NG NS NR < <(python tools/profile_step.py --config $CFG --count 2>/dev/null | tail -1)
  echo "$CFG launches/step=$N gemm=$NG shrink=$NS reduce=$NR"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32.sum \
      --clock-control none -k regex:"gemm_lora|lora_|expand_" -s $N -c $N --csv --log-file $OUT/launches_$CFG.csv \
      python tools/profile_step.py --config $CFG 2>&1 | tail -1
done
