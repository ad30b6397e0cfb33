#!/bin/bash
# Quick GPU round trip (under gpurun): GPU tests, a short bench line, the per-kernel launch list
# of one step.  usage: bash tools/gpu_quick.sh TAG [config] [pytest -k expr]
TAG=${1:-dev}; CFG=${2:-llama2-7b}; K=${3:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then timeout 600 python -m pytest tests/ -m gpu -x -q -k "$K" 2>&1 | tail -5
else timeout 600 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -5; fi
timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err
read N NG NS NR < <(python tools/profile_step.py --config $CFG --count 2>/dev/null | tail -1)
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"gemm_lora|lora_|expand_" -s $N -c $N --csv --log-file gpurun_out/launches_$TAG.csv \
   python tools/profile_step.py --config $CFG 2>&1 | tail -1
