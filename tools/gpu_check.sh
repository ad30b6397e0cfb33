#!/bin/bash
# One gpurun round trip: GPU tests, a short 7B bench line, and the ncu launch list of one step.
# usage (under gpurun): bash tools/gpu_check.sh [tag] [config]
TAG=${1:-dev}; CFG=${2:-llama2-7b}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -4
timeout 400 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_lora|lora_|expand_" -s ${SKIP:-641} -c ${COUNT:-641} --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --config $CFG 2>&1 | tail -1
