#!/bin/bash
# Round-2 GPU check (under gpurun, 1 GPU): full GPU test suite with durations, the default bench
# line, then the evidence captures of tools/profile_r02.sh.
OUT=gpurun_out/r02; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests/ -m gpu -q --durations=25 > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?"; tail -40 $OUT/pytest_gpu.txt | grep -E "passed|failed|error" | tail -3
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
echo "bench rc=$?"; cat $OUT/bench_default.json | head -c 600; echo
if [ "${EVIDENCE:-1}" = 1 ]; then timeout 2400 bash tools/profile_r02.sh > $OUT/profile.log 2>&1; echo "profile rc=$?"; fi
