#!/bin/bash
# Round-2 final check (under gpurun, 1 GPU): the full GPU suite, smoke(), the default bench line,
# the reference arm's line.
OUT=gpurun_out/r02f; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests/ -m gpu -q --durations=15 > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?"; grep -E "passed|failed|error" $OUT/pytest_gpu.txt | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
echo "bench rc=$?"; head -c 700 $OUT/bench_default.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
echo "ref rc=$?"; head -c 400 $OUT/bench_reference.json; echo
