#!/bin/bash
# Per-kernel checks of the round-2 tcgen05 kernels (under gpurun, 1 GPU): their parity tests,
# then graph-timed microbenchmarks at the BASELINE shapes —
#   K9 forward / backward (tools/flash_bench.py) and the backward's breakdown with the
#   COLLM_DEBUG_FB switches (1: no MMAs, 2: no elementwise work, 3: neither) under ncu;
#   K5 per layer (tools/reduce_bench.py, tcgen05 vs mma.sync);
#   K1 vs K1' on the whole GPU (tools/shrink_bench.py, TC=148).
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x -k "flash or attention or reduce or shrink" 2>&1 | tail -1
timeout 300 python tools/flash_bench.py 2>&1 | tail -3
for d in 0 1 2 3; do echo "COLLM_DEBUG_FB=$d"; COLLM_DEBUG_FB=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flash_bwd" -c 2 --csv python tools/flash_bench.py llama2-13b 2>/dev/null | grep -E "flash" | awk -F'","' '{print $5, $NF}'; done
for c in llama2-7b llama3-8b llama2-13b; do
  CFG=$c timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  CFG=$c COLLM_K5_TC=0 timeout 300 python tools/reduce_bench.py 2>&1 | tail -1
  for tc in 0 148; do CFG=$c TC=$tc timeout 300 python tools/shrink_bench.py 2>&1 | tail -1; done
done
