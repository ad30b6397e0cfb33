#!/bin/bash
# bench.py with K9 attention inside the step for the three single-GPU BASELINE configs
OUT=gpurun_out/attn; mkdir -p $OUT
timeout 900 python bench.py --steps 10 --warmup 3 --attention --no-cpu-baseline > $OUT/bench_7b_attn.json 2> $OUT/bench_7b_attn.err; echo "7b rc=$?"
timeout 1500 python bench.py --config llama3-8b --steps 4 --warmup 3 --attention --no-cpu-baseline > $OUT/bench_8b_attn.json 2> $OUT/bench_8b_attn.err; echo "8b rc=$?"
timeout 1500 python bench.py --config llama2-13b --steps 4 --warmup 3 --attention --no-cpu-baseline > $OUT/bench_13b_attn.json 2> $OUT/bench_13b_attn.err; echo "13b rc=$?"
for f in 7b 8b 13b; do python -c "
import json; d=json.load(open('$OUT/bench_${f}_attn.json'))
print('$f attn', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None, d['clocks'])" 2>&1 | tail -1; done
