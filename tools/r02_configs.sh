# Round-2 bench lines of the three BASELINE single-GPU configs (default mode) + 7B with attention
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_7b.json 2> $OUT/bench_7b.err; echo "7b rc=$?"
timeout 1200 python bench.py --config llama3-8b --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_8b.json 2> $OUT/bench_8b.err; echo "8b rc=$?"
timeout 1500 python bench.py --config llama2-13b --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_13b.json 2> $OUT/bench_13b.err; echo "13b rc=$?"
for f in 7b 8b 13b; do python -c "
import json; d=json.load(open('$OUT/bench_$f.json'))
print('$f', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None, 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), 'lora', round(d['roofline_lora']['frac'],3), d['clocks'])" 2>&1 | tail -1; done
