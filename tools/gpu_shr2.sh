OUT=gpurun_out/shr2; mkdir -p $OUT
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 1200 python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline > $OUT/$tag.json 2> $OUT/$tag.err
  python -c "
import json; d=json.load(open('$OUT/$tag.json'))
print('$tag', round(d['value']), round(d['ms_per_step'],2), 'lora', round(d['roofline_lora']['frac'],3), round(d['roofline_lora']['lora_ms_per_step'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1
}
for CFG in llama3-8b llama2-13b; do
  export CFG
  run ${CFG}_base X=0
  run ${CFG}_f148 COLLM_SHRINK_TC_FWD=148
  run ${CFG}_f148_d148 COLLM_SHRINK_TC_FWD=148 COLLM_SHRINK_TC_DH=148
  run ${CFG}_f148_d64 COLLM_SHRINK_TC_FWD=148 COLLM_SHRINK_TC_DH=64
done
