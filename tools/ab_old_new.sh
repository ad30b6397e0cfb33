set -x
cd $GRAFT_REPO_ROOT
echo "=== NEW tree"
python tools/reduce_bench.py
COLLM_K5_MINB=3 python tools/reduce_bench.py
python tools/shrink_bench.py
NO_LO=1 python tools/shrink_bench.py
echo "=== OLD tree"
(cd build/old_tree && python tools/reduce_bench.py && python tools/shrink_bench.py)
echo "=== NEW bench"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-lm-head --no-e2e > gpurun_out/ab_new.json 2>gpurun_out/ab_new.err
COLLM_K5_MINB=3 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-lm-head --no-e2e > gpurun_out/ab_new3.json 2>>gpurun_out/ab_new.err
(cd build/old_tree && python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-lm-head --no-e2e > ../../gpurun_out/ab_old.json 2>../../gpurun_out/ab_old.err)
for f in ab_new ab_new3 ab_old; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), round(d['roofline_lora']['lora_ms_per_step'],3), d['clocks'])"; done
