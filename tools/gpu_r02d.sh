mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stack.py -q -x -k "flash or attention" > gpurun_out/r02d/attn.txt 2>&1; echo "attn tests rc=$?"; tail -4 gpurun_out/r02d/attn.txt
timeout 300 python tools/flash_bench.py 2>&1 | tail -3 | tee gpurun_out/r02d/flash_bench.txt
timeout 600 python bench.py --attention --no-cpu-baseline --no-e2e > gpurun_out/r02d/bench_attn.json 2> gpurun_out/r02d/bench_attn.err; echo "bench attn rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02d/bench_attn.json'));print(d['value'],d['ms_per_step'])"
