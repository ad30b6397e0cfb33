mkdir -p gpurun_out/r02b
timeout 600 python -m pytest tests/test_gpu_many_adapters.py -q -x > gpurun_out/r02b/many.txt 2>&1; echo "many rc=$?"; tail -5 gpurun_out/r02b/many.txt
for r in 16 64; do timeout 300 python tools/many_adapter_bench.py $r 2>&1 | tail -1; done | tee gpurun_out/r02b/many_bench.txt
