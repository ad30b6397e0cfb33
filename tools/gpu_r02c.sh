mkdir -p gpurun_out/r02c
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "flash" > gpurun_out/r02c/flash.txt 2>&1; echo "flash rc=$?"; tail -25 gpurun_out/r02c/flash.txt
timeout 600 python -m pytest tests/test_gpu_many_adapters.py -q -x > gpurun_out/r02c/many.txt 2>&1; echo "many rc=$?"; tail -3 gpurun_out/r02c/many.txt
