cd $GRAFT_REPO_ROOT
for gn in 1 4 8 16; do echo "== GN=$gn"; COLLM_GEMM_RASTER_GN=$gn python tools/tensor_pipe_check.py 2>&1 | grep collm; COLLM_GEMM_RASTER_GN=$gn timeout 900 python tools/gemm_table.py llama3-8b llama2-13b 2>&1 | grep fwd\\\|dX; done
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_kernels.py -q -p no:cacheprovider 2>&1 | tail -3
