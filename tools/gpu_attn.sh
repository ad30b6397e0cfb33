timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "paged_attention" 2>&1 | tail -2
COLLM_ATTN_TC=0 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "paged_attention" 2>&1 | tail -2
for shape in "256 1024 32 32" "256 1024 32 8" "64 1024 64 8"; do echo "$shape: $(timeout 300 python tools/attn_bench.py $shape 2>&1 | tail -1)"; done
