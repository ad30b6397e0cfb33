"""Validate the ncu tensor-pipe counters for tcgen05 on B200: run a cuBLAS bf16 8192^3 matmul and
our GEMM on the same shape plus two Llama-2-7B step shapes, each 3x (profile the 3rd launch of
each under ncu with the candidate metrics; compare metric % with achieved FLOP/s / peak from the
timed run printed here).

  python tools/tensor_pipe_check.py            # timing (CUDA events) -> achieved TFLOP/s
  ncu --metrics <list> -k regex:'gemm|nvjet|cutlass|sm100' python tools/tensor_pipe_check.py --once
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402

SHAPES = [("sq8192", 8192, 8192, 8192), ("7b_fwd_qkv", 1024, 12288, 4096),
          ("7b_dx_gate_up", 512, 4096, 22016)]
once = "--once" in sys.argv
_lib.load()
for name, M, N, K in SHAPES:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for impl in ("cublas", "collm"):
        fn = (lambda: torch.matmul(A, W.t(), out=Y)) if impl == "cublas" else \
             (lambda: ops.gemm_lora(A, W, Y))
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if once:
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(f"{name:14s} {impl:7s} {us:9.1f} us  {2 * M * N * K / us / 1e6:7.1f} TFLOP/s", flush=True)
