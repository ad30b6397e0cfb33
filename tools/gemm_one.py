"""Run one GEMM shape a few times (for ncu).  usage: gemm_one.py M N K [bn] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    ops.gemm_lora(A, W, Y, bn=bn)
torch.cuda.synchronize()
