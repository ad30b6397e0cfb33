"""Time the collm GEMM alone on Llama-7B projection shapes (CUDA events, L2-sized inputs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

SHAPES = [("qkv", 1024, 12288, 4096), ("o", 1024, 4096, 4096), ("gate_up", 1024, 22016, 4096),
          ("down", 1024, 4096, 11008), ("dX_qkv", 512, 4096, 12288), ("dX_o", 512, 4096, 4096),
          ("dX_gu", 512, 4096, 22016), ("dX_down", 512, 11008, 4096)]


def main():
    bns = [int(b) for b in os.environ.get("BNS", "0").split(",")]
    for name, M, N, K in SHAPES:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
        Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for bn in bns:
            for i in range(3):
                ops.gemm_lora(A, Ws[i % 3], Y, bn=bn)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 30
            e0.record()
            for i in range(reps):
                ops.gemm_lora(A, Ws[i % 3], Y, bn=bn)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / reps * 1e3
            tf = 2 * M * N * K / (us * 1e-6) / 1e12
            print(f"{os.environ.get('COLLM_GEMM_SCHED','hybrid'):6s} bn={bn:3d} {name:8s} M={M:5d} N={N:6d} K={K:6d} {us:8.1f} us {tf:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
