"""Which cuBLAS kernels (name, grid, block) torch.matmul picks for the step's GEMM shapes."""
import torch
from torch.profiler import ProfilerActivity, profile

SHAPES = [("dX_qkv", 512, 4096, 12288), ("dX_o", 512, 4096, 4096), ("dX_gu", 512, 4096, 22016),
          ("dX_down", 512, 11008, 4096), ("o", 1024, 4096, 4096)]
for name, M, N, K in SHAPES:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, W.t(), out=Y)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.matmul(A, W.t(), out=Y)
        torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type.name == "CUDA":
            print(name, e.name[:150], getattr(e, "kernel_grid", None) if hasattr(e, "kernel_grid") else "")
    for ev in prof.profiler.kineto_results.events():
        if ev.device_type().name == "CUDA":
            print("   ", ev.name()[:160], ev.duration_ns() / 1e3 if hasattr(ev, "duration_ns") else "")
