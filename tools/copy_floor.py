"""Practical HBM floor for transfers of the LoRA kernels' sizes: torch copy_ (read+write bytes)
of several sizes, 30 back-to-back copies captured in a CUDA graph (no launch gaps)."""
import torch

for mb in (2, 6, 10, 17, 40, 100, 1000):
    n = mb * (1 << 20) // 2
    xs = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(4)]
    ys = [torch.empty_like(x) for x in xs]
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for i in range(30):
            ys[i % 4].copy_(xs[i % 4])
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 30 * 1e3
    print(f"copy {2 * mb:5d} MB traffic: {us:8.1f} us  {2 * mb * 1.048576 / us:6.2f} TB/s")
