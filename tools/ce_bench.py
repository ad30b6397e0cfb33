"""K7 cross-entropy alone at the 7B LM-head shape (512 x 32000 bf16 logits): graph-timed us and
achieved GB/s of the algorithmic bytes (logits read once + dlogits written).  usage: ce_bench.py [T V]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

T, V = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (512, 32000)
z = [(torch.randn(T, V, device="cuda") * 4).to(torch.bfloat16) for _ in range(4)]
y = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
rows = torch.empty(T, device="cuda")
mean = torch.empty(1, device="cuda")
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
dz = torch.empty(T, V, dtype=torch.bfloat16, device="cuda")


def run(i):
    ops.cross_entropy(z[i % 4], y, V, loss_rows=rows, loss_mean=mean, counter=cnt, dlogits=dz,
                      grad_scale=1.0 / T)


for i in range(3):
    run(i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    for i in range(20):
        run(i)
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"CE T={T} V={V}: {us:.1f} us, {4 * T * V / us / 1e3:.0f} GB/s")
