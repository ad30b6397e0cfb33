"""K8 paged attention alone: a decode batch of B rows with context C each over a paged cache
(7B: 32 query / 32 KV heads; 8B: 32 / 8), graph-timed; achieved GB/s of the algorithmic bytes
(every K/V byte of every context read once).  usage: attn_bench.py [B C n_heads n_kv]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402

B, C, H, KV = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (256, 1024, 32, 32)
D, page = 128, 64
npg = (C + page - 1) // page
n_pages = B * npg
kc = torch.randn(n_pages, KV, page, D, device="cuda").to(torch.bfloat16)
vc = torch.randn(n_pages, KV, page, D, device="cuda").to(torch.bfloat16)
bt = torch.randperm(n_pages, device="cuda").to(torch.int32).view(B, npg)
q = torch.randn(B, H * D, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
rs = torch.arange(B, device="cuda", dtype=torch.int32)
rp = torch.full((B,), C - 1, device="cuda", dtype=torch.int32)


def run():
    ops.paged_attention(q, kc, vc, bt, rs, rp, out, n_heads=H, n_kv_heads=KV, max_ctx=C)


run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    for _ in range(10):
        run()
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 10 * 1e3
nbytes = 2 * B * C * KV * D * 2
print(f"K8 decode B={B} ctx={C} heads {H}/{KV}: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s "
      f"({nbytes / 1e6:.0f} MB of K/V)")
