"""Many-adapter decode at the Llama-2-7B q|k|v shape: 256 decode rows of
256 distinct adapters (one 256-row slot tile with 256 LoRA slots) vs the same rows on 1 and 32
adapters and vs the base GEMM alone — forward (shrink + GEMM with the fused expand), graph-timed.
usage: many_adapter_bench.py [rank]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops, segments  # noqa: E402
from paper_2604_16400_b200.domain import InferenceItem, RowRole  # noqa: E402
from paper_2604_16400_b200.layer import LoraProjection, ProjectionSpec  # noqa: E402

rank = int(sys.argv[1]) if len(sys.argv) > 1 else 16
K, subs, T = 4096, (4096, 4096, 4096), 256
n_ad = 256
spec = ProjectionSpec("qkv", K, subs, rank, alpha=2.0 * rank)
proj = LoraProjection(spec, n_ad)
for t in (proj.W, proj.A, proj.B):
    t.normal_(0, 0.02)
proj.scale.fill_(2.0)
X = torch.randn(T, K, device="cuda").to(torch.bfloat16)
Y = torch.empty(T, sum(subs), device="cuda", dtype=torch.bfloat16)


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


res = {}
res["base GEMM only"] = timed(lambda: ops.gemm_lora(X, proj.W, Y, M=T))
for n_distinct, expand_rows in ((1, True), (32, True), (256, False), (256, True)):
    os.environ["COLLM_EXPAND_ROWS_SLOTS"] = "32" if expand_rows else "100000"
    items = [InferenceItem(i, i * n_distinct // T, 1, RowRole.DECODE) for i in range(T)]
    mb = segments.build_mixed_batch(None, items)
    tc = int(os.environ.get("TC", "0"))  # K1' on this many CTAs (0: the default selection)
    plan = segments.DevicePlan(segments.plan_segments(mb.seg_start, mb.seg_adapter),
                               tc_ctas=tc or None)
    torch.cuda.synchronize()
    tag = f"{n_distinct} adapters" + (" [per-row expand]" if plan.n_expand_tiles else "")
    res[f"{tag}: shrink+GEMM"] = timed(lambda: proj.forward(X, plan, Y))
    cache = proj.forward_lora(X, plan)
    res[f"{tag}: GEMM+expand"] = timed(lambda: proj.forward_gemm(cache, plan, Y))
    res[f"{tag}: shrink"] = timed(lambda: proj.forward_lora(X, plan))
print(f"rank {rank}: " + " | ".join(f"{k} {v:.1f} us" for k, v in res.items()))
