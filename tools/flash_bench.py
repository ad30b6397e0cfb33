"""K9 timing at the BASELINE step shapes: forward over every sequence of the pass (packed
64-row tiles) and backward over the training sequences, graph-timed, with the algorithmic
FLOPs (fwd 4*P*D*H, bwd 10*P_tr*D*H, P = sum L(L+1)/2).  usage: flash_bench.py [config...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.segments import build_mixed_batch  # noqa: E402


def timed(fn, reps=20):
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


for key in sys.argv[1:] or ["llama2-7b", "llama3-8b", "llama2-13b"]:
    cfg = CONFIGS[key]
    train, items = cfg.batch(0)
    mb = build_mixed_batch(train, items)
    T, Ttr = mb.n_rows, mb.n_train_rows
    bounds = list(range(0, Ttr + 1, train.seq_len))
    for t in range(Ttr + 1, T):
        if mb.row_request[t] != mb.row_request[t - 1]:
            bounds.append(t)
    bounds.append(T)
    H, Hk, D = cfg.model.hidden // 128, cfg.model.kv_dim // 128, 128
    rows = ops.seq_rows(bounds, "cuda")
    qkv = torch.randn(T, (H + 2 * Hk) * D, device="cuda").to(torch.bfloat16)
    q, k, v = qkv[:, :H * D], qkv[:, H * D:(H + Hk) * D], qkv[:, (H + Hk) * D:]
    out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(H, T, device="cuda")
    dout = torch.randn(T, H * D, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(H, T, device="cuda")
    kw = dict(n_heads=H, n_kv_heads=Hk)
    t_f = timed(lambda: ops.flash_attention(q, k, v, out, lse, *rows, T=T, **kw))
    t_b = timed(lambda: ops.flash_attention_bwd(
        q[:Ttr], k[:Ttr], v[:Ttr], out[:Ttr], dout[:Ttr], lse, delta, dqkv[:Ttr, :H * D],
        dqkv[:Ttr, H * D:(H + Hk) * D], dqkv[:Ttr, (H + Hk) * D:], *rows, T=Ttr, stat_ld=T, **kw))
    P = sum((b - a) * (b - a + 1) // 2 for a, b in zip(bounds[:-1], bounds[1:]))
    P_tr = sum((b - a) * (b - a + 1) // 2 for a, b in zip(bounds[:-1], bounds[1:]) if b <= Ttr)
    f_f, f_b = 4 * P * D * H, 10 * P_tr * D * H
    print(f"{key}: T={T} seqs={len(bounds) - 1} heads {H}/{Hk}: fwd {t_f:.1f} us "
          f"({f_f / t_f / 1e6:.0f} TFLOP/s), bwd(train {Ttr}) {t_b:.1f} us ({f_b / t_b / 1e6:.0f} TFLOP/s)")
