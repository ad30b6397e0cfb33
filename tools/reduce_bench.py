"""Time K5 (one launch = one Llama-2-7B layer's dB/dA^T reductions + fused AdamW) alone, graph-
replayed over rotating layers' buffers (inputs > L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.layer import ForwardCache, LoraProjection, OptimizerState  # noqa: E402

cfg = CONFIGS[os.environ.get("CFG", "llama2-7b")]
_tr, _items = cfg.batch(0)
Ttr = _tr.batch * _tr.seq_len
T = Ttr + sum(it.n_rows for it in _items)
NL = int(os.environ.get("LAYERS", "4"))
opt = OptimizerState()
opt.advance()
layers = []
for l in range(NL):
    groups = []
    for spec in cfg.projections:
        pr = LoraProjection(spec, 2, "cuda")
        pr.W.normal_(0, 0.02)
        pr.refresh_transpose()
        pr.make_trainable(0)
        X = torch.randn(T, spec.in_features, device="cuda").to(torch.bfloat16)
        H16 = torch.randn(T, spec.R, device="cuda").to(torch.bfloat16)
        pr._dh_buffer(Ttr).normal_()
        dY = torch.randn(Ttr, spec.out_features, device="cuda").to(torch.bfloat16)
        cache = ForwardCache(X=X, H16=H16, n_train=Ttr)
        groups += pr.grad_groups(dY, cache, optimizer=opt)
        layers.append((pr, dY, cache))
    layers_groups = groups
    layers.append(groups)
groups_per_layer = [x for x in layers if isinstance(x, list)]
nbytes = 0
for gs in groups_per_layer[:1]:
    for g in gs:
        nbytes += 2 * Ttr * (g.P + g.Q) + 32 * g.P * g.Q
lean = os.environ.get("LEAN", "0") == "1"
_lib.load().collm_set_gemm_lean(1 if lean else 0)
for gs in groups_per_layer:
    ops.lora_reduce(Ttr, gs, _lib.MODE_ADAMW, adamw=opt.args)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
n = 20
with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
    for i in range(n):
        ops.lora_reduce(Ttr, groups_per_layer[i % len(groups_per_layer)], _lib.MODE_ADAMW, adamw=opt.args)
torch.cuda.current_stream().wait_stream(s)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
print(f"K5 one {cfg.key} layer (lean={lean}): {us:.1f} us, ~{nbytes / 1e6:.0f} MB algorithmic "
      f"-> {nbytes / us / 1e6:.2f} TB/s")
