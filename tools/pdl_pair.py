"""Does the shrink -> GEMM programmatic-dependent-launch overlap work?  Layer 0's four forward
projections (K1 shrink + K2 GEMM each) replayed from CUDA graphs: with PDL, serialized, GEMMs
alone, shrinks alone.  usage: pdl_pair.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ENTRY, ReplicaStack  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
st = ReplicaStack(cfg, "cuda")
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()
a = st._acts
layer = st.layers[0]
_lib.load().collm_set_gemm_lean(1)


def fwd(pdl):
    for _ in range(reps):
        for proj in layer:
            name = proj.spec.name
            X = a["X"][0] if name in ENTRY else (a["Xo"][0] if name == "o" else a["Xd"][0])
            Y = a["X"][1] if name == "down" else a["Y"][name]
            cache = proj.forward_lora(X, plan.device, n_train=plan.n_train)
            proj.forward_gemm(cache, plan.device, Y, pdl=pdl)


def timed(fn, kinds=None):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        if kinds:
            with ops.only(*kinds), torch.cuda.graph(g, stream=s):
                fn()
        else:
            with torch.cuda.graph(g, stream=s):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5 / reps * 1e3


res = {
    "pdl": timed(lambda: fwd(True)),
    "serial": timed(lambda: fwd(False)),
    "gemm only": timed(lambda: fwd(False), ("gemm", "plan")),
    "shrink only": timed(lambda: fwd(False), ("shrink", "plan")),
}
print(f"layer forward (4 projections, mode {os.environ.get('COLLM_OVERLAP_MODE', 'pdl')}), us: " + "  ".join(f"{k} {v:.1f}" for k, v in res.items()))
