"""Debug: the overlapped forward projection by projection (sync + print after each)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg0 = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"]
cfg = dataclasses.replace(cfg0, model=dataclasses.replace(cfg0.model, layers=1))
st = ReplicaStack(cfg, "cuda")
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.advance_step(False)
sig = st._signals(4)
plan.device.expand()
side = torch.cuda.Stream()
_lib.load().collm_set_gemm_lean(1)
order = os.environ.get("ORDER", "shrink_first")
torch.cuda.synchronize()
a = st._acts
if os.environ.get("MAINSTREAM"):  # run the GEMMs on a non-default stream too
    ms = torch.cuda.Stream()
    torch.cuda.set_stream(ms)
for pi, proj in enumerate(st.layers[0]):
    name = proj.spec.name
    X = a["X"][0] if name in ("qkv", "gate_up") else (a["Xo"][0] if name == "o" else a["Xd"][0])
    Y = a["X"][1] if name == "down" else a["Y"][name]
    s = (sig[pi], st._gen)
    box = {}
    if order == "shrink_first":
        with torch.cuda.stream(side):
            box["c"] = proj.forward_lora(X, plan.device, n_train=plan.n_train, signal=s)
        proj.forward_gemm(box["c"], plan.device, Y, wait=s)
        if os.environ.get("ONE"):
            torch.cuda.synchronize(); print(name, "ok", sig[pi].tolist(), flush=True); break
    else:  # GEMM enqueued first: the shrink must co-reside with a running, waiting GEMM
        proj._buffers(plan.n_rows, plan.device.n_slots)
        from paper_2604_16400_b200.layer import ForwardCache
        c = ForwardCache(X=X, H16=proj._H16, n_train=plan.n_train)
        proj.forward_gemm(c, plan.device, Y, wait=s)
        with torch.cuda.stream(side):
            if os.environ.get("TRIVIAL"):
                sig[pi][1:2].copy_(st._gen)  # a trivial kernel sets the flag
            else:
                proj.forward_lora(X, plan.device, n_train=plan.n_train, signal=s)
    torch.cuda.synchronize()
    print(name, "ok", sig[pi].tolist(), flush=True)
