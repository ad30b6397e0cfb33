"""Debug: does one shrink launch set its completion signal?  (8B q|k|v forward shrink alone)"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

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
for pi, proj in enumerate(st.layers[0]):
    name = proj.spec.name
    X = st._acts["X"][0] if name in ("qkv", "gate_up") else (st._acts["Xo"][0] if name == "o" else st._acts["Xd"][0])
    proj.forward_lora(X, plan.device, n_train=plan.n_train, signal=(sig[pi], st._gen))
    torch.cuda.synchronize()
    print(name, "signal after shrink:", sig[pi].tolist(), "gen", st._gen.item(), flush=True)
