"""Per-GEMM flag-wait totals in the overlapped 7B forward/backward (projection by projection:
shrink on the side stream + GEMM on main, synchronized between projections)."""
import ctypes
import os
import sys

os.environ["COLLM_GEMM_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg = CONFIGS["llama2-7b"]
st = ReplicaStack(cfg, "cuda")
st.overlap = True
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()
lib = _lib.load()
ns, n = ctypes.c_ulonglong(), ctypes.c_ulonglong()
lib.collm_gemm_wait_stats(ctypes.byref(ns), ctypes.byref(n))
side = st._side_stream()
sig = st._signals(8)
st.advance_step(False)
a = st._acts
lib.collm_set_gemm_lean(1)
for rep in range(2):
    for pi, proj in enumerate(st.layers[1]):
        name = proj.spec.name
        X = a["X"][1] if name in ("qkv", "gate_up") else (a["Xo"][1] if name == "o" else a["Xd"][1])
        Y = a["X"][2] if name == "down" else a["Y"][name]
        s = (sig[pi], st._gen)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            c = proj.forward_lora(X, plan.device, n_train=plan.n_train, signal=s)
        proj.forward_gemm(c, plan.device, Y, wait=s)
        torch.cuda.synchronize()
        lib.collm_gemm_wait_stats(ctypes.byref(ns), ctypes.byref(n))
        if rep == 1:
            print(f"fwd {name:8s}: {n.value:4d} waiting producers, avg {ns.value / max(n.value, 1) / 1e3:6.2f} us", flush=True)
        st.advance_step(False)
