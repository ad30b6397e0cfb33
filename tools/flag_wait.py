"""How long GEMM producers wait for the concurrent shrink's flag in an overlapped step
(COLLM_GEMM_DEBUG=1: the kernels also record a timeline, negligible cost)."""
import ctypes
import os
import sys

os.environ["COLLM_GEMM_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"]
st = ReplicaStack(cfg, "cuda")
st.overlap = True
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
for _ in range(3):
    st.run_step(plan)
torch.cuda.synchronize()
lib = _lib.load()
ns, n = ctypes.c_ulonglong(), ctypes.c_ulonglong()
lib.collm_gemm_wait_stats(ctypes.byref(ns), ctypes.byref(n))
st.run_step(plan)
torch.cuda.synchronize()
lib.collm_gemm_wait_stats(ctypes.byref(ns), ctypes.byref(n))
print(f"one step: {n.value} producer flag waits, total {ns.value / 1e6:.2f} ms "
      f"(avg {ns.value / max(n.value, 1) / 1e3:.2f} us per waiting producer thread)")
