"""Main-loop rate of one GEMM from the debug timeline (COLLM_GEMM_DEBUG): per CTA the first
TMA issue, first stage ready, 32nd stage ready, last MMA issue, epilogue done (us from the first
CTA's start).  usage: gemm_rate.py M N K   (variant via COLLM_GEMM_CG/BN/SCHED/MC)"""
import ctypes
import os
import statistics
import sys

os.environ["COLLM_GEMM_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
lib = _lib.load()
for i in range(6):
    ops.gemm_lora(A, Ws[i % 3], Y)
torch.cuda.synchronize()
arr = (ctypes.c_uint64 * (256 * 32))()
assert lib.collm_gemm_debug_copy(ctypes.byref(arr), ctypes.c_size_t(256 * 32 * 8)) == 0
t = [list(arr[i * 32:(i + 1) * 32]) for i in range(256)]
rows = [r for r in t if r[0]]
t0 = min(r[0] for r in rows)
cols = {"begin": 0, "tma0": 15, "ready0": 4, "ready32": 8, "last_mma": 12, "epi_acc": 2,
        "s2_stored": 16, "s2_fenced/peer": 17, "s2_flag/in": 18, "s2_in0/own": 19, "s2_in3": 22,
        "done": 13}
out = {k: [(r[i] - t0) / 1e3 for r in rows if r[i]] for k, i in cols.items()}
print(f"M={M} N={N} K={K} CTAs={len(rows)} " + os.environ.get("COLLM_GEMM_CG", "") + ":" +
      os.environ.get("COLLM_GEMM_BN", "") + ":" + os.environ.get("COLLM_GEMM_SCHED", "") + ":" +
      os.environ.get("COLLM_GEMM_MC", ""))
for k, v in out.items():
    if v:
        print(f"  {k:9s} min {min(v):6.2f} med {statistics.median(v):6.2f} max {max(v):6.2f}")
r32 = [(r[8] - r[4]) / 1e3 / 32 for r in rows if r[8] and r[4]]
if r32:
    print(f"  steady us/stage (ready0->ready32)/32: med {statistics.median(r32):.3f}")
