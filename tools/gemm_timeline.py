"""Per-CTA timeline of one stream-K GEMM (COLLM_GEMM_DEBUG=1)."""
import ctypes
import os
import sys

os.environ["COLLM_GEMM_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib, ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
Y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
lib = _lib.load()
for _ in range(3):
    ops.gemm_lora(A, W, Y, bn=256)
torch.cuda.synchronize()
arr = (ctypes.c_uint64 * (256 * 32))()
assert lib.collm_gemm_debug_copy(ctypes.byref(arr), ctypes.c_size_t(256 * 32 * 8)) == 0
t = [list(arr[i * 32:(i + 1) * 32]) for i in range(256)]
mask = (1 << 60) - 1
t0 = min(r[0] for r in t if r[0])
for r in t:  # the segment-start stamps carry the mode in bits 60+
    pass
for c, r in enumerate(t[:148]):
    segs = []
    for i in range(3):
        if r[1 + 4 * i]:
            mode = r[1 + 4 * i] >> 60
            segs.append(f"m{mode}: start {((r[1+4*i]&mask)-t0)/1e3:6.1f} mma {(r[2+4*i]-t0)/1e3:6.1f} end {(r[3+4*i]-t0)/1e3:6.1f}")
    extra = ""
    if r[14]:
        extra += f" flags {(r[14]-t0)/1e3:6.1f}"
    if r[16]:
        extra += " chunks(ld,done): " + " ".join(f"{(r[24+k]-t0)/1e3:.1f},{(r[16+k]-t0)/1e3:.1f}" for k in range(8) if r[16+k])
    print(f"cta {c:3d} begin {(r[0]-t0)/1e3:5.1f}  " + " | ".join(segs) + f"  done {(r[13]-t0)/1e3:6.1f}" + extra)
