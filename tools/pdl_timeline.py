"""Timeline of one forward projection's shrink -> GEMM programmatic-dependent-launch pair
(COLLM_SHRINK_DEBUG / COLLM_GEMM_DEBUG=2 stamps, globaltimer): when the shrink CTAs run, when
the GEMM CTAs start, get their first stage, pass the LoRA wait and finish.
usage: pdl_timeline.py [projection] [pdl 0/1]"""
import ctypes
import os
import statistics
import sys

os.environ["COLLM_SHRINK_DEBUG"] = "1"
os.environ["COLLM_GEMM_DEBUG"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import _lib  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ENTRY, ReplicaStack  # noqa: E402

want = sys.argv[1] if len(sys.argv) > 1 else "qkv"
pdl = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
cfg = CONFIGS["llama2-7b"]
st = ReplicaStack(cfg, "cuda")
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()
a = st._acts
lib = _lib.load()
GRAPH = os.environ.get("GRAPH", "0") == "1"  # replay the pairs from a CUDA graph (no CPU gaps)
lib.collm_set_gemm_lean(0 if (GRAPH and pdl) else 1)
proj = [p for p in st.layers[0] if p.spec.name == want][0]
X = a["X"][0] if want in ENTRY else (a["Xo"][0] if want == "o" else a["Xd"][0])
Y = a["X"][1] if want == "down" else a["Y"][want]


def pairs():
    for _ in range(4):
        cache = proj.forward_lora(X, plan.device, n_train=plan.n_train)
        proj.forward_gemm(cache, plan.device, Y, pdl=pdl)


if GRAPH:
    pairs()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
        pairs()
    torch.cuda.current_stream().wait_stream(s)
    gr.replay()
else:
    pairs()
torch.cuda.synchronize()
sh = (ctypes.c_uint64 * (4096 * 2))()
assert lib.collm_shrink_debug_copy(ctypes.byref(sh), ctypes.c_size_t(4096 * 16)) == 0
gm = (ctypes.c_uint64 * (256 * 32))()
assert lib.collm_gemm_debug_copy(ctypes.byref(gm), ctypes.c_size_t(256 * 32 * 8)) == 0
s_start = [sh[2 * i] for i in range(4096) if sh[2 * i]]
s_end = [sh[2 * i + 1] for i in range(4096) if sh[2 * i + 1]]
g = [list(gm[i * 32:(i + 1) * 32]) for i in range(256)]
g = [r for r in g if r[0] and r[0] >= min(s_start) - 10**6]
t0 = min(s_start)


def dist(name, v):
    v = sorted((x - t0) / 1e3 for x in v)
    if v:
        print(f"  {name:16s} n={len(v):4d} min {v[0]:7.2f} med {statistics.median(v):7.2f} max {v[-1]:7.2f}")


print(f"{want} pdl={pdl}: shrink CTAs {len(s_start)}, GEMM CTAs {len(g)}")
dist("shrink start", s_start)
dist("shrink end", s_end)
dist("gemm begin", [r[0] for r in g])
dist("gemm tma0", [r[15] for r in g if r[15]])
dist("gemm ready0", [r[4] for r in g if r[4]])
dist("gemm lora wait", [r[20] for r in g if r[20]])
dist("gemm last mma", [r[12] for r in g if r[12]])
dist("gemm done", [r[13] for r in g if r[13]])
