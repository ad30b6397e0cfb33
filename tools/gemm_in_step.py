"""Per-GEMM device time inside the real step (eager, CUDA events around every GEMM launch),
grouped by shape, next to the same shape replayed alone by tools/gemm_bench.py.
usage: gemm_in_step.py [config] [nolora]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"]
kinds = ("gemm", "plan") + (("nolora",) if "nolora" in sys.argv else ())
st = ReplicaStack(cfg, "cuda")
st.overlap = False
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()

records = []
orig = ops.gemm_lora


def timed(A, B, Y, **kw):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig(A, B, Y, **kw)
    e1.record()
    M = kw.get("M") or A.shape[0]
    records.append(((M, B.shape[0], A.shape[1]), e0, e1))


ops.gemm_lora = timed
import paper_2604_16400_b200.layer as _layer  # noqa: E402

if hasattr(_layer, "ops"):
    _layer.ops.gemm_lora = timed
with ops.only(*kinds):
    for _ in range(3):
        records.clear()
        st.run_step(plan, advance=True)
        torch.cuda.synchronize()
agg = collections.defaultdict(list)
for shape, e0, e1 in records:
    agg[shape].append(e0.elapsed_time(e1) * 1e3)
tot = 0.0
for shape, ts in agg.items():
    ts.sort()
    tot += sum(ts)
    M, N, K = shape
    print(f"M={M:5d} N={N:6d} K={K:6d} n={len(ts):3d} median {ts[len(ts) // 2]:7.1f}us "
          f"min {ts[0]:7.1f} max {ts[-1]:7.1f}  {2 * M * N * K / (ts[len(ts) // 2] * 1e-6) / 1e12:6.0f} TF/s")
print(f"sum {tot / 1e3:.2f} ms over {len(records)} GEMMs ({kinds})")
