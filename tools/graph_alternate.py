"""Is alternating two captured step graphs (double-buffered inputs) slower than replaying one?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg = CONFIGS["llama2-7b"]
st = ReplicaStack(cfg, "cuda")
st.overlap = True
plan = st.plan(*cfg.batch(0))
a = st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()
g_a = st.capture(plan)
L = cfg.model.layers
orig = (a["X"][0], a["dY_top"], a["X"][L])
alt = (orig[0].clone(), orig[1].clone(), torch.empty_like(orig[2]))
a["X"][0], a["dY_top"], a["X"][L] = alt
g_b = st.capture(plan)
a["X"][0], a["dY_top"], a["X"][L] = orig


def timeit(seq, n=20):
    for g in seq[:2]:
        st.advance_step(True)
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(n):
        st.advance_step(True)
        seq[k % len(seq)].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(2):
    print(f"one graph {timeit([g_a]):.2f} ms   alternating {timeit([g_a, g_b]):.2f} ms   "
          f"g_b only {timeit([g_b]):.2f} ms")
