"""Where the step time goes: CUDA-graph replays of the full step and of the step with kernel
kinds removed (ops.only), same overlap schedule.  usage: step_breakdown.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
st = ReplicaStack(cfg, "cuda")
st.overlap = os.environ.get("OVERLAP", "1") == "1"
plan = st.plan(*cfg.batch(0))
st.allocate(plan)
st.run_step(plan)
torch.cuda.synchronize()
variants = [("full", None), ("gemm only", ("gemm", "plan")),
            ("base gemm", ("gemm", "plan", "nolora")), ("gemm+shrink", ("gemm", "plan", "shrink")),
            ("gemm+reduce", ("gemm", "plan", "reduce")), ("lora only", ("plan", "lora"))]
graphs = {}
for name, kinds in variants:
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        if kinds:
            with ops.only(*kinds), torch.cuda.graph(g, stream=s):
                st.run_step(plan, advance=False)
        else:
            with torch.cuda.graph(g, stream=s):
                st.run_step(plan, advance=False)
    torch.cuda.current_stream().wait_stream(s)
    graphs[name] = g
for rnd in range(2):
    out = []
    for name, _ in variants:
        g = graphs[name]
        st.advance_step(True)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            st.advance_step(True)
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.append(f"{name} {e0.elapsed_time(e1) / reps:.2f}")
    print(f"[overlap={st.overlap}] " + " | ".join(out) + " ms")
