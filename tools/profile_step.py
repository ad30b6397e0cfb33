"""Run warm-up eager steps of a config, then exactly one profiled step (for ncu launch lists).

  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'gemm|lora|expand' \
      -s <launches to skip> --csv --log-file out.csv python tools/profile_step.py --config llama2-7b
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_16400_b200 import ops  # noqa: E402
from paper_2604_16400_b200.configs import CONFIGS  # noqa: E402
from paper_2604_16400_b200.replica import ReplicaStack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama2-7b")
ap.add_argument("--warm", type=int, default=1)
ap.add_argument("--kinds", default="")
ap.add_argument("--count", action="store_true", help="print launches per step (total gemm shrink reduce)")
a = ap.parse_args()
cfg = CONFIGS[a.config]
stack = ReplicaStack(cfg, "cuda")
plan = stack.plan(*cfg.batch(0))
stack.allocate(plan)
for _ in range(a.warm):
    stack.run_step(plan)
torch.cuda.synchronize()
if a.count:
    counts = []
    for kinds in (None, ("gemm",), ("lora",)):
        c0 = ops.launch_count()
        if kinds:
            with ops.only(*kinds):
                stack.run_step(plan)
        else:
            stack.run_step(plan)
        counts.append(ops.launch_count() - c0)
    n_lora = counts[2]
    n_reduce = sum(1 for p in stack.projections()) // len(stack.specs) if plan.n_train else 0
    print(counts[0], counts[1], n_lora - n_reduce, n_reduce)
    sys.exit(0)
c0 = ops.launch_count()
if a.kinds:
    with ops.only(*a.kinds.split(",")):
        stack.run_step(plan)
else:
    stack.run_step(plan)
torch.cuda.synchronize()
print(f"launches in profiled step: {ops.launch_count() - c0} (warm-up steps: {a.warm})", file=sys.stderr)
