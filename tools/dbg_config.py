import os, sys, time, dataclasses
sys.path.insert(0, "/root/repo")
import torch
from paper_2604_16400_b200.configs import CONFIGS, ModelShape
from paper_2604_16400_b200.replica import ReplicaStack
cfg0 = CONFIGS[sys.argv[1]]
model = dataclasses.replace(cfg0.model, layers=2)
cfg = dataclasses.replace(cfg0, model=model)
st = ReplicaStack(cfg, "cuda")
st.overlap = sys.argv[2] == "1"
plan = st.plan(*cfg.batch(0))
print("rows", plan.n_rows, "train", plan.n_train, "shrink tiles", plan.device.n_shrink_tiles, "slots", plan.device.n_slots, flush=True)
st.allocate(plan)
t0 = time.time()
st.run_step(plan, backward=os.environ.get("BWD", "1") == "1")
torch.cuda.synchronize()
print("step ok", sys.argv[1:], round(time.time() - t0, 2), "s", flush=True)
