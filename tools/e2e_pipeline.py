"""e2e step with host copies: serial (H2D, step, D2H on one stream) vs pipelined (step k's H2D
and step k-1's D2H on a copy stream, two captured buffer sets), alternated."""
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
L = cfg.model.layers
g_a = st.capture(plan)
sets = [(a["X"][0], a["dY_top"], a["X"][L])]
alt = (sets[0][0].clone(), sets[0][1].clone(), torch.empty_like(sets[0][2]))
a["X"][0], a["dY_top"], a["X"][L] = alt
g_b = st.capture(plan)
a["X"][0], a["dY_top"], a["X"][L] = sets[0]
sets.append(alt)
graphs = [g_a, g_b]
x_host = sets[0][0].cpu().pin_memory()
dy_host = sets[0][1].cpu().pin_memory()
out_host = torch.empty(sets[0][2].shape, dtype=torch.bfloat16).pin_memory()
main = torch.cuda.current_stream()
cs = torch.cuda.Stream()


def serial(n):
    for _ in range(n):
        sets[0][0].copy_(x_host, non_blocking=True)
        sets[0][1].copy_(dy_host, non_blocking=True)
        plan.device.upload()
        plan.train_device.upload()
        st.advance_step(True)
        g_a.replay()
        out_host.copy_(sets[0][2], non_blocking=True)


def pipelined(n):
    done = [None, None]
    out_done = [None, None]

    def h2d(k):
        i = k % 2
        with torch.cuda.stream(cs):
            if done[i] is not None:
                cs.wait_event(done[i])
            sets[i][0].copy_(x_host, non_blocking=True)
            sets[i][1].copy_(dy_host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        return ev
    ready = h2d(0)
    for k in range(n):
        i = k % 2
        main.wait_event(ready)
        if out_done[i] is not None:
            main.wait_event(out_done[i])
        plan.device.upload()
        plan.train_device.upload()
        st.advance_step(True)
        graphs[i].replay()
        ev = torch.cuda.Event()
        ev.record(main)
        done[i] = ev
        if k + 1 < n:
            ready = h2d(k + 1)
        with torch.cuda.stream(cs):
            cs.wait_event(ev)
            out_host.copy_(sets[i][2], non_blocking=True)
            od = torch.cuda.Event()
            od.record(cs)
        out_done[i] = od
    main.wait_stream(cs)


def plain(n):
    for _ in range(n):
        st.advance_step(True)
        g_a.replay()


def timeit(fn, n=20):
    fn(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(n)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(3):
    print(f"plain {timeit(plain):.2f}  serial e2e {timeit(serial):.2f}  pipelined e2e {timeit(pipelined):.2f} ms")
