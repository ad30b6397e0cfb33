"""GPU: the grad-mode cross-replica sync machinery on one device.

* Per-layer gradient buckets handed to a comm stream by external events recorded INSIDE the
  captured step graph (``run_step(grad_events=...)``): what the comm stream reads after waiting on
  layer l's event is exactly the gradient the step wrote (bitwise equal to an eager step's), for
  every layer, step after step (the step's input changes between replays).
* ``bench.py`` multi-replica flow (2 ranks under torchrun, both on cuda:0 with gloo — the test
  hook; NCCL itself needs one GPU per rank): per-layer bucket allreduce + per-layer AdamW apply
  (grad mode) and FedAvg rounds (fedavg mode) run end to end and print one JSON line.
"""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    _lib.load()


def _cfg(key="llama2-7b", layers=3):
    import dataclasses

    from paper_2604_16400_b200.configs import CONFIGS
    c = CONFIGS[key]
    return dataclasses.replace(c, model=dataclasses.replace(c.model, layers=layers))


def test_grad_bucket_events_inside_graph():
    from paper_2604_16400_b200.replica import ReplicaStack
    cfg = _cfg()
    st = ReplicaStack(cfg, "cuda", seed=0)
    st.overlap = True
    plan = st.plan(*cfg.batch(0))
    a = st.allocate(plan, distinct_synthetic=True)
    L = cfg.model.layers
    x0 = a["X"][0].clone()
    inputs = [x0, (x0.float() * 0.5).to(torch.bfloat16), (x0.float() + 0.25).to(torch.bfloat16)]
    # eager reference gradients per input
    want = []
    for x in inputs:
        a["X"][0].copy_(x)
        st.run_step(plan, optimizer_step=False)
        torch.cuda.synchronize()
        want.append([b.clone() for b in st.grad_buckets()])
    assert not torch.equal(want[0][0], want[1][0])
    events = [torch.cuda.Event(external=True) for _ in range(L)]
    main = torch.cuda.current_stream()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(main)
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        st.run_step(plan, optimizer_step=False, advance=False, grad_events=events)
    main.wait_stream(s)
    comm = torch.cuda.Stream()
    buckets = st.grad_buckets()
    snaps = [torch.empty_like(b) for b in buckets]
    for it, x in enumerate(inputs):
        a["X"][0].copy_(x)
        st.advance_step(False)
        g.replay()
        for l in range(L - 1, -1, -1):
            comm.wait_event(events[l])
            with torch.cuda.stream(comm):
                snaps[l].copy_(buckets[l])
        main.wait_stream(comm)
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(snaps[l], want[it][l]), f"step {it} layer {l}"


def _torchrun(args, env_extra, timeout=600):
    env = dict(os.environ, COLLM_BENCH_ONE_GPU="1", COLLM_BENCH_DIST_BACKEND="gloo", **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", *args]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0]), p.stderr


@pytest.mark.parametrize("mode", ["grad", "fedavg"])
def test_bench_two_replicas(mode):
    common = ["--config", "tiny", "--steps", "4", "--warmup", "3", "--no-cpu-baseline",
              "--no-lm-head", "--no-roofline", "--sync", mode, "--round-steps", "2"]
    line, err = _torchrun(common, {})
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert "communicator" in err and err.count("communicator") == 2
    assert line["syncs_in_timed_region"] == (4 if mode == "grad" else 2)
