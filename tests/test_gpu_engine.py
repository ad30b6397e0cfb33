"""GPU: the reference engine (coserve, unmodified, from baseline/_ref) driving the CUDA backend.

``backend.make_engine(coserve.engine, CudaLoraBackend(...))`` runs the reference's
determinism.yaml scenario (4 replicas of one family, bursty chat stream, FL fine-tuning enabled)
with every inference batch and every training step executed as real co-batched passes on this GPU
(tiny config): the dispatcher's requests become prefill/decode rows on their tenant's adapter,
training steps co-batch with the in-flight decode rows, every replica trains its own adapter slot,
round boundaries FedAvg the reporting replicas' adapters on the device and hand the mean back.
"""

import numpy as np
import pytest
import torch

import oracle
from paper_2604_16400_b200.reference import import_coserve

coserve = import_coserve()
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(coserve is None, reason="reference (coserve) not installed")]


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2604_16400_b200 import _lib, build
    build.build()
    _lib.load()


def _scenario(duration):
    from pathlib import Path

    import coserve.scenario as scenario
    here = Path(coserve.__file__).resolve()
    cands = [here.parents[2] / "configs" / "determinism.yaml",
             Path("/root/reference/pkg/configs/determinism.yaml")]
    path = next((p for p in cands if p.is_file()), None)
    if path is None:  # the installed package has no configs: the same scenario inline
        sc = scenario.scenario_from_dict({
            "duration_s": duration,
            "workloads": [{"stream_id": "chat", "family": "llama", "kind": "bursty",
                           "base_rate": 15.0, "scale": 1.0, "slo_s": 0.5}],
            "cluster": [{"family": "llama", "count": 4, "profile": {"noise_cv": 0.05}}],
            "training": {"enabled": True}, "coordinator": {"scale_a": 300.0}})
    else:
        sc = scenario.load_scenario(path)
    sc.duration_s = duration
    return sc


def _backend(sc, **kw):
    from paper_2604_16400_b200.backend import CudaLoraBackend
    from paper_2604_16400_b200.configs import CONFIGS
    from paper_2604_16400_b200.layer import AdamWConfig
    streams = sorted(sc.stream_map)
    fams = {s: c.family for s, c in sc.stream_map.items()}
    n_rep = sum(g.count for g in sc.cluster)
    return CudaLoraBackend(CONFIGS["tiny"], streams, n_rep, families=fams,
                           optimizer=AdamWConfig(lr=1e-3), **kw)


def test_engine_runs_on_the_cuda_backend():
    import coserve.engine as engine

    from paper_2604_16400_b200.backend import MeasuredWorkLog, make_engine
    # device time is scaled so a batch of 8 requests x 100 tokens takes 30 ms simulated
    import coserve.domain as domain
    sc = _scenario(30.0)
    be = _backend(sc, noise_every=5)
    assert be.calibrate(0.03) > 0
    handed_back = []
    orig = be.aggregate

    def checked(family, reporting):  # right after each FedAvg: every reporter holds the mean
        orig(family, reporting)
        fl = [be.stack.trainers[("replica", r)].flat_master for r in reporting]
        handed_back.append(all(torch.equal(fl[0], f) for f in fl))

    be.aggregate = checked
    eng = make_engine(engine, be)(sc, 3)
    # The reference's idle detection (state.py thresholds over utilization / queue / batch EWMAs)
    # decides when an FL process starts in a replay, and it depends on the load level; to run the
    # FL path deterministically here, the first state scan puts three replicas Idle, after which
    # the reference's own launcher scan (scan_and_trigger, launcher.py:112-120) starts the process.
    orig_scan = eng._launcher_scan
    forced = []

    def scan():
        if not forced:
            for rid in (1, 2, 3):
                eng.replicas[rid].set_state(domain.ReplicaState.IDLE, eng.now)
            forced.append(eng.now)
        orig_scan()

    eng._launcher_scan = scan
    led = eng.run()  # the reference's request-conservation check runs inside
    assert be.passes > 0 and be.gpu_seconds > 0
    served = [r for r in led.requests if r.complete is not None]
    assert served, "no request completed"
    # FL ran on real passes: per-replica trainers, real losses, FedAvg handed back
    assert led.fl_rounds, "no FL round"
    tr = {k: t for k, t in be.stack.trainers.items()}
    assert len(tr) >= 3 and len({t.slot for t in tr.values()}) == len(tr)
    rnd = led.fl_rounds[-1]
    losses = list(rnd["client_losses"].values())
    assert all(np.isfinite(losses)) and all(0.0 < v < 20.0 for v in losses)
    reporting = [int(k) for k in rnd["client_losses"]]
    assert handed_back and all(handed_back)
    # measured gradient-noise scale and GPU busy-time utilization
    # (the estimator was fed from real gradient norms; B_simple itself may be undefined when the
    # noise dominates at these tiny batches, then the coordinator gets the stand-in's value)
    assert any(r in be._noise and be._noise[r].g2 is not None for r in reporting)
    assert all(be.noise_scale(r) is None or be.noise_scale(r) >= 0.0 for r in reporting)
    assert all(isinstance(r.work, MeasuredWorkLog) for r in eng.replicas.values())
    assert led.util_rows and all(0.0 <= u <= 1.0 for _, _, u in led.util_rows)
    # the first round's mean loss vs the last: training on the fixed synthetic targets descends
    # (the first round starts from the scenario's nominal loss; compare measured round means)
    same = [r for r in led.fl_rounds if r["process_id"] == rnd["process_id"]]
    assert len(same) >= 2, "expected several rounds of one FL process"
    losses = [round(r["mean_loss"], 4) for r in same]
    assert same[-1]["mean_loss"] < same[0]["mean_loss"], losses


def test_aggregate_is_fedavg_and_hands_back():
    """backend.aggregate: the device mean of the reporting replicas' fp32 masters equals the
    oracle's fedavg (launcher.py:68-80 semantics) and every reporting replica gets it (masters and
    bf16 copies); a non-reporting replica keeps its own adapter."""
    from types import SimpleNamespace
    sc = _scenario(10.0)
    be = _backend(sc)
    st = be.stack
    reps = [SimpleNamespace(id=i, family="llama") for i in range(4)]
    for r in reps:
        tr = be._use_trainer(r)
        g = torch.Generator(device="cuda")
        g.manual_seed(100 + r.id)
        tr.flat_master.normal_(0.0, 0.1, generator=g)
    before3 = st.trainers[("replica", 3)].flat_master.clone()
    clients = [st.trainers[("replica", i)].flat_master.cpu().numpy().astype(np.float64)
               for i in range(3)]
    want, _ = oracle.fedavg([(c, c[:1]) for c in clients])
    be.aggregate("llama", [0, 1, 2])
    torch.cuda.synchronize()
    for i in range(3):
        t = st.trainers[("replica", i)]
        got = t.flat_master.cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-7)
        for p, s in zip(st.projections(), t.states):  # bf16 copies follow the masters
            assert torch.equal(p.B[t.slot], s.master_B.to(torch.bfloat16))
    assert torch.equal(st.trainers[("replica", 3)].flat_master, before3)


def test_infer_step_composes_the_dispatched_requests():
    """infer_step turns the dispatched requests into rows on their tenants' adapters and charges
    one prefill pass plus one real pass per distinct set of still-decoding requests."""
    from types import SimpleNamespace

    import coserve.domain as domain
    sc = _scenario(10.0)
    be = _backend(sc, latency_scale=1.0)
    reqs = [domain.Request(i, 0.0, 1.0, n, "chat") for i, n in enumerate((1, 3, 3, 7))]
    p0 = be.passes
    sec = be.infer_step(SimpleNamespace(id=0, family="llama"), reqs, 0.0)
    assert sec > 0
    assert be.passes - p0 == 3  # prefill + decode sets {3,3,7} (x2 iters) and {7} (x4 iters)
    bad = [domain.Request(9, 0.0, 1.0, 1, "unknown")]
    with pytest.raises(domain.ConfigurationError):
        be.infer_step(SimpleNamespace(id=0, family="llama"), bad, 0.0)
