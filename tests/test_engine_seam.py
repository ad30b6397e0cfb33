"""CPU: the drop-in seam into the reference engine (needs /root/reference; skipped elsewhere).

A passthrough backend installed at the seam must leave a reference run byte-identical (the
reference's own determinism criterion, tests/test_acceptance.py:390-398); a different latency
model installed at the same seam must change the run (the seam is really used)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
CFG = "/root/reference/pkg/configs/determinism.yaml"

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def coserve():
    sys.path.insert(0, REF)
    import coserve.engine as engine
    import coserve.perf as perf
    import coserve.scenario as scenario
    yield engine, perf, scenario
    sys.path.remove(REF)


def _run(engine, scenario, seed=3):
    sc = scenario.load_scenario(CFG)
    sc.duration_s = min(sc.duration_s, 60.0)
    led = engine.Engine(sc, seed).run()
    return [(r.id, r.replica, r.start, r.complete, r.outcome) for r in led.requests], led.fl_rounds


def test_passthrough_is_byte_identical(coserve):
    from paper_2604_16400_b200.backend import PassthroughBackend, install
    engine, perf, scenario = coserve
    base = _run(engine, scenario)
    with install(engine, PassthroughBackend(perf)):
        seam = _run(engine, scenario)
    assert seam == base
    assert engine.true_infer_latency is perf.true_infer_latency  # restored


def test_seam_is_used(coserve):
    from paper_2604_16400_b200.backend import install
    engine, perf, scenario = coserve

    class Faster:
        def true_infer_latency(self, profile, cfg, rng=None):
            return 0.5 * perf.true_infer_latency(profile, cfg, rng)

        def true_train_latency(self, profile, cfg, rng=None):
            return 0.5 * perf.true_train_latency(profile, cfg, rng)

    base = _run(engine, scenario)
    with install(engine, Faster()):
        fast = _run(engine, scenario)
    assert fast != base
