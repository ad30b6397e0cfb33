"""CPU: the drop-in seam into the reference engine (coserve from baseline/_ref or the environment;
skipped where the reference is not installed).

* An engine built by ``backend.make_engine`` on the reference's own perf model
  (``SimulatedBackend``) reproduces a reference run byte for byte — the overrides of
  ``_start_batch`` / ``_handle_train_start`` / ``_handle_train_done`` / ``_handle_round_boundary``
  only pass numbers into the reference's handler bodies (the reference's determinism criterion,
  tests/test_acceptance.py:390-398).
* A different number at the same seam changes the run (the seam is really used).
* Errors: the package's ConfigurationError / AggregationError ARE the reference's classes, so a
  COLLM_EINVAL from the C ABI inside an engine run makes the reference's experiment runner return
  its configuration exit code 2 (experiment.py:43-48).
* ``MeasuredWorkLog`` (GPU busy time) keeps WorkLog's interface and clamping.
"""

import dataclasses
import os

import pytest

from paper_2604_16400_b200.reference import import_coserve

coserve = import_coserve(("/root/reference/pkg/src",))
pytestmark = pytest.mark.skipif(coserve is None, reason="reference (coserve) not installed")


def _cfg_path():
    from pathlib import Path
    here = Path(coserve.__file__).resolve()
    for p in (here.parents[2] / "configs" / "determinism.yaml",
              Path("/root/reference/pkg/configs/determinism.yaml")):
        if p.is_file():
            return str(p)
    return None


def _scenario(duration=60.0):
    import coserve.scenario as scenario
    path = _cfg_path()
    if path is None:
        pytest.skip("determinism.yaml not found")
    sc = scenario.load_scenario(path)
    sc.duration_s = min(sc.duration_s, duration)
    return sc


def _digest(led):
    return ([(r.id, r.replica, r.start, r.complete, r.outcome, r.loss_at_serve) for r in led.requests],
            led.fl_rounds, led.util_rows, led.sweep_rows)


def test_simulated_backend_engine_is_byte_identical():
    import coserve.domain as domain
    import coserve.engine as engine
    import coserve.perf as perf

    from paper_2604_16400_b200.backend import SimulatedBackend, make_engine
    base = engine.Engine(_scenario(), 3).run()
    Eng = make_engine(engine, SimulatedBackend(perf, domain))
    seam = Eng(_scenario(), 3).run()
    assert _digest(seam) == _digest(base)
    assert base.fl_rounds, "the scenario must exercise FL rounds (train start/done, boundary)"
    assert engine.true_infer_latency is perf.true_infer_latency  # every rebinding restored
    assert engine.train_step is perf.train_step


def test_seam_is_used():
    import coserve.domain as domain
    import coserve.engine as engine
    import coserve.perf as perf

    from paper_2604_16400_b200.backend import SimulatedBackend, make_engine

    class Faster(SimulatedBackend):
        def infer_step(self, replica, requests, now):
            return 0.5 * super().infer_step(replica, requests, now)

    base = engine.Engine(_scenario(), 3).run()
    fast = make_engine(engine, Faster(perf, domain))(_scenario(), 3).run()
    assert _digest(fast) != _digest(base)


def test_error_classes_are_the_references():
    import coserve.domain as domain
    import coserve.launcher as launcher

    from paper_2604_16400_b200 import domain as d
    from paper_2604_16400_b200 import sync
    assert d.USING_REFERENCE_CLASSES
    assert d.ConfigurationError is domain.ConfigurationError
    assert d.InvariantViolation is domain.InvariantViolation
    assert d.Request is domain.Request and d.BatchConfig is domain.BatchConfig
    assert sync.AggregationError is launcher.AggregationError


def test_abi_einval_maps_to_experiment_exit_code_2(tmp_path):
    """A COLLM_EINVAL status raised inside the engine's replica step (through _lib.check, the
    ABI's error mapping) is the reference's ConfigurationError: run_experiment returns 2."""
    import coserve.domain as domain
    import coserve.engine as engine
    import coserve.experiment as experiment
    import coserve.perf as perf

    from paper_2604_16400_b200 import _lib
    from paper_2604_16400_b200.backend import SimulatedBackend, install, make_engine

    class Failing(SimulatedBackend):
        def infer_step(self, replica, requests, now):
            st = _lib.load().collm_plan_segments(None, None, 0, 0, None, None, 0, None, None, 0,
                                                 None)
            _lib.check(st, "collm_plan_segments")  # COLLM_EINVAL -> ConfigurationError
            raise AssertionError("unreachable")

    with install(experiment, make_engine(engine, Failing(perf, domain))):
        rc = experiment.run_experiment(_cfg_path(), 3, "subflow", tmp_path / "out")
    assert rc == experiment.EXIT_CONFIG == 2
    assert experiment.Engine is engine.Engine  # restored


def test_measured_worklog_interface():
    from paper_2604_16400_b200.backend import MeasuredWorkLog
    w = MeasuredWorkLog(50.0)
    w.record(0.0, 0.25, 10.0)
    w.record(0.5, 0.75)
    assert w.sample(1.0, 1.0) == pytest.approx(0.5)
    assert w.sample(0.75, 0.5) == pytest.approx(0.25 / 0.5)
    w.record(0.8, 3.0)
    assert w.sample(2.0, 1.0) == 1.0  # clamped
    w.prune(0.9)
    assert w.busy(1.0, 1.0) == pytest.approx(0.2)
    from paper_2604_16400_b200.domain import ConfigurationError
    with pytest.raises(ConfigurationError):
        w.record(1.0, 1.0)


def test_noise_estimator_recovers_b_simple():
    """McCandlish's two-batch-size estimator on exact expectations: E|G_B|^2 = |G|^2 + tr(S)/B."""
    from paper_2604_16400_b200.backend import _NoiseEstimator
    g2, tr = 4.0, 96.0  # B_simple = 24
    est = _NoiseEstimator()
    for _ in range(5):
        est.update(4, g2 + tr / 4, 16, g2 + tr / 16)
    assert est.b_noise == pytest.approx(24.0)
    assert _NoiseEstimator().b_noise is None
