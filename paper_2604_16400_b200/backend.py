"""Drop-in seam into the reference engine (coserve): latency and optimizer stand-ins -> B200 layer.

The reference engine imports its hardware model by NAME (``from .perf import ...
true_infer_latency, true_train_latency, train_step``, /root/reference/pkg/src/coserve/engine.py:40)
and calls those names from the replica-step handlers (engine.py:315-317, :379-383, :395); FedAvg is
the module global ``fedavg`` of launcher.py (called at :226).  The least invasive drop-in is to
rebind exactly those names for the duration of a run — the reference's loop, dispatcher,
coordinator and launcher run unmodified:

    with install(engine_module, MeasuredLatencyBackend(cfg)):
        ledger = Engine(scenario, seed).run()

``MeasuredLatencyBackend`` answers ``true_infer_latency(profile, BatchConfig(B, b), rng)`` with the
measured CUDA-event time of a real co-batched pass on this GPU (b decode rows over the tenant
adapters + B training sequences, forward only) and ``true_train_latency`` with a full training
step (forward + backward + fused AdamW of the B sequences while b inference rows co-run), keeping
the coordinator's (B, b, t) sample interface (coordinator.py:284-288) unchanged.
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass, field

from .domain import ConfigurationError


@dataclass
class PassthroughBackend:
    """Delegates to the reference's own functions (used to prove the seam is transparent)."""

    perf_module: object

    def true_infer_latency(self, profile, cfg, rng=None):
        return self.perf_module.true_infer_latency(profile, cfg, rng)

    def true_train_latency(self, profile, cfg, rng=None):
        return self.perf_module.true_train_latency(profile, cfg, rng)


@dataclass
class MeasuredLatencyBackend:
    """Measured latencies of the B200 unified layer for the reference's (B, b) interface."""

    cfg: object                 # configs.LayerConfig
    device: str = "cuda"
    seed: int = 0
    reps: int = 3
    _stack: object = None
    _cache: dict = field(default_factory=dict)

    def _replica(self):
        if self._stack is None:
            from .replica import ReplicaStack
            self._stack = ReplicaStack(self.cfg, self.device, seed=self.seed)
        return self._stack

    def _measure(self, B: int, b: int, train: bool) -> float:
        import torch

        from .domain import InferenceItem, RowRole, TrainItem
        key = (B, b, train)
        if key in self._cache:
            return self._cache[key]
        st = self._replica()
        items = [InferenceItem(i, i % self.cfg.n_adapters, 1, RowRole.DECODE) for i in range(b)]
        tr = TrainItem(self.cfg.train_adapter, B, self.cfg.train_seq) if B > 0 else None
        if tr is None and not items:
            raise ConfigurationError("empty pass")
        plan = st.plan(tr, items)
        st.allocate(plan, distinct_synthetic=False)
        opt = train and B > 0
        st.run_step(plan, optimizer_step=opt)  # warm (sizes workspaces)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(self.reps):
            st.run_step(plan, optimizer_step=opt, backward=train)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / self.reps / 1e3
        self._cache[key] = sec
        return sec

    def true_infer_latency(self, profile, cfg, rng=None):
        if cfg.infer_batch < 1:
            raise ConfigurationError("infer_batch must be >= 1")
        return self._measure(cfg.train_batch, cfg.infer_batch, train=False)

    def true_train_latency(self, profile, cfg, rng=None):
        if cfg.train_batch < 1:
            raise ConfigurationError("train_batch must be >= 1")
        return self._measure(cfg.train_batch, cfg.infer_batch, train=True)


@dataclass
class RealTrainingBackend(MeasuredLatencyBackend):
    """Also replaces the convergence stand-in ``train_step`` (perf.py:111-126, called at
    engine.py:395): every call runs a real co-batched training step (B sequences of the trainable
    adapter, LM head + next-token CE, fused AdamW) and returns the reference's ``TrainState`` with
    the MEASURED loss — ``last_decrement`` = previous loss - new loss, so the coordinator's
    record_decrement / record_noise_scale (engine.py:396-397) consume real training signal;
    ``noise_scale`` keeps the reference's own definition on top of the real loss."""

    optimizer: object = None    # layer.AdamWConfig (None: its defaults)
    _train_stack: object = None
    _train_plans: dict = field(default_factory=dict)

    def _trainer(self):
        if self._train_stack is None:
            from .replica import ReplicaStack
            self._train_stack = ReplicaStack(self.cfg, self.device, seed=self.seed,
                                             optimizer=self.optimizer, lm_head=True)
        return self._train_stack

    def train_step(self, state, batch: int, rng=None):
        import dataclasses

        from .domain import TrainItem
        if batch < 1:
            raise ConfigurationError("training batch must be >= 1")
        st = self._trainer()
        if batch not in self._train_plans:
            plan = st.plan(TrainItem(self.cfg.train_adapter, batch, self.cfg.train_seq), [])
            st.allocate(plan, distinct_synthetic=False)
            self._train_plans[batch] = plan
        plan = self._train_plans[batch]
        if st._plan is not plan:
            st.allocate(plan, distinct_synthetic=False)
        st.run_step(plan, optimizer_step=True)
        loss = st.last_loss()
        if state.steps == 0:  # the stand-in's initial loss is a guess: anchor it to the real one
            return dataclasses.replace(state, loss=loss, initial_loss=loss, steps=1,
                                       last_decrement=0.0)
        return dataclasses.replace(state, loss=loss, steps=state.steps + 1,
                                   last_decrement=state.loss - loss)


@contextlib.contextmanager
def install(engine_module, backend):
    """Rebind the engine module's imported latency functions (and, when the backend provides
    it, ``train_step``) to ``backend`` for the block."""
    names = ["true_infer_latency", "true_train_latency"]
    if hasattr(backend, "train_step"):
        names.append("train_step")
    saved = {n: getattr(engine_module, n) for n in names}
    try:
        for n in names:
            setattr(engine_module, n, getattr(backend, n))
        yield backend
    finally:
        for n, f in saved.items():
            setattr(engine_module, n, f)
