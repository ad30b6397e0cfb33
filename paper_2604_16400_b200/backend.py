"""The drop-in seam: the reference engine's replica step runs on the B200 unified layer.

The reference (coserve) is a discrete-event simulator whose replica step asks a hardware model
for numbers: ``true_infer_latency`` at ``Engine._start_batch`` (engine.py:312-333),
``true_train_latency`` at ``_handle_train_start`` (:372-388), the convergence stand-in
``train_step`` at ``_handle_train_done`` (:391-408) and the toy ``fedavg`` of ``AdapterParams`` in
``FLProcess.finalize_round`` (launcher.py:215-246, :226).  :func:`make_engine` builds an ``Engine``
subclass that overrides exactly those handlers and routes them through a :class:`ReplicaBackend`;
the reference's loop, dispatcher, coordinator, state machine and launcher run unmodified (the
override passes each measured number into the reference's own handler body, so no reference
logic is restated here):

* :class:`SimulatedBackend` answers with the reference's own perf model (byte-identical runs —
  the seam is transparent).
* :class:`CudaLoraBackend` runs the real co-batched passes on this GPU: ``infer_step`` composes a
  ``MixedBatch`` from the DISPATCHED requests (``Request.stream_id`` -> the tenant's adapter slot,
  ``output_tokens`` -> decode iterations), ``train_step`` runs the replica's training micro-batch
  co-batched with the decode rows of its in-flight inference batch (forward + backward + fused
  AdamW + LM-head CE: the measured loss), each simulated replica trains ITS OWN adapter slot
  (per-replica fp32 masters / AdamW state), ``aggregate`` averages the reporting replicas'
  adapters on the device and hands the mean back to every participant (the broadcast the
  reference omits, engine.py:478-480).  Latencies are CUDA-event times; the gradient-noise scale
  fed to ``Coordinator.record_noise_scale`` (coordinator.py:293-294) is McCandlish's B_simple
  estimated from gradient norms at two batch sizes; replica utilization (``WorkLog``,
  perf.py:129-158) becomes measured GPU busy time (:class:`MeasuredWorkLog`).

    from paper_2604_16400_b200.backend import CudaLoraBackend, make_engine
    Engine = make_engine(coserve.engine, CudaLoraBackend(cfg, streams, n_replicas))
    ledger = Engine(scenario, seed).run()
"""

from __future__ import annotations

import contextlib
import dataclasses
import math
from typing import Protocol

from .domain import ConfigurationError

# --------------------------------------------------------------------------- backend protocol


class ReplicaBackend(Protocol):
    def infer_step(self, replica, requests, now: float) -> float:
        """Run (or model) one inference batch of the dispatched ``requests`` on ``replica``;
        return its latency in seconds."""

    def train_step(self, replica, train_batch: int, concurrent_b: int, now: float) -> float:
        """Run (or model) one training step of ``train_batch`` samples while ``concurrent_b``
        inference rows of the replica's in-flight batch co-run; return its latency (s)."""

    def train_result(self, replica, train_batch: int):
        """(new reference TrainState, measured gradient-noise scale or None) of the step that
        finished (``_handle_train_done``)."""

    def aggregate(self, family: str, reporting: list[int]) -> None:
        """Round boundary: combine the reporting replicas' adapters (FedAvg) and hand the result
        back to them."""


@dataclasses.dataclass
class SimulatedBackend:
    """The reference's own hardware model (perf.py), consuming the replica RNG streams exactly as
    the reference handlers do: an engine built on it is byte-identical to the reference."""

    perf: object  # the coserve.perf module
    domain: object  # the coserve.domain module

    def infer_step(self, replica, requests, now):
        return self.perf.true_infer_latency(
            replica.profile, self.domain.BatchConfig(replica.interference_train_batch, len(requests)),
            replica.latency_rng)

    def train_step(self, replica, train_batch, concurrent_b, now):
        return self.perf.true_train_latency(
            replica.profile, self.domain.BatchConfig(train_batch, concurrent_b), replica.latency_rng)

    def train_result(self, replica, train_batch):
        return self.perf.train_step(replica.train, train_batch, replica.train_rng), None

    def aggregate(self, family, reporting):
        return None


# --------------------------------------------------------------------------- engine subclass


@contextlib.contextmanager
def _rebind(module, name: str, value):
    saved = getattr(module, name)
    setattr(module, name, value)
    try:
        yield
    finally:
        setattr(module, name, saved)


class MeasuredWorkLog:
    """``perf.WorkLog`` (perf.py:129-158) on measured GPU busy time: every recorded interval is a
    pass whose duration was timed with CUDA events, so utilization over a window is the fraction
    of the window the replica's GPU work covered (clamped to [0, 1]); the reference's work units
    and capacity are not needed."""

    def __init__(self, capacity: float | None = None) -> None:
        self.capacity = capacity
        self._entries: list[tuple[float, float]] = []

    def record(self, start: float, end: float, units: float = 0.0) -> None:
        if end <= start:
            raise ConfigurationError("work interval must have positive duration")
        self._entries.append((start, end))

    def prune(self, horizon: float) -> None:
        self._entries = [e for e in self._entries if e[1] > horizon]

    def busy(self, now: float, window: float) -> float:
        lo = now - window
        return sum(max(0.0, min(e, now) - max(s, lo)) for s, e in self._entries)

    def sample(self, now: float, window: float) -> float:
        if window <= 0:
            raise ConfigurationError("utilization window must be positive")
        return min(1.0, self.busy(now, window) / window)


def make_engine(engine_module, backend: ReplicaBackend, measured_worklog: bool | None = None):
    """An ``Engine`` subclass of the reference ``engine_module`` (coserve.engine) whose replica
    step goes through ``backend``.  Each override computes the backend's number first and then
    runs the reference's own handler with the engine module's hardware-model names rebound to
    return it, so the reference's bookkeeping (busy time, ledger stamps, coordinator samples,
    event scheduling, FL round protocol) is unchanged."""
    base = engine_module.Engine
    if measured_worklog is None:
        measured_worklog = isinstance(backend, CudaLoraBackend)

    class CollmEngine(base):
        collm_backend = backend

        def __init__(self, scenario, seed, policy_name="subflow"):
            super().__init__(scenario, seed, policy_name)
            if measured_worklog:
                for r in self.replicas.values():
                    r.work = MeasuredWorkLog(r.profile.capacity)
            hook = getattr(backend, "attach", None)
            if hook is not None:
                hook(self)

        # engine.py:312-333
        def _start_batch(self, replica, requests, now):
            latency = backend.infer_step(replica, requests, now)
            with _rebind(engine_module, "true_infer_latency", lambda *a, **k: latency):
                super()._start_batch(replica, requests, now)

        # engine.py:372-388
        def _handle_train_start(self, ev):
            replica = self.replicas[ev.payload]
            runtime = self.processes.get(replica.family)
            if runtime is None or replica.round_steps_left <= 0:
                return
            latency = backend.train_step(replica, replica.batch_cfg.train_batch,
                                         replica.current_infer_b, self.now)
            with _rebind(engine_module, "true_train_latency", lambda *a, **k: latency):
                super()._handle_train_start(ev)

        # engine.py:391-408
        def _handle_train_done(self, ev):
            replica = self.replicas[ev.payload]
            runtime = self.processes.get(replica.family)
            if runtime is None:
                return
            state, noise = backend.train_result(replica, replica.batch_cfg.train_batch)
            coord = runtime.coordinator
            patched = noise is not None
            if patched:  # the measured B_noise instead of the stand-in's property (perf.py:105-108)
                orig = coord.record_noise_scale
                coord.record_noise_scale = lambda _v: orig(noise)
            try:
                with _rebind(engine_module, "train_step", lambda *a, **k: state):
                    super()._handle_train_done(ev)
            finally:
                if patched:
                    del coord.record_noise_scale

        # engine.py:415-466 (FLProcess.finalize_round -> fedavg, launcher.py:215-246)
        def _handle_round_boundary(self, ev):
            family = ev.payload
            runtime = self.processes.get(family)
            reporting = None
            if runtime is not None and runtime.process.round_done:
                proc = runtime.process
                reporting = [rid for rid in proc._round.participants if rid in proc._clients]
            super()._handle_round_boundary(ev)
            if reporting:
                backend.aggregate(family, reporting)

    CollmEngine.__name__ = CollmEngine.__qualname__ = "CollmEngine"
    return CollmEngine


@contextlib.contextmanager
def install(module, engine_cls):
    """Rebind ``module.Engine`` (e.g. coserve.experiment, which builds ``Engine(...)`` by name at
    experiment.py:21-28) to ``engine_cls`` for the block: the reference's CLI / experiment runner
    then drives the CUDA backend unchanged, including its exit-code mapping."""
    with _rebind(module, "Engine", engine_cls):
        yield engine_cls


# --------------------------------------------------------------------------- the CUDA backend


@dataclasses.dataclass
class _NoiseEstimator:
    """McCandlish et al.'s unbiased estimates from gradient norms at two batch sizes (App. A):
    |G|^2 ~ (B_big |G_big|^2 - B_small |G_small|^2) / (B_big - B_small),
    tr(S) ~ (|G_small|^2 - |G_big|^2) / (1/B_small - 1/B_big); both smoothed by EMA, then
    B_simple = tr(S) / |G|^2 (in the units of B: training samples)."""

    decay: float = 0.9
    g2: float | None = None
    trace: float | None = None

    def update(self, b_small: float, g2_small: float, b_big: float, g2_big: float) -> None:
        g2 = (b_big * g2_big - b_small * g2_small) / (b_big - b_small)
        tr = (g2_small - g2_big) / (1.0 / b_small - 1.0 / b_big)
        self.g2 = g2 if self.g2 is None else self.decay * self.g2 + (1 - self.decay) * g2
        self.trace = tr if self.trace is None else self.decay * self.trace + (1 - self.decay) * tr

    @property
    def b_noise(self) -> float | None:
        if self.g2 is None or self.trace is None or self.g2 <= 0:
            return None  # noise dominates the signal: B_simple undefined (unbounded)
        return max(0.0, self.trace) / self.g2  # tr(S) <= 0: no measurable noise


class CudaLoraBackend:
    """Real co-batched passes for every simulated replica of one engine on this GPU.

    One frozen base model (a :class:`ReplicaStack`) is shared by the engine's replicas (one
    device); adapter slots [0, n_streams) hold the tenants' adapters (stream_id -> slot, sorted),
    slots [n_streams, n_streams + n_replicas) each replica's own trainable adapter (initialised
    from its family's tenant adapter when the replica first trains).  An inference request
    contributes ``prompt_tokens`` prefill rows on its tenant's adapter and ``output_tokens - 1``
    decode iterations; a batch's latency is its prefill pass plus, for every distinct set of
    still-decoding requests, one REAL decode pass of that set times the iterations it lasts
    (passes over the same rows do the same projection work).  ``latency_scale`` maps device
    seconds to simulated seconds (1.0: measured time as is)."""

    def __init__(self, cfg, streams, n_replicas: int, device="cuda", seed: int = 0,
                 prompt_tokens: int = 16, latency_scale: float = 1.0, optimizer=None,
                 lm_head: bool = True, noise_every: int = 10, families: dict | None = None,
                 dataset_seqs: int = 8):
        from .replica import ReplicaStack
        streams = sorted(streams)
        if not streams or n_replicas < 1:
            raise ConfigurationError("need >= 1 stream and >= 1 replica")
        if prompt_tokens < 1 or latency_scale <= 0:
            raise ConfigurationError("prompt_tokens >= 1 and latency_scale > 0 required")
        self.slot_of_stream = {s: i for i, s in enumerate(streams)}
        self.n_streams = len(streams)
        self.family_slot = {}
        for s, fam in (families or {}).items():
            self.family_slot.setdefault(fam, self.slot_of_stream[s])
        n_ad = self.n_streams + n_replicas
        self.cfg = dataclasses.replace(cfg, n_adapters=n_ad, train_adapter=self.n_streams)
        self.stack = ReplicaStack(self.cfg, device, seed=seed, optimizer=optimizer,
                                  lm_head=lm_head, trainer=False)
        self.prompt_tokens = prompt_tokens
        self.latency_scale = latency_scale
        self.noise_every = max(1, noise_every)
        self.dataset_seqs = max(1, dataset_seqs)
        self._data = None
        self._cursor = 0
        self._inflight: dict[int, list] = {}
        self._results: dict[int, tuple] = {}
        self._losses: dict[int, float] = {}
        self._noise: dict[int, _NoiseEstimator] = {}
        self._steps: dict[int, int] = {}
        self.gpu_seconds = 0.0
        self.passes = 0
        self._engine = None

    # -- wiring
    def attach(self, engine) -> None:
        self._engine = engine
        for sid, scfg in engine.stream_map.items():
            if sid not in self.slot_of_stream:
                raise ConfigurationError(f"stream {sid!r} has no tenant adapter slot")
            self.family_slot.setdefault(scfg.family, self.slot_of_stream[sid])
        if len(engine.replicas) > self.cfg.n_adapters - self.n_streams:
            raise ConfigurationError(f"{len(engine.replicas)} replicas, backend sized for "
                                     f"{self.cfg.n_adapters - self.n_streams}")
        # every replica starts from its family's adapter: anchor the reference's nominal initial
        # loss (scenario training.initial_loss) to the MEASURED loss of that adapter on the
        # training data, so FL rounds (early stop, quality updates, launcher.py:171-246) compare
        # real losses with real losses
        from .domain import TrainItem
        for fam in sorted({r.family for r in engine.replicas.values()}):
            reps = sorted((r for r in engine.replicas.values() if r.family == fam),
                          key=lambda r: r.id)
            tr = self._use_trainer(reps[0])
            self._pass(TrainItem(tr.slot, 1, self.cfg.train_seq), [], backward=True,
                       optimizer_step=False)
            l0 = self.stack.last_loss()
            for r in reps:
                r.train = dataclasses.replace(r.train, loss=l0, initial_loss=l0)
                self._losses[r.id] = l0

    def calibrate(self, target_seconds: float, batch: int = 8, output_tokens: int = 100) -> float:
        """Set ``latency_scale`` so that an inference batch of ``batch`` requests generating
        ``output_tokens`` tokens each (on the first tenant) takes ``target_seconds`` simulated —
        e.g. the reference profile's latency for that batch (``perf.true_infer_latency``), so a
        reference scenario replays at its own load level on a model much smaller or faster than
        the one its profile describes.  Returns the scale."""
        from types import SimpleNamespace

        from .domain import Request
        if target_seconds <= 0 or batch < 1 or output_tokens < 1:
            raise ConfigurationError("calibrate: positive target, batch and output_tokens")
        stream = next(iter(self.slot_of_stream))
        reqs = [Request(-1 - i, 0.0, 1.0, output_tokens, stream) for i in range(batch)]
        saved, self.latency_scale = self.latency_scale, 1.0
        probe = SimpleNamespace(id=-1, family=None)
        self.infer_step(probe, reqs, 0.0)  # warm (buffers, workspaces)
        sec = self.infer_step(probe, reqs, 0.0)
        self._inflight.pop(-1, None)
        self.latency_scale = target_seconds / sec if sec > 0 else saved
        return self.latency_scale

    def trainer_slot(self, replica_id: int) -> int:
        return self.n_streams + replica_id

    def _use_trainer(self, replica):
        st = self.stack
        key = ("replica", replica.id)
        if key not in st.trainers:
            src = self.family_slot.get(replica.family, 0)
            st.add_trainer(key, self.trainer_slot(replica.id), copy_from=src)
        return st.use_trainer(key)

    # -- one measured pass
    def _pass(self, train, items, backward: bool, optimizer_step: bool = True) -> float:
        import torch
        st = self.stack
        plan = st.plan(train, items)
        a = st.allocate(plan, distinct_synthetic=False, reuse=True)
        if plan.n_train:
            self._load_training_data(a, plan.n_train)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st.run_step(plan, optimizer_step=optimizer_step, backward=backward)
        e1.record()
        e1.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        self.gpu_seconds += sec
        self.passes += 1
        return sec

    def _load_training_data(self, acts, n_rows: int) -> None:
        """The training rows of a pass read a fixed synthetic dataset of ``dataset_seqs``
        sequences (seeded: the layer-0 hidden states, the path's attention-output / MLP-activation
        stand-ins that feed o / down (replica.py), and the next-token targets) in epoch order:
        sequence j of the micro-batch is dataset sequence (cursor + j) mod dataset_seqs, the
        cursor advancing by the micro-batch size every step — whatever micro-batch size the
        coordinator picks, every sequence is visited and the loss is measured on the same data
        (no checkpoints or corpora offline: the 'fine-tuning task' is fitting these targets)."""
        import torch
        seq = self.cfg.train_seq
        if self._data is None:
            g = torch.Generator(device=self.stack.device)
            g.manual_seed(7919)
            n = self.dataset_seqs * seq
            dev, m = self.stack.device, self.cfg.model

            def rnd(cols):
                return torch.randn(n, cols, device=dev, generator=g).to(torch.bfloat16)
            y = torch.randint(0, m.vocab, (n,), device=dev, generator=g, dtype=torch.int32)
            self._data = {"X0": rnd(m.hidden), "Xo": rnd(m.hidden), "Xd": rnd(m.intermediate),
                          "labels": y}
        D = self._data
        targets = [(acts["X"][0], D["X0"])]
        targets += [(t, D["Xo"]) for t in acts["Xo"]] + [(t, D["Xd"]) for t in acts["Xd"]]
        if "labels" in acts:
            targets.append((acts["labels"], D["labels"]))
        for j, r0 in enumerate(range(0, n_rows, seq)):
            d = ((self._cursor + j) % self.dataset_seqs) * seq
            k = min(seq, n_rows - r0)
            for dst, src in targets:
                dst[r0:r0 + k].copy_(src[d:d + k])

    def _decode_items(self, requests):
        from .domain import InferenceItem, RowRole
        return [InferenceItem(r.id, self.slot_of_stream[r.stream_id], 1, RowRole.DECODE)
                for r in requests]

    # -- ReplicaBackend
    def infer_step(self, replica, requests, now):
        from .domain import InferenceItem, RowRole
        for r in requests:
            if r.stream_id not in self.slot_of_stream:
                raise ConfigurationError(f"request {r.id}: stream {r.stream_id!r} has no adapter")
        self._inflight[replica.id] = list(requests)
        items = [InferenceItem(r.id, self.slot_of_stream[r.stream_id], self.prompt_tokens,
                               RowRole.PREFILL) for r in requests]
        sec = self._pass(None, items, backward=False)
        # decode iterations: request r decodes output_tokens - 1 more tokens after the prefill
        left = sorted(requests, key=lambda r: (r.output_tokens, r.id))
        done = 1
        i = 0
        while i < len(left):
            active = left[i:]
            upto = active[0].output_tokens
            if upto > done:
                sec += self._pass(None, self._decode_items(active), backward=False) * (upto - done)
                done = upto
            while i < len(left) and left[i].output_tokens <= done:
                i += 1
        return sec * self.latency_scale

    def train_step(self, replica, train_batch, concurrent_b, now):
        from .domain import TrainItem
        if train_batch < 1:
            raise ConfigurationError("training batch must be >= 1")
        tr = self._use_trainer(replica)
        seq = self.cfg.train_seq
        co = self._decode_items(self._inflight.get(replica.id, [])[:concurrent_b])
        k = self._steps.get(replica.id, 0)
        self._steps[replica.id] = k + 1
        self._cursor = (k * train_batch) % self.dataset_seqs
        if k % self.noise_every == 0:
            sec = self._train_with_noise_estimate(replica, tr, train_batch, seq, co)
        else:
            sec = self._pass(TrainItem(tr.slot, train_batch, seq), co, backward=True)
        loss = self.stack.last_loss()
        prev = self._losses.get(replica.id)
        self._losses[replica.id] = loss
        self._results[replica.id] = (loss, None if prev is None else prev - loss)
        return sec * self.latency_scale

    def _train_with_noise_estimate(self, replica, tr, B, seq, co) -> float:
        """One training step that also measures |G|^2 at two batch sizes: the gradient of a
        half-size sub-batch (first half of the sequences, or of the tokens when B = 1) and of
        the full micro-batch, both stored (not applied); then the AdamW step is applied from the
        full gradient.  Only the full pass is charged as the step's latency."""
        import torch

        from .domain import TrainItem
        st = self.stack
        if B >= 2:
            small, b_small, b_big = TrainItem(tr.slot, B // 2, seq), B // 2, B
        else:
            small, b_small, b_big = TrainItem(tr.slot, 1, max(1, seq // 2)), 0.5, 1.0
        self._pass(small, [], backward=True, optimizer_step=False)
        g2_small = self._loss_grad_norm2(tr)
        sec = self._pass(TrainItem(tr.slot, B, seq), co, backward=True, optimizer_step=False)
        g2_big = self._loss_grad_norm2(tr)
        st.opt.advance()
        st.apply_optimizer()
        if b_big != b_small:
            self._noise.setdefault(replica.id, _NoiseEstimator()).update(b_small, g2_small,
                                                                         b_big, g2_big)
        return sec

    def _loss_grad_norm2(self, tr) -> float:
        """|G|^2 over the parameters whose gradient is the true mean gradient of the training
        loss: the top layer's last projection (its dY is the LM head's dX, normalised by the
        number of target tokens).  The other projections' output grads are synthetic stand-ins
        of the path (replica.py), whose row SUMS would grow with the batch and bias the estimate."""
        import torch
        st = tr.states[-1]
        return float(torch.dot(st.grad_B.reshape(-1), st.grad_B.reshape(-1))
                     + torch.dot(st.grad_AT.reshape(-1), st.grad_AT.reshape(-1)))

    def noise_scale(self, replica_id: int) -> float | None:
        est = self._noise.get(replica_id)
        return None if est is None else est.b_noise

    def train_result(self, replica, train_batch):
        loss, dec = self._results.pop(replica.id)
        s = replica.train
        if dec is None:  # first real step of this replica: anchor the stand-in's initial loss
            new = dataclasses.replace(s, loss=loss, initial_loss=loss, steps=s.steps + 1,
                                      last_decrement=0.0)
        else:
            # the real (noisy, possibly negative) drop: the coordinator EWMA-smooths it
            # (coordinator.py:324-334)
            new = dataclasses.replace(s, loss=loss, steps=s.steps + 1,
                                      last_decrement=s.loss - loss if math.isfinite(loss) else 0.0)
        return new, self.noise_scale(replica.id)

    def aggregate(self, family, reporting):
        """FedAvg of the reporting replicas' fp32 master adapters (launcher.py:68-80: element-wise
        mean of B and of A), on the device, handed back to every reporting replica (bf16 copies
        rewritten).  One replica per GPU would do this with ``sync.fedavg_params`` (NCCL
        allreduce) + ``registry.broadcast_adapter``; here the engine's replicas share a GPU."""
        import torch
        st = self.stack
        trs = [st.trainers[("replica", r)] for r in reporting if ("replica", r) in st.trainers]
        if not trs:
            return
        mean = torch.stack([t.flat_master for t in trs]).mean(dim=0)
        for t in trs:
            t.flat_master.copy_(mean)
            st.use_trainer(t.key)
            st.refresh_from_master()
