"""One replica's co-batched step through the whole LoRA-augmented projection stack.

This is the B200 body of the reference's replica step: ``Engine._start_batch`` (inference,
/root/reference/pkg/src/coserve/engine.py:312-333) and ``_handle_train_start`` /
``_handle_train_done`` (training, engine.py:372-408), which today call the latency surfaces
``true_infer_latency`` / ``true_train_latency`` and the convergence stand-in ``train_step``
(perf.py:62-126).  Here one pass runs the forward of every row (inference + training) through
every projection of every layer and the backward + fused AdamW of the training rows, over frozen
bf16 base weights resident in HBM.

Data flow per layer l (attention / MLP nonlinearities are outside this hot path):
  X_l --qkv--> ;  Xo_l --o--> ;  X_l --gate_up--> ;  Xd_l --down--> X_{l+1}
where Xo_l / Xd_l (attention output / MLP activation) are synthetic device-resident stand-ins.
Backward runs from the top: dY(down_l) = dX(qkv_{l+1}) (dY_top for the last layer); the other
projections' output grads are synthetic stand-ins.  Every projection computes dX, dA, dB and its
fused AdamW step, as the metric's FLOP count assumes.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import _lib, ops
from .configs import LayerConfig
from .domain import ConfigurationError, InferenceItem, MixedBatch, TrainItem
from .layer import AdamWConfig, LMHead, LoraProjection, OptimizerState, TrainState
from .segments import DevicePlan, HostPlan, build_mixed_batch, plan_segments, uniform_plan

ENTRY = ("qkv", "q", "k", "v", "gate_up", "gate", "up")


@dataclass
class Trainer:
    """One trainable adapter of the replica (the reference's per-replica ``adapter``,
    engine.py:92, trained by that replica's FL client): its device slot, the per-projection fp32
    masters / AdamW moments / gradients (re-homed at creation into ONE flat master buffer and ONE
    flat gradient buffer, so a cross-replica sync is a single collective) and its optimizer step."""

    key: object
    slot: int
    states: list[TrainState]
    opt: OptimizerState
    flat_master: torch.Tensor
    flat_grad: torch.Tensor


@dataclass
class StepPlan:
    batch: MixedBatch
    host: HostPlan
    device: DevicePlan
    train_host: HostPlan | None
    train_device: DevicePlan | None
    # K9 attention (ReplicaStack(attention=True)): sequences of the pass as row ranges — the
    # training sequences (train.batch x train.seq_len) then each inference request's rows — and
    # the training sequences alone (the backward); device int32 + the longest length
    attn_seq: list | None = None           # sequence boundaries [0, ..., T] (host)
    attn_rows: tuple | None = None         # (row_start, row_end) int32 [T] on the device

    @property
    def n_rows(self) -> int:
        return self.batch.n_rows

    @property
    def n_train(self) -> int:
        return self.batch.n_train_rows


class ReplicaStack:
    def __init__(self, cfg: LayerConfig, device: torch.device | str = "cuda", seed: int = 0,
                 optimizer: AdamWConfig | None = None, init: bool = True, lm_head: bool = False,
                 trainer: bool = True, attention: bool = False):
        self.cfg = cfg
        # attention: K9 causal attention between q|k|v and o (its output IS o's input; its
        # backward turns o's dX into q|k|v's dY) over the pass's sequences
        self.attention = attention
        if attention:
            if cfg.projections[0].name != "qkv" or cfg.model.hidden % 128 or cfg.model.kv_dim % 128:
                raise ConfigurationError("attention needs a fused q|k|v projection and 128-wide heads")
            self.n_heads = cfg.model.hidden // 128
            self.n_kv_heads = cfg.model.kv_dim // 128
        self.device = torch.device(device)
        self.specs = cfg.projections
        L = cfg.model.layers
        self.layers: list[list[LoraProjection]] = [
            [LoraProjection(spec, cfg.n_adapters, self.device) for spec in self.specs]
            for _ in range(L)]
        # lm_head: the training rows' real next-token CE (K7) drives the backward from the top
        # (dY_top = its dX) and gives the step's training loss; without it dY_top is synthetic
        self.head = LMHead(cfg.model.hidden, cfg.model.vocab, self.device) if lm_head else None
        self._loss: torch.Tensor | None = None
        self.optimizer_cfg = optimizer
        self.trainers: dict[object, Trainer] = {}
        self.active: Trainer | None = None
        self.seed = seed
        self._graph: torch.cuda.CUDAGraph | None = None
        self._make_default_trainer = trainer
        self._acts: dict | None = None
        if init:
            self.init_synthetic(seed)
        self._side: torch.cuda.Stream | None = None
        self.overlap = False
        # how a projection's shrink overlaps its GEMM: "pdl" (default) = same stream, the GEMM
        # launched programmatically dependent on the shrink (deadlock-free by construction,
        # 2-3 % faster); "flag" = shrink on the side stream + a device completion flag
        self.overlap_mode = os.environ.get("COLLM_OVERLAP_MODE", "pdl")
        self._gen: torch.Tensor | None = None
        self._gen_count = 0
        self._sig: torch.Tensor | None = None

    # ------------------------------------------------------------------ weights
    @torch.no_grad()
    def init_synthetic(self, seed: int) -> None:
        """Random-init weights of the named architecture (no checkpoints offline):
        W ~ N(0, 0.02^2); A ~ U(+-1/sqrt(K)); B ~ N(0, 0.02^2) (non-zero, so the expand path is
        exercised); scale = alpha / r."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        r = self.cfg.rank
        for layer in self.layers:
            for proj in layer:
                sp = proj.spec
                K, rp = sp.in_features, sp.r_pad
                proj.W.normal_(0.0, 0.02, generator=g)
                proj.refresh_transpose()
                lim = 1.0 / (K ** 0.5)
                proj.A.zero_()
                proj.B.zero_()
                bnd = sp.sub_bounds
                for s in range(len(sp.subs)):
                    a = torch.empty(self.cfg.n_adapters, r, K, device=self.device)
                    a.uniform_(-lim, lim, generator=g)
                    proj.A[:, s * rp:s * rp + r] = a.to(torch.bfloat16)
                    b = torch.empty(self.cfg.n_adapters, sp.subs[s], r, device=self.device)
                    b.normal_(0.0, 0.02, generator=g)
                    proj.B[:, bnd[s]:bnd[s + 1], :r] = b.to(torch.bfloat16)
                proj.scale.fill_(sp.alpha / r)
        if self.head is not None:
            self.head.W.normal_(0.0, 0.02, generator=g)
            self.head.refresh_transpose()
        self.trainers.clear()
        self.active = None
        if self._make_default_trainer:
            self.add_trainer("default", self.cfg.train_adapter)

    # ------------------------------------------------------------------ trainable adapters
    @property
    def opt(self) -> OptimizerState:
        return self._require_trainer().opt

    @property
    def train_slot(self) -> int:
        return self._require_trainer().slot

    def _require_trainer(self) -> Trainer:
        if self.active is None:
            raise ConfigurationError("no trainable adapter (add_trainer)")
        return self.active

    def add_trainer(self, key, slot: int, copy_from: int | None = None) -> Trainer:
        """Start fine-tuning device slot ``slot`` as trainer ``key``: fp32 masters from the slot's
        bf16 weights (after copying adapter ``copy_from``'s weights into it, when given), fresh
        AdamW state, and the flat master / gradient buffers — built here, once, so nothing later
        re-homes tensors a captured graph points at.  The new trainer becomes the active one."""
        if not 0 <= slot < self.cfg.n_adapters:
            raise ConfigurationError(f"trainer slot {slot} outside [0, {self.cfg.n_adapters})")
        if any(t.slot == slot and k != key for k, t in self.trainers.items()):
            raise ConfigurationError(f"slot {slot} is already trained by another trainer")
        if self._graph is not None:
            raise ConfigurationError("add trainers before capturing a graph")
        states = []
        with torch.no_grad():
            for p in self.projections():
                if copy_from is not None and copy_from != slot:
                    p.A[slot].copy_(p.A[copy_from])
                    p.B[slot].copy_(p.B[copy_from])
                    p.scale[slot:slot + 1].copy_(p.scale[copy_from:copy_from + 1])
                states.append(p.make_trainable(slot))
        flat_m = self._flatten(states, ("master_B", "master_AT"), copy=True)
        flat_g = self._flatten(states, ("grad_B", "grad_AT"), copy=False)
        tr = Trainer(key, slot, states, OptimizerState(self.optimizer_cfg, self.device), flat_m,
                     flat_g)
        self.trainers[key] = tr
        self.use_trainer(key)
        return tr

    def use_trainer(self, key) -> Trainer:
        """Make trainer ``key`` the one the next steps train (eager steps; a captured graph is
        bound to the trainer active at capture)."""
        tr = self.trainers.get(key)
        if tr is None:
            raise ConfigurationError(f"unknown trainer {key!r}")
        for p, st in zip(self.projections(), tr.states):
            p.train_state = st
        self.active = tr
        return tr

    def _flatten(self, states, names, copy: bool) -> torch.Tensor:
        total = sum(getattr(st, n).numel() for st in states for n in names)
        flat = torch.zeros(total, dtype=torch.float32, device=self.device)
        off = 0
        for st in states:
            for n in names:
                t = getattr(st, n)
                view = flat[off:off + t.numel()].view(t.shape)
                if copy:
                    view.copy_(t)
                setattr(st, n, view)
                off += t.numel()
        return flat

    def projections(self):
        for layer in self.layers:
            yield from layer

    def trainable_tensors(self, which: str = "master") -> list[torch.Tensor]:
        """The active trainer's fp32 tensors across the stack (for cross-replica sync):
        'master' = parameters (fedavg mode), 'grad' = gradients (grad-sync mode)."""
        out = []
        for st in self._require_trainer().states:
            out += [st.master_B, st.master_AT] if which == "master" else [st.grad_B, st.grad_AT]
        return out

    @property
    def flat_grad(self) -> torch.Tensor:
        """The active trainer's gradients as ONE flat fp32 buffer (every projection's grad_B /
        grad_AT are views of it): the cross-replica sync is a single NCCL allreduce."""
        return self._require_trainer().flat_grad

    def grad_buckets(self) -> list[torch.Tensor]:
        """Per-layer views of the active trainer's flat gradient buffer (layer l's projections
        are contiguous in it): the buckets a grad-mode sync reduces as soon as layer l's K5 has
        written them, overlapping the backward of the layers below."""
        tr = self._require_trainer()
        per_layer = len(self.specs)
        out, off = [], 0
        for l in range(self.cfg.model.layers):
            n = sum(st.grad_B.numel() + st.grad_AT.numel()
                    for st in tr.states[l * per_layer:(l + 1) * per_layer])
            out.append(tr.flat_grad[off:off + n])
            off += n
        return out

    def apply_optimizer_layer(self, l: int) -> None:
        """AdamW of layer ``l``'s projections from their grad buffers (current stream)."""
        for p in self.layers[l]:
            p.apply_optimizer(self.opt)

    @property
    def flat_master(self) -> torch.Tensor:
        """The active trainer's fp32 master parameters as ONE flat buffer (fedavg mode)."""
        return self._require_trainer().flat_master

    def refresh_from_master(self) -> None:
        """Rewrite every bf16 copy of the active trainer's adapter from its fp32 masters (after
        an average / broadcast of ``flat_master``)."""
        for p in self.projections():
            p.refresh_from_master()

    def apply_optimizer(self) -> None:
        """AdamW of the active trainer from its (e.g. allreduced) gradient buffers, on the
        current stream, using the step ``opt.advance()`` already set."""
        for p in self.projections():
            p.apply_optimizer(self.opt)

    # ------------------------------------------------------------------ plans
    def _shrink_tc_ctas(self) -> tuple[int | None, int | None]:
        """CTAs of the K1' (TMA + tcgen05) shrink for the forward and the dH pass: the rank-space
        partition when one is set (None: DevicePlan takes collm_get_rank_sms), else the
        whole-GPU override COLLM_SHRINK_TC_FWD / COLLM_SHRINK_TC_DH (0 = the mma.sync K1)."""
        env = os.environ
        return tuple(int(env[k]) if env.get(k) else None
                     for k in ("COLLM_SHRINK_TC_FWD", "COLLM_SHRINK_TC_DH"))

    def plan(self, train: TrainItem | None, items: list[InferenceItem]) -> StepPlan:
        for it in items:
            if it.adapter >= self.cfg.n_adapters:
                raise ConfigurationError(
                    f"request {it.request_id}: adapter {it.adapter} is not a registered slot "
                    f"(n_adapters={self.cfg.n_adapters})")
        mb = build_mixed_batch(train, items)
        hp = plan_segments(mb.seg_start, mb.seg_adapter)
        fwd_ctas, dh_ctas = self._shrink_tc_ctas()
        dp = DevicePlan(hp, self.device, expand=False, tc_ctas=fwd_ctas)
        th = td = None
        if mb.n_train_rows:
            if mb.train_adapter != self.train_slot:
                raise ConfigurationError(
                    f"training rows use adapter {mb.train_adapter}, the replica trains "
                    f"{self.train_slot}")
            th = uniform_plan(mb.n_train_rows, mb.train_adapter)
            td = DevicePlan(th, self.device, tc_ctas=dh_ctas)
        sp = StepPlan(mb, hp, dp, th, td)
        if self.attention:
            # sequences: training sequences of seq_len rows, then maximal runs of one request
            bounds = []
            if train is not None:
                bounds = list(range(0, mb.n_train_rows + 1, train.seq_len))
            else:
                bounds = [0]
            req = mb.row_request
            for t in range(mb.n_train_rows + 1, mb.n_rows):
                if req[t] != req[t - 1]:
                    bounds.append(t)
            if mb.n_rows > bounds[-1]:
                bounds.append(mb.n_rows)
            sp.attn_seq = bounds
            sp.attn_rows = ops.seq_rows(bounds, self.device)
        return sp

    # ------------------------------------------------------------------ activations
    def allocate(self, plan: StepPlan, distinct_synthetic: bool | None = None, seed: int = 1,
                 reuse: bool = False) -> dict:
        """Device buffers of one pass.  Synthetic stand-ins (Xo, Xd, the non-chained output grads)
        are per layer when they fit comfortably in HBM, else shared across layers (same traffic,
        inputs are far larger than L2 either way).  ``reuse``: keep the current buffers when they
        have room for this plan's rows (every kernel takes its row counts from the plan), so a
        serving loop changing its batch every pass does not reallocate."""
        T, Ttr = plan.n_rows, plan.n_train
        a = self._acts
        if (reuse and a is not None and a["cap"] >= T and a["cap_train"] >= Ttr
                and (distinct_synthetic is None or a["distinct_synthetic"] == distinct_synthetic)):
            self._plan = plan
            if Ttr and "labels" in a:
                a["n_valid"] = Ttr
            return a
        old = None
        if reuse and a is not None:  # grow to cover both the old and the new sizes
            T, Ttr = max(T, a["cap"]), max(Ttr, a["cap_train"])
            distinct_synthetic = a["distinct_synthetic"]
            old, self._acts, a = a, None, None
        h = self.cfg.model.hidden
        i = self.cfg.model.intermediate
        L = self.cfg.model.layers
        dev = self.device
        bf = torch.bfloat16
        per_layer_bytes = 2 * (T * h + T * i + Ttr * sum(s.out_features for s in self.specs))
        if self.attention:  # per-layer q|k|v outputs and their gradients (the attention backward)
            per_layer_bytes += 2 * (T + Ttr) * self.specs[0].out_features
        if distinct_synthetic is None:
            free, _ = torch.cuda.mem_get_info(dev)
            distinct_synthetic = per_layer_bytes * L < 0.5 * free
        g = torch.Generator(device=dev)
        g.manual_seed(seed)

        def rnd(*shape):
            return torch.randn(*shape, device=dev, generator=g, dtype=torch.float32).to(bf)

        n_syn = L if distinct_synthetic else 1
        acts = {
            "cap": T, "cap_train": Ttr,
            "distinct_synthetic": distinct_synthetic,
            "X": [torch.empty(T, h, dtype=bf, device=dev) for _ in range(L + 1)],
            "Xo": [rnd(T, h) for _ in range(n_syn)],
            "Xd": [rnd(T, i) for _ in range(n_syn)],
            "dY": [{s.name: rnd(Ttr, s.out_features) for s in self.specs
                    if s.name != "down"} for _ in range(n_syn)] if Ttr else [],
            "dY_top": rnd(Ttr, h) if Ttr else None,
            "Y": {s.name: torch.empty(T, s.out_features, dtype=bf, device=dev)
                  for s in self.specs if s.name != "down"},
            "dX_first": [torch.empty(Ttr, h, dtype=bf, device=dev) for _ in range(L)] if Ttr else [],
            "dX": {s.name: torch.empty(Ttr, s.in_features, dtype=bf, device=dev)
                   for s in self.specs} if Ttr else {},
        }
        acts["X"][0].copy_(rnd(T, h))
        if self.attention:
            nq = self.specs[0].out_features
            # attention outputs (o's inputs) per layer, written by K9 every pass
            acts["Xo"] = [torch.empty(T, h, dtype=bf, device=dev) for _ in range(L)]
            acts["Yqkv"] = [torch.empty(T, nq, dtype=bf, device=dev) for _ in range(L)]
            acts["lse"] = torch.zeros(L, self.n_heads, T, dtype=torch.float32, device=dev)
            acts["dqkv"] = [torch.empty(Ttr, nq, dtype=bf, device=dev) for _ in range(L)] if Ttr else []
            acts["delta"] = torch.zeros(self.n_heads, max(1, T), dtype=torch.float32, device=dev)
        if self.head is not None and Ttr:
            # next-token targets of the training rows (synthetic token ids; no dataset offline)
            acts["labels"] = torch.randint(0, self.cfg.model.vocab, (Ttr,), device=dev,
                                           generator=g, dtype=torch.int32)
            acts["n_valid"] = plan.n_train  # every synthetic target is a real token id
        if old is not None:
            # growth keeps the data already there (the rows a pass sees first keep their inputs
            # and next-token targets: a replica trains on a stable dataset across regrowth)
            def keep(new, prev):
                if new is not None and prev is not None:
                    n = min(new.shape[0], prev.shape[0])
                    new[:n].copy_(prev[:n])
            keep(acts["X"][0], old["X"][0])
            keep(acts.get("dY_top"), old.get("dY_top"))
            keep(acts.get("labels"), old.get("labels"))
            for k in ("Xo", "Xd"):
                for n_, p_ in zip(acts[k], old[k]):
                    keep(n_, p_)
            for dn, dp in zip(acts["dY"], old["dY"]):
                for name in dn:
                    keep(dn[name], dp.get(name))
            del old
            torch.cuda.empty_cache()
        self._acts = acts
        self._plan = plan
        return acts

    # ------------------------------------------------------------------ the step
    def run_step(self, plan: StepPlan | None = None, optimizer_step: bool = True,
                 advance: bool = True, overlap: bool | None = None,
                 backward: bool = True, grad_events: list | None = None) -> torch.Tensor:
        """Enqueue one full co-batched step on the current stream; returns the final hidden state
        buffer (device).  With ``advance`` the optimizer step counter and the step generation are
        bumped first (keep it False inside CUDA-graph capture; ``replay()`` bumps them).
        ``backward=False``: forward of every row only (an inference-only pass).
        ``grad_events[l]`` (optional, ``torch.cuda.Event(external=True)`` when capturing): recorded
        on the stream of layer l's K5 right after it, so a comm stream can reduce that layer's
        gradient bucket while the backward continues below (grad-mode sync).

        Projections run in data-flow order: a projection's shrink (K1) and GEMM (K2/K3) start
        only after the previous projection's GEMM (its input exists only then, as in the real
        model).  ``overlap``: the shrink runs on a side stream CONCURRENTLY with its own GEMM's
        base main loop (which needs only X); the GEMM's LoRA k-stages come last and wait for the
        shrink's completion signal (device flag == step generation).  The weight-gradient
        reductions + fused AdamW (K5) of a layer run on the side stream after the layer's last
        dX GEMM, queued behind the next projection's dH shrink.  The GEMMs then use their lean
        pipelines so one rank-space CTA fits next to each GEMM CTA."""
        plan = plan or self._plan
        a = self._acts
        if a is None:
            raise ConfigurationError("allocate() the step buffers first")
        if overlap is None:
            overlap = self.overlap
        L = self.cfg.model.layers
        Ttr = plan.n_train
        if advance:
            self.advance_step(optimizer_step and backward and Ttr > 0)
        main = torch.cuda.current_stream(self.device)
        side = self._side_stream() if overlap else main
        # pdl: every shrink CTA is resident before its GEMM launches and the GEMM waits for nothing
        # that needs SM room, so all kernels keep their standalone configuration (deep GEMM
        # pipelines, default carveouts: measured 1.5-2 % faster than fitting a rank-space CTA next
        # to each GEMM CTA); flag: the side-stream shrink may need room next to GEMM CTAs spinning
        # on its flag (1 = lean GEMMs + max-shared carveouts)
        lean = (0 if self.overlap_mode == "pdl" else 1) if overlap else 0
        _lib.load().collm_set_gemm_lean(int(os.environ.get("COLLM_LEAN_MODE", lean)))
        n_sig = 0

        pdl = overlap and self.overlap_mode == "pdl"

        def signal():
            nonlocal n_sig
            if not overlap or pdl:
                return None
            sig = (self._signals(n_sig + 1)[n_sig], self._gen)
            n_sig += 1
            return sig

        def after(stream_from) -> torch.cuda.Event:
            e = torch.cuda.Event()
            e.record(stream_from)
            return e

        def on_side(fn, wait_ev):
            if overlap:
                side.wait_event(wait_ev)
            with torch.cuda.stream(side):
                fn()

        plan.device.expand()
        prev = after(main)
        first = self.specs[0].name
        # ---------------- forward of every row: K1 on the side stream || K2 main loop
        caches: list[dict] = [dict() for _ in range(L)]
        for l, layer in enumerate(self.layers):
            syn = l if a["distinct_synthetic"] else 0
            for proj in layer:
                name = proj.spec.name
                if self.attention and name == "o":
                    X = a["Xo"][l]
                else:
                    X = a["X"][l] if name in ENTRY else (a["Xo"][syn] if name == "o" else a["Xd"][syn])
                Y = a["X"][l + 1] if name == "down" else a["Y"][name]
                if self.attention and name == "qkv":
                    Y = a["Yqkv"][l]
                sig = signal()
                if pdl:
                    cache = proj.forward_lora(X, plan.device, n_train=Ttr)
                    proj.forward_gemm(cache, plan.device, Y, pdl=True)
                    caches[l][name] = cache
                    if self.attention and name == "qkv":
                        self._attention_fwd(l, plan)
                    continue
                box = {}
                on_side(lambda: box.setdefault("c", proj.forward_lora(X, plan.device, n_train=Ttr,
                                                                    signal=sig)), prev)
                caches[l][name] = box["c"]
                proj.forward_gemm(box["c"], plan.device, Y, wait=sig)
                if self.attention and name == "qkv":
                    self._attention_fwd(l, plan)
                prev = after(main)
        if Ttr and backward and self.head is not None:
            # K2 logits -> K7 softmax-CE fwd+bwd -> K3 dX: the real dY entering the top layer
            self._loss = self.head.forward_backward(a["X"][L][:Ttr], a["labels"][:Ttr],
                                                    a["dY_top"], n_valid=Ttr)
        if Ttr and backward:
            opt = self.opt if optimizer_step else None
            mode = _lib.MODE_ADAMW if opt is not None else _lib.MODE_STORE_GRAD
            pending = None  # (layer, groups, event) of the last finished layer's K5

            def flush_k5():
                nonlocal pending
                if pending is not None:
                    lk, grp, ev = pending

                    # K5 of a whole layer in one launch, after the layer's last dX GEMM: the
                    # fused optimizer rewrites A_t^T, which those GEMMs read
                    def k5():
                        ops.lora_reduce(Ttr, grp, mode, adamw=opt.args if opt is not None else None,
                                        device=self.device)
                        if grad_events is not None:
                            grad_events[lk].record(torch.cuda.current_stream(self.device))
                    on_side(k5, ev)
                    pending = None

            for l in range(L - 1, -1, -1):
                syn = l if a["distinct_synthetic"] else 0
                groups: list = []
                for proj in reversed(self.layers[l]):
                    name = proj.spec.name
                    dY = (a["dY_top"] if l == L - 1 else a["dX_first"][l + 1]) if name == "down" \
                        else a["dY"][syn][name]
                    if self.attention and name == "qkv":
                        # K9 backward: o's dX (the gradient of the attention output) -> q|k|v's dY
                        self._attention_bwd(l, plan)
                        dY = a["dqkv"][l]
                        prev = after(main)  # the side-stream dH shrink reads this dY
                    dX = a["dX_first"][l] if name == first else a["dX"][name]
                    cache = caches[l][name]
                    sig = signal()
                    if pdl:
                        proj.backward_dh(dY, cache, plan.train_device)
                        proj.backward_dx(dY, cache, plan.train_device, dX, pdl=True)
                        flush_k5()
                        prev = after(main)
                    else:
                        on_side(lambda: proj.backward_dh(dY, cache, plan.train_device, signal=sig),
                                prev)
                        flush_k5()  # the previous layer's K5 queues behind this dH shrink
                        proj.backward_dx(dY, cache, plan.train_device, dX, wait=sig)
                        prev = after(main)
                    groups += proj.grad_groups(dY, cache, optimizer=opt)
                pending = (l, groups, prev)
            flush_k5()
        if overlap:
            main.wait_stream(side)
        return a["X"][L]

    def _qkv_views(self, t: torch.Tensor):
        H, Hk, D = self.n_heads, self.n_kv_heads, 128
        return t[:, :H * D], t[:, H * D:(H + Hk) * D], t[:, (H + Hk) * D:]

    def _attention_fwd(self, l: int, plan: StepPlan) -> None:
        """K9 forward of layer l over every sequence of the pass: q|k|v output -> o's input."""
        a = self._acts
        T = plan.n_rows
        q, k, v = self._qkv_views(a["Yqkv"][l][:T])
        ops.flash_attention(q, k, v, a["Xo"][l][:T], a["lse"][l], *plan.attn_rows, T=T,
                            n_heads=self.n_heads, n_kv_heads=self.n_kv_heads,
                            stat_ld=a["lse"].shape[-1])

    def _attention_bwd(self, l: int, plan: StepPlan) -> None:
        """K9 backward of layer l over the training sequences: o's dX -> q|k|v's dY."""
        a = self._acts
        Ttr = plan.n_train
        q, k, v = self._qkv_views(a["Yqkv"][l][:Ttr])
        dq, dk, dv = self._qkv_views(a["dqkv"][l][:Ttr])
        # the training sequences are rows [0, Ttr): the same per-row bounds, first Ttr rows
        ops.flash_attention_bwd(q, k, v, a["Xo"][l][:Ttr], a["dX"]["o"][:Ttr], a["lse"][l],
                                a["delta"], dq, dk, dv, *plan.attn_rows, T=Ttr,
                                n_heads=self.n_heads, n_kv_heads=self.n_kv_heads,
                                stat_ld=a["lse"].shape[-1])

    def last_loss(self) -> float:
        """Training loss of the last step that ran the LM head (reads the device scalar back)."""
        if self._loss is None:
            raise ConfigurationError("no step with the LM head has run (lm_head=True, training rows)")
        return float(self._loss.item())

    # ------------------------------------------------------------------ step generation
    def advance_step(self, optimizer_step: bool = True) -> None:
        """Per-step host->device bookkeeping (outside any captured graph, on the current stream):
        the optimizer's step block and the step generation the shrink->GEMM signals carry."""
        if optimizer_step:
            self.opt.advance()
        if self._gen is None:
            self._gen = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._gen_count += 1
        # fresh pinned staging per step (see OptimizerState.advance)
        host = torch.tensor([self._gen_count], dtype=torch.int32).pin_memory()
        self._gen.copy_(host, non_blocking=True)

    def _signals(self, n: int) -> torch.Tensor:
        """int32 [n, 2] shrink->GEMM completion signals (zeroed once; the kernels restore the
        counters and the flags carry the step generation).  Sized before graph capture."""
        if self._sig is None or self._sig.shape[0] < n:
            if torch.cuda.is_current_stream_capturing():
                raise ConfigurationError("run one eager step before capturing (signal buffers)")
            n_max = max(n, 2 * sum(1 for _ in self.projections()))
            self._sig = torch.zeros(n_max, 2, dtype=torch.int32, device=self.device)
        return self._sig

    def _side_stream(self) -> torch.cuda.Stream:
        if self._side is None:
            # high priority: the rank-space CTAs a spinning GEMM waits for are scheduled first
            prio = int(os.environ.get("COLLM_SIDE_PRIORITY", "-1"))
            self._side = torch.cuda.Stream(self.device, priority=prio)
        return self._side

    # ------------------------------------------------------------------ graphs
    def capture(self, plan: StepPlan | None = None, optimizer_step: bool = True) -> torch.cuda.CUDAGraph:
        """Capture one step into a CUDA graph (buffers and workspaces must already be sized: run
        one eager step first)."""
        plan = plan or self._plan
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.run_step(plan, optimizer_step=optimizer_step, advance=False)
        torch.cuda.current_stream().wait_stream(s)
        self._graph = g
        return g

    def replay(self, optimizer_step: bool = True) -> torch.Tensor:
        if self._graph is None:
            raise ConfigurationError("capture() first")
        self.advance_step(optimizer_step and self._plan.n_train > 0)
        self._graph.replay()
        return self._acts["X"][self.cfg.model.layers]

    # ------------------------------------------------------------------ accounting
    def step_flops(self, plan: StepPlan | None = None) -> int:
        """Algorithmic tensor-pipe FLOPs of one step: 2*K*N*(T + T_tr) summed over projections."""
        plan = plan or self._plan
        T, Ttr = plan.n_rows, plan.n_train
        return sum(2 * s.in_features * s.out_features * (T + Ttr)
                   for s in self.specs) * self.cfg.model.layers

    def lora_bytes(self, plan: StepPlan | None = None) -> dict:
        """Algorithmic HBM bytes of the rank-space (LoRA) kernels per step, counted
        as the unique minimum each pass must move (ranks unpadded, cache re-reads not counted):
          forward  (K1): X read, every distinct adapter's A read once, H written once;
          backward (K1 dH + K5): dY read once, X_tr and H_tr read, B_t read, dH written once,
                   and the fused AdamW's fp32 master/m/v read+write (24 B/param) plus the four
                   bf16 working copies it rewrites (8 B/param).
        The adapters' B matrices of the forward expand are read by the tensor-core GEMM (fused
        epilogue K-steps) and are counted there, not here."""
        plan = plan or self._plan
        T, Ttr = plan.n_rows, plan.n_train
        n_distinct = len({a for a in plan.batch.seg_adapter if a >= 0})
        fwd = bwd = 0
        for s in self.specs:
            K, N, r = s.in_features, s.out_features, s.rank
            nsub = len(s.subs)
            fwd += 2 * T * K + n_distinct * 2 * nsub * r * K + 2 * T * nsub * r
            if Ttr:
                params = r * N + nsub * r * K
                bwd += (2 * Ttr * N + 2 * Ttr * K + 2 * Ttr * nsub * r + 2 * r * N
                        + 2 * Ttr * nsub * r + 32 * params)
        L = self.cfg.model.layers
        return {"fwd": fwd * L, "bwd": bwd * L, "total": (fwd + bwd) * L}
