"""The unified PEFT projection: one LoRA-augmented linear layer serving a mixed row batch.

``LoraProjection`` owns the frozen base weight of one (optionally fused: q|k|v, gate|up)
projection, the adapter registry slice for it (every tenant's A/B), and the trainable adapter's
optimizer state.  Its ``forward`` / ``backward`` are the hot path:

  forward (all rows)   : K1 shrink  H = s_a . X . A_a^T  -> per-tile LoRA slot blocks
                         K2 tcgen05 GEMM  Y = X . W^T + sum_slots H_slot . B_a^T   (one write of Y)
  backward (train rows): K1 shrink  dH = s . dY . B_t           (one rank group per sub-projection)
                         K3 tcgen05 GEMM  dX = dY . W + dH . A_t  (W^T kept resident)
                         K5 reductions dB = dY^T . H, dA^T = X^T . dH with fused AdamW

Adapter layout follows the reference (`AdapterParams`, /root/reference/pkg/src/coserve/
launcher.py:28-47): b_mat (d, r) = (out, rank), a_mat (r, l) = (rank, in); dW = b_mat @ a_mat;
scale s_a = lora_alpha / r per adapter.  Ranks are zero-padded to r_pad (a multiple of 16) so the
rank dimension is a whole number of tensor-core K-steps; padding contributes exact zeros.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from . import _lib, ops
from .domain import ConfigurationError
from .segments import TILE_M, DevicePlan, HostPlan


def pad_rank(r: int) -> int:
    if r < 1:
        raise ConfigurationError(f"LoRA rank must be >= 1, got {r}")
    return 16 * math.ceil(r / 16)


@dataclass(frozen=True)
class ProjectionSpec:
    """Shape of one (fused) projection: ``subs`` are the output widths of the fused members."""

    name: str
    in_features: int
    subs: tuple[int, ...]
    rank: int
    alpha: float

    @property
    def out_features(self) -> int:
        return sum(self.subs)

    @property
    def r_pad(self) -> int:
        return pad_rank(self.rank)

    @property
    def R(self) -> int:
        return len(self.subs) * self.r_pad

    @property
    def sub_bounds(self) -> list[int]:
        b = [0]
        for n in self.subs:
            b.append(b[-1] + n)
        return b


@dataclass
class AdamWConfig:
    """AdamW hyper-parameters (torch.optim.AdamW semantics; HF Trainer's default optimizer)."""

    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0

    def args(self, step: int) -> list[float]:
        return [self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                1.0 - self.beta1 ** step, 1.0 - self.beta2 ** step]


class OptimizerState:
    """Step counter + the device-resident 7-float argument block the fused AdamW kernels read.

    ``advance()`` bumps the step and enqueues a 28-byte H2D copy on the current stream, so the
    same captured CUDA graph replays correctly step after step."""

    def __init__(self, cfg: AdamWConfig | None = None, device: torch.device | str = "cuda"):
        self.cfg = cfg or AdamWConfig()
        self.step = 0
        self.args = torch.zeros(7, dtype=torch.float32, device=device)

    def advance(self) -> None:
        self.step += 1
        # a fresh pinned staging tensor per step: the caching host allocator keeps it alive until
        # the async copy has run, so a CPU running steps ahead never overwrites a pending copy
        host = torch.tensor(self.cfg.args(self.step), dtype=torch.float32).pin_memory()
        self.args.copy_(host, non_blocking=True)


@dataclass
class TrainState:
    """fp32 master copies + AdamW moments of the trainable adapter, in the layouts the gradient
    reductions produce (B: [N, r_pad]; A^T: [K, R]), plus the extra bf16 layouts the backward
    kernels read (A^T for dX, B^T for dH)."""

    adapter: int
    master_B: torch.Tensor
    master_AT: torch.Tensor
    m_B: torch.Tensor
    v_B: torch.Tensor
    m_AT: torch.Tensor
    v_AT: torch.Tensor
    grad_B: torch.Tensor
    grad_AT: torch.Tensor
    AT16: torch.Tensor
    BT16: torch.Tensor


@dataclass
class ForwardCache:
    """What backward needs from forward: the training rows' input and rank-space activations."""

    X: torch.Tensor
    H16: torch.Tensor
    n_train: int


class LoraProjection:
    def __init__(self, spec: ProjectionSpec, n_adapters: int, device: torch.device | str = "cuda",
                 weight: torch.Tensor | None = None, keep_transpose: bool = True):
        self.spec = spec
        self.n_adapters = n_adapters
        self.device = torch.device(device)
        K, N, R, rp = spec.in_features, spec.out_features, spec.R, spec.r_pad
        for v, what in ((K, "in_features"), (N, "out_features")):
            if v % 8:
                raise ConfigurationError(f"{spec.name}: {what}={v} must be a multiple of 8")
        self.W = (weight if weight is not None else
                  torch.empty(N, K, dtype=torch.bfloat16, device=self.device))
        self.WT = torch.empty(K, N, dtype=torch.bfloat16, device=self.device) if keep_transpose else None
        self.A = torch.zeros(n_adapters, R, K, dtype=torch.bfloat16, device=self.device)
        self.B = torch.zeros(n_adapters, N, rp, dtype=torch.bfloat16, device=self.device)
        self.scale = torch.zeros(n_adapters, dtype=torch.float32, device=self.device)
        self.train_state: TrainState | None = None
        self._H16: torch.Tensor | None = None
        self._Hslots: torch.Tensor | None = None
        self._dH16: torch.Tensor | None = None
        self._dH16lo: torch.Tensor | None = None

    # ------------------------------------------------------------------ weights / registry
    def refresh_transpose(self) -> None:
        if self.WT is not None:
            self.WT.copy_(self.W.t())

    def set_adapter(self, slot: int, b_mats, a_mats, alpha: float | None = None) -> None:
        """Load adapter ``slot`` from per-sub (b_mat (d_s, r), a_mat (r, K)) pairs — the
        reference's AdapterParams layout (launcher.py:28-33)."""
        spec = self.spec
        if len(b_mats) != len(spec.subs) or len(a_mats) != len(spec.subs):
            raise ConfigurationError(f"{spec.name}: expected {len(spec.subs)} (b, a) pairs")
        r, rp = spec.rank, spec.r_pad
        bnd = spec.sub_bounds
        self.A[slot].zero_()
        self.B[slot].zero_()
        for s, (b, a) in enumerate(zip(b_mats, a_mats)):
            b = torch.as_tensor(b)
            a = torch.as_tensor(a)
            if tuple(b.shape) != (spec.subs[s], r) or tuple(a.shape) != (r, spec.in_features):
                raise ConfigurationError(
                    f"{spec.name}[{s}]: adapter dimensions {tuple(b.shape)}/{tuple(a.shape)} do "
                    f"not match ({spec.subs[s]}, {r})/({r}, {spec.in_features})")
            self.A[slot, s * rp:s * rp + r] = a.to(self.device, torch.bfloat16)
            self.B[slot, bnd[s]:bnd[s + 1], :r] = b.to(self.device, torch.bfloat16)
        self.scale[slot] = (alpha if alpha is not None else spec.alpha) / r

    def get_adapter(self, slot: int):
        """Inverse of set_adapter: per-sub (b_mat (d_s, r), a_mat (r, K)) float32 CPU tensors."""
        spec = self.spec
        r, rp = spec.rank, spec.r_pad
        bnd = spec.sub_bounds
        return [(self.B[slot, bnd[s]:bnd[s + 1], :r].float().cpu(),
                 self.A[slot, s * rp:s * rp + r].float().cpu()) for s in range(len(spec.subs))]

    def make_trainable(self, slot: int) -> TrainState:
        """Start fine-tuning adapter ``slot``: fp32 masters from its current bf16 weights."""
        K, N, R, rp = self.spec.in_features, self.spec.out_features, self.spec.R, self.spec.r_pad
        if self.WT is None:
            raise ConfigurationError(f"{self.spec.name}: training needs the resident W^T copy")
        dev = self.device
        mB = self.B[slot].float().contiguous()
        mAT = self.A[slot].float().t().contiguous()
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)  # noqa: E731
        st = TrainState(adapter=slot, master_B=mB, master_AT=mAT, m_B=z(N, rp), v_B=z(N, rp),
                        m_AT=z(K, R), v_AT=z(K, R), grad_B=z(N, rp), grad_AT=z(K, R),
                        AT16=self.A[slot].t().contiguous(),
                        BT16=torch.zeros(R, N, dtype=torch.bfloat16, device=dev))
        bnd = self.spec.sub_bounds
        for s in range(len(self.spec.subs)):
            st.BT16[s * rp:(s + 1) * rp, bnd[s]:bnd[s + 1]] = self.B[slot, bnd[s]:bnd[s + 1]].t()
        self.train_state = st
        return st

    # ------------------------------------------------------------------ buffers
    def _buffers(self, T: int, n_slots: int):
        R = self.spec.R
        if self._H16 is None or self._H16.shape[0] < T:
            self._H16 = torch.zeros(T, R, dtype=torch.bfloat16, device=self.device)
        rows = max(1, n_slots) * TILE_M
        if self._Hslots is None or self._Hslots.shape[0] < rows:
            self._Hslots = torch.zeros(rows, R, dtype=torch.bfloat16, device=self.device)
        return self._H16, self._Hslots

    def _dh_buffer(self, T: int) -> torch.Tensor:
        """dH = s.dY.B_t as a bf16 hi+lo pair: ``_dH16`` (hi, the dX GEMM's LoRA operand) and
        ``_dH16lo`` = bf16(dH - hi) (the dA reduction adds it: X^T (hi + lo))."""
        if self._dH16 is None or self._dH16.shape[0] < T:
            self._dH16 = torch.zeros(T, self.spec.R, dtype=torch.bfloat16, device=self.device)
            self._dH16lo = torch.zeros(T, self.spec.R, dtype=torch.bfloat16, device=self.device)
        return self._dH16[:T]

    def _dh_lo(self, T: int) -> torch.Tensor:
        self._dh_buffer(T)
        return self._dH16lo[:T]

    # ------------------------------------------------------------------ hot path
    def forward(self, X: torch.Tensor, plan: DevicePlan, Y: torch.Tensor | None = None,
                n_train: int = 0) -> tuple[torch.Tensor, ForwardCache]:
        """K1 + K2 over all rows of the pass: Y = X.W^T + per-row s_a.(X.A_a^T).B_a^T."""
        cache = self.forward_lora(X, plan, n_train)
        return self.forward_gemm(cache, plan, Y), cache

    def _check_plan(self, plan: DevicePlan) -> None:
        # the kernels index A / B / scale by adapter id: an unknown tenant must be a
        # ConfigurationError, not an out-of-bounds read
        if plan.max_adapter >= self.n_adapters:
            raise ConfigurationError(
                f"{self.spec.name}: adapter {plan.max_adapter} is not a registered slot "
                f"(n_adapters={self.n_adapters})")

    def forward_lora(self, X: torch.Tensor, plan: DevicePlan, n_train: int = 0,
                     signal: tuple | None = None) -> ForwardCache:
        """K1 (rank space): H16 and the GEMM's LoRA slot blocks for every row of the pass.
        ``signal`` = (int32[2] device signal, device step generation): publish completion so this
        projection's GEMM can run concurrently on another stream (``forward_gemm(wait=...)``)."""
        spec = self.spec
        T = plan.n_rows
        if X.shape[0] < T or X.shape[1] != spec.in_features:
            raise ConfigurationError(f"{spec.name}: X {tuple(X.shape)} vs T={T}, K={spec.in_features}")
        self._check_plan(plan)
        H16, Hslots = self._buffers(T, plan.n_slots)
        R, K = spec.R, spec.in_features
        if plan.n_slots:
            Hs = Hslots[: plan.n_slots * TILE_M]
            groups = [(g, min(64, R - g), 0, K) for g in range(0, R, 64)]
            tc = ops.shrink_tc_groups(groups) if plan.tc_ctas and signal is None else None
            units = plan.tc_units(tc[0][1]) if tc else None
            if units:  # the rank-space SM partition (collm_lora_shrink_tc)
                ops.lora_shrink_tc(X, self.A, *units, plan.tc_ctas, plan.row_adapter,
                                   self.scale, tc, R, H16=H16, Hslots=Hs,
                                   slot_of_row=plan.slot_of_row, tile_slot_ptr=plan.tile_slot_ptr)
            else:
                ops.lora_shrink(X, self.A, plan.shrink_tiles, plan.n_shrink_tiles, self.scale,
                                groups, R, H16=H16, Hslots=Hs, slot_of_row=plan.slot_of_row,
                                tile_slot_ptr=plan.tile_slot_ptr,
                                signal=signal[0] if signal else None,
                                gen=signal[1] if signal else None)
        return ForwardCache(X=X, H16=H16, n_train=n_train)

    def forward_gemm(self, cache: ForwardCache, plan: DevicePlan,
                     Y: torch.Tensor | None = None, wait: tuple | None = None,
                     pdl: bool = False) -> torch.Tensor:
        """K2: the base projection with the multi-adapter expand fused into the accumulator.
        ``wait`` = the shrink's (signal, generation): this GEMM may run before that shrink has
        finished (another stream); it loads the LoRA operand only after the signal.  ``pdl``: the
        shrink was the previous launch on this stream; overlap it by programmatic dependent launch
        instead (the LoRA stages wait for that grid)."""
        spec = self.spec
        T = plan.n_rows
        X = cache.X
        if Y is None:
            Y = torch.empty(T, spec.out_features, dtype=torch.bfloat16, device=self.device)
        rp = spec.r_pad
        self._check_plan(plan)
        if plan.n_slots:
            Hs = self._Hslots[: plan.n_slots * TILE_M]
            bnd = spec.sub_bounds
            ops.gemm_lora(X, self.W, Y, M=T, Hslots=Hs, h_rows=Hs.shape[0],
                          LB=self.B.view(self.n_adapters * spec.out_features, rp),
                          lb_rows=self.n_adapters * spec.out_features,
                          tile_slot_ptr=plan.tile_slot_ptr, slot_adapter=plan.slot_adapter,
                          lora_rank=rp, lb_rows_per_adapter=spec.out_features, sub_n_start=bnd,
                          sub_h_col=[s * rp for s in range(len(spec.subs))],
                          lora_flag=wait[0][1:] if wait else None, gen=wait[1] if wait else None,
                          lora_pdl=pdl, tile_skip=plan.tile_skip)
            if plan.n_expand_tiles:  # many-adapter tiles: per-row expand after the base GEMM
                ops.lora_expand_rows(Y, cache.H16, self.B, plan.row_adapter, plan.expand_tiles,
                                     plan.n_expand_tiles, T, r_pad=rp, sub_n_start=bnd,
                                     sub_h_col=[s * rp for s in range(len(spec.subs))])
        else:
            ops.gemm_lora(X, self.W, Y, M=T)
        return Y

    def _grad_groups(self, dY=None, X_tr=None, H_tr=None, dH16=None, dH16lo=None, *,
                     targets: str):
        """The K5 group table of this projection: dB per sub-projection (U = dY, V = H16) and
        dA^T in <=64-wide rank chunks (U = X_tr, V = dH16 hi, V2 = dH16lo), with their optimizer
        targets."""
        st = self.train_state
        spec = self.spec
        K, N, R, rp = spec.in_features, spec.out_features, spec.R, spec.r_pad
        bnd = spec.sub_bounds
        full = targets != "grad"
        groups = []
        for s in range(len(spec.subs)):
            groups.append(ops.reduce_group(
                dY, H_tr, u_off=bnd[s], P=spec.subs[s], v_off=s * rp, Q=rp, ldc=rp,
                c_row_off=bnd[s], grad=st.grad_B,
                master=st.master_B if full else None, m=st.m_B if full else None,
                v=st.v_B if full else None, out_same=self.B[st.adapter] if full else None,
                out_trans=st.BT16 if full else None, ld_trans=N, t_row_off=s * rp,
                t_col_off=bnd[s]))
        for q in range(0, R, 64):
            groups.append(ops.reduce_group(
                X_tr, dH16, V2=dH16lo, u_off=0, P=K, v_off=q, Q=min(64, R - q), ldc=R, c_col_off=q,
                grad=st.grad_AT, master=st.master_AT if full else None,
                m=st.m_AT if full else None, v=st.v_AT if full else None,
                out_same=st.AT16 if full else None, out_trans=self.A[st.adapter] if full else None,
                ld_trans=K, t_row_off=q))
        return groups

    def backward(self, dY: torch.Tensor, cache: ForwardCache, train_plan: DevicePlan,
                 dX: torch.Tensor | None = None, *, optimizer: OptimizerState | None = None,
                 accumulate: bool = False, grad_scale: float = 1.0,
                 need_dx: bool = True) -> torch.Tensor | None:
        """Backward of the training rows [0, n_train).  ``optimizer`` given -> fused AdamW step
        (after adding the gradient already accumulated when ``accumulate``) using the step the
        caller already advanced (``OptimizerState.advance``); otherwise the gradient is stored (or
        added, ``accumulate``) into the grad buffers, e.g. for a cross-replica allreduce followed
        by :meth:`apply_optimizer`."""
        if cache.n_train <= 0:
            return None
        self.backward_dh(dY, cache, train_plan)
        if need_dx:
            dX = self.backward_dx(dY, cache, train_plan, dX)
        self.backward_grads(dY, cache, optimizer=optimizer, accumulate=accumulate,
                            grad_scale=grad_scale)
        return dX

    def _require_train(self) -> TrainState:
        st = self.train_state
        if st is None:
            raise ConfigurationError(f"{self.spec.name}: no trainable adapter (make_trainable)")
        return st

    def backward_dh(self, dY: torch.Tensor, cache: ForwardCache, train_plan: DevicePlan,
                    signal: tuple | None = None) -> torch.Tensor:
        """K1: dH = s * dY . B_t (bf16 hi + lo), one rank group per sub-projection (its own N
        range)."""
        st = self._require_train()
        spec = self.spec
        Ttr = cache.n_train
        rp, R = spec.r_pad, spec.R
        bnd = spec.sub_bounds
        dH16 = self._dh_buffer(Ttr)
        groups = [(s * rp + g, min(64, rp - g), bnd[s], bnd[s + 1])
                  for s in range(len(spec.subs)) for g in range(0, rp, 64)]
        tc = ops.shrink_tc_groups(groups) if train_plan.tc_ctas and signal is None else None
        units = train_plan.tc_units(tc[0][1]) if tc else None
        if units:  # the rank-space SM partition (collm_lora_shrink_tc)
            ops.lora_shrink_tc(dY, st.BT16, *units, train_plan.tc_ctas, train_plan.row_adapter,
                               self.scale, tc, R, a_stride=0, H16=dH16, H16lo=self._dh_lo(Ttr))
        else:
            ops.lora_shrink(dY, st.BT16, train_plan.shrink_tiles, train_plan.n_shrink_tiles,
                            self.scale, groups, R, a_stride=0, H16=dH16, H16lo=self._dh_lo(Ttr),
                            signal=signal[0] if signal else None,
                            gen=signal[1] if signal else None)
        return dH16

    def backward_dx(self, dY: torch.Tensor, cache: ForwardCache, train_plan: DevicePlan,
                    dX: torch.Tensor | None = None, wait: tuple | None = None,
                    pdl: bool = False) -> torch.Tensor:
        """K3: dX = dY . W + dH . A_t (reads A_t^T: run before this projection's optimizer step)."""
        st = self._require_train()
        spec = self.spec
        Ttr = cache.n_train
        K, R = spec.in_features, spec.R
        if dX is None:
            dX = torch.empty(Ttr, K, dtype=torch.bfloat16, device=self.device)
        dH16 = self._dh_buffer(Ttr)
        ops.gemm_lora(dY, self.WT, dX, M=Ttr, Hslots=dH16, h_rows=Ttr, LB=st.AT16, lb_rows=K,
                      tile_slot_ptr=train_plan.tile_slot_ptr, slot_adapter=train_plan.slot_adapter,
                      lora_rank=R, lb_rows_per_adapter=0,
                      lora_flag=wait[0][1:] if wait else None, gen=wait[1] if wait else None,
                      lora_pdl=pdl)
        return dX

    def grad_groups(self, dY: torch.Tensor, cache: ForwardCache, *,
                    optimizer: OptimizerState | None = None) -> list:
        """This projection's K5 group table (dB per sub, dA^T chunks) for a given dY — so a caller
        can reduce several projections (a whole layer) in ONE launch (`ops.lora_reduce`)."""
        self._require_train()
        Ttr = cache.n_train
        dH16 = self._dh_buffer(Ttr)
        return self._grad_groups(dY, cache.X[:Ttr], cache.H16[:Ttr], dH16, self._dh_lo(Ttr),
                                 targets="full" if optimizer is not None else "grad")

    def backward_grads(self, dY: torch.Tensor, cache: ForwardCache, *,
                       optimizer: OptimizerState | None = None, accumulate: bool = False,
                       grad_scale: float = 1.0) -> None:
        """K5: dB = dY^T . H16 (per sub), dA^T = X^T . (dH16 + dH16lo) — one launch, fused AdamW
        or store."""
        rg = self.grad_groups(dY, cache, optimizer=optimizer)
        mode = _lib.MODE_ADAMW if optimizer is not None else _lib.MODE_STORE_GRAD
        ops.lora_reduce(cache.n_train, rg, mode, accum_in=accumulate, grad_scale=grad_scale,
                        adamw=optimizer.args if optimizer is not None else None,
                        device=self.device)

    def apply_optimizer(self, optimizer: OptimizerState) -> None:
        """AdamW from the grad buffers (after a cross-replica allreduce of the gradients)."""
        ops.lora_apply(self._grad_groups(targets="full"), _lib.MODE_ADAMW, adamw=optimizer.args)

    def refresh_from_master(self) -> None:
        """Rewrite every bf16 copy of the trainable adapter from the fp32 masters (after a
        parameter average across replicas — the reference's fedavg, launcher.py:68-80)."""
        ops.lora_apply(self._grad_groups(targets="full"), _lib.MODE_COPY_ONLY)


class LMHead:
    """Frozen LM head + next-token cross-entropy of the training rows: the
    real training signal behind the reference's convergence stand-in (`perf.train_step`,
    perf.py:92-126).  logits = X_top . W^T (K2 GEMM, no LoRA), K7 softmax-CE forward + backward,
    dX_top = dlogits . W (K3-shaped GEMM on the kept W^T) — the dY that enters the top layer's
    LoRA backward.  W [V, h] bf16 (nn.Linear layout), W^T [h, V] bf16."""

    def __init__(self, hidden: int, vocab: int, device: torch.device | str = "cuda",
                 weight: torch.Tensor | None = None):
        if hidden % 8 or vocab % 8:
            raise ConfigurationError(f"LM head: hidden={hidden} and vocab={vocab} must be x8")
        self.hidden, self.vocab = hidden, vocab
        self.device = torch.device(device)
        self.W = (weight if weight is not None else
                  torch.empty(vocab, hidden, dtype=torch.bfloat16, device=self.device))
        self.WT = torch.empty(hidden, vocab, dtype=torch.bfloat16, device=self.device)
        self._bufs: dict = {}

    def refresh_transpose(self) -> None:
        self.WT.copy_(self.W.t())

    def _buffers(self, T: int) -> dict:
        b = self._bufs
        if not b or b["logits"].shape[0] < T:
            dev = self.device
            b.update(logits=torch.empty(T, self.vocab, dtype=torch.bfloat16, device=dev),
                     dlogits=torch.empty(T, self.vocab, dtype=torch.bfloat16, device=dev),
                     loss_rows=torch.zeros(T, dtype=torch.float32, device=dev),
                     loss=torch.zeros(1, dtype=torch.float32, device=dev),
                     counter=torch.zeros(1, dtype=torch.int32, device=dev))
        return b

    def forward_backward(self, X: torch.Tensor, labels: torch.Tensor, dX: torch.Tensor,
                         n_valid: int | None = None) -> torch.Tensor:
        """Mean CE of the rows of X [T, h] against labels [T] (int32, < 0 or >= V ignored) and
        its gradient w.r.t. X into dX [T, h].  Returns the device loss (fp32 [1]).  The gradient is
        that of the reported mean, so it is scaled by 1 / n_valid (the count of non-ignored
        labels); pass ``n_valid`` when the caller knows it (the step path does) — otherwise it is
        counted here from the device labels, which reads one scalar back (a host sync)."""
        T = labels.shape[0]
        if X.shape[0] < T or X.shape[1] != self.hidden or dX.shape[0] < T:
            raise ConfigurationError(f"LM head: X {tuple(X.shape)} / dX {tuple(dX.shape)} vs T={T}")
        if T == 0:
            raise ConfigurationError("LM head: no training rows")
        b = self._buffers(T)
        if n_valid is None:
            n = int(((labels >= 0) & (labels < self.vocab)).sum().item())
        else:
            n = n_valid
        ops.gemm_lora(X, self.W, b["logits"], M=T)
        ops.cross_entropy(b["logits"], labels, self.vocab, loss_rows=b["loss_rows"],
                          loss_mean=b["loss"], counter=b["counter"], dlogits=b["dlogits"],
                          grad_scale=1.0 / max(n, 1))
        ops.gemm_lora(b["dlogits"], self.WT, dX, M=T)
        return b["loss"]
