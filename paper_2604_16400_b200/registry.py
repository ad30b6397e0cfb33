"""Adapter registry lifecycle: host-resident adapters paged into the
replica's device slots, save / load in the reference's layout, and the global-adapter broadcast.

The paper keeps adapters in host memory and swaps them into the GPU asynchronously;
the reference's ``AdapterParams`` (launcher.py:28-47) is the per-client (b_mat (d, r), a_mat (r, l))
pair and its round protocol never pushes the aggregate back to the replicas (engine.py:468-480).

B200 design: every registered adapter lives in PINNED host memory in exactly the device slot
layout of each projection (A [R, K], B [N, r_pad] bf16, scale fp32), so paging an adapter in is
one async H2D copy per tensor on a dedicated copy stream (the DMA engines, no SM work) that
overlaps the running step.  The device slots are an LRU cache: a slot is reused only after (a)
the copy stream has waited for the last compute-stream step that read it (``mark_used``) and
(b) the compute stream waits for the copy's completion event before a step reads it
(``ensure``).  Nothing on this path synchronises the host with the device.
"""

from __future__ import annotations

import collections
import os

import torch

from .domain import ConfigurationError
from .layer import LoraProjection


class AdapterPager:
    """Host store + device slot cache for one ReplicaStack's adapter registry."""

    def __init__(self, stack, pinned_slots: tuple[int, ...] | None = None):
        self.stack = stack
        self.projs: list[LoraProjection] = list(stack.projections())
        self.n_slots = stack.cfg.n_adapters
        # trainable adapters' slots are never evicted (their masters / optimizer state live there)
        self.pinned = set(pinned_slots if pinned_slots is not None
                          else (t.slot for t in stack.trainers.values()))
        self.host: dict[object, list[tuple[torch.Tensor, torch.Tensor, torch.Tensor]]] = {}
        self.slot_of: collections.OrderedDict = collections.OrderedDict()  # adapter id -> slot, LRU
        self.held: list[object | None] = [None] * self.n_slots
        self.copy_stream = torch.cuda.Stream(stack.device)
        self._ready: list[torch.cuda.Event | None] = [None] * self.n_slots
        self._last_use: list[torch.cuda.Event | None] = [None] * self.n_slots

    # ------------------------------------------------------------------ host store
    def register(self, adapter_id, per_projection, alpha: float | None = None) -> None:
        """Store adapter ``adapter_id`` on the host.  ``per_projection``: one list per projection
        of the stack (stack.projections() order) of per-sub (b_mat (d_s, r), a_mat (r, K)) pairs —
        the reference's AdapterParams layout (launcher.py:28-33)."""
        if len(per_projection) != len(self.projs):
            raise ConfigurationError(f"expected {len(self.projs)} projections, got {len(per_projection)}")
        entry = []
        for proj, pairs in zip(self.projs, per_projection):
            sp = proj.spec
            if len(pairs) != len(sp.subs):
                raise ConfigurationError(f"{sp.name}: expected {len(sp.subs)} (b, a) pairs")
            A = torch.zeros(sp.R, sp.in_features, dtype=torch.bfloat16)
            B = torch.zeros(sp.out_features, sp.r_pad, dtype=torch.bfloat16)
            bnd = sp.sub_bounds
            for s, (b, a) in enumerate(pairs):
                b, a = torch.as_tensor(b), torch.as_tensor(a)
                if tuple(b.shape) != (sp.subs[s], sp.rank) or tuple(a.shape) != (sp.rank, sp.in_features):
                    raise ConfigurationError(
                        f"{sp.name}[{s}]: adapter dimensions {tuple(b.shape)}/{tuple(a.shape)} do not "
                        f"match ({sp.subs[s]}, {sp.rank})/({sp.rank}, {sp.in_features})")
                A[s * sp.r_pad:s * sp.r_pad + sp.rank] = a.to(torch.bfloat16)
                B[bnd[s]:bnd[s + 1], :sp.rank] = b.to(torch.bfloat16)
            sc = torch.tensor([(alpha if alpha is not None else sp.alpha) / sp.rank], dtype=torch.float32)
            entry.append((A.pin_memory(), B.pin_memory(), sc.pin_memory()))
        self.host[adapter_id] = entry

    def register_from_slot(self, adapter_id, slot: int) -> None:
        """Snapshot device slot ``slot`` (e.g. a freshly fine-tuned adapter) into the host store
        (synchronous D2H; not on the step path)."""
        entry = []
        for proj in self.projs:
            entry.append((proj.A[slot].cpu().pin_memory(), proj.B[slot].cpu().pin_memory(),
                          proj.scale[slot:slot + 1].cpu().pin_memory()))
        self.host[adapter_id] = entry

    def adapter(self, adapter_id):
        """The stored adapter in the reference layout: per projection, per-sub (b, a) fp32."""
        out = []
        for proj, (A, B, _) in zip(self.projs, self.host[adapter_id]):
            sp = proj.spec
            bnd = sp.sub_bounds
            out.append([(B[bnd[s]:bnd[s + 1], :sp.rank].float(),
                         A[s * sp.r_pad:s * sp.r_pad + sp.rank].float()) for s in range(len(sp.subs))])
        return out

    def save(self, adapter_id, path: str | os.PathLike) -> None:
        """Write the adapter in the reference layout (per projection, per sub: b_mat (d, r),
        a_mat (r, l) — launcher.py:28-33) plus its scales."""
        torch.save({"format": "collm-lora-v1",
                    "projections": [p.spec.name for p in self.projs],
                    "adapter": self.adapter(adapter_id),
                    "scale": [float(e[2][0]) for e in self.host[adapter_id]]}, path)

    def load(self, adapter_id, path: str | os.PathLike) -> None:
        d = torch.load(path, weights_only=True)
        if d.get("format") != "collm-lora-v1" or d["projections"] != [p.spec.name for p in self.projs]:
            raise ConfigurationError(f"{path}: not an adapter of this stack's projections")
        self.register(adapter_id, d["adapter"])
        for e, sc in zip(self.host[adapter_id], d["scale"]):
            e[2][0] = sc

    # ------------------------------------------------------------------ device slots
    def ensure(self, adapter_ids) -> dict:
        """Make every adapter of ``adapter_ids`` resident; returns adapter id -> device slot.
        Missing adapters are copied (async, copy stream) into least-recently-used unpinned slots
        not needed by this call; the CURRENT stream then waits for those copies."""
        want = list(dict.fromkeys(adapter_ids))
        missing = [a for a in want if a not in self.slot_of]
        for a in want:
            if a not in self.host and a not in self.slot_of:
                raise ConfigurationError(f"adapter {a!r} is not registered")
        keep = {self.slot_of[a] for a in want if a in self.slot_of}
        free = [s for s in range(self.n_slots) if self.held[s] is None and s not in self.pinned]
        victims = [self.slot_of[a] for a in self.slot_of
                   if self.slot_of[a] not in keep and self.slot_of[a] not in self.pinned]
        candidates = free + victims
        if len(missing) > len(candidates):
            raise ConfigurationError(f"{len(want)} adapters requested, only "
                                     f"{self.n_slots - len(self.pinned)} pageable device slots")
        compute = torch.cuda.current_stream(self.stack.device)
        for a, slot in zip(missing, candidates):
            old = self.held[slot]
            if old is not None:
                del self.slot_of[old]
            with torch.cuda.stream(self.copy_stream):
                if self._last_use[slot] is not None:
                    self.copy_stream.wait_event(self._last_use[slot])  # the last reader is done
                for proj, (A, B, sc) in zip(self.projs, self.host[a]):
                    proj.A[slot].copy_(A, non_blocking=True)
                    proj.B[slot].copy_(B, non_blocking=True)
                    proj.scale[slot:slot + 1].copy_(sc, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            self._ready[slot] = ev
            self.held[slot] = a
            self.slot_of[a] = slot
        for a in want:
            self.slot_of.move_to_end(a)
            ev = self._ready[self.slot_of[a]]
            if ev is not None:
                compute.wait_event(ev)
        return {a: self.slot_of[a] for a in want}

    def mark_used(self, slots) -> None:
        """Record that the work just enqueued on the current stream reads ``slots`` (call after
        enqueueing the step): their next eviction waits for it."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.stack.device))
        for s in set(slots):
            self._last_use[s] = ev


def broadcast_adapter(stack, src: int = 0, group=None) -> None:
    """Push the global (e.g. FedAvg-aggregated) trainable adapter from rank ``src`` to every
    replica of the group: one broadcast of the flat fp32 masters, then each replica rewrites its
    bf16 copies (collm_lora_apply COPY_ONLY).  The reference stores the aggregate but never pushes
    it back (engine.py:468-480); this closes that loop."""
    import torch.distributed as dist
    flat = stack.flat_master  # built once with the trainer (never re-homed behind a graph)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(flat, src=src, group=group)
    stack.refresh_from_master()
