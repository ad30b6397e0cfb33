"""K6 — cross-replica synchronisation of the shared training adapter (the path's only collective).

Each GPU is an independent replica (one process per GPU, ``torch.distributed`` with NCCL over
NVLink/NVSwitch).  Replicas fine-tuning the same adapter exchange it in one of two ways:

* ``grad`` mode (north star): every optimizer step, the flat fp32 LoRA-gradient buffer of the
  trainable adapter (all layers, all projections — :attr:`ReplicaStack.flat_grad`) is
  averaged with ONE ``all_reduce(AVG)``; then the AdamW apply kernel runs on every replica, so
  all replicas keep identical adapters.
* ``fedavg`` mode (reference semantics, /root/reference/pkg/src/coserve/launcher.py:68-80 called
  from FLProcess.finalize_round :226): replicas take local fused-AdamW steps and, at each round
  boundary, the fp32 master parameters are averaged (``fedavg``: element-wise mean of B and of A)
  and the bf16 working copies are rewritten (``collm_lora_apply`` COPY_ONLY).  Unlike the
  reference, the averaged adapter IS handed back to every participant (the reference stores
  ``global_adapter`` but never broadcasts it, engine.py:478-480).

Participant groups follow the reference's FL process: the replicas of one family that joined the
process (``launcher.scan_and_trigger``, min_participants = 3 by default).  ``new_group`` builds the
communicator for a participant list; a single participant short-circuits like ``fedavg`` does for
one client (launcher.py:76-77).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .domain import ConfigurationError
from .reference import coserve_module

_ref_launcher = coserve_module("launcher")


class _LocalAggregationError(ValueError):
    """Stand-in for launcher.AggregationError (launcher.py:24-25) without the reference."""


# the reference's own class when coserve is importable (the drop-in), else the stand-in
AggregationError = _ref_launcher.AggregationError if _ref_launcher is not None else _LocalAggregationError


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def new_group(participants: list[int]):
    """Communicator over the given ranks (all ranks must call it, torch.distributed semantics)."""
    if not participants:
        raise ConfigurationError("no participants")
    if len(set(participants)) != len(participants):
        raise ConfigurationError("duplicate participant")
    _, ws = world()
    if ws == 1:
        return None
    return dist.new_group(ranks=sorted(participants))


def _avg_(t: torch.Tensor, group=None) -> torch.Tensor:
    n = dist.get_world_size(group) if group is not None else dist.get_world_size()
    if t.is_cuda:
        dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
    else:  # gloo has no AVG
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t.div_(n)
    return t


def allreduce_grads(flat_grad: torch.Tensor, group=None) -> torch.Tensor:
    """grad mode: in-place average of the flat fp32 gradient buffer across the group."""
    if flat_grad.dtype != torch.float32:
        raise ConfigurationError("LoRA gradients are synchronised in fp32")
    _, ws = world()
    if ws == 1:
        return flat_grad
    return _avg_(flat_grad, group)


def fedavg_params(flat_master: torch.Tensor, shapes: list[tuple[int, ...]] | None = None,
                  group=None) -> torch.Tensor:
    """fedavg mode: in-place element-wise mean of the flat fp32 master parameters.

    ``shapes`` (optional) are the per-tensor shapes this rank holds; they are compared across the
    group first so a mismatch raises AggregationError naming the offending client, like the
    reference (launcher.py:73-75)."""
    if flat_master.dtype != torch.float32:
        raise ConfigurationError("master parameters are averaged in fp32")
    rank, ws = world()
    if ws == 1:
        return flat_master
    n = torch.tensor([flat_master.numel()], dtype=torch.int64, device=flat_master.device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size(group) if group else ws)]
    dist.all_gather(sizes, n, group=group)
    for idx, s in enumerate(sizes):
        if int(s.item()) != int(sizes[0].item()):
            raise AggregationError(f"client {idx} adapter dimensions do not match the first client")
    return _avg_(flat_master, group)
