"""K0 — batch composition for the unified pass: mixed rows -> segment table -> device plan.

Replaces the reference's single-stream batch formation (``domain.Batch``,
/root/reference/pkg/src/coserve/domain.py:64-86; ``StreamQueue.pop_up_to``, dispatcher.py:66-82)
with the mixed-adapter row table the unified PEFT layer consumes:

    rows = [training rows of adapter t] ++ [inference rows sorted by (adapter, request id, pos)]

Segments are maximal runs of rows with the same (adapter, role).  The per-128-row-tile LoRA slot
lists and the shrink work list are planned by the native host planner (``collm_plan_segments``);
``row_adapter`` / ``slot_of_row`` are expanded on the device (``collm_expand_segments``).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .domain import ConfigurationError, InferenceItem, MixedBatch, RowRole, TrainItem

TILE_M = 256  # LoRA slot-plan granularity (kSlotTileM in csrc/common.cuh)
SHRINK_TILE = 16


def build_mixed_batch(train: TrainItem | None, items: list[InferenceItem]) -> MixedBatch:
    """Compose one mixed pass.  Deterministic: inference items are ordered by
    (adapter, request_id); ties on request_id are rejected (a request appears once per pass)."""
    seen: set[int] = set()
    for it in items:
        if it.request_id in seen:
            raise ConfigurationError(f"request {it.request_id} appears twice in one pass")
        seen.add(it.request_id)
    if train is None and not items:
        raise ConfigurationError("a pass needs training rows or inference rows")
    seg_start = [0]
    seg_adapter: list[int] = []
    seg_role: list[int] = []
    row_req: list[int] = []
    row_pos: list[int] = []

    def push(adapter: int, role: int, n: int) -> None:
        if seg_adapter and seg_adapter[-1] == adapter and seg_role[-1] == role:
            seg_start[-1] += n
        else:
            seg_adapter.append(adapter)
            seg_role.append(role)
            seg_start.append(seg_start[-1] + n)

    n_train = 0
    if train is not None:
        n_train = train.rows
        push(train.adapter, int(RowRole.TRAIN), n_train)
        row_req.extend([-1] * n_train)
        row_pos.extend(range(n_train))
    for it in sorted(items, key=lambda i: (i.adapter, i.request_id)):
        push(it.adapter, int(it.role), it.n_rows)
        row_req.extend([it.request_id] * it.n_rows)
        row_pos.extend(range(it.n_rows))
    return MixedBatch(
        seg_start=tuple(seg_start),
        seg_adapter=tuple(seg_adapter),
        seg_role=tuple(seg_role),
        row_request=tuple(row_req),
        row_pos=tuple(row_pos),
        n_train_rows=n_train,
        train_adapter=train.adapter if train is not None else -1,
    )


@dataclass
class HostPlan:
    """Host arrays of a planned batch (int32)."""

    seg_start: np.ndarray
    seg_adapter: np.ndarray
    tile_slot_ptr: np.ndarray
    slot_adapter: np.ndarray
    shrink_tiles: np.ndarray  # [n, 3]

    @property
    def n_slots(self) -> int:
        return int(self.slot_adapter.shape[0])

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.seg_start, self.seg_adapter, self.tile_slot_ptr,
                                      self.slot_adapter, self.shrink_tiles))


def plan_segments(seg_start, seg_adapter) -> HostPlan:
    """Native host planner (collm_plan_segments): tile slot lists + shrink work list."""
    ss = np.ascontiguousarray(np.asarray(seg_start, dtype=np.int32))
    sa = np.ascontiguousarray(np.asarray(seg_adapter, dtype=np.int32))
    n_seg = int(sa.shape[0])
    if ss.shape[0] != n_seg + 1:
        raise ConfigurationError("seg_start must have n_segments + 1 entries")
    n_rows = int(ss[-1])
    n_tiles = (n_rows + TILE_M - 1) // TILE_M
    slot_cap = n_tiles + n_seg
    tile_cap = n_rows // SHRINK_TILE + n_seg + 1
    tsp = np.zeros(n_tiles + 1, np.int32)
    slots = np.zeros(slot_cap, np.int32)
    tiles = np.zeros((tile_cap, 3), np.int32)
    ns = C.c_int32(0)
    nt = C.c_int32(0)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    _lib.call("collm_plan_segments", ip(ss), ip(sa), n_seg, n_rows, ip(tsp), ip(slots), slot_cap,
              C.byref(ns), ip(tiles), tile_cap, C.byref(nt))
    return HostPlan(ss, sa, tsp, slots[: ns.value].copy(), tiles[: nt.value].copy())


SHRINK_TC_MIN_ROWS = int(os.environ.get("COLLM_SHRINK_TC_MIN_ROWS", "4096"))


def default_tc_ctas(n_rows: int, rank_sms: int, num_sms: int) -> int:
    """CTAs of the K1' shrink for a pass of n_rows rows (0 = the mma.sync K1): the rank-space
    partition when one is set, else the whole GPU (even: TPC pairs) for passes of
    >= SHRINK_TC_MIN_ROWS rows."""
    if rank_sms:
        return rank_sms
    return num_sms // 2 * 2 if n_rows >= SHRINK_TC_MIN_ROWS else 0
TC_RANKS = (16, 32, 48, 64, 96, 128, 192, 256)  # group widths the K1' units are planned for


def plan_shrink_windows(host: HostPlan, nr: int, n_ctas: int):
    """collm_plan_shrink_windows: K1' work chunks (128-row windows x runs of consecutive adapter
    ids stacked in the MMA's N <= 256 for groups of ``nr`` ranks, big units split along K),
    assigned longest-first to ``n_ctas`` CTAs -> (chunks [n, 8], cta_ptr [n_ctas + 1])."""
    tiles = np.ascontiguousarray(host.shrink_tiles.reshape(-1, 3).astype(np.int32))
    nt = int(tiles.shape[0])
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
    cap = max(1, 8 * (2 * (int(host.seg_start[-1]) // 128 + 1) + nt))
    items = np.zeros((cap, 8), np.int32)
    ptr = np.zeros(n_ctas + 1, np.int32)
    n = C.c_int32(0)
    _lib.call("collm_plan_shrink_windows", ip(tiles), nt, nr, n_ctas, ip(items), cap, C.byref(n),
              ip(ptr))
    return items[: max(1, n.value)].copy(), ptr


def uniform_plan(n_rows: int, adapter: int) -> HostPlan:
    """Plan for rows [0, n_rows) that all use one adapter (the training rows' backward)."""
    return plan_segments([0, n_rows], [adapter])


class DevicePlan:
    """Device-resident plan of one pass, shared by every projection of every layer."""

    def __init__(self, host: HostPlan, device: torch.device | str = "cuda",
                 stream: torch.cuda.Stream | None = None, expand: bool = True,
                 tc_ctas: int | None = None):
        self.host = host
        self.n_rows = int(host.seg_start[-1])
        self.n_tiles_m = (self.n_rows + TILE_M - 1) // TILE_M
        dev = torch.device(device)
        if tc_ctas is None:
            # the rank-space partition of this device (collm_set_rank_sms); without one, passes of
            # >= SHRINK_TC_MIN_ROWS rows take K1' on the whole GPU (the TMA + tcgen05 shrink
            # streams the large X near HBM rate; small passes are MMA-latency-bound there and
            # keep the mma.sync K1)
            from . import ops
            tc_ctas = 0
            if dev.type == "cuda":
                tc_ctas = default_tc_ctas(self.n_rows, ops.rank_sms(dev), ops.num_sms(dev))
        self.tc_ctas = int(tc_ctas)
        # K1' units per group width (the rank-space partition, collm_set_rank_sms)
        tc_plans = [plan_shrink_windows(host, nr, self.tc_ctas) for nr in TC_RANKS] \
            if self.tc_ctas else []
        # many-adapter slot tiles: more LoRA slots than this and the tile's expand leaves the GEMM
        # (whose fused expand costs slots x r / 64 extra k-stages) for the per-row expand kernel
        slots = np.diff(host.tile_slot_ptr)
        thr = int(os.environ.get("COLLM_EXPAND_ROWS_SLOTS", "32"))
        skip = (slots > thr).astype(np.int32)
        expand_tiles = np.nonzero(skip)[0].astype(np.int32)
        self.n_expand_tiles = int(expand_tiles.size)
        # one packed upload: [seg_start | seg_adapter | tile_slot_ptr | slot_adapter | shrink_tiles
        #                     | shrink items | item ranges per CTA]
        parts = [host.seg_start, host.seg_adapter, host.tile_slot_ptr,
                 host.slot_adapter if host.n_slots else np.zeros(1, np.int32),
                 host.shrink_tiles.reshape(-1) if host.shrink_tiles.size else np.zeros(3, np.int32),
                 skip if skip.size else np.zeros(1, np.int32),
                 expand_tiles if expand_tiles.size else np.zeros(1, np.int32)]
        for it, ptr in tc_plans:
            parts += [it.reshape(-1), ptr]
        sizes = [p.size for p in parts]
        packed = torch.from_numpy(np.concatenate(parts).astype(np.int32)).pin_memory()
        self.h2d_bytes = packed.numel() * 4
        buf = torch.empty(packed.numel(), dtype=torch.int32, device=dev)
        buf.copy_(packed, non_blocking=True)
        offs = np.cumsum([0] + sizes)
        self._pinned = packed
        self._buf = buf
        self.seg_start = buf[offs[0]:offs[1]]
        self.seg_adapter = buf[offs[1]:offs[2]]
        self.tile_slot_ptr = buf[offs[2]:offs[3]]
        self.slot_adapter = buf[offs[3]:offs[4]]
        self.shrink_tiles = buf[offs[4]:offs[5]]
        self.tile_skip = buf[offs[5]:offs[6]] if self.n_expand_tiles else None
        self.expand_tiles = buf[offs[6]:offs[7]]
        self._tc = {nr: (buf[offs[7 + 2 * k]:offs[8 + 2 * k]], buf[offs[8 + 2 * k]:offs[9 + 2 * k]])
                    for k, nr in enumerate(TC_RANKS)} if self.tc_ctas else {}
        self.n_slots = host.n_slots
        self.max_adapter = int(host.seg_adapter.max()) if host.seg_adapter.size else -1
        self.n_shrink_tiles = int(host.shrink_tiles.shape[0])
        self.row_adapter = torch.empty(self.n_rows, dtype=torch.int32, device=dev)
        self.slot_of_row = torch.empty(self.n_rows, dtype=torch.int32, device=dev)
        if expand:
            self.expand(stream)

    def tc_units(self, nr: int):
        """(units, cta_ptr) of K1' for groups of ``nr`` ranks, or None (no partition / width)."""
        return self._tc.get(nr)

    def upload(self) -> int:
        """Re-send the (pinned) host tables to the same device buffers on the current stream —
        what a serving loop does once per pass; returns the bytes copied."""
        self._buf.copy_(self._pinned, non_blocking=True)
        return self.h2d_bytes

    def expand(self, stream: torch.cuda.Stream | None = None) -> None:
        from . import ops
        if not ops._launch("plan"):
            return
        st = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.call("collm_expand_segments", self.seg_start.data_ptr(), self.seg_adapter.data_ptr(),
                  len(self.host.seg_adapter), self.n_rows, self.tile_slot_ptr.data_ptr(),
                  self.slot_adapter.data_ptr(), self.row_adapter.data_ptr(),
                  self.slot_of_row.data_ptr(), st)
