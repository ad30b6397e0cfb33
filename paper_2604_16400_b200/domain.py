"""Value types of the co-batched LoRA layer, named after the reference's domain.

The reference's error classes (ConfigurationError domain.py:15-16, InvariantViolation :19-20) and
value types (``Request`` :45-61, ``BatchConfig`` :89-98) ARE the reference's own classes whenever
``coserve`` is importable (see :mod:`.reference`): an error the CUDA path raises is then caught by
the reference's handlers (experiment.py:43-48).  Without the reference, same-named local classes
with the same validation and messages stand in.  The one new type the unified layer needs is a
*mixed* row batch: the reference's ``Batch`` refuses to mix streams (domain.py:75-77); the unified
PEFT layer mixes adapters by design, so its row table is ``MixedBatch``, not a ``Batch``.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

from .reference import coserve_module

_ref_domain = coserve_module("domain")


class _LocalConfigurationError(ValueError):
    """Bad input or configuration detected before the kernels run."""


class _LocalInvariantViolation(RuntimeError):
    """Internal consistency check failed; indicates a bug, never expected."""


@dataclass(frozen=True)
class _LocalRequest:
    """One inference query (reference domain.py:45-61), plus its prompt/decode shape."""

    id: int
    arrival: float
    deadline: float
    output_tokens: int
    stream_id: str = "default"

    def __post_init__(self) -> None:
        if self.deadline <= self.arrival:
            raise ConfigurationError(
                f"request {self.id}: deadline {self.deadline} must exceed arrival {self.arrival}"
            )
        if self.output_tokens < 1:
            raise ConfigurationError(f"request {self.id}: output_tokens must be >= 1")


@dataclass(frozen=True)
class _LocalBatchConfig:
    """Per-replica batch sizing knobs: training micro-batch and inference batch (domain.py:89-98)."""

    train_batch: int = 0
    infer_batch: int = 0

    def __post_init__(self) -> None:
        if self.train_batch < 0 or self.infer_batch < 0:
            raise ConfigurationError("batch sizes must be non-negative")


if _ref_domain is not None:  # the drop-in: the reference's own classes
    ConfigurationError = _ref_domain.ConfigurationError
    InvariantViolation = _ref_domain.InvariantViolation
    Request = _ref_domain.Request
    BatchConfig = _ref_domain.BatchConfig
else:
    ConfigurationError = _LocalConfigurationError
    InvariantViolation = _LocalInvariantViolation
    Request = _LocalRequest
    BatchConfig = _LocalBatchConfig
USING_REFERENCE_CLASSES = _ref_domain is not None


class RowRole(enum.IntEnum):
    """Role of a segment of rows in the mixed pass."""

    TRAIN = 0
    PREFILL = 1
    DECODE = 2


@dataclass(frozen=True)
class InferenceItem:
    """Rows one inference request contributes to this pass: ``n_rows`` prompt tokens (prefill) or
    one token (decode), served with ``adapter`` (the tenant's adapter slot, -1 = base model)."""

    request_id: int
    adapter: int
    n_rows: int
    role: RowRole = RowRole.DECODE

    def __post_init__(self) -> None:
        if self.n_rows < 1:
            raise ConfigurationError(f"request {self.request_id}: n_rows must be >= 1")
        if self.role is RowRole.DECODE and self.n_rows != 1:
            raise ConfigurationError(f"request {self.request_id}: a decode item has exactly 1 row")
        if self.role is RowRole.TRAIN:
            raise ConfigurationError("inference items cannot have role TRAIN")


@dataclass(frozen=True)
class TrainItem:
    """The co-running fine-tuning micro-batch: ``batch`` sequences of ``seq_len`` tokens trained
    on ``adapter``."""

    adapter: int
    batch: int
    seq_len: int

    def __post_init__(self) -> None:
        if self.adapter < 0:
            raise ConfigurationError("the training adapter must be a registered slot (>= 0)")
        if self.batch < 1 or self.seq_len < 1:
            raise ConfigurationError("training micro-batch must have batch, seq_len >= 1")

    @property
    def rows(self) -> int:
        return self.batch * self.seq_len


@dataclass(frozen=True)
class MixedBatch:
    """The row table of one unified pass (built by :func:`segments.build_mixed_batch`).

    Rows are ``[training rows] ++ [inference rows sorted by (adapter, request id, position)]``;
    ``seg_start[s]:seg_start[s+1]`` uses adapter ``seg_adapter[s]`` in role ``seg_role[s]``;
    ``row_src[t] = (request id, position)`` for inference rows and ``(-1, i)`` for training rows.
    """

    seg_start: tuple[int, ...]
    seg_adapter: tuple[int, ...]
    seg_role: tuple[int, ...]
    row_request: tuple[int, ...]
    row_pos: tuple[int, ...]
    n_train_rows: int
    train_adapter: int
    extra: dict = field(default_factory=dict, compare=False)

    @property
    def n_rows(self) -> int:
        return self.seg_start[-1]

    @property
    def n_segments(self) -> int:
        return len(self.seg_adapter)

    @property
    def n_infer_rows(self) -> int:
        return self.n_rows - self.n_train_rows
