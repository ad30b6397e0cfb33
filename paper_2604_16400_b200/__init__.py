"""B200-native co-batched LoRA layer (CoLLM's unified PEFT layer, arxiv 2604.16400).

One forward/backward pass in which a replica's frozen base weights serve a mixed token batch:
inference rows (prefill + decode, each tagged with its tenant's adapter) and the training rows of
the co-running fine-tuning micro-batch.  The compute path is the C-ABI library ``libcollm.so``
(hand-written sm_100a kernels, see ``include/collm.h``); this package is the Python host side
mirroring the reference's API (/root/reference/pkg/src/coserve).
"""

from .domain import (BatchConfig, ConfigurationError, InferenceItem, InvariantViolation,
                     MixedBatch, Request, RowRole, TrainItem)

__all__ = [
    "BatchConfig", "ConfigurationError", "InferenceItem", "InvariantViolation", "MixedBatch",
    "Request", "RowRole", "TrainItem",
]
