"""The BASELINE.json configurations of the co-batched LoRA layer stack.

Each config fixes the model shape (Llama projections per layer), the adapter population (count,
rank, alpha) and the mixed row batch of one pass (training micro-batch + inference rows drawn
deterministically from a PCG64 seed, like the reference's workload generator,
/root/reference/pkg/src/coserve/workload.py:86-106).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .domain import ConfigurationError, InferenceItem, RowRole, TrainItem
from .layer import ProjectionSpec


@dataclass(frozen=True)
class ModelShape:
    name: str
    layers: int
    hidden: int
    intermediate: int
    kv_dim: int
    vocab: int = 32000  # LM head (K7 training loss)

    def projections(self, rank: int, alpha: float, fuse: bool = True) -> list[ProjectionSpec]:
        """Per-layer projections.  q|k|v and gate|up are fused into one GEMM when their boundaries
        are multiples of 128 (the GEMM's N tile); otherwise they stay separate launches."""
        h, i, kv = self.hidden, self.intermediate, self.kv_dim
        out: list[ProjectionSpec] = []
        if fuse and h % 128 == 0 and (h + kv) % 128 == 0:
            out.append(ProjectionSpec("qkv", h, (h, kv, kv), rank, alpha))
        else:
            out += [ProjectionSpec("q", h, (h,), rank, alpha), ProjectionSpec("k", h, (kv,), rank, alpha),
                    ProjectionSpec("v", h, (kv,), rank, alpha)]
        out.append(ProjectionSpec("o", h, (h,), rank, alpha))
        if fuse and i % 128 == 0:
            out.append(ProjectionSpec("gate_up", h, (i, i), rank, alpha))
        else:
            out += [ProjectionSpec("gate", h, (i,), rank, alpha), ProjectionSpec("up", h, (i,), rank, alpha)]
        out.append(ProjectionSpec("down", i, (h,), rank, alpha))
        return out

    def flops_per_row(self) -> int:
        """Forward base-projection FLOPs per row per step over all layers (2*K*N summed)."""
        h, i, kv = self.hidden, self.intermediate, self.kv_dim
        per_layer = 2 * (h * (h + 2 * kv) + h * h + 2 * h * i + i * h)
        return per_layer * self.layers


TINY = ModelShape("tiny-llama", 2, 256, 688, 256, 512)
LLAMA2_7B = ModelShape("llama-2-7b", 32, 4096, 11008, 4096, 32000)
LLAMA3_8B = ModelShape("llama-3-8b", 32, 4096, 14336, 1024, 128256)
LLAMA2_13B = ModelShape("llama-2-13b", 40, 5120, 13824, 5120, 32000)


@dataclass(frozen=True)
class LayerConfig:
    """One BASELINE config: model, adapters and the mixed pass."""

    key: str
    model: ModelShape
    n_adapters: int
    rank: int
    alpha: float
    train_adapter: int
    train_batch: int
    train_seq: int
    description: str

    def batch(self, seed: int = 0) -> tuple[TrainItem | None, list[InferenceItem]]:
        return _BATCHERS[self.key](self, np.random.Generator(np.random.PCG64(seed)))

    @property
    def projections(self) -> list[ProjectionSpec]:
        return self.model.projections(self.rank, self.alpha)


def _tiny_batch(cfg, g):
    # 16 decode rows, 4 per adapter; train micro-batch 2 x 64
    items = [InferenceItem(i, i % cfg.n_adapters, 1, RowRole.DECODE) for i in range(16)]
    return TrainItem(cfg.train_adapter, cfg.train_batch, cfg.train_seq), items


def _split_rows(g, total: int, parts: int, lo: int, hi: int) -> list[int]:
    """`parts` positive counts in [lo, hi] summing to `total` (deterministic given g)."""
    if not (parts * lo <= total <= parts * hi):
        raise ConfigurationError("infeasible row split")
    counts = np.full(parts, lo, dtype=np.int64)
    rest = total - parts * lo
    while rest > 0:
        i = int(g.integers(0, parts))
        if counts[i] < hi:
            counts[i] += 1
            rest -= 1
    return counts.tolist()


def _7b_batch(cfg, g):
    # 32 adapters, rows per adapter in [1, 32] summing to 512: one prefill segment per adapter
    # with >= 2 rows, single rows are decode steps
    counts = _split_rows(g, 512, cfg.n_adapters, 1, 32)
    items = []
    rid = 0
    for a, n in enumerate(counts):
        n_dec = int(g.integers(0, n + 1)) if n > 1 else 1
        for _ in range(n_dec):
            items.append(InferenceItem(rid, a, 1, RowRole.DECODE))
            rid += 1
        if n - n_dec > 0:
            items.append(InferenceItem(rid, a, n - n_dec, RowRole.PREFILL))
            rid += 1
    return TrainItem(cfg.train_adapter, cfg.train_batch, cfg.train_seq), items


def _8b_batch(cfg, g):
    # 64 prefill segments, lengths lognormal(ln 256, 0.5) clipped to [16, 1024]
    lens = np.clip(np.round(g.lognormal(np.log(256.0), 0.5, cfg.n_adapters)), 16, 1024).astype(int)
    items = [InferenceItem(a, a, int(n), RowRole.PREFILL) for a, n in enumerate(lens)]
    return TrainItem(cfg.train_adapter, cfg.train_batch, cfg.train_seq), items


def _13b_batch(cfg, g):
    # training-heavy: 256 decode rows over 4 adapters
    items = [InferenceItem(i, int(g.integers(0, cfg.n_adapters)), 1, RowRole.DECODE)
             for i in range(256)]
    return TrainItem(cfg.train_adapter, cfg.train_batch, cfg.train_seq), items


_BATCHERS = {"tiny": _tiny_batch, "llama2-7b": _7b_batch, "llama3-8b": _8b_batch,
             "llama2-13b": _13b_batch}

CONFIGS: dict[str, LayerConfig] = {
    "tiny": LayerConfig("tiny", TINY, 4, 8, 16.0, 0, 2, 64,
                        "tiny Llama-style (2 layers, hidden 256, rank-8 LoRA, 4 adapters), "
                        "16 decode + 2x64 train rows"),
    "llama2-7b": LayerConfig("llama2-7b", LLAMA2_7B, 32, 16, 32.0, 0, 1, 512,
                             "Llama-2-7B, 32 inference adapters r=16 (512 mixed prefill/decode "
                             "rows) + 1x512 fine-tuning micro-batch"),
    "llama3-8b": LayerConfig("llama3-8b", LLAMA3_8B, 64, 32, 64.0, 0, 8, 1024,
                             "Llama-3-8B, prefill-heavy, 64 adapters r=32 + 8x1024 fine-tuning"),
    "llama2-13b": LayerConfig("llama2-13b", LLAMA2_13B, 4, 64, 128.0, 0, 8, 2048,
                              "Llama-2-13B, r=64, training-heavy: 8x2048 train + 256 decode rows"),
}
