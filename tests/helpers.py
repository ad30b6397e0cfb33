"""Shared synthetic-input builders for the parity tests (seeded numpy PCG64, bf16-rounded)."""

from __future__ import annotations

import numpy as np

from oracle import bf16_round


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def mixed_items(g: np.random.Generator, n_adapters: int, n_decode: int, n_prefill: int,
                prefill_len=(2, 40), base_rows: int = 0):
    """(request_id, adapter, n_rows, role) items: decode rows (1 row) and prefill segments."""
    items = []
    rid = 0
    for _ in range(n_decode):
        items.append((rid, int(g.integers(0, n_adapters)), 1, 2))
        rid += 1
    for _ in range(n_prefill):
        items.append((rid, int(g.integers(0, n_adapters)), int(g.integers(*prefill_len)), 1))
        rid += 1
    for _ in range(base_rows):
        items.append((rid, -1, 1, 2))
        rid += 1
    return items


def projection_inputs(g: np.random.Generator, T: int, T_tr: int, K: int, subs, rank: int,
                      r_pad: int, n_adapters: int, alpha: float = 16.0):
    """bf16-valued float32 arrays for one fused projection (SURVEY §8(d) init: W ~ N(0, .02^2),
    A ~ U(+-1/sqrt(K)), B ~ N(0, .02^2) non-zero so the expand is exercised, X ~ N(0,1))."""
    N = int(sum(subs))
    R = len(subs) * r_pad
    X = bf16_round(g.standard_normal((T, K), dtype=np.float32))
    W = bf16_round(0.02 * g.standard_normal((N, K), dtype=np.float32))
    A = np.zeros((n_adapters, R, K), np.float32)
    B = np.zeros((n_adapters, N, r_pad), np.float32)
    bnd = np.cumsum([0] + list(subs))
    lim = 1.0 / np.sqrt(K)
    for a in range(n_adapters):
        for s in range(len(subs)):
            A[a, s * r_pad:s * r_pad + rank] = bf16_round(
                g.uniform(-lim, lim, (rank, K)).astype(np.float32))
            B[a, bnd[s]:bnd[s + 1], :rank] = bf16_round(
                0.02 * g.standard_normal((subs[s], rank), dtype=np.float32))
    scale = np.array([alpha / rank * (1 + 0.25 * a) for a in range(n_adapters)], np.float32)
    dY = bf16_round(g.standard_normal((T_tr, N), dtype=np.float32))
    return dict(X=X, W=W, A=A, B=B, scale=scale, dY=dY)
