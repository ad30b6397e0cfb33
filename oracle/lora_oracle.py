"""numpy restatement of the unified PEFT layer — TEST INFRASTRUCTURE ONLY (see __init__.py).

Every function restates one step of the algorithm the device path implements, with exact
(float64) arithmetic apart from the rounding points that DEFINE the computed function: the bf16
inputs, the forward's rank-space activation H16 = bf16(s.X.A^T) (the forward really multiplies
B by the rounded H, so Y and dB = dY^T.H16 are exact derivatives of that function) and the bf16
working copies of the adapter.  The backward's dH = s.dY.B_t is NOT rounded by default
(``dh_mode="exact"``): the device carries it as a bf16 hi+lo pair into the dA reduction, so dA
must match exact math to SURVEY §8(c)'s 1e-3; ``dh_mode="bf16"`` restates the single-rounding
variant (round 1's device algorithm) for comparison.

Reference anchors (/root/reference):
  * adapter layout  b_mat (d, r), a_mat (r, l), update = b_mat @ a_mat ... pkg/src/coserve/launcher.py:28-47
  * LoRA on a frozen W_pre, FedAvg of B and A separately .................. PAPER.md:359-366
  * fedavg semantics (identity for 1 client, AggregationError naming client) launcher.py:68-80
  * batch composition (replaced: single-stream Batch) ...................... domain.py:64-86
  * AdamW: the HF Trainer default optimizer; the paper keeps .backward() ... PAPER.md:578
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "bf16_round", "bf16_to_bits", "bits_to_f32", "build_rows", "expand_segments", "tile_slots",
    "slot_of_row", "shrink_tiles", "lora_shrink", "lora_forward", "lora_backward", "adamw_step", "AdamWState",
    "fedavg", "AggregationError", "projection_flops", "cross_entropy", "paged_attention",
    "causal_attention",
]


# --------------------------------------------------------------------------- bf16 helpers
def bf16_to_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern, round-to-nearest-even (NaN kept quiet)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    nan = np.isnan(f)
    out = rounded.astype(np.uint16)
    out[nan] = 0x7FC0
    return out


def bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Values of x rounded to bf16 (returned as float32)."""
    return bits_to_f32(bf16_to_bits(np.asarray(x, dtype=np.float32)))


# --------------------------------------------------------------------------- K0: rows/segments
def build_rows(train, items):
    """Row table of one mixed pass.

    train: None or (adapter, n_rows).  items: iterable of (request_id, adapter, n_rows, role).
    Rows = training rows first, then inference rows ordered by (adapter, request_id); segments are
    maximal runs of equal (adapter, role).  Returns (seg_start, seg_adapter, seg_role, row_request,
    row_pos) as python lists.
    """
    rows = []  # (adapter, role, request, pos)
    if train is not None:
        ad, n = train
        rows += [(ad, 0, -1, i) for i in range(n)]
    for rid, ad, n, role in sorted(items, key=lambda it: (it[1], it[0])):
        rows += [(ad, int(role), rid, i) for i in range(n)]
    seg_start, seg_adapter, seg_role = [0], [], []
    for i, (ad, role, _, _) in enumerate(rows):
        if i == 0 or (ad, role) != (rows[i - 1][0], rows[i - 1][1]):
            if i:
                seg_start.append(i)
            seg_adapter.append(ad)
            seg_role.append(role)
    seg_start.append(len(rows))
    return (seg_start, seg_adapter, seg_role, [r[2] for r in rows], [r[3] for r in rows])


def expand_segments(seg_start, seg_adapter) -> np.ndarray:
    out = np.empty(seg_start[-1], dtype=np.int32)
    for s, a in enumerate(seg_adapter):
        out[seg_start[s]:seg_start[s + 1]] = a
    return out


def tile_slots(row_adapter: np.ndarray, tile_m: int = 256):
    """Distinct adapters (>= 0) of each tile_m-row tile, in order of first appearance."""
    ptr, slots = [0], []
    for m0 in range(0, len(row_adapter), tile_m):
        seen = []
        for a in row_adapter[m0:m0 + tile_m].tolist():
            if a >= 0 and a not in seen:
                seen.append(a)
        slots += seen
        ptr.append(len(slots))
    return np.array(ptr, np.int32), np.array(slots, np.int32)


def slot_of_row(row_adapter, tile_slot_ptr, slot_adapter, tile_m: int = 256) -> np.ndarray:
    out = np.full(len(row_adapter), -1, np.int32)
    for t, a in enumerate(row_adapter.tolist()):
        if a < 0:
            continue
        m = t // tile_m
        for s in range(tile_slot_ptr[m], tile_slot_ptr[m + 1]):
            if slot_adapter[s] == a:
                out[t] = s
                break
    return out


def shrink_tiles(seg_start, seg_adapter, tile: int = 16) -> np.ndarray:
    """Maximal runs of equal adapter (base-only runs too, adapter -1), cut into <= tile-row items."""
    out = []
    s = 0
    while s < len(seg_adapter):
        e = s + 1
        while e < len(seg_adapter) and seg_adapter[e] == seg_adapter[s]:
            e += 1
        for r in range(seg_start[s], seg_start[e], tile):
            out.append((r, min(tile, seg_start[e] - r), seg_adapter[s]))
        s = e
    return np.array(out, np.int32).reshape(-1, 3)


# --------------------------------------------------------------------------- projection fwd/bwd
def _sub_bounds(sub_sizes):
    b = [0]
    for n in sub_sizes:
        b.append(b[-1] + n)
    return b


def lora_shrink(X, A, scale, row_adapter, chunk=4096):
    """K1's restatement: H16[t] = bf16(scale[a] * X[t] . A[a]^T) for a = row_adapter[t] >= 0 (0
    for base-only rows).  X [T, K], A [n_ad, R, K], float32 holding bf16 values; rows of one
    adapter are processed in chunks (float64 products).  Returns float32 [T, R]."""
    T = X.shape[0]
    R = A.shape[1]
    H16 = np.zeros((T, R), np.float32)
    for a in np.unique(row_adapter):
        if a < 0:
            continue
        rows = np.nonzero(row_adapter == a)[0]
        Aa = A[a].astype(np.float64).T
        for c in range(0, len(rows), chunk):
            rr = rows[c:c + chunk]
            H = float(scale[a]) * (X[rr].astype(np.float64) @ Aa)
            H16[rr] = bf16_round(H.astype(np.float32))
    return H16


def lora_forward(X, W, A, B, scale, row_adapter, sub_sizes, r_pad):
    """Forward of one (possibly fused) LoRA projection over the mixed rows.

    X [T, K], W [N, K] (N = sum(sub_sizes)), A [n_ad, R, K] (R = n_sub * r_pad; rank rows of sub s
    at s*r_pad), B [n_ad, N, r_pad], scale [n_ad]; all float32 holding bf16 values.
      H16[t]     = bf16(scale[a] * X[t] . A[a]^T)                       (a = row_adapter[t] >= 0)
      Y[t, n_s]  = X[t] . W[n_s]^T + H16[t, s*r_pad:(s+1)*r_pad] . B[a][n_s]^T
    Rows are independent: pass X[rows], row_adapter[rows] to evaluate a subset of rows.
    Returns Y (float64, before the output rounding) and H16 (float32 bf16 values; 0 for a < 0).
    """
    X64 = X.astype(np.float64)
    bounds = _sub_bounds(sub_sizes)
    Y = X64 @ W.astype(np.float64).T
    H16 = lora_shrink(X, A, scale, row_adapter)
    for a in np.unique(row_adapter):
        if a < 0:
            continue
        rows = np.nonzero(row_adapter == a)[0]
        for s in range(len(sub_sizes)):
            cols = slice(bounds[s], bounds[s + 1])
            Y[np.ix_(rows, np.arange(bounds[s], bounds[s + 1]))] += (
                H16[rows, s * r_pad:(s + 1) * r_pad].astype(np.float64)
                @ B[a][cols].astype(np.float64).T)
    return Y, H16


def lora_backward(dY, X_tr, H16_tr, W, A_t, B_t, s, sub_sizes, r_pad, dh_mode="exact",
                  dx_rows=None, chunk=2048):
    """Backward of the training rows (all on adapter t, scale s) through one projection.

      dH[:, sub s]   = s * dY[:, n_s] . B_t[n_s]                  (dh_mode "bf16": rounded)
      dX             = dY . W + dH . A_t
      dB[n_s]        = dY[:, n_s]^T . H16_tr[:, sub s]            ([N, r_pad], B_t's layout)
      dA^T           = X_tr^T . dH                                ([K, R], A_t^T's layout)
    (d/dW of the frozen base is not formed; the forward's H16 rounding is straight-through.)
    The T reductions run over row chunks (float64 partial products); ``dx_rows`` restricts dX to
    those rows (the dense dY.W term dominates the cost at BASELINE shapes).
    Returns float64 dX ([len(dx_rows) or T, K]), dB, dAT and dH (float64; float32 bf16 values
    in "bf16" mode).
    """
    if dh_mode not in ("exact", "bf16"):
        raise ValueError(f"dh_mode {dh_mode!r}")
    bounds = _sub_bounds(sub_sizes)
    T = dY.shape[0]
    R = len(sub_sizes) * r_pad
    K = X_tr.shape[1]
    dH = np.zeros((T, R), np.float64)
    dB = np.zeros((bounds[-1], r_pad))
    dAT = np.zeros((K, R))
    Bt64 = B_t.astype(np.float64)
    for c in range(0, T, chunk):
        rr = slice(c, min(T, c + chunk))
        dY64 = dY[rr].astype(np.float64)
        for si in range(len(sub_sizes)):
            ns = slice(bounds[si], bounds[si + 1])
            rs = slice(si * r_pad, (si + 1) * r_pad)
            d = s * (dY64[:, ns] @ Bt64[ns])
            dH[rr, rs] = bf16_round(d.astype(np.float32)) if dh_mode == "bf16" else d
            dB[ns] += dY64[:, ns].T @ H16_tr[rr, rs].astype(np.float64)
        dAT += X_tr[rr].astype(np.float64).T @ dH[rr]
    rows = np.arange(T) if dx_rows is None else np.asarray(dx_rows)
    dX = dY[rows].astype(np.float64) @ W.astype(np.float64) + dH[rows] @ A_t.astype(np.float64)
    return dX, dB, dAT, (dH.astype(np.float32) if dh_mode == "bf16" else dH)


def projection_flops(T, T_tr, K, N):
    """Algorithmic tensor-pipe FLOPs of one projection per step: forward of all rows + dX of the
    training rows (the frozen base has no dW) — SURVEY.md §8(d)."""
    return 2 * K * N * (T + T_tr)


# --------------------------------------------------------------------------- optimizer
@dataclass
class AdamWState:
    m: np.ndarray
    v: np.ndarray
    step: int = 0


def adamw_step(p, g, st: AdamWState, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0):
    """torch.optim.AdamW (single-tensor path) in float32: decoupled weight decay, bias-corrected."""
    p = p.astype(np.float32).copy()
    g = g.astype(np.float32)
    st.step += 1
    p *= np.float32(1.0 - lr * wd)
    st.m = (st.m + (g - st.m) * np.float32(1.0 - beta1)).astype(np.float32)
    st.v = (st.v * np.float32(beta2) + np.float32(1.0 - beta2) * g * g).astype(np.float32)
    bc1 = 1.0 - beta1 ** st.step
    bc2 = 1.0 - beta2 ** st.step
    denom = np.sqrt(st.v) / np.float32(math.sqrt(bc2)) + np.float32(eps)
    p -= np.float32(lr / bc1) * st.m / denom
    return p


# --------------------------------------------------------------------------- LM-head CE (K7)
def cross_entropy(logits, labels, grad_scale=None):
    """Next-token softmax cross-entropy of the training rows — the real loss behind the
    reference's convergence stand-in (perf.py:92-126: TrainState.loss / train_step); the paper's
    fine-tuning uses the HF Trainer's causal-LM loss.  ``logits`` [T, V] (the bf16
    GEMM output, as float), ``labels`` [T] int (< 0 or >= V: ignored row).  Returns float64
    (loss_rows [T], mean over valid rows, dlogits [T, V] = grad_scale * (softmax - onehot), zero
    for ignored rows; grad_scale defaults to 1 / #valid, the gradient of the mean)."""
    z = np.asarray(logits, dtype=np.float64)
    y = np.asarray(labels).astype(np.int64)
    T, V = z.shape
    valid = (y >= 0) & (y < V)
    m = z.max(axis=1, keepdims=True)
    lse = (m + np.log(np.exp(z - m).sum(axis=1, keepdims=True)))[:, 0]
    picked = np.where(valid, z[np.arange(T), np.clip(y, 0, V - 1)], 0.0)
    loss_rows = np.where(valid, lse - picked, 0.0)
    n = int(valid.sum())
    mean = loss_rows[valid].sum() / n if n else 0.0
    g = (1.0 / max(n, 1)) if grad_scale is None else grad_scale
    d = np.exp(z - lse[:, None])
    d[np.arange(T)[valid], y[valid]] -= 1.0
    d *= g
    d[~valid] = 0.0
    return loss_rows, mean, d


# --------------------------------------------------------------------------- attention (K9)
def causal_attention(q, k, v, seq_start, n_heads, n_kv_heads, scale=None, dout=None):
    """Causal self-attention of packed sequences (row ranges seq_start[s]..seq_start[s+1]; row i
    attends to rows [seq_start[s], i]) and, with ``dout``, its backward — float64 restatement of
    the standard softmax attention gradient (dV = P^T dO, dP = dO V^T, dS = P (dP - rowsum(dO O)),
    dQ = scale dS K, dK = scale dS^T Q; GQA: dK/dV summed over the G heads of a kv head).
    q [T, n_heads*D], k / v [T, n_kv_heads*D].  Returns out, lse2 [n_heads, T] (base-2
    log-sum-exp of scale*log2(e)*scores) and, with dout, (dq, dk, dv)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    T = q.shape[0]
    D = q.shape[1] // n_heads
    G = n_heads // n_kv_heads
    sc = D ** -0.5 if scale is None else scale
    out = np.zeros_like(q)
    lse2 = np.zeros((n_heads, T))
    grads = None
    if dout is not None:
        dout = np.asarray(dout, np.float64)
        grads = (np.zeros_like(q), np.zeros_like(k), np.zeros_like(v))
    for s in range(len(seq_start) - 1):
        a, b = int(seq_start[s]), int(seq_start[s + 1])
        n = b - a
        mask = np.tril(np.ones((n, n), bool))
        for h in range(n_heads):
            hk = h // G
            Q = q[a:b, h * D:(h + 1) * D]
            K = k[a:b, hk * D:(hk + 1) * D]
            V = v[a:b, hk * D:(hk + 1) * D]
            S = np.where(mask, Q @ K.T * sc, -np.inf)
            m = S.max(axis=1, keepdims=True)
            E = np.exp(S - m)
            Z = E.sum(axis=1, keepdims=True)
            P = E / Z
            O = P @ V
            out[a:b, h * D:(h + 1) * D] = O
            lse2[h, a:b] = (m[:, 0] + np.log(Z[:, 0])) / np.log(2.0)
            if grads is not None:
                dO = dout[a:b, h * D:(h + 1) * D]
                dP = dO @ V.T
                dS = P * (dP - (dO * O).sum(axis=1, keepdims=True))
                grads[0][a:b, h * D:(h + 1) * D] += sc * dS @ K
                grads[1][a:b, hk * D:(hk + 1) * D] += sc * dS.T @ Q
                grads[2][a:b, hk * D:(hk + 1) * D] += P.T @ dO
    return (out, lse2) if grads is None else (out, lse2, grads)


# --------------------------------------------------------------------------- attention (K8)
def paged_attention(q, k_cache, v_cache, block_table, row_seq, row_pos, n_heads, n_kv_heads,
                    scale=None):
    """Causal attention of each query row over tokens [0, pos] of its sequence's paged KV cache
    (the step either side of the LoRA projections; the reference has no
    attention).  q [T, n_heads*D]; caches [n_pages, n_kv_heads, page, D]; block_table
    [n_seq, max_pages].  float64, returns [T, n_heads*D]."""
    q = np.asarray(q, np.float64)
    kc = np.asarray(k_cache, np.float64)
    vc = np.asarray(v_cache, np.float64)
    page, D = kc.shape[2], kc.shape[3]
    G = n_heads // n_kv_heads
    sc = D ** -0.5 if scale is None else scale
    out = np.zeros((q.shape[0], n_heads * D))
    for t in range(q.shape[0]):
        n = int(row_pos[t]) + 1
        j = np.arange(n)
        pages = np.asarray(block_table)[int(row_seq[t])][j // page]
        K = kc[pages, :, j % page]  # [n, n_kv_heads, D]
        V = vc[pages, :, j % page]
        for h in range(n_heads):
            s = K[:, h // G] @ q[t, h * D:(h + 1) * D] * sc
            p = np.exp(s - s.max())
            out[t, h * D:(h + 1) * D] = (p / p.sum()) @ V[:, h // G]
    return out


# --------------------------------------------------------------------------- FedAvg
class AggregationError(ValueError):
    pass


def fedavg(clients):
    """Element-wise mean of B and of A, separately (launcher.py:68-80).  ``clients`` is a list of
    (b_mat, a_mat).  One client returns that client's arrays unchanged (launcher.py:76-77); a
    shape mismatch raises AggregationError naming the client index (launcher.py:73-75)."""
    if not clients:
        raise AggregationError("no adapters to aggregate")
    b0, a0 = clients[0]
    for idx, (b, a) in enumerate(clients):
        if b.shape != b0.shape or a.shape != a0.shape:
            raise AggregationError(f"client {idx} adapter dimensions do not match the first client")
    if len(clients) == 1:
        return b0, a0
    return (np.mean(np.stack([c[0] for c in clients]), axis=0),
            np.mean(np.stack([c[1] for c in clients]), axis=0))
