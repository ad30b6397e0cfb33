"""Typed torch-tensor wrappers over the collm C ABI (one function per ABI entry point).

Torch is plumbing here (device memory, streams); every computation is a collm kernel.  Each
wrapper validates dtypes/devices, picks the split factors, and launches on the current stream.
"""

from __future__ import annotations

import math
import threading
from contextlib import contextmanager

import torch

from . import _lib


class _LaunchFilter(threading.local):
    """Per-thread launch accounting: which op kinds are issued ('plan', 'lora', 'gemm') and how
    many collm kernels were launched.  Used by bench.py to build GEMM-only / LoRA-only graphs
    of the same step (per-kernel roofline timing) and to count launches."""

    def __init__(self) -> None:
        self.kinds: set[str] | None = None
        self.count = 0


_filter = _LaunchFilter()


@contextmanager
def only(*kinds: str):
    prev = _filter.kinds
    _filter.kinds = set(kinds)
    try:
        yield
    finally:
        _filter.kinds = prev


def enabled(kind: str) -> bool:
    """'lora' stands for both rank-space kinds ('shrink' = K1, 'reduce' = K5 + apply); 'head' (K7
    cross-entropy) rides with 'gemm' (the LM-head GEMMs)."""
    k = _filter.kinds
    return (k is None or kind in k or (kind in ("shrink", "reduce") and "lora" in k)
            or (kind == "head" and "gemm" in k))


def launch_count() -> int:
    return _filter.count


def _launch(kind: str) -> bool:
    if not enabled(kind):
        return False
    _filter.count += 1
    return True

NUM_SMS_DEFAULT = 148
# timing experiments only: GEMMs ignore the shrink completion flag (results are then undefined)
_NO_WAIT = __import__("os").environ.get("COLLM_DEBUG_NO_FLAG_WAIT") == "1"
_sms_cache: dict[int, int] = {}


def num_sms(device: torch.device | None = None) -> int:
    d = (device or torch.device("cuda")).index or 0
    if d not in _sms_cache:
        _sms_cache[d] = torch.cuda.get_device_properties(d).multi_processor_count
    return _sms_cache[d]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if t.dtype != dtype or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA {dtype} tensor, got {t.dtype} on {t.device}")
    if t.stride(-1) != 1:
        raise TypeError(f"{name}: innermost dimension must be contiguous")


class Workspace:
    """Grow-only, zero-initialised scratch for the split-K / split-T ordered reductions.

    The kernels restore their arrival counters to zero, so the buffer stays valid across launches
    and CUDA-graph replays.  Size it (call once outside capture) before capturing a graph."""

    def __init__(self) -> None:
        self._bufs: dict[int, torch.Tensor] = {}
        self._lock = threading.Lock()

    def get(self, nbytes: int, device: torch.device) -> torch.Tensor | None:
        if nbytes <= 0:
            return None
        d = device.index or 0
        with self._lock:
            buf = self._bufs.get(d)
            if buf is None or buf.numel() < nbytes:
                if torch.cuda.is_current_stream_capturing():
                    raise RuntimeError("collm workspace must be sized before CUDA graph capture")
                nb = max(nbytes, 1 << 20)
                buf = torch.zeros(nb, dtype=torch.uint8, device=device)
                self._bufs[d] = buf
            return buf


_reduce_ws = Workspace()
_gemm_ws = Workspace()
_shrink_tc_ws = Workspace()  # its own: a partition shrink runs concurrently with a GEMM


def lora_shrink(X: torch.Tensor, A: torch.Tensor, tiles: torch.Tensor, n_tiles: int,
                scale: torch.Tensor, groups: list[tuple[int, int, int, int]], ldh: int, *,
                a_stride: int | None = None, H32: torch.Tensor | None = None,
                H16: torch.Tensor | None = None, H16lo: torch.Tensor | None = None,
                Hslots: torch.Tensor | None = None,
                slot_of_row: torch.Tensor | None = None,
                tile_slot_ptr: torch.Tensor | None = None, signal: torch.Tensor | None = None,
                gen: torch.Tensor | None = None) -> None:
    """K1: H[t, ranks of g] = scale[a] * X[t, K-range of g] . A_a[ranks of g]^T (see collm.h).
    ``H16lo``: also write bf16(h - H16), the lo half of a bf16 hi+lo pair.
    ``signal``/``gen``: publish completion for a GEMM consuming the output on another stream."""
    _need(X, torch.bfloat16, "X")
    _need(A, torch.bfloat16, "A")
    if n_tiles == 0 or not _launch("shrink"):
        return
    lda = A.stride(-2)
    if a_stride is None:
        a_stride = A.stride(0) if A.dim() == 3 else 0
    flat = [v for g in groups for v in g]
    _lib.call("collm_lora_shrink", X.data_ptr(), X.stride(0), A.data_ptr(), int(a_stride), lda,
              tiles.data_ptr(), n_tiles, scale.data_ptr(), _lib.int_array(flat), len(groups),
              _p(H32), _p(H16), _p(H16lo), ldh, _p(Hslots), _p(slot_of_row), _p(tile_slot_ptr), _p(signal),
              _p(gen), _stream())


_rank_sms: dict[int, int] = {}


def set_rank_sms(n: int, device: torch.device | None = None) -> None:
    """Reserve ``n`` SMs (even, whole TPCs) of ``device`` for the rank-space kernels
    (collm_set_rank_sms): shrinks then run as ``collm_lora_shrink_tc`` on that partition and every
    GEMM grid is capped at the remaining SMs.  0 switches back to the whole-GPU shrink."""
    d = (device or torch.device("cuda", torch.cuda.current_device())).index or 0
    with torch.cuda.device(d):
        _lib.call("collm_set_rank_sms", int(n))
    _rank_sms[d] = int(n)


def set_flash_impl(tc: int) -> None:
    """K9 forward kernel: 1 = tcgen05/TMEM (default), 0 = mma.sync (collm_set_flash_impl)."""
    _lib.call("collm_set_flash_impl", int(tc))


def flash_impl() -> int:
    return int(_lib.load().collm_get_flash_impl())


def rank_sms(device: torch.device | None = None) -> int:
    d = (device or torch.device("cuda", torch.cuda.current_device())).index or 0
    if d not in _rank_sms:
        n = int(__import__("os").environ.get("COLLM_RANK_SMS", "0"))
        if n:
            set_rank_sms(n, torch.device("cuda", d))
        else:
            _rank_sms[d] = 0
    return _rank_sms[d]


def shrink_tc_groups(groups: list[tuple[int, int, int, int]]) -> list[tuple[int, int, int, int]] | None:
    """The group table for collm_lora_shrink_tc, or None when it does not apply: adjacent groups
    over the same K range merge into one (<= 256 ranks), every group must then have the same
    width (a multiple of 16) and 64-aligned K ranges."""
    out: list[list[int]] = []
    for ro, nr, klo, khi in groups:
        if out and out[-1][2] == klo and out[-1][3] == khi and out[-1][0] + out[-1][1] == ro \
                and out[-1][1] + nr <= 256:
            out[-1][1] += nr
        else:
            out.append([ro, nr, klo, khi])
    if len({g[1] for g in out}) != 1 or len(out) > 8:
        return None
    if any(g[1] % 16 or g[2] % 64 or g[3] % 64 for g in out):
        return None
    return [tuple(g) for g in out]


def lora_shrink_tc(X: torch.Tensor, A: torch.Tensor, items: torch.Tensor, cta_ptr: torch.Tensor,
                   n_ctas: int, row_adapter: torch.Tensor, scale: torch.Tensor,
                   groups: list[tuple[int, int, int, int]],
                   ldh: int, *, a_stride: int | None = None, H32: torch.Tensor | None = None,
                   H16: torch.Tensor | None = None, H16lo: torch.Tensor | None = None,
                   Hslots: torch.Tensor | None = None, slot_of_row: torch.Tensor | None = None,
                   tile_slot_ptr: torch.Tensor | None = None) -> None:
    """K1 on the rank-space SM partition (collm_lora_shrink_tc): same outputs as lora_shrink;
    ``groups`` from :func:`shrink_tc_groups`, units / cta_ptr from ``plan.tc_units(nr)``,
    ``row_adapter`` the plan's device expansion."""
    _need(X, torch.bfloat16, "X")
    _need(A, torch.bfloat16, "A")
    if not _launch("shrink"):
        return
    lda = A.stride(-2)
    if a_stride is None:
        a_stride = A.stride(0) if A.dim() == 3 else 0
    a_rows = A.numel() // lda
    flat = [v for g in groups for v in g]
    n_chunks = items.numel() // 8
    ws = _shrink_tc_ws.get(_lib.load().collm_shrink_tc_workspace_bytes(n_chunks, len(groups)),
                           X.device)
    _lib.call("collm_lora_shrink_tc", X.data_ptr(), X.stride(0), X.shape[0], A.data_ptr(),
              int(a_stride), lda, a_rows, items.data_ptr(), cta_ptr.data_ptr(), n_ctas, n_chunks,
              row_adapter.data_ptr(), scale.data_ptr(), _lib.int_array(flat), len(groups), _p(H32),
              _p(H16), _p(H16lo), ldh, _p(Hslots), _p(slot_of_row), _p(tile_slot_ptr), _p(ws),
              0 if ws is None else ws.numel(), _stream())


def gemm_lora(A: torch.Tensor, B: torch.Tensor, Y: torch.Tensor, *, M: int | None = None,
              Hslots: torch.Tensor | None = None, h_rows: int = 0, LB: torch.Tensor | None = None,
              lb_rows: int = 0, tile_slot_ptr: torch.Tensor | None = None,
              slot_adapter: torch.Tensor | None = None, lora_rank: int = 0,
              lb_rows_per_adapter: int = 0, sub_n_start: list[int] | None = None,
              sub_h_col: list[int] | None = None, bn: int = 0,
              lora_flag: torch.Tensor | None = None, gen: torch.Tensor | None = None,
              lora_pdl: bool = False, tile_skip: torch.Tensor | None = None) -> None:
    """K2/K3: Y[M,N] = A[M,K] . B[N,K]^T (+ fused multi-adapter LoRA expand), bf16 -> bf16.
    ``lora_flag``/``gen``: wait for a concurrently running shrink's signal before the LoRA
    stages (see collm.h); ``lora_pdl``: launch programmatically dependent on the shrink launched
    just before on the same stream instead (see collm.h)."""
    for t, n in ((A, "A"), (B, "B"), (Y, "Y")):
        _need(t, torch.bfloat16, n)
    M = A.shape[0] if M is None else M
    K = A.shape[1]
    N = B.shape[0]
    if B.shape[1] != K or Y.shape[1] < N or Y.shape[0] < M:
        raise ValueError(f"gemm_lora shapes: A {tuple(A.shape)} B {tuple(B.shape)} Y {tuple(Y.shape)}")
    if not _launch("gemm"):
        return
    lora = tile_slot_ptr is not None
    if _filter.kinds is not None and "nolora" in _filter.kinds:  # timing only: base GEMM alone
        lora = False
    if not enabled("shrink") or _NO_WAIT:  # a timing graph without the shrinks: nothing to wait for
        lora_flag = gen = None
        lora_pdl = False
    n_sub = len(sub_n_start) - 1 if (lora and sub_n_start) else 1
    ws = _gemm_ws.get(_lib.load().collm_gemm_workspace_bytes(0), A.device)
    _lib.call(
        "collm_gemm_lora_ex", A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), Y.data_ptr(),
        Y.stride(0), M, N, K,
        _p(Hslots) if lora else None, Hslots.stride(0) if lora else 0, h_rows,
        _p(LB) if lora else None, LB.stride(-2) if lora else 0, lb_rows,
        _p(tile_slot_ptr) if lora else None, _p(slot_adapter) if lora else None, lora_rank,
        lb_rows_per_adapter, n_sub,
        _lib.int_array(sub_n_start) if (lora and sub_n_start) else None,
        _lib.int_array(sub_h_col) if (lora and sub_h_col) else None, bn, _p(ws),
        0 if ws is None else ws.numel(), _p(lora_flag) if lora else None,
        _p(gen) if lora else None, int(bool(lora_pdl and lora)),
        _p(tile_skip) if lora else None, _stream())


def lora_expand_rows(Y: torch.Tensor, H16: torch.Tensor, B: torch.Tensor, row_adapter: torch.Tensor,
                     tiles: torch.Tensor, n_tiles: int, T: int, *, r_pad: int,
                     sub_n_start: list[int] | None = None,
                     sub_h_col: list[int] | None = None) -> None:
    """Per-row expand of the many-adapter slot tiles the GEMM skipped (collm_lora_expand_rows):
    Y[t] += H16[t, sub's ranks] . B_{a(t)}^T.  B = the registry's [n_adapters, N, r_pad]."""
    for t, n in ((Y, "Y"), (H16, "H16"), (B, "B")):
        _need(t, torch.bfloat16, n)
    if n_tiles == 0 or not _launch("shrink"):  # rank-space work (timing kinds, see enabled())
        return
    N = B.shape[-2]
    n_sub = len(sub_n_start) - 1 if sub_n_start else 1
    _lib.call("collm_lora_expand_rows", Y.data_ptr(), Y.stride(0), N, H16.data_ptr(),
              H16.stride(0), B.data_ptr(), r_pad, row_adapter.data_ptr(), tiles.data_ptr(),
              n_tiles, T, n_sub, _lib.int_array(sub_n_start) if sub_n_start else None,
              _lib.int_array(sub_h_col) if sub_h_col else None, _stream())


def set_reduce_impl(tc: int) -> None:
    """K5 kernel: 1 = TMA + tcgen05 stream (default), 0 = mma.sync (collm_set_reduce_impl)."""
    _lib.call("collm_set_reduce_impl", int(tc))


def reduce_impl() -> int:
    return int(_lib.load().collm_get_reduce_impl())


def reduce_tsplit(T: int, n_tiles: int, device: torch.device) -> int:
    if reduce_impl():
        # persistent, one CTA per SM: ~8 units per CTA keeps the static share balanced; parts are
        # whole 128-row chunks
        # (static share per CTA balanced to within ~8 %; parts of >= 8 whole 128-row chunks, so
        # the partial round trip stays small next to the stream)
        chunks, sms = math.ceil(T / 128), num_sms(device)
        env = __import__("os").environ.get("COLLM_K5_TSPLIT")
        if env:
            return max(1, min(int(env), chunks))
        for ts in range(1, 129):
            if chunks < 8 * ts:
                break
            units = n_tiles * ts / sms
            if math.ceil(units) <= 1.08 * units:
                return ts
        return 1
    # one wave: the kernel keeps 3 CTAs/SM resident; keep >= 3 32-row chunks per split
    chunks = math.ceil(T / 32)
    want = (3 * num_sms(device)) // max(1, n_tiles)
    return max(1, min(want, chunks // 3, 128))


def reduce_group(U=None, V=None, *, u_off=0, P, v_off=0, Q, ldc, c_row_off=0, c_col_off=0,
                 grad=None, master=None, m=None, v=None, out_same=None, out_trans=None,
                 ld_trans=0, t_row_off=0, t_col_off=0, V2=None) -> _lib.ReduceGroup:
    """One ``collm_reduce_group``: C[p,q] = sum_t U[t,u_off+p] (V + V2)[t,v_off+q] and its
    targets (``V2`` optional, same layout as V: the lo half of a bf16 hi+lo pair)."""
    if V2 is not None and (V is None or V2.stride(0) != V.stride(0)):
        raise ValueError("V2 must have V's layout")
    return _lib.ReduceGroup(
        _p(U), _p(V), _p(grad), _p(master), _p(m), _p(v), _p(out_same), _p(out_trans),
        U.stride(0) if U is not None else 0, V.stride(0) if V is not None else 0,
        u_off, P, v_off, Q, ldc, ld_trans, c_row_off, c_col_off, t_row_off, t_col_off, _p(V2))


def lora_reduce(T: int, groups: list, mode: int, *, accum_in: bool = False,
                grad_scale: float = 1.0, adamw: torch.Tensor | None = None,
                tsplit: int | None = None, device: torch.device | None = None) -> None:
    """K5: C = U^T V per group -> grad store or fused AdamW, one launch (see collm.h)."""
    if not _launch("reduce"):
        return
    arr = (_lib.ReduceGroup * len(groups))(*groups)
    device = device or torch.device("cuda", torch.cuda.current_device())
    if tsplit is None:
        n_tiles = sum(math.ceil(g.P / 128) for g in groups)
        tsplit = reduce_tsplit(T, n_tiles, device)
    ws_bytes = _lib.load().collm_reduce_workspace_bytes(arr, len(groups), tsplit)
    ws = _reduce_ws.get(ws_bytes, device)
    _lib.call("collm_lora_reduce", T, arr, len(groups), mode, int(accum_in), float(grad_scale),
              _p(adamw), tsplit, _p(ws), 0 if ws is None else ws.numel(), _stream())


def lora_apply(groups: list, mode: int, *, adamw: torch.Tensor | None = None) -> None:
    if not _launch("reduce"):
        return
    arr = (_lib.ReduceGroup * len(groups))(*groups)
    _lib.call("collm_lora_apply", arr, len(groups), mode, _p(adamw), _stream())


def cross_entropy(logits: torch.Tensor, labels: torch.Tensor, V: int, *,
                  loss_rows: torch.Tensor, loss_mean: torch.Tensor | None = None,
                  counter: torch.Tensor | None = None, dlogits: torch.Tensor | None = None,
                  grad_scale: float = 1.0) -> None:
    """K7: per-row softmax cross-entropy of bf16 logits [T, >=V] against int32 labels (< 0 =
    ignored), the row-ordered mean over valid rows, and dlogits = grad_scale*(softmax - onehot)."""
    _need(logits, torch.bfloat16, "logits")
    _need(labels, torch.int32, "labels")
    _need(loss_rows, torch.float32, "loss_rows")
    T = labels.shape[0]
    if logits.shape[0] < T or loss_rows.shape[0] < T:
        raise ValueError(f"cross_entropy: logits {tuple(logits.shape)} / loss_rows vs T={T}")
    if dlogits is not None:
        _need(dlogits, torch.bfloat16, "dlogits")
    if not _launch("head"):
        return
    _lib.call("collm_cross_entropy", logits.data_ptr(), logits.stride(0), T, V, labels.data_ptr(),
              loss_rows.data_ptr(), _p(loss_mean), _p(counter), _p(dlogits),
              dlogits.stride(0) if dlogits is not None else 0, float(grad_scale), _stream())


_attn_ws = Workspace()


def paged_attention(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                    block_table: torch.Tensor, row_seq: torch.Tensor, row_pos: torch.Tensor,
                    out: torch.Tensor, *, n_heads: int, n_kv_heads: int, max_ctx: int,
                    scale: float | None = None) -> None:
    """K8: out[t, h] = causal attention of query row t over tokens [0, row_pos[t]] of its
    sequence's paged KV cache (see collm.h).  q / out [T, n_heads*128] bf16, caches
    [n_pages, n_kv_heads, page, 128] bf16 (head-major pages), block_table [n_seq, max_pages] int32."""
    for t, n in ((q, "q"), (k_cache, "k_cache"), (v_cache, "v_cache"), (out, "out")):
        _need(t, torch.bfloat16, n)
    for t, n in ((block_table, "block_table"), (row_seq, "row_seq"), (row_pos, "row_pos")):
        _need(t, torch.int32, n)
    T = row_pos.shape[0]
    D = k_cache.shape[-1]
    if k_cache.shape != v_cache.shape or k_cache.shape[1] != n_kv_heads:
        raise ValueError(f"paged_attention: caches {tuple(k_cache.shape)} / {tuple(v_cache.shape)}")
    if not _launch("attention"):
        return
    ws_bytes = _lib.load().collm_attention_workspace_bytes(T, n_heads, n_kv_heads, max_ctx)
    ws = _attn_ws.get(ws_bytes, q.device)
    _lib.call("collm_paged_attention", q.data_ptr(), q.stride(0), T, n_heads, n_kv_heads, D,
              k_cache.data_ptr(), v_cache.data_ptr(), k_cache.shape[2], block_table.data_ptr(),
              block_table.stride(0), row_seq.data_ptr(), row_pos.data_ptr(), max_ctx,
              float(scale if scale is not None else D ** -0.5), out.data_ptr(), out.stride(0),
              _p(ws), 0 if ws is None else ws.numel(), _stream())


def seq_rows(bounds, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-row sequence bounds for K9 from sequence boundaries [0, b1, ..., T]: (row_start,
    row_end) int32 [T] on ``device``."""
    import numpy as np
    b = np.asarray(bounds, np.int64)
    lens = np.diff(b)
    rs = np.repeat(b[:-1], lens).astype(np.int32)
    re = np.repeat(b[1:], lens).astype(np.int32)
    return torch.from_numpy(rs).to(device), torch.from_numpy(re).to(device)


def flash_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
                    lse: torch.Tensor, row_start: torch.Tensor, row_end: torch.Tensor, *, T: int,
                    n_heads: int, n_kv_heads: int, scale: float | None = None,
                    stat_ld: int = 0) -> None:
    """K9 forward: causal attention of the packed sequences (see collm.h).  q / k / v / out may be
    column views of the fused q|k|v output (row stride = its width); lse fp32 [n_heads, stat_ld];
    row_start / row_end from :func:`seq_rows`."""
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _need(t, torch.bfloat16, n)
    _need(lse, torch.float32, "lse")
    _need(row_start, torch.int32, "row_start")
    _need(row_end, torch.int32, "row_end")
    if not _launch("attention"):
        return
    D = 128
    _lib.call("collm_flash_attention_fwd", q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0),
              v.data_ptr(), v.stride(0), out.data_ptr(), out.stride(0), lse.data_ptr(), T,
              n_heads, n_kv_heads, D, row_start.data_ptr(), row_end.data_ptr(),
              float(scale if scale is not None else D ** -0.5), stat_ld or lse.stride(0), _stream())


def flash_attention_bwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
                        dout: torch.Tensor, lse: torch.Tensor, delta: torch.Tensor,
                        dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor,
                        row_start: torch.Tensor, row_end: torch.Tensor, *, T: int, n_heads: int,
                        n_kv_heads: int, scale: float | None = None, stat_ld: int = 0) -> None:
    """K9 backward: dq / dk / dv of :func:`flash_attention` over rows [0, T) (deterministic;
    delta fp32 [n_heads, stat_ld] workspace)."""
    for t, n in ((q, "q"), (k, "k"), (v, "v"), (out, "out"), (dout, "dout"), (dq, "dq"),
                 (dk, "dk"), (dv, "dv")):
        _need(t, torch.bfloat16, n)
    _need(lse, torch.float32, "lse")
    _need(delta, torch.float32, "delta")
    if not _launch("attention"):
        return
    D = 128
    _lib.call("collm_flash_attention_bwd", q.data_ptr(), q.stride(0), k.data_ptr(), k.stride(0),
              v.data_ptr(), v.stride(0), out.data_ptr(), out.stride(0), dout.data_ptr(),
              dout.stride(0), lse.data_ptr(), delta.data_ptr(), dq.data_ptr(), dq.stride(0),
              dk.data_ptr(), dk.stride(0), dv.data_ptr(), dv.stride(0), T, n_heads, n_kv_heads, D,
              row_start.data_ptr(), row_end.data_ptr(),
              float(scale if scale is not None else D ** -0.5), stat_ld or lse.stride(0), _stream())
