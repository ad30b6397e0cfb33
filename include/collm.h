/* collm.h — C ABI of the B200 co-batched LoRA layer (CoLLM unified PEFT layer).
 *
 * The drop-in boundary for the reference's replica-step hot path.  The reference (coserve,
 * /root/reference/pkg/src/coserve) is pure Python and binds no native code; the functions below are
 * what its Python seam calls (via ctypes) in place of the stand-ins it uses
 * today:
 *
 *   perf.true_infer_latency      perf.py:62-74     -> collm_lora_shrink + collm_gemm_lora (forward)
 *   perf.true_train_latency      perf.py:77-89     -> forward + collm_lora_shrink (dH) +
 *                                                     collm_gemm_lora (dX) + collm_lora_reduce
 *   perf.train_step              perf.py:111-126   -> collm_lora_reduce(mode=ADAMW) (real update)
 *   AdapterParams.perturbed      launcher.py:43-47 -> collm_lora_reduce(mode=ADAMW)
 *   fedavg                       launcher.py:68-80 -> NCCL allreduce(avg) + collm_lora_apply(COPY)
 *   domain.Batch / pop_up_to     domain.py:64-86, dispatcher.py:66-82
 *                                                  -> collm_plan_segments + collm_expand_segments
 *   TrainState.loss / train_step perf.py:92-126    -> collm_cross_entropy (real LM-head loss)
 *
 * Conventions: plain C types, device pointers for tensors (bf16 = 2-byte bfloat16, row-major,
 * leading dimensions in ELEMENTS), `stream` is a cudaStream_t passed as void*.  All launches are
 * asynchronous on `stream`; nothing allocates or frees on the hot path (workspaces are
 * caller-owned, sized by the *_workspace_bytes functions, zero-filled once before first use).
 * Every function returns a collm_status; the message of the last failure on the calling thread is
 * available from collm_last_error().  The error classes mirror the reference's exceptions:
 * COLLM_EINVAL -> ConfigurationError (domain.py:15-16), COLLM_EINTERNAL -> InvariantViolation
 * (domain.py:19-20), COLLM_ECUDA -> RuntimeError.  No function aborts the process.
 */
#ifndef COLLM_H_
#define COLLM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  COLLM_OK = 0,
  COLLM_EINVAL = 1,       /* bad shape / rank / segment table: ConfigurationError */
  COLLM_EINTERNAL = 2,    /* internal invariant broken: InvariantViolation */
  COLLM_ECUDA = 3,        /* CUDA runtime/driver error */
  COLLM_EUNSUPPORTED = 4, /* not an sm_100 device, or a configuration this build does not cover */
} collm_status;

enum { COLLM_MODE_STORE_GRAD = 0, COLLM_MODE_ADAMW = 1, COLLM_MODE_COPY_ONLY = 2 };

/* ---- library / device --------------------------------------------------------------------- */
int collm_version(void);
const char* collm_last_error(void);
/* Load every kernel of the library now (call once per process before the first step): CUDA lazy
 * loading would load a kernel at its first launch, which can implicitly synchronize the device —
 * a deadlock when a running GEMM waits for the shrink being launched on another stream. */
int collm_preload(void);
/* Fills compute capability and SM count; COLLM_EUNSUPPORTED unless sm_100. */
int collm_device_info(int device, int* sm_major, int* sm_minor, int* num_sms);

/* ---- K0: batch composition (host planning + device expansion) -------------------------------
 * Segment table of the mixed batch: rows [seg_start[s], seg_start[s+1]) use adapter
 * seg_adapter[s] (-1 = base model only).  Replaces domain.Batch (domain.py:64-86), which may not
 * mix streams (domain.py:75-77).
 *
 * collm_plan_segments (HOST, pure CPU): per 256-row slot tile the distinct adapters in order of first
 * appearance (tile_slot_ptr[n_tiles+1], slot_adapter[n_slots]) — the LoRA "slots" the GEMM folds
 * into its accumulator — and the shrink work list: maximal same-adapter runs cut into <=16-row
 * tiles (shrink_tiles[3*i] = row_start, n_rows, adapter; base-only runs included with adapter
 * -1).  Capacities are checked (COLLM_EINVAL). */
int collm_plan_segments(const int32_t* seg_start, const int32_t* seg_adapter, int n_seg,
                        int n_rows, int32_t* tile_slot_ptr, int32_t* slot_adapter, int slot_cap,
                        int32_t* n_slots, int32_t* shrink_tiles, int shrink_tile_cap,
                        int32_t* n_shrink_tiles);

/* DEVICE: row_adapter[t], slot_of_row[t] (either may be NULL). */
int collm_expand_segments(const int32_t* seg_start, const int32_t* seg_adapter, int n_seg,
                          int n_rows, const int32_t* tile_slot_ptr, const int32_t* slot_adapter,
                          int32_t* row_adapter, int32_t* slot_of_row, void* stream);

/* ---- K1: LoRA shrink (SGMV) ------------------------------------------------------------------
 * H[t, g.rank_off + j] = scale[a] * sum_{k in [g.k_lo, g.k_hi)} X[t,k] * A[a][g.rank_off + j, k]
 * for each shrink tile (rows of one adapter a; a = -1 -> no LoRA, zeros) and each rank group g
 * (groups: n_groups x 4 ints rank_off, n_ranks (multiple of 8, <= 64), k_lo, k_hi).  Outputs
 * (each optional): H32 fp32 [T, ldh]; H16 bf16 [T, ldh]; H16lo bf16 [T, ldh] = bf16(h - H16), so
 * H16 + H16lo carries the fp32 result to ~2^-16 relative (the backward's dH feeding the dA
 * reduction: collm_reduce_group.V2); Hslots bf16 [n_slots*256, ldh] — the
 * GEMM's LoRA slot blocks, written completely: row t's value at row slot_of_row[t]*256 + t%256 and
 * zeros in the other slots of its 256-row slot tile (tile_slot_ptr).  One CTA per (tile, group) covers
 * the whole K range; the reduction is in-CTA and fixed-order (deterministic, no workspace).
 * Optional completion signal (signal and gen both non-NULL, device memory): signal = 2 int32,
 * zeroed once; gen = the current step generation.  When every output is written the kernel sets
 * signal[1] = *gen (release, gpu scope) and restores signal[0] = 0: the GEMM consuming Hslots /
 * H16 on another stream waits for exactly that (collm_gemm_lora lora_flag), so the shrink runs
 * concurrently with that GEMM's main loop.
 * Replaces: the inference half of perf.true_infer_latency (perf.py:62-74). */
int collm_lora_shrink(const void* X, int ldx, const void* A, long long a_stride, int lda,
                      const int32_t* tiles, int n_tiles, const float* scale, const int32_t* groups,
                      int n_groups, float* H32, void* H16, void* H16lo, int ldh, void* Hslots,
                      const int32_t* slot_of_row, const int32_t* tile_slot_ptr, int32_t* signal,
                      const int32_t* gen, void* stream);

/* ---- K1 on a rank-space SM partition (TMA + tcgen05) -----------------------------------------
 * collm_set_rank_sms(n): reserve n SMs (even: whole TPCs; 0 = off, the default) of the caller's
 * current device for collm_lora_shrink_tc; every GEMM grid is capped at the other SMs, so a
 * shrink and the GEMM it overlaps are always co-resident.
 * collm_plan_shrink_windows (HOST): work units over windows of 128 consecutive rows; the distinct
 * adapters of a window (from collm_plan_segments' shrink tiles) are cut into runs of consecutive
 * ids whose span rounded up to 2^c keeps 2^c * nr <= 256; base-only rows get a zero unit
 * (a_lo = -1); big units' K ranges are split into S <= 8 parts (about 2 chunks per CTA); chunks
 * (items[8*i] = row0, n_rows, a_lo, c, S, part, first chunk of the unit, unit) are assigned
 * longest-first to n_ctas CTAs (CTA k: chunks [cta_ptr[k], cta_ptr[k+1])).
 * collm_lora_shrink_tc: the collm_lora_shrink contract (same outputs, same group table; here every
 * group has the same n_ranks, a multiple of 16 <= 256, and 64-aligned K ranges) computed by n_ctas
 * CTAs (the rank-space partition): per unit and 64 K, one TMA box of the window's X rows and one of
 * the 2^c adapters' rank rows, ONE tcgen05.mma per 16 K with the adapters stacked in N (a row
 * keeps its own adapter's columns); accumulators in TMEM; split units: each part stores its fp32
 * partial in `workspace` (collm_shrink_tc_workspace_bytes(n_chunks, n_groups), zero-filled once:
 * arrival counters are restored) and the last part to arrive sums them in part order
 * (deterministic).  row_adapter [T] (the plan's device expansion).  x_rows / a_rows bound the X / A row ranges (rows past them read as zero); A row of
 * (adapter a, rank j) = a * (a_stride / lda) + j.  The kernel lets a programmatically dependent
 * GEMM launch at once (collm_gemm_lora lora_pdl = 1).
 * Replaces: the inference half of perf.true_infer_latency (perf.py:62-74). */
int collm_set_rank_sms(int n);
int collm_get_rank_sms(void);
int collm_plan_shrink_windows(const int32_t* tiles, int n_tiles, int nr, int n_ctas,
                              int32_t* items, int item_cap, int32_t* n_items, int32_t* cta_ptr);
size_t collm_shrink_tc_workspace_bytes(int n_chunks, int n_groups);
int collm_lora_shrink_tc(const void* X, int ldx, int x_rows, const void* A, long long a_stride,
                         int lda, int a_rows, const int32_t* items, const int32_t* cta_ptr,
                         int n_ctas, int n_chunks, const int32_t* row_adapter, const float* scale,
                         const int32_t* groups, int n_groups, float* H32, void* H16, void* H16lo,
                         int ldh, void* Hslots, const int32_t* slot_of_row,
                         const int32_t* tile_slot_ptr, void* workspace, size_t ws_bytes,
                         void* stream);

/* ---- K2 / K3: base projection on tcgen05 with the LoRA expand fused into the accumulator ------
 * Y[M,N] = A[M,K] . B[N,K]^T + sum over the LoRA slots s of each 256-row slot tile of
 *          Hslots[s*256 + r%256 (r = the tile's rows), hcol(n) : hcol(n)+lora_rank] . LB[a(s)*lb_rows_per_adapter + n,
 *          0 : lora_rank]^T,
 * hcol(n) = sub_h_col[i] for the sub-projection i with sub_n_start[i] <= n < sub_n_start[i+1].
 * Pass tile_slot_ptr = NULL for a plain GEMM.  lora_rank a multiple of 16.  bn = 0 picks the
 * N tile (128/256).  Requirements: K, N, lda, ldb, ldy, ldh, ld_lb multiples of 8; 16-byte aligned
 * pointers; sub-projection boundaries multiples of the N tile.
 * Forward: A = X, B = W [N,K], Hslots from collm_lora_shrink, LB = adapters' B [n_ad*N, r].
 * Backward dX: A = dY, B = W^T [K_in, N], Hslots = s*dY.B_t [T_tr, R] with one slot per tile,
 *              LB = A_t^T [K_in, R].
 * Persistent stream-K schedule (one CTA per SM): boundary tiles are combined through fp32
 * partials in `workspace` (zero-filled once; flags are reset by their consumers) in a fixed
 * order, so results are bitwise deterministic.  collm_gemm_workspace_bytes(bn) sizes it (0 = max).
 * Each tile runs its K/64 main blocks first and its LoRA k-stages last.  With lora_flag / gen
 * (device, optional) the producer waits for *lora_flag == *gen before loading the LoRA operand, so
 * the shrink writing Hslots may run concurrently on another stream (collm_lora_shrink signal).
 * Alternatively lora_pdl = 1: the GEMM is launched programmatically dependent on the preceding
 * kernel of the SAME stream (that shrink, which lets it start at once) and its LoRA stages wait
 * for that grid's completion (griddepcontrol.wait) — the same overlap with no flag.
 * Replaces: perf.true_infer_latency / true_train_latency (perf.py:62-89). */
size_t collm_gemm_workspace_bytes(int bn);
int collm_gemm_lora(const void* A, int lda, const void* B, int ldb, void* Y, int ldy, int M, int N,
                    int K, const void* Hslots, int ldh, int h_rows, const void* LB, int ld_lb,
                    int lb_rows, const int32_t* tile_slot_ptr, const int32_t* slot_adapter,
                    int lora_rank, int lb_rows_per_adapter, int n_sub, const int32_t* sub_n_start,
                    const int32_t* sub_h_col, int bn, void* workspace, size_t ws_bytes,
                    const int32_t* lora_flag, const int32_t* gen, int lora_pdl, void* stream);

/* Same, with tile_skip (device int32 per 256-row slot tile, may be NULL): tiles marked 1 get no
 * fused expand (only their base GEMM) — for many-adapter tiles, expanded afterwards by
 * collm_lora_expand_rows. */
int collm_gemm_lora_ex(const void* A, int lda, const void* B, int ldb, void* Y, int ldy, int M,
                       int N, int K, const void* Hslots, int ldh, int h_rows, const void* LB,
                       int ld_lb, int lb_rows, const int32_t* tile_slot_ptr,
                       const int32_t* slot_adapter, int lora_rank, int lb_rows_per_adapter,
                       int n_sub, const int32_t* sub_n_start, const int32_t* sub_h_col, int bn,
                       void* workspace, size_t ws_bytes, const int32_t* lora_flag,
                       const int32_t* gen, int lora_pdl, const int32_t* tile_skip, void* stream);

/* Per-row LoRA expand of the 256-row slot tiles listed in `tiles` (device int32, n_tiles):
 *   Y[t, n] += sum_j H16[t, sub_h_col[s(n)] + j] * B[row_adapter[t]][n, j]   (j < r_pad)
 * B = [n_adapters, N, r_pad] bf16 (the registry layout), H16 = the shrink's s_a-scaled output.
 * HBM-bound on the rows' adapters' B (one warp per row and 256 columns); the many-adapter
 * alternative to the GEMM's fused expand (whose cost grows with slots x r).  Deterministic. */
int collm_lora_expand_rows(void* Y, int ldy, int N, const void* H16, int ldh, const void* B,
                           int r_pad, const int32_t* row_adapter, const int32_t* tiles, int n_tiles,
                           int T, int n_sub, const int32_t* sub_n_start, const int32_t* sub_h_col,
                           void* stream);

/* Co-residence mode of the kernels (process-wide): 0 (default) -> deepest GEMM pipelines, default
 * carveouts; 1 -> lean GEMM pipelines (~181 KB shared memory per CTA) and the rank-space kernels
 * (shrink, K5) configured to fit next to a GEMM CTA (max-shared carveout, shallower K5 ring) — for
 * a shrink running concurrently on a second stream next to GEMM CTAs that wait for it; 2 -> only
 * the rank-space half of 1 (the programmatic-dependent-launch overlap: every shrink CTA is
 * resident before its GEMM starts, so the GEMM keeps its deeper pipeline). */
int collm_set_gemm_lean(int lean);

/* ---- K5: LoRA weight-gradient reductions with fused AdamW ------------------------------------
 * One group = one reduction C[p,q] = sum_t U[t, u_off+p] * V[t, v_off+q] (p < P, q < Q <= 64;
 * P, Q multiples of 8) and the tensors it updates.  Element (p,q) lives at fp32 index
 * (c_row_off+p)*ldc + c_col_off+q of grad / master / m / v and of out_same (bf16), and at
 * (t_row_off+q)*ld_trans + t_col_off+p of out_trans (bf16).  One launch serves up to 16 groups
 * — all projections of a layer (per projection: dB per sub-projection, U = dY, V = H16; dA^T in
 * <= 64-rank chunks, U = X_tr, V = dH16, V2 = dH16lo); all groups share T.
 * Replaces: AdapterParams.perturbed (launcher.py:43-47) and perf.train_step (perf.py:111-126). */
typedef struct {
  const void* U;     /* bf16 [T, ldu] */
  const void* V;     /* bf16 [T, ldv] */
  float* grad;       /* fp32, may be NULL unless STORE_GRAD / accum_in / apply(ADAMW) */
  float* master;     /* fp32 master weights (ADAMW / COPY_ONLY) */
  float* m;          /* AdamW first moment */
  float* v;          /* AdamW second moment */
  void* out_same;    /* bf16 copy in the master layout, may be NULL */
  void* out_trans;   /* bf16 transposed copy, may be NULL */
  int ldu, ldv;
  int u_off, P, v_off, Q;
  int ldc, ld_trans;
  int c_row_off, c_col_off, t_row_off, t_col_off;
  const void* V2;    /* optional bf16 [T, ldv]: C = U^T (V + V2) (the lo half of a hi+lo pair) */
} collm_reduce_group;

/* mode STORE_GRAD: grad = C*grad_scale (+grad if accum_in).  mode ADAMW: the same gradient drives
 * an AdamW step on master/m/v (PyTorch semantics) and the bf16 copies are rewritten.  `adamw` is
 * a DEVICE pointer to 7 floats {lr, beta1, beta2, eps, weight_decay, 1-beta1^step, 1-beta2^step}
 * so a captured CUDA graph can be replayed with a changing step.  Deterministic (split-T partials
 * reduced in a fixed order by the last-arriving CTA).
 * Kernel: by default the persistent TMA -> tcgen05.mma -> TMEM stream (one CTA per SM, units of
 * 128 P rows x a range of 128-row T chunks, T split into at most `tsplit` parts of whole chunks,
 * accumulators double-buffered in TMEM so the AdamW finalize overlaps the next unit's stream);
 * collm_set_reduce_impl(0) (or COLLM_K5_TC=0) selects the mma.sync kernel (32-row T chunks), which
 * also serves launches with more than 40 distinct U / V tensors. */
int collm_set_reduce_impl(int tc); /* 1 = tcgen05 (default), 0 = mma.sync; caller's current device */
int collm_get_reduce_impl(void);
size_t collm_reduce_workspace_bytes(const collm_reduce_group* groups, int n_groups, int tsplit);
int collm_lora_reduce(int T, const collm_reduce_group* groups, int n_groups, int mode,
                      int accum_in, float grad_scale, const float* adamw, int tsplit,
                      void* workspace, size_t ws_bytes, void* stream);
/* Elementwise update over the same groups from `grad` (mode ADAMW, e.g. after a cross-replica
 * gradient allreduce) or master -> bf16 copies only (mode COPY_ONLY, after fedavg; replaces
 * fedavg's result hand-back, launcher.py:68-80 / :226). */
int collm_lora_apply(const collm_reduce_group* groups, int n_groups, int mode,
                     const float* adamw, void* stream);

/* ---- K8: attention of the mixed batch over a paged KV cache (forward) -------------------------
 * Every query row t (decode, prefill or training token) attends causally to tokens
 * [0, row_pos[t]] of its sequence row_seq[t], whose K/V already sit in the paged cache:
 *   out[t, h] = sum_j softmax_j(scale * q[t, h] . K[j, h/G]) V[j, h/G],  G = n_heads / n_kv_heads
 * q [T, ldq] / out [T, ldo] bf16 (head h at columns h*head_dim); k_cache, v_cache bf16
 * [n_pages, n_kv_heads, page_size, head_dim] (head-major pages); block_table [n_seq, bt_stride]
 * int32 page ids;
 * max_ctx >= every row_pos + 1.  head_dim 128, G <= 8, page_size a power of two.  fp32 softmax,
 * deterministic (split partials combined in split order by the last CTA; workspace counters
 * zeroed once and restored).  Replaces: nothing in the reference (which has no attention); the
 * step either side of the LoRA projections. */
size_t collm_attention_workspace_bytes(int T, int n_heads, int n_kv_heads, int max_ctx);
int collm_paged_attention(const void* q, int ldq, int T, int n_heads, int n_kv_heads,
                          int head_dim, const void* k_cache, const void* v_cache, int page_size,
                          const int32_t* block_table, int bt_stride, const int32_t* row_seq,
                          const int32_t* row_pos, int max_ctx, float scale, void* out, int ldo,
                          void* workspace, size_t ws_bytes, void* stream);

/* ---- K9: causal self-attention of packed sequences, forward + backward ------------------------
 * Sequences are row ranges of the mixed batch (training sequences, prefill segments, decode rows)
 * given per row: row_start[t] / row_end[t] (device int32 [T]) = first / one-past-last row of row
 * t's sequence (sequences contiguous and in row order); row t attends to rows [row_start[t], t].
 * Forward: by default the tcgen05/TMEM kernel (128 query rows per CTA: TMA-fed Q K^T and P V on
 * the tensor core, S / O accumulators in TMEM, 8 softmax warps); collm_set_flash_impl(0) (or
 * COLLM_FA_TC=0) selects the mma.sync kernel (64 rows per CTA).  Backward: mma.sync kernels.
 * CTAs take consecutive rows (packed: short sequences share a tile).  q [T, ldq] (head h at columns h*128), k / v [T, ldk/ldv]
 * (kv head h/G), typically column blocks of the fused q|k|v projection output.  head_dim 128; GQA with n_heads a multiple of n_kv_heads.
 * fwd: out [T, ldo] bf16, lse [n_heads, stat_ld] fp32 = base-2 log-sum-exp of
 *      scale*log2(e)*scores (kept for the backward); stat_ld <= 0 means T.
 * bwd: over the sequences given (e.g. the training rows [0, T) of a pass whose forward covered
 *      more rows: stat_ld = the forward's row count); delta [n_heads, stat_ld] fp32 workspace; dq / dk / dv bf16 (dk/dv per kv head: the G query heads
 *      of a group summed in a fixed order).  Deterministic: no atomics (dK/dV and dQ in separate
 *      kernels, each output element owned by one CTA).  fp32 softmax and accumulation.
 * Replaces: nothing in the reference (it has no attention); SURVEY §8(f) row 1. */
int collm_set_flash_impl(int tc); /* 1 = tcgen05 (default), 0 = mma.sync; caller's current device */
int collm_get_flash_impl(void);
int collm_flash_attention_fwd(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                              void* out, int ldo, float* lse, int T, int n_heads, int n_kv_heads,
                              int head_dim, const int32_t* row_start, const int32_t* row_end,
                              float scale, int stat_ld, void* stream);
int collm_flash_attention_bwd(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                              const void* out, int ldo, const void* dout, int lddo, const float* lse,
                              float* delta, void* dq, int lddq, void* dk, int lddk, void* dv, int lddv,
                              int T, int n_heads, int n_kv_heads, int head_dim,
                              const int32_t* row_start, const int32_t* row_end, float scale,
                              int stat_ld, void* stream);

/* ---- K7: softmax cross-entropy forward + backward over LM-head logits ------------------------
 * For each row t of logits [T, ld] (bf16, V used columns, V and ld multiples of 8):
 *   loss_rows[t] = logsumexp(z_t) - z_t[labels[t]]  (0 when labels[t] < 0 or >= V: ignored)
 *   dlogits[t, v] = grad_scale * (softmax(z_t)[v] - [v == labels[t]])  (bf16; 0 for ignored rows;
 *                   dlogits may be NULL = forward only; it must not alias logits)
 *   *loss_mean = mean of loss_rows over the valid rows, summed in row order by the last CTA
 *                (loss_mean may be NULL; otherwise `counter` = 1 device int32, zeroed once,
 *                restored by the kernel).  fp32 softmax arithmetic, deterministic.
 * Replaces: the convergence stand-in perf.train_step (perf.py:111-126) — TrainState.loss becomes
 * the measured next-token cross-entropy of the training rows. */
int collm_cross_entropy(const void* logits, int ld, int T, int V, const int32_t* labels,
                        float* loss_rows, float* loss_mean, int32_t* counter, void* dlogits,
                        int ld_d, float grad_scale, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COLLM_H_ */
