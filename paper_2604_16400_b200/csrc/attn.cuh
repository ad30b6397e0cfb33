// attn.cuh — K8: attention of the mixed batch's query rows over a paged KV cache (forward),
// HBM-bound.  SURVEY §8(f) row 1 (the step either side of the projections): every row — a decode
// token, a prefill token or a training token — attends causally to the tokens [0, pos] of its own
// sequence, whose K/V already sit in the paged cache (the layer appends the batch's K/V first).
//
//   o[t, h, :] = sum_{j <= pos_t} softmax_j(scale * q[t, h, :] . k[seq_t, j, h/G, :]) v[seq_t, j, h/G, :]
//
// GQA: G = n_heads / n_kv_heads query heads share one KV head; one CTA handles (row, KV head,
// split of <= kAttnSplit tokens) for all G heads, so each K/V byte of the split is read once.
// Each CTA streams its split as 8 half-warp flash-decoding streams (below).  Splits of one (row, KV head) combine in split order in the CTA that finishes
// last (arrival counter, restored): (m, l, acc) rescaled exactly like flash-decoding —
// deterministic, no float atomics.  fp32 softmax / accumulation, bf16 in and out, D = 128.
//
// Bytes (§8(d)-style, algorithmic): per (row, KV head) 2 * (pos + 1) * D * 2 (K and V read
// once) + the queries and outputs.
#pragma once
#include "common.cuh"
#include "flash_attn.cuh"

namespace collm {

constexpr int kAttnD = 128;
constexpr int kAttnThreads = 128;
constexpr int kAttnSplit = 256;  // tokens per split (<= 2 per thread in the score phase)
constexpr int kAttnMaxG = 8;

struct AttnParams {
  const bf16* q;  // [T, n_heads, D] (row stride ldq elements)
  int ldq;
  const bf16* k_cache;  // [n_pages, n_kv_heads, page, D] (head-major pages: a CTA's rows contiguous)
  const bf16* v_cache;
  int page_shift;  // log2(tokens per page)
  int n_heads, n_kv_heads;
  const int32_t* block_table;  // [n_seq, bt_stride] page ids
  int bt_stride;
  const int32_t* row_seq;  // [T] sequence of each query row
  const int32_t* row_pos;  // [T] position of the row's token (attends to [0, pos])
  bf16* out;               // [T, n_heads, D]
  int ldo;
  float scale;
  float* part;        // [T, n_kv_heads, max_splits, G, D + 2] split partials (m, l, acc)
  int32_t* counters;  // [T, n_kv_heads] arrival counters (0 on entry, restored)
  int max_splits;
};

// Half-warp streams: lanes 0-15 of a warp walk one token, lanes 16-31 the next, each lane owning 8
// of the 128 dims (16-byte loads: a half-warp reads a whole K row, then the same token's V row).
// Per stream an online softmax (m, l, acc[8] per head) — no block-wide phases; the 8 streams of
// the CTA merge through shared memory at the end (fixed order).
template <int G>
__global__ void __launch_bounds__(kAttnThreads) paged_attention_kernel(const AttnParams p) {
  constexpr float kLog2e = 1.4426950408889634f;
  constexpr int kStreams = 2 * kAttnThreads / 32;  // 8 half-warps
  const int t = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int pos = p.row_pos[t];
  // a row_pos beyond max_ctx (host cannot check device positions) is clamped to the launched
  // split count: the last split's combine always runs and restores its arrival counter, so one
  // bad row never corrupts the shared workspace of later launches
  const int n_tok = min(pos + 1, p.max_splits * kAttnSplit);
  const int n_splits = (n_tok + kAttnSplit - 1) / kAttnSplit;
  if (split >= n_splits) return;  // this row's context is shorter
  const int seq = p.row_seq[t];
  const int j0 = split * kAttnSplit, j1 = min(n_tok, j0 + kAttnSplit);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hl = lane & 15, stream = warp * 2 + (lane >> 4);
  const int psz = 1 << p.page_shift;
  const int32_t* bt = p.block_table + (size_t)seq * p.bt_stride;
  const int h0 = kvh * G;

  // this lane's 8 query dims of each head, pre-scaled by scale * log2(e) (exp2 softmax)
  float qf[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint4 u = ld_global_nc_v4(p.q + (size_t)t * p.ldq + (h0 + g) * kAttnD + 8 * hl);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      qf[g][2 * k] = __uint_as_float(w[k] << 16) * p.scale * kLog2e;
      qf[g][2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u) * p.scale * kLog2e;
    }
  }
  float m[G], l[G], acc[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < 8; ++d) acc[g][d] = 0.f;
  }
  auto row_of = [&](const bf16* cache, int j) {
    const int pg = bt[j >> p.page_shift];
    return cache + (((size_t)pg * p.n_kv_heads + kvh) * psz + (j & (psz - 1))) * kAttnD + 8 * hl;
  };
  constexpr int kU = G >= 4 ? 1 : 2;  // tokens per stream in flight (registers: G x 8 accumulators)
  // warp-uniform trip count (the half-warp shuffles need both halves): a half whose token is
  // past the split end computes on zeros and skips its state update
  for (int jw = j0 + warp * 2; jw < j1; jw += kStreams * kU) {
    uint4 kr[kU], vr[kU];
    bool ok[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = jw + (lane >> 4) + u * kStreams;
      ok[u] = j < j1;
      kr[u] = ok[u] ? ld_global_nc_v4(row_of(p.k_cache, j)) : make_uint4(0, 0, 0, 0);
      vr[u] = ok[u] ? ld_global_nc_v4(row_of(p.v_cache, j)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      float kf[8], vf[8];
      const uint32_t kw[4] = {kr[u].x, kr[u].y, kr[u].z, kr[u].w};
      const uint32_t vw[4] = {vr[u].x, vr[u].y, vr[u].z, vr[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        kf[2 * k] = __uint_as_float(kw[k] << 16);
        kf[2 * k + 1] = __uint_as_float(kw[k] & 0xffff0000u);
        vf[2 * k] = __uint_as_float(vw[k] << 16);
        vf[2 * k + 1] = __uint_as_float(vw[k] & 0xffff0000u);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float sdot = 0.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) sdot = fmaf(qf[g][d], kf[d], sdot);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
        if (!ok[u]) continue;
        // online softmax in base 2 (scores already carry log2 e)
        const float mn = fmaxf(m[g], sdot);
        const float corr = exp2f(m[g] - mn);  // m = -inf at first: exp2(-inf) = 0
        const float pr = exp2f(sdot - mn);
        l[g] = l[g] * corr + pr;
#pragma unroll
        for (int d = 0; d < 8; ++d) acc[g][d] = fmaf(acc[g][d], corr, pr * vf[d]);
        m[g] = mn;
      }
    }
  }

  // merge the 8 streams (fixed order) through shared memory: (m, l) per stream and head, acc
  __shared__ float sml[kStreams][G][2];
  __shared__ __align__(16) float sacc[kStreams][G][kAttnD];
  __shared__ bool s_last;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (hl == 0) {
      sml[stream][g][0] = m[g];
      sml[stream][g][1] = l[g];
    }
    *reinterpret_cast<float4*>(&sacc[stream][g][8 * hl]) = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
    *reinterpret_cast<float4*>(&sacc[stream][g][8 * hl + 4]) = make_float4(acc[g][4], acc[g][5], acc[g][6], acc[g][7]);
  }
  __syncthreads();
  float M[G], L[G], A[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    M[g] = -INFINITY;
    for (int s2 = 0; s2 < kStreams; ++s2) M[g] = fmaxf(M[g], sml[s2][g][0]);
    L[g] = 0.f;
    A[g] = 0.f;
    for (int s2 = 0; s2 < kStreams; ++s2) {
      const float ms = sml[s2][g][0];
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M[g]);
      L[g] += f * sml[s2][g][1];
      A[g] += f * sacc[s2][g][tid];
    }
  }
  if (n_splits == 1) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      p.out[(size_t)t * p.ldo + (h0 + g) * kAttnD + tid] = __float2bfloat16_rn(A[g] / L[g]);
    return;
  }
  // split partial (m in base 2, l, acc) -> workspace; the last split CTA combines in split order
  const size_t stride_g = kAttnD + 2;
  float* mine = p.part + (((size_t)t * p.n_kv_heads + kvh) * p.max_splits + split) * G * stride_g;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    mine[g * stride_g + 2 + tid] = A[g];
    if (tid == 0) {
      mine[g * stride_g] = M[g];
      mine[g * stride_g + 1] = L[g];
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    int32_t* c = p.counters + (size_t)t * p.n_kv_heads + kvh;
    s_last = atomicAdd(c, 1) == n_splits - 1;
    if (s_last) *c = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = p.part + ((size_t)t * p.n_kv_heads + kvh) * p.max_splits * G * stride_g;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float Mx = -INFINITY;
    for (int s2 = 0; s2 < n_splits; ++s2) Mx = fmaxf(Mx, __ldcg(base + ((size_t)s2 * G + g) * stride_g));
    float Ls = 0.f, As = 0.f;
    for (int s2 = 0; s2 < n_splits; ++s2) {
      const float* b = base + ((size_t)s2 * G + g) * stride_g;
      const float f = exp2f(__ldcg(b) - Mx);
      Ls += f * __ldcg(b + 1);
      As += f * __ldcg(b + 2 + tid);
    }
    p.out[(size_t)t * p.ldo + (h0 + g) * kAttnD + tid] = __float2bfloat16_rn(As / Ls);
  }
}


// Tensor-core variant (the default): the G query heads of a KV head are the rows of ONE m16n8k16
// MMA (rows G..15 zero), so each K/V element feeds G heads through the tensor pipe instead of G
// shuffle-reduced dot products (the CUDA-core kernel above is issue-bound at G = 4: 1.4 TB/s).
// Each of the 4 warps stages 64 tokens of the split into its own 16 KB XOR-swizzled tile (cp.async,
// zero-filled past the split end): K first — S = Q K^T (64 MMAs) and a local base-2 softmax per
// head row — then V in the same tile — O = P V (64 MMAs, P from the score fragments); 64 KB per
// CTA keeps 3 CTAs (12 warps, ~190 KB of loads) in flight per SM.  The warps merge in fixed order
// through the tiles' space and splits combine exactly as above (deterministic).  Measured
// (tools/attn_bench.py, 256 rows): 7B decode ctx 1024 5.26 TB/s (0.81 of HBM; CUDA-core 4.07),
// GQA G = 4 4.79 TB/s (CUDA-core 1.44), G = 8 3.4 TB/s (0.55).
constexpr int kAttnTcSmem = 4 * 16384;  // one 16 KB tile per warp: K, then V in the same buffer

template <int G>
__global__ void __launch_bounds__(kAttnThreads, 1) paged_attention_tc_kernel(const AttnParams p) {
  constexpr float kLog2e = 1.4426950408889634f;
  constexpr int kW = kAttnThreads / 32;  // 4 warps x 64 tokens = one 256-token split
  extern __shared__ __align__(128) uint8_t asm_[];
  const int t = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int pos = p.row_pos[t];
  const int n_tok = min(pos + 1, p.max_splits * kAttnSplit);
  const int n_splits = (n_tok + kAttnSplit - 1) / kAttnSplit;
  if (split >= n_splits) return;
  const int seq = p.row_seq[t];
  const int j0 = split * kAttnSplit, j1 = min(n_tok, j0 + kAttnSplit);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int psz = 1 << p.page_shift;
  const int32_t* bt = p.block_table + (size_t)seq * p.bt_stride;
  const int h0 = kvh * G;
  const int jw0 = j0 + warp * 64;
  const int nvalid = max(0, min(64, j1 - jw0));
  // one 16 KB tile per warp (3 CTAs fit an SM): this warp's 64 tokens of K, then of V
  uint8_t* Ts = asm_ + warp * 16384;
  auto stage = [&](const bf16* cache) {  // rows past the split end zero-filled
    for (int i = lane; i < 64 * 16; i += 32) {
      const int row = i >> 4, ch = i & 15;
      const bool ok = row < nvalid;
      const int j = ok ? jw0 + row : j0;
      const size_t off = (((size_t)bt[j >> p.page_shift] * p.n_kv_heads + kvh) * psz + (j & (psz - 1))) *
                         kAttnD + ch * 8;
      cp_async_16(Ts + fa_off(row, ch * 8), cache + off, ok);
    }
    cp_async_commit();
  };
  stage(p.k_cache);
  // Q fragments: rows = the group's heads (rows >= G zero), 8 k-steps over the 128 dims
  uint32_t qa[8][4];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t* qp = reinterpret_cast<const uint32_t*>(p.q + (size_t)t * p.ldq + (h0 + g) * kAttnD + kk * 16 + 2 * c);
    qa[kk][0] = g < G ? __ldg(qp) : 0u;
    qa[kk][1] = 0u;
    qa[kk][2] = g < G ? __ldg(qp + 4) : 0u;
    qa[kk][3] = 0u;
  }
  cp_async_wait<0>();
  __syncwarp();
  const uint32_t kb = smem_u32(Ts), vb = kb;
  float sc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
#pragma unroll
    for (int jn = 0; jn < 4; ++jn) {
      uint32_t b[4];
      fa_ldb_nk(b, kb, jn * 16, kk * 16, lane);
      mma16816(sc[2 * jn], qa[kk], b[0], b[1]);
      mma16816(sc[2 * jn + 1], qa[kk], b[2], b[3]);
    }
  // local softmax of head row g over this warp's tokens (base 2)
  float m = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool ok = nt * 8 + 2 * c + e < nvalid;
      sc[nt][e] = ok ? sc[nt][e] * p.scale * kLog2e : -INFINITY;
      m = fmaxf(m, sc[nt][e]);
      sc[nt][2 + e] = 0.f;  // rows g+8: no head
    }
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
  m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
  float l = 0.f;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float v = m == -INFINITY ? 0.f : exp2f(sc[nt][e] - m);
      sc[nt][e] = v;
      l += v;
    }
  l += __shfl_xor_sync(0xffffffffu, l, 1);
  l += __shfl_xor_sync(0xffffffffu, l, 2);
  __syncwarp();  // every lane's K fragments are read: the tile takes V
  stage(p.v_cache);
  cp_async_wait<0>();
  __syncwarp();
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t pa[4];
    fa_c2a(pa, sc[2 * kk], sc[2 * kk + 1]);
#pragma unroll
    for (int jd = 0; jd < 8; ++jd) {
      uint32_t b[4];
      fa_ldb_kn(b, vb, jd * 16, kk * 16, lane);
      mma16816(o[2 * jd], pa, b[0], b[1]);
      mma16816(o[2 * jd + 1], pa, b[2], b[3]);
    }
  }
  // merge the 4 warps (fixed order) through shared memory (the tiles' space, all MMAs done)
  __syncthreads();
  float (*sml)[kAttnMaxG][2] = reinterpret_cast<float (*)[kAttnMaxG][2]>(asm_);
  float (*sacc)[kAttnMaxG][kAttnD] = reinterpret_cast<float (*)[kAttnMaxG][kAttnD]>(asm_ + 1024);
  __shared__ bool s_last;
  if (g < G) {
    if (c == 0) {
      sml[warp][g][0] = m;
      sml[warp][g][1] = l;
    }
#pragma unroll
    for (int dt = 0; dt < 16; ++dt) {
      sacc[warp][g][dt * 8 + 2 * c] = o[dt][0];
      sacc[warp][g][dt * 8 + 2 * c + 1] = o[dt][1];
    }
  }
  __syncthreads();
  float M[G], L[G], A[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    M[h] = -INFINITY;
    for (int w = 0; w < kW; ++w) M[h] = fmaxf(M[h], sml[w][h][0]);
    L[h] = 0.f;
    A[h] = 0.f;
    for (int w = 0; w < kW; ++w) {
      const float ms = sml[w][h][0];
      const float f = ms == -INFINITY ? 0.f : exp2f(ms - M[h]);
      L[h] += f * sml[w][h][1];
      A[h] += f * sacc[w][h][tid];
    }
  }
  if (n_splits == 1) {
#pragma unroll
    for (int h = 0; h < G; ++h)
      p.out[(size_t)t * p.ldo + (h0 + h) * kAttnD + tid] = __float2bfloat16_rn(A[h] / L[h]);
    return;
  }
  const size_t stride_g = kAttnD + 2;
  float* mine = p.part + (((size_t)t * p.n_kv_heads + kvh) * p.max_splits + split) * G * stride_g;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    mine[h * stride_g + 2 + tid] = A[h];
    if (tid == 0) {
      mine[h * stride_g] = M[h];
      mine[h * stride_g + 1] = L[h];
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    int32_t* cn = p.counters + (size_t)t * p.n_kv_heads + kvh;
    s_last = atomicAdd(cn, 1) == n_splits - 1;
    if (s_last) *cn = 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = p.part + ((size_t)t * p.n_kv_heads + kvh) * p.max_splits * G * stride_g;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float Mx = -INFINITY;
    for (int s2 = 0; s2 < n_splits; ++s2) Mx = fmaxf(Mx, __ldcg(base + ((size_t)s2 * G + h) * stride_g));
    float Ls = 0.f, As = 0.f;
    for (int s2 = 0; s2 < n_splits; ++s2) {
      const float* b = base + ((size_t)s2 * G + h) * stride_g;
      const float f = exp2f(__ldcg(b) - Mx);
      Ls += f * __ldcg(b + 1);
      As += f * __ldcg(b + 2 + tid);
    }
    p.out[(size_t)t * p.ldo + (h0 + h) * kAttnD + tid] = __float2bfloat16_rn(As / Ls);
  }
}

}  // namespace collm
