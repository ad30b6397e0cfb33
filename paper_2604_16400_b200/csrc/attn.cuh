// attn.cuh — K8: attention of the mixed batch's query rows over a paged KV cache (forward),
// HBM-bound.  SURVEY §8(f) row 1 (the step either side of the projections): every row — a decode
// token, a prefill token or a training token — attends causally to the tokens [0, pos] of its own
// sequence, whose K/V already sit in the paged cache (the layer appends the batch's K/V first).
//
//   o[t, h, :] = sum_{j <= pos_t} softmax_j(scale * q[t, h, :] . k[seq_t, j, h/G, :]) v[seq_t, j, h/G, :]
//
// GQA: G = n_heads / n_kv_heads query heads share one KV head; one CTA handles (row, KV head,
// split of <= kAttnSplit tokens) for all G heads, so each K/V byte of the split is read once.
// Three phases per CTA: scores (one thread per token: 16-byte loads of its K row, G dot products
// against the row's queries staged in shared memory), max / sum of exp over the split (block
// reduction), then P.V (each warp a quarter of the tokens, a lane 4 of the 128 dims: a warp reads
// one whole 256-byte V row per token).  Splits of one (row, KV head) combine in split order in the CTA that finishes
// last (arrival counter, restored): (m, l, acc) rescaled exactly like flash-decoding —
// deterministic, no float atomics.  fp32 softmax / accumulation, bf16 in and out, D = 128.
//
// Bytes (§8(d)-style, algorithmic): per (row, KV head) 2 * (pos + 1) * D * 2 (K and V read
// once) + the queries and outputs.
#pragma once
#include "common.cuh"

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

__global__ void __launch_bounds__(kAttnThreads) paged_attention_kernel(const AttnParams p) {
  const int t = blockIdx.x, kvh = blockIdx.y, split = blockIdx.z;
  const int G = p.n_heads / p.n_kv_heads;
  const int pos = p.row_pos[t];
  const int n_tok = pos + 1;
  const int n_splits = (n_tok + kAttnSplit - 1) / kAttnSplit;
  if (split >= n_splits) return;  // this row's context is shorter
  const int seq = p.row_seq[t];
  const int j0 = split * kAttnSplit, j1 = min(n_tok, j0 + kAttnSplit);
  const int n = j1 - j0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int psz = 1 << p.page_shift;
  const int32_t* bt = p.block_table + (size_t)seq * p.bt_stride;

  __shared__ float sq[kAttnMaxG][kAttnD];
  __shared__ float ss[kAttnMaxG][kAttnSplit];
  __shared__ float red[kAttnMaxG][kAttnThreads / 32];
  __shared__ float s_m[kAttnMaxG], s_l[kAttnMaxG];
  __shared__ bool s_last;

  // queries of the G heads of this KV head (pre-scaled)
  for (int e = tid; e < G * kAttnD; e += kAttnThreads) {
    const int g = e / kAttnD, d = e % kAttnD;
    sq[g][d] = p.scale * __bfloat162float(p.q[(size_t)t * p.ldq + (kvh * G + g) * kAttnD + d]);
  }
  __syncthreads();

  // phase 1: scores, one thread per token
  auto kv_row = [&](const bf16* cache, int j) {
    const int pg = bt[j >> p.page_shift];
    return cache + (((size_t)pg * p.n_kv_heads + kvh) * psz + (j & (psz - 1))) * kAttnD;
  };
  for (int i = tid; i < n; i += kAttnThreads) {
    const bf16* kr = kv_row(p.k_cache, j0 + i);
    float acc[kAttnMaxG];
#pragma unroll
    for (int g = 0; g < kAttnMaxG; ++g) acc[g] = 0.f;
#pragma unroll 4
    for (int v8 = 0; v8 < kAttnD / 8; ++v8) {
      const uint4 u = ld_global_nc_v4(kr + 8 * v8);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __uint_as_float(w[k] << 16), b = __uint_as_float(w[k] & 0xffff0000u);
#pragma unroll
        for (int g = 0; g < kAttnMaxG; ++g)
          if (g < G) acc[g] += a * sq[g][8 * v8 + 2 * k] + b * sq[g][8 * v8 + 2 * k + 1];
      }
    }
#pragma unroll
    for (int g = 0; g < kAttnMaxG; ++g)
      if (g < G) ss[g][i] = acc[g];
  }
  __syncthreads();

  // phase 2: per head max and sum of exp over the split
  for (int g = 0; g < G; ++g) {
    float m = -INFINITY;
    for (int i = tid; i < n; i += kAttnThreads) m = fmaxf(m, ss[g][i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[g][warp] = m;
  }
  __syncthreads();
  if (tid < G) {
    float m = red[tid][0];
    for (int w = 1; w < kAttnThreads / 32; ++w) m = fmaxf(m, red[tid][w]);
    s_m[tid] = m;
  }
  __syncthreads();
  for (int g = 0; g < G; ++g) {
    const float m = s_m[g];
    float l = 0.f;
    for (int i = tid; i < n; i += kAttnThreads) {
      const float e = __expf(ss[g][i] - m);
      ss[g][i] = e;
      l += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) red[g][warp] = l;
  }
  __syncthreads();
  if (tid < G) {
    float l = 0.f;
    for (int w = 0; w < kAttnThreads / 32; ++w) l += red[tid][w];
    s_l[tid] = l;
  }
  __syncthreads();

  // phase 3: P.V — warp w takes the tokens i = w (mod 4), lane the 4 dims [4 lane, 4 lane + 4)
  // (8-byte loads, a warp reads a whole 256-byte V row); the 4 warp partials meet in smem
  float pacc[kAttnMaxG][4];
#pragma unroll
  for (int g = 0; g < kAttnMaxG; ++g) pacc[g][0] = pacc[g][1] = pacc[g][2] = pacc[g][3] = 0.f;
#pragma unroll 4
  for (int i = warp; i < n; i += kAttnThreads / 32) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(kv_row(p.v_cache, j0 + i) + 4 * lane));
    const float v0 = __uint_as_float(u.x << 16), v1 = __uint_as_float(u.x & 0xffff0000u);
    const float v2 = __uint_as_float(u.y << 16), v3 = __uint_as_float(u.y & 0xffff0000u);
#pragma unroll
    for (int g = 0; g < kAttnMaxG; ++g)
      if (g < G) {
        const float pr = ss[g][i];
        pacc[g][0] += pr * v0;
        pacc[g][1] += pr * v1;
        pacc[g][2] += pr * v2;
        pacc[g][3] += pr * v3;
      }
  }
  __shared__ __align__(16) float wacc[kAttnThreads / 32][kAttnMaxG][kAttnD];
#pragma unroll
  for (int g = 0; g < kAttnMaxG; ++g)
    if (g < G)
      *reinterpret_cast<float4*>(&wacc[warp][g][4 * lane]) =
          make_float4(pacc[g][0], pacc[g][1], pacc[g][2], pacc[g][3]);
  __syncthreads();
  float acc[kAttnMaxG];
#pragma unroll
  for (int g = 0; g < kAttnMaxG; ++g)
    acc[g] = g < G ? (wacc[0][g][tid] + wacc[1][g][tid]) + (wacc[2][g][tid] + wacc[3][g][tid]) : 0.f;

  const int h0 = kvh * G;
  if (n_splits == 1) {  // whole context in one split: normalise and store
#pragma unroll
    for (int g = 0; g < kAttnMaxG; ++g)
      if (g < G) p.out[(size_t)t * p.ldo + (h0 + g) * kAttnD + tid] = __float2bfloat16_rn(acc[g] / s_l[g]);
    return;
  }
  // split partial: (m, l, acc) -> workspace; the last split CTA combines in split order
  const size_t stride_g = kAttnD + 2;
  float* mine = p.part + (((size_t)t * p.n_kv_heads + kvh) * p.max_splits + split) * G * stride_g;
#pragma unroll
  for (int g = 0; g < kAttnMaxG; ++g)
    if (g < G) {
      mine[g * stride_g + 2 + tid] = acc[g];
      if (tid == 0) {
        mine[g * stride_g] = s_m[g];
        mine[g * stride_g + 1] = s_l[g];
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
  for (int g = 0; g < G; ++g) {
    float M = -INFINITY;
    for (int s = 0; s < n_splits; ++s) M = fmaxf(M, __ldcg(base + ((size_t)s * G + g) * stride_g));
    float L = 0.f, A = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float* b = base + ((size_t)s * G + g) * stride_g;
      const float f = __expf(__ldcg(b) - M);
      L += f * __ldcg(b + 1);
      A += f * __ldcg(b + 2 + tid);
    }
    p.out[(size_t)t * p.ldo + (h0 + g) * kAttnD + tid] = __float2bfloat16_rn(A / L);
  }
}

}  // namespace collm
