// flash_attn.cuh — K9: causal self-attention of the packed prefill / training sequences of the
// mixed batch, forward + backward (the step either side of the LoRA
// projections; the reference has no attention — PAPER.md:171 "cached KV tokens").
//
//   out[i, h] = sum_{j in seq(i), j <= i} softmax_j(scale * q[i,h] . k[j,h/G]) v[j,h/G]
//
// Sequences are row ranges of the mixed batch (a training sequence, a prefill segment, a decode
// row), given per row as row_start[t] / row_end[t]; q / k / v are column blocks of the fused q|k|v
// projection output (any row stride), GQA with G = n_heads / n_kv_heads, head_dim 128.  Decode
// rows' cached context is the paged KV cache's (K8, attn.cuh).
//
// Packed tiling: CTAs take 64 CONSECUTIVE ROWS of the batch, not of a sequence, so a tile of
// short prefill / decode sequences costs one CTA (keys: from the first row's sequence start to
// the tile's last row, masked by same-sequence-and-causal) — grid = T/64 x heads whatever the
// sequence mix (7B step: 293 sequences in 1024 rows -> 16 tiles per head).
//
// Tensor-core flash attention (mma.sync m16n8k16 bf16 -> fp32, ldmatrix from XOR-swizzled shared
// memory, cp.async double buffers) — the legacy warp-level MMA path, not tcgen05: attention is
// 0.3 % of the 7B step's FLOPs (2.1 GFLOP fwd per layer vs 620 GFLOP of projections) and 5.7 % at
// 13B (8 x 2048-token training sequences); measured (tools/flash_bench.py) 64-69 TFLOP/s at the
// 7B shape, 126-157 at 8B, 157-211 at 13B — a tcgen05/TMEM version is the next step for the
// long-sequence configs.
//   forward : CTA = (64 rows, head); online base-2 softmax; writes out and the base-2
//             log-sum-exp of the scaled scores (lse [n_heads, T]) for the backward.
//   backward: delta = rowsum(dout * out); dK/dV: CTA = (64 keys, kv head) looping over the G query
//             heads of its group and the query tiles from its first key to the end of its last
//             key's sequence (recomputing P from lse);
//             dQ: CTA = (64 queries, head) looping over the key tiles up to the diagonal.  Every
//             output element is owned by one CTA and accumulated in a fixed order: bitwise
//             deterministic (no atomics).
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kFaD = 128;   // head dim
constexpr int kFaBM = 64;   // rows per tile (4 warps x 16)
constexpr int kFaThreads = 128;

struct FlashParams {
  const bf16* q; const bf16* k; const bf16* v;
  int ldq, ldk, ldv;
  bf16* out; int ldo;
  float* lse;            // [n_heads, stat_ld] base-2 log-sum-exp of scale*log2(e)*scores
  const bf16* dout; int lddo;
  float* delta;          // [n_heads, stat_ld]
  bf16* dq; bf16* dk; bf16* dv;
  int lddq, lddk, lddv;
  const int32_t* row_start;  // [T] first row of each row's sequence
  const int32_t* row_end;    // [T] one past the last row of each row's sequence
  int T, n_heads, n_kv_heads;
  int stat_ld;           // row stride of lse / delta per head (>= the rows indexed)
  float scale_log2;      // scale * log2(e)
  float scale;
};

// [64 rows][128 cols] bf16 tile, 256-byte rows, 16-byte chunks XOR-swizzled by (row % 8)
__device__ __forceinline__ uint32_t fa_off(int row, int col) {
  return (uint32_t)(row * 256 + ((((col >> 3) ^ (row & 7))) << 4) + ((col & 7) << 1));
}

// cp.async a [64 x 128] tile (rows r0.. of a row-major matrix with leading dim ld, column c0);
// rows >= n_valid are zero-filled
__device__ __forceinline__ void fa_load_tile(uint8_t* s, const bf16* g, int ld, int r0, int n_valid,
                                             int c0) {
  for (int i = threadIdx.x; i < kFaBM * 16; i += kFaThreads) {
    const int row = i >> 4, ch = i & 15;
    const bool ok = row < n_valid;
    const bf16* src = g + (size_t)(r0 + (ok ? row : 0)) * ld + c0 + ch * 8;
    cp_async_16(s + fa_off(row, ch * 8), src, ok);
  }
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                          uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

// A fragment (16 rows x 16 k) of a row-major swizzled tile at (r0, k0)
__device__ __forceinline__ void fa_lda(uint32_t (&a)[4], uint32_t base, int r0, int k0, int lane) {
  const int row = r0 + (lane & 7) + (((lane >> 3) & 1) << 3);
  const int col = k0 + ((lane >> 4) << 3);
  ldsm_x4(a[0], a[1], a[2], a[3], base + fa_off(row, col));
}
// B fragments of two n8 tiles (n0, n0+8) x k16 at k0 from a tile stored [n][k] ("col" B)
__device__ __forceinline__ void fa_ldb_nk(uint32_t (&b)[4], uint32_t base, int n0, int k0, int lane) {
  const int row = n0 + (lane & 7) + ((lane >> 4) << 3);
  const int col = k0 + (((lane >> 3) & 1) << 3);
  ldsm_x4(b[0], b[1], b[2], b[3], base + fa_off(row, col));  // b0,b1 tile n0; b2,b3 tile n0+8
}
// B fragments of two n8 tiles (n0, n0+8) x k16 at k0 from a tile stored [k][n] (row-major B)
__device__ __forceinline__ void fa_ldb_kn(uint32_t (&b)[4], uint32_t base, int n0, int k0, int lane) {
  const int row = k0 + (lane & 7) + (((lane >> 3) & 1) << 3);
  const int col = n0 + ((lane >> 4) << 3);
  ldsm_x4_t(b[0], b[1], b[2], b[3], base + fa_off(row, col));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  mma_m16n8k16_bf16(d, a[0], a[1], a[2], a[3], b0, b1);
}

// C fragments (two n8 tiles j, j+1 of a 16-row strip) -> A fragment of the k16 step they span
__device__ __forceinline__ void fa_c2a(uint32_t (&a)[4], const float (&c0)[4], const float (&c1)[4]) {
  a[0] = pack_bf16x2(c0[0], c0[1]);
  a[1] = pack_bf16x2(c0[2], c0[3]);
  a[2] = pack_bf16x2(c1[0], c1[1]);
  a[3] = pack_bf16x2(c1[2], c1[3]);
}

// ----------------------------------------------------------------------------------- forward
// ST = 2: K/V double-buffered (80 KB, 2 CTAs/SM); ST = 1: one K/V stage (48 KB, 3 CTAs/SM —
// other CTAs hide the load latency instead of the prefetch)
template <int ST>
__global__ void __launch_bounds__(kFaThreads, ST == 1 ? 3 : 2) flash_fwd_kernel(const FlashParams p) {
  extern __shared__ __align__(128) uint8_t fsm[];
  // packed tiling: a CTA takes 64 consecutive rows of the batch whatever their sequences; its
  // keys run from the first row's sequence start to its last row, masked per (query, key) by
  // "same sequence and not after the query" — short prefill / decode sequences share a tile
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * kFaBM;
  if (q0 >= p.T) return;
  const int hk = h / (p.n_heads / p.n_kv_heads);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  uint8_t* Qs = fsm;
  uint8_t* Ks = fsm + 16384;                     // [ST] stages
  uint8_t* Vs = fsm + 16384 + ST * 16384;         // [ST] stages
  const uint32_t qb = smem_u32(Qs), kb0 = smem_u32(Ks), vb0 = smem_u32(Vs);
  const int nq = min(kFaBM, p.T - q0);
  const int kstart = p.row_start[q0], kend = q0 + nq;
  const int n_kt = (kend - kstart + kFaBM - 1) / kFaBM;

  fa_load_tile(Qs, p.q, p.ldq, q0, nq, h * kFaD);
  fa_load_tile(Ks, p.k, p.ldk, kstart, min(kFaBM, kend - kstart), hk * kFaD);
  fa_load_tile(Vs, p.v, p.ldv, kstart, min(kFaBM, kend - kstart), hk * kFaD);
  cp_async_commit();
  const int qrow0 = q0 + warp * 16 + g;  // this thread's rows qrow0, qrow0 + 8 (batch rows)
  int qs[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) qs[r] = qrow0 + r * 8 < p.T ? p.row_start[qrow0 + r * 8] : 0x7fffffff;

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_i[2] = {-INFINITY, -INFINITY}, l_i[2] = {0.f, 0.f};

  for (int j = 0; j < n_kt; ++j) {
    if constexpr (ST == 2) {
      if (j + 1 < n_kt) {
        const int kr = kstart + (j + 1) * kFaBM;
        fa_load_tile(Ks + ((j + 1) & 1) * 16384, p.k, p.ldk, kr, min(kFaBM, kend - kr), hk * kFaD);
        fa_load_tile(Vs + ((j + 1) & 1) * 16384, p.v, p.ldv, kr, min(kFaBM, kend - kr), hk * kFaD);
      }
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      if (j > 0) {  // every warp is done with the previous tile (the loop-end barrier)
        const int kr = kstart + j * kFaBM;
        fa_load_tile(Ks, p.k, p.ldk, kr, min(kFaBM, kend - kr), hk * kFaD);
        fa_load_tile(Vs, p.v, p.ldv, kr, min(kFaBM, kend - kr), hk * kFaD);
        cp_async_commit();
      }
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t kb = kb0 + (ST == 2 ? (j & 1) * 16384 : 0), vb = vb0 + (ST == 2 ? (j & 1) * 16384 : 0);
    float sc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a[4];
      fa_lda(a, qb, warp * 16, kk * 16, lane);
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        uint32_t b[4];
        fa_ldb_nk(b, kb, jn * 16, kk * 16, lane);
        mma16816(sc[2 * jn], a, b[0], b[1]);
        mma16816(sc[2 * jn + 1], a, b[2], b[3]);
      }
    }
    // scale, causal / length mask, online softmax (rows g and g+8 of the warp's strip)
    float mx[2] = {m_i[0], m_i[1]};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kstart + j * kFaBM + nt * 8 + 2 * c + (e & 1);
        const int qr = qrow0 + (e >> 1) * 8;
        const bool ok = key <= qr && key >= qs[e >> 1];
        sc[nt][e] = ok ? sc[nt][e] * p.scale_log2 : -INFINITY;
        mx[e >> 1] = fmaxf(mx[e >> 1], sc[nt][e]);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float alpha[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) alpha[r] = (mx[r] == -INFINITY) ? 1.f : exp2f(m_i[r] - mx[r]);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = (mx[e >> 1] == -INFINITY) ? 0.f : exp2f(sc[nt][e] - mx[e >> 1]);
        sc[nt][e] = v;
        rs[e >> 1] += v;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l_i[r] = l_i[r] * alpha[r] + rs[r];
      m_i[r] = mx[r];
    }
#pragma unroll
    for (int dt = 0; dt < 16; ++dt) {
      o[dt][0] *= alpha[0]; o[dt][1] *= alpha[0];
      o[dt][2] *= alpha[1]; o[dt][3] *= alpha[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4];
      fa_c2a(a, sc[2 * kk], sc[2 * kk + 1]);
#pragma unroll
      for (int jd = 0; jd < 8; ++jd) {
        uint32_t b[4];
        fa_ldb_kn(b, vb, jd * 16, kk * 16, lane);
        mma16816(o[2 * jd], a, b[0], b[1]);
        mma16816(o[2 * jd + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();  // this stage's K/V are consumed before the next prefetch overwrites them
  }
  cp_async_wait<0>();
  // normalize, write out and lse
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qr = qrow0 + r * 8;
    if (qr >= p.T) continue;
    const float inv = 1.f / l_i[r];
    bf16* dst = p.out + (size_t)qr * p.ldo + h * kFaD;
#pragma unroll
    for (int dt = 0; dt < 16; ++dt)
      *reinterpret_cast<uint32_t*>(dst + dt * 8 + 2 * c) =
          pack_bf16x2(o[dt][2 * r] * inv, o[dt][2 * r + 1] * inv);
    if (c == 0) p.lse[(size_t)h * p.stat_ld + qr] = m_i[r] + log2f(l_i[r]);
  }
}

// ----------------------------------------------------------------------------------- backward
// delta[h, i] = sum_d dout[i, h, d] * out[i, h, d]   (one warp per (row, head))
__global__ void flash_delta_kernel(const FlashParams p) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= p.T * p.n_heads) return;
  const int i = w / p.n_heads, h = w % p.n_heads;
  const uint2 a = *reinterpret_cast<const uint2*>(p.dout + (size_t)i * p.lddo + h * kFaD + lane * 4);
  const uint2 b = *reinterpret_cast<const uint2*>(p.out + (size_t)i * p.ldo + h * kFaD + lane * 4);
  const float2 a0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.x));
  const float2 a1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a.y));
  const float2 b0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b.x));
  const float2 b1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&b.y));
  float v = a0.x * b0.x + a0.y * b0.y + a1.x * b1.x + a1.y * b1.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) p.delta[(size_t)h * p.stat_ld + i] = v;
}

// dK, dV of 64 keys of one kv head: for every query head of the group and every query tile at or
// after the key tile, recompute P^T = exp2(scale_log2 * K Q^T - lse), dP^T = V dO^T,
// dS^T = P^T (dP^T - delta); dV += P^T dO, dK += dS^T Q (warp w owns keys 16w..16w+15).
__global__ void __launch_bounds__(kFaThreads) flash_bwd_dkdv_kernel(const FlashParams p) {
  extern __shared__ __align__(128) uint8_t fsm[];
  const int hk = blockIdx.y;
  const int k0 = blockIdx.x * kFaBM;
  if (k0 >= p.T) return;
  const int G = p.n_heads / p.n_kv_heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  uint8_t* Ks = fsm;
  uint8_t* Vs = fsm + 16384;
  uint8_t* Qs = fsm + 32768;    // [2]
  uint8_t* Os = fsm + 65536;    // [2] dO
  float* lse_s = reinterpret_cast<float*>(fsm + 98304);    // [2][64]
  float* dl_s = lse_s + 2 * kFaBM;                          // [2][64]
  int* qs_s = reinterpret_cast<int*>(dl_s + 2 * kFaBM);     // [2][64] queries' sequence starts
  const uint32_t kb = smem_u32(Ks), vb = smem_u32(Vs), qb0 = smem_u32(Qs), ob0 = smem_u32(Os);
  const int nk = min(kFaBM, p.T - k0);
  fa_load_tile(Ks, p.k, p.ldk, k0, nk, hk * kFaD);
  fa_load_tile(Vs, p.v, p.ldv, k0, nk, hk * kFaD);

  // queries that see these keys: rows [k0, row_end of the last key) (row_end is non-decreasing)
  const int qend = p.row_end[k0 + nk - 1];
  const int per_head = (qend - k0 + kFaBM - 1) / kFaBM, total = G * per_head;
  auto issue = [&](int it, int buf) {
    const int hq = hk * G + it / per_head;
    const int qr = k0 + (it % per_head) * kFaBM, nq = min(kFaBM, qend - qr);
    fa_load_tile(Qs + buf * 16384, p.q, p.ldq, qr, nq, hq * kFaD);
    fa_load_tile(Os + buf * 16384, p.dout, p.lddo, qr, nq, hq * kFaD);
    for (int i = threadIdx.x; i < kFaBM; i += kFaThreads) {
      const bool ok = i < nq;
      lse_s[buf * kFaBM + i] = ok ? p.lse[(size_t)hq * p.stat_ld + qr + i] : 0.f;
      dl_s[buf * kFaBM + i] = ok ? p.delta[(size_t)hq * p.stat_ld + qr + i] : 0.f;
      qs_s[buf * kFaBM + i] = ok ? p.row_start[qr + i] : 0x7fffffff;
    }
  };
  issue(0, 0);
  cp_async_commit();

  float dk[16][4], dv[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i)
    dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
  const int key_r0 = k0 + warp * 16 + g;  // this thread's keys key_r0, key_r0 + 8

  for (int it = 0; it < total; ++it) {
    if (it + 1 < total) issue(it + 1, (it + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const int buf = it & 1;
    const int qr = k0 + (it % per_head) * kFaBM;
    const uint32_t qb = qb0 + buf * 16384, ob = ob0 + buf * 16384;
    const float* lse_b = lse_s + buf * kFaBM;
    const float* dl_b = dl_s + buf * kFaBM;
    const int* qs_b = qs_s + buf * kFaBM;
    // S^T = K_w Q^T and dP^T = V_w dO^T  (16 keys x 64 queries each)
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      st[i][0] = st[i][1] = st[i][2] = st[i][3] = dpt[i][0] = dpt[i][1] = dpt[i][2] = dpt[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t ak[4], av[4];
      fa_lda(ak, kb, warp * 16, kk * 16, lane);
      fa_lda(av, vb, warp * 16, kk * 16, lane);
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        uint32_t bq[4], bo[4];
        fa_ldb_nk(bq, qb, jn * 16, kk * 16, lane);
        fa_ldb_nk(bo, ob, jn * 16, kk * 16, lane);
        mma16816(st[2 * jn], ak, bq[0], bq[1]);
        mma16816(st[2 * jn + 1], ak, bq[2], bq[3]);
        mma16816(dpt[2 * jn], av, bo[0], bo[1]);
        mma16816(dpt[2 * jn + 1], av, bo[2], bo[3]);
      }
    }
    // P^T, dS^T  (rows = keys, columns = queries)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + 2 * c + (e & 1);  // query within the tile
        const int key = key_r0 + (e >> 1) * 8;
        const int q = qr + ql;
        const bool ok = key <= q && q < qend && qs_b[ql] <= key;
        const float pv = ok ? exp2f(st[nt][e] * p.scale_log2 - lse_b[ql]) : 0.f;
        st[nt][e] = pv;
        dpt[nt][e] = pv * (dpt[nt][e] - dl_b[ql]);
      }
    // dV += P^T dO ; dK += dS^T Q   (k16 steps over the 64 queries)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t ap[4], as[4];
      fa_c2a(ap, st[2 * kk], st[2 * kk + 1]);
      fa_c2a(as, dpt[2 * kk], dpt[2 * kk + 1]);
#pragma unroll
      for (int jd = 0; jd < 8; ++jd) {
        uint32_t bo[4], bq[4];
        fa_ldb_kn(bo, ob, jd * 16, kk * 16, lane);
        fa_ldb_kn(bq, qb, jd * 16, kk * 16, lane);
        mma16816(dv[2 * jd], ap, bo[0], bo[1]);
        mma16816(dv[2 * jd + 1], ap, bo[2], bo[3]);
        mma16816(dk[2 * jd], as, bq[0], bq[1]);
        mma16816(dk[2 * jd + 1], as, bq[2], bq[3]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key_r0 + r * 8;
    if (key >= p.T) continue;
    bf16* dkd = p.dk + (size_t)key * p.lddk + hk * kFaD;
    bf16* dvd = p.dv + (size_t)key * p.lddv + hk * kFaD;
#pragma unroll
    for (int dt = 0; dt < 16; ++dt) {
      *reinterpret_cast<uint32_t*>(dkd + dt * 8 + 2 * c) =
          pack_bf16x2(dk[dt][2 * r] * p.scale, dk[dt][2 * r + 1] * p.scale);
      *reinterpret_cast<uint32_t*>(dvd + dt * 8 + 2 * c) = pack_bf16x2(dv[dt][2 * r], dv[dt][2 * r + 1]);
    }
  }
}

// dQ of 64 query rows of one head: over the key tiles up to the diagonal, P = exp2(scale_log2 *
// Q K^T - lse), dP = dO V^T, dS = P (dP - delta), dQ += dS K (warp w owns queries 16w..16w+15).
// (a single K/V stage with 3 CTAs/SM, which helps the forward, measured 4-13 % slower here)
__global__ void __launch_bounds__(kFaThreads) flash_bwd_dq_kernel(const FlashParams p) {
  extern __shared__ __align__(128) uint8_t fsm[];
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * kFaBM;
  if (q0 >= p.T) return;
  const int hk = h / (p.n_heads / p.n_kv_heads);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  uint8_t* Qs = fsm;
  uint8_t* Os = fsm + 16384;
  uint8_t* Ks = fsm + 32768;  // [2]
  uint8_t* Vs = fsm + 65536;  // [2]
  const uint32_t qb = smem_u32(Qs), ob = smem_u32(Os), kb0 = smem_u32(Ks), vb0 = smem_u32(Vs);
  const int nq = min(kFaBM, p.T - q0);
  const int kstart = p.row_start[q0], kend = q0 + nq;
  const int n_kt = (kend - kstart + kFaBM - 1) / kFaBM;
  fa_load_tile(Qs, p.q, p.ldq, q0, nq, h * kFaD);
  fa_load_tile(Os, p.dout, p.lddo, q0, nq, h * kFaD);
  fa_load_tile(Ks, p.k, p.ldk, kstart, min(kFaBM, kend - kstart), hk * kFaD);
  fa_load_tile(Vs, p.v, p.ldv, kstart, min(kFaBM, kend - kstart), hk * kFaD);
  cp_async_commit();
  const int qrow0 = q0 + warp * 16 + g;
  float lse_r[2], dl_r[2];
  int qs[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qr = qrow0 + r * 8;
    const bool ok = qr < p.T;
    lse_r[r] = ok ? p.lse[(size_t)h * p.stat_ld + qr] : 0.f;
    dl_r[r] = ok ? p.delta[(size_t)h * p.stat_ld + qr] : 0.f;
    qs[r] = ok ? p.row_start[qr] : 0x7fffffff;
  }
  float dq[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int j = 0; j < n_kt; ++j) {
    if (j + 1 < n_kt) {
      const int kr = kstart + (j + 1) * kFaBM;
      fa_load_tile(Ks + ((j + 1) & 1) * 16384, p.k, p.ldk, kr, min(kFaBM, kend - kr), hk * kFaD);
      fa_load_tile(Vs + ((j + 1) & 1) * 16384, p.v, p.ldv, kr, min(kFaBM, kend - kr), hk * kFaD);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t kb = kb0 + (j & 1) * 16384, vb = vb0 + (j & 1) * 16384;
    float sc[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t aq[4], ao[4];
      fa_lda(aq, qb, warp * 16, kk * 16, lane);
      fa_lda(ao, ob, warp * 16, kk * 16, lane);
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        uint32_t bk[4], bv[4];
        fa_ldb_nk(bk, kb, jn * 16, kk * 16, lane);
        fa_ldb_nk(bv, vb, jn * 16, kk * 16, lane);
        mma16816(sc[2 * jn], aq, bk[0], bk[1]);
        mma16816(sc[2 * jn + 1], aq, bk[2], bk[3]);
        mma16816(dp[2 * jn], ao, bv[0], bv[1]);
        mma16816(dp[2 * jn + 1], ao, bv[2], bv[3]);
      }
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kstart + j * kFaBM + nt * 8 + 2 * c + (e & 1);
        const int qr = qrow0 + (e >> 1) * 8;
        const bool ok = key <= qr && key >= qs[e >> 1] && qr < p.T;
        const float pv = ok ? exp2f(sc[nt][e] * p.scale_log2 - lse_r[e >> 1]) : 0.f;
        dp[nt][e] = pv * (dp[nt][e] - dl_r[e >> 1]);
      }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t as[4];
      fa_c2a(as, dp[2 * kk], dp[2 * kk + 1]);
#pragma unroll
      for (int jd = 0; jd < 8; ++jd) {
        uint32_t bk[4];
        fa_ldb_kn(bk, kb, jd * 16, kk * 16, lane);
        mma16816(dq[2 * jd], as, bk[0], bk[1]);
        mma16816(dq[2 * jd + 1], as, bk[2], bk[3]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qr = qrow0 + r * 8;
    if (qr >= p.T) continue;
    bf16* dst = p.dq + (size_t)qr * p.lddq + h * kFaD;
#pragma unroll
    for (int dt = 0; dt < 16; ++dt)
      *reinterpret_cast<uint32_t*>(dst + dt * 8 + 2 * c) =
          pack_bf16x2(dq[dt][2 * r] * p.scale, dq[dt][2 * r + 1] * p.scale);
  }
}

}  // namespace collm
