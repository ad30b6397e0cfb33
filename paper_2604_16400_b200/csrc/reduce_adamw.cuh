// reduce_adamw.cuh — K5: LoRA weight gradients as deterministic T-reductions, with the AdamW
// step fused into the final reduction stage.
//
//   C[p, q] = sum_t U[t, u_off + p] * V[t, v_off + q]        (fp32 accumulation)
//
//   dB_s   = dY[:, n-range of sub s]^T . H16[:, s*r : (s+1)*r]     (P = N_s, Q = r)
//   dA^T   = X^T . (dH16 + dH16lo)                                 (P = K,   Q = R)
//
// A group may carry a second V operand V2 (same layout) reduced into the same accumulator:
// C = U^T (V + V2).  The dA^T groups use it for the bf16 hi+lo pair of dH (the shrink writes
// dH16 = bf16(dH) and dH16lo = bf16(dH - dH16)), so the gradient sees dH to ~2^-16 relative
// instead of one bf16 rounding (LoRA grads within 1e-3 of the exact math).
//
// The trainable adapter's fp32 master copies live in these C layouts (B: [N, r], A^T: [K, R]),
// so the optimizer is elementwise on the reduced tile; the bf16 working copies the forward and
// backward kernels read are written from the same registers in both layouts the kernels need
// (B [N,r] + B^T [R,N]; A^T [K,R] + A [R,K]).  Replaces the reference's optimizer stand-in
// `AdapterParams.perturbed` (/root/reference/pkg/src/coserve/launcher.py:43-47, called at
// engine.py:402-403) and the convergence stand-in `perf.train_step` (perf.py:111-126).
//
// Tiling: CTA = 4 warps = 64 (P) x QT (Q); T streamed in 32-row chunks through a cp.async double
// buffer; operand fragments via ldmatrix.trans (both operands are t-major in HBM); mma.sync
// m16n8k16.  T is split across CTAs; the last CTA of a tile sums the splits in index order, so the
// result is bitwise reproducible (no float atomics).
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kReduceMaxGroups = 16;  // ABI limit per launch: a whole layer's projections
constexpr int kReduceMaxQ = 64;       // widest group a CTA reduces (wider ABI groups are split)
constexpr int kReduceMaxInner = 32;   // groups after that split
constexpr int kReducePT = 128;     // P rows per CTA tile (8 warps x 16)
constexpr int kReduceTC = 32;      // T rows per pipeline stage
constexpr int kReduceMaxStages = 4;  // cp.async ring depth (runtime: fits the smem budget)
constexpr int kReduceThreads = 256;

enum ReduceMode : int {
  kModeStoreGrad = 0,  // grad = C (* grad_scale) [+ grad]
  kModeAdamW = 1,      // g = C (* grad_scale) [+ grad]; AdamW on master/m/v; write bf16 copies
  kModeCopyOnly = 2,   // (apply kernel only) master -> bf16 copies
};

// One reduction problem: its operands, its placement, and the optimizer state it updates.
// AdamW hyper-parameters live in DEVICE memory ({lr, beta1, beta2, eps, weight_decay,
// 1-beta1^step, 1-beta2^step}) so a captured CUDA graph can be replayed step after step with the
// host updating only this 28-byte block.
struct ReduceGroup {
  const bf16* U;
  const bf16* V;
  const bf16* V2;  // optional second V operand (same ldv / v_off): C = U^T (V + V2)
  float* grad;
  float* master;
  float* m;
  float* v;
  bf16* out_same;
  bf16* out_trans;
  int ldu, ldv;
  int u_off, P, v_off, Q;
  int ldc, ld_trans;
  int c_row_off, c_col_off;  // placement in the fp32 (grad/master/m/v) layout, ld = ldc
  int t_row_off, t_col_off;  // placement of the transposed bf16 copy, ld = ld_trans
  int tile_begin;            // first CTA tile of this group (kReducePT-row P tiles)
};

struct ReduceParams {
  int T;
  int n_groups;
  ReduceGroup groups[kReduceMaxInner];
  int n_tiles;
  int tsplit;
  int stages;
  int mode;
  int accum_in;      // add the existing grad buffer contents
  float grad_scale;  // applied to the freshly reduced C
  const float* opt;  // device [7]
  float* partials;   // [tsplit][n_tiles][kReducePT*64]
  int32_t* counters;
};

__device__ __forceinline__ void ldsm_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                              uint32_t& r3, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t& r0, uint32_t& r1, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(smem_u32(p)));
}

// Finalize one element: gradient bookkeeping + (optionally) the AdamW step, PyTorch semantics
// (decoupled weight decay; step_size = lr / bc1; denom = sqrt(v)/sqrt(bc2) + eps).  Returns the
// bf16 weight written to the copies (for the transposed write-out by the caller).
__device__ __forceinline__ bf16 finalize_elem(const ReduceParams& p, const ReduceGroup& gr, int pp,
                                              int q, float c, bool have_c) {
  const size_t idx = (size_t)(gr.c_row_off + pp) * gr.ldc + gr.c_col_off + q;
  if (p.mode == kModeCopyOnly) {
    const bf16 wb = __float2bfloat16_rn(gr.master[idx]);
    if (gr.out_same) gr.out_same[idx] = wb;
    return wb;
  }
  float g = have_c ? c * p.grad_scale : 0.f;
  if (!have_c || p.accum_in) g += gr.grad[idx];
  if (p.mode == kModeStoreGrad) {
    gr.grad[idx] = g;
    return __float2bfloat16_rn(0.f);
  }
  float w = gr.master[idx];
  const float lr = __ldg(p.opt + 0), beta1 = __ldg(p.opt + 1), beta2 = __ldg(p.opt + 2);
  const float eps = __ldg(p.opt + 3), wd = __ldg(p.opt + 4);
  const float bc1 = __ldg(p.opt + 5), bc2 = __ldg(p.opt + 6);
  w -= lr * wd * w;
  const float m = beta1 * gr.m[idx] + (1.f - beta1) * g;
  const float v = beta2 * gr.v[idx] + (1.f - beta2) * g * g;
  gr.m[idx] = m;
  gr.v[idx] = v;
  const float denom = sqrtf(v) / sqrtf(bc2) + eps;
  w -= (lr / bc1) * (m / denom);
  gr.master[idx] = w;
  const bf16 wb = __float2bfloat16_rn(w);
  if (gr.out_same) gr.out_same[idx] = wb;
  return wb;
}

// Vectorized finalize of a reduced tile: every thread owns float4 groups of 4 consecutive q and
// issues all loads (partials, grad, m, v, master) of UNR groups before using any of them, so the
// tail of the split reduction runs at memory parallelism instead of one latency per element.
// `cs` is the CTA's own tile in shared memory (tsplit == 1) or null (sum the global partials).
template <int QT, int UNR = 1>
__device__ __forceinline__ void finalize_tile(const ReduceParams& p, const ReduceGroup& gr, int p0,
                                              int prow, const float (*cs)[QT + 1],
                                              const float* parts, size_t part_stride,
                                              bf16 (*Ct)[kReducePT + 8], bool trans) {
  const int Q = gr.Q, nq4 = Q >> 2, nvec = prow * nq4;
  const bool adam = p.mode == kModeAdamW, store = p.mode == kModeStoreGrad;
  const bool read_grad = store ? (p.accum_in != 0) : (adam && p.accum_in);
  float lr = 0.f, beta1 = 0.f, beta2 = 0.f, eps = 0.f, wd = 0.f, bc1 = 1.f, bc2 = 1.f;
  if (adam) {
    lr = __ldg(p.opt + 0); beta1 = __ldg(p.opt + 1); beta2 = __ldg(p.opt + 2);
    eps = __ldg(p.opt + 3); wd = __ldg(p.opt + 4); bc1 = __ldg(p.opt + 5); bc2 = __ldg(p.opt + 6);
  }
  const float step_size = lr / bc1, inv_sqrt_bc2 = rsqrtf(bc2);
  for (int base = threadIdx.x; base < nvec; base += kReduceThreads * UNR) {
    float4 c[UNR], gv[UNR], mv[UNR], vv[UNR], wv[UNR];
    size_t idx[UNR];
    int pp[UNR], qq[UNR];
    bool ok[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int v4 = base + u * kReduceThreads;
      ok[u] = v4 < nvec;
      pp[u] = ok[u] ? v4 / nq4 : 0;
      qq[u] = ok[u] ? (v4 % nq4) * 4 : 0;
      idx[u] = (size_t)(gr.c_row_off + p0 + pp[u]) * gr.ldc + gr.c_col_off + qq[u];
      c[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!ok[u]) continue;
      if (cs) {
        c[u] = make_float4(cs[pp[u]][qq[u]], cs[pp[u]][qq[u] + 1], cs[pp[u]][qq[u] + 2],
                           cs[pp[u]][qq[u] + 3]);
      } else {
        for (int s = 0; s < p.tsplit; ++s) {
          const float4 t = __ldcg(reinterpret_cast<const float4*>(parts + s * part_stride +
                                                                  pp[u] * Q + qq[u]));
          c[u].x += t.x; c[u].y += t.y; c[u].z += t.z; c[u].w += t.w;
        }
      }
      if (read_grad) gv[u] = *reinterpret_cast<const float4*>(gr.grad + idx[u]);
      if (adam) {
        mv[u] = *reinterpret_cast<const float4*>(gr.m + idx[u]);
        vv[u] = *reinterpret_cast<const float4*>(gr.v + idx[u]);
        wv[u] = *reinterpret_cast<const float4*>(gr.master + idx[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (!ok[u]) continue;
      float g[4] = {c[u].x * p.grad_scale, c[u].y * p.grad_scale, c[u].z * p.grad_scale,
                    c[u].w * p.grad_scale};
      if (read_grad) { g[0] += gv[u].x; g[1] += gv[u].y; g[2] += gv[u].z; g[3] += gv[u].w; }
      if (store) {
        *reinterpret_cast<float4*>(gr.grad + idx[u]) = make_float4(g[0], g[1], g[2], g[3]);
        continue;
      }
      float m[4] = {mv[u].x, mv[u].y, mv[u].z, mv[u].w};
      float v[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
      float w[4] = {wv[u].x, wv[u].y, wv[u].z, wv[u].w};
      bf16 wb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        w[k] -= lr * wd * w[k];
        m[k] = beta1 * m[k] + (1.f - beta1) * g[k];
        v[k] = beta2 * v[k] + (1.f - beta2) * g[k] * g[k];
        w[k] -= step_size * (m[k] / (sqrtf(v[k]) * inv_sqrt_bc2 + eps));
        wb[k] = __float2bfloat16_rn(w[k]);
      }
      *reinterpret_cast<float4*>(gr.m + idx[u]) = make_float4(m[0], m[1], m[2], m[3]);
      *reinterpret_cast<float4*>(gr.v + idx[u]) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(gr.master + idx[u]) = make_float4(w[0], w[1], w[2], w[3]);
      if (gr.out_same) {
        __nv_bfloat162 lo = __halves2bfloat162(wb[0], wb[1]), hi = __halves2bfloat162(wb[2], wb[3]);
        uint2 pk = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
        *reinterpret_cast<uint2*>(gr.out_same + idx[u]) = pk;
      }
      if (trans) {
#pragma unroll
        for (int k = 0; k < 4; ++k) Ct[qq[u] + k][pp[u]] = wb[k];
      }
    }
  }
}

__device__ __forceinline__ int find_group(const ReduceParams& p, int tile) {
  int gi = 0;
  for (int i = 1; i < p.n_groups; ++i)
    if (tile >= p.groups[i].tile_begin) gi = i;
  return gi;
}

template <int QT>
struct ReduceSmem {
  static constexpr int kUP = kReducePT + 8, kVP = QT + 8;  // padded rows: conflict-free ldmatrix
  static constexpr size_t kUStage = (size_t)kReduceTC * kUP * 2;
  static constexpr size_t kVStage = (size_t)kReduceTC * kVP * 2;
  static constexpr size_t kCBytes = (size_t)kReducePT * (QT + 1) * 4;
  static constexpr size_t kTBytes = (size_t)QT * (kReducePT + 8) * 2;
  static constexpr size_t kEpi = kCBytes + kTBytes;
  static size_t total(int stages) {
    const size_t pipe = (size_t)stages * (kUStage + 2 * kVStage);  // V and V2 rings
    return (pipe > kEpi ? pipe : kEpi) + 16;
  }
};

// MINB = resident CTAs per SM the register budget is sized for (4: 64 registers, 3: 80)
template <int QT, int MINB = 4>
__global__ void __launch_bounds__(kReduceThreads, MINB) lora_reduce_kernel(const ReduceParams p) {
  using S = ReduceSmem<QT>;
  constexpr int PT = kReducePT, TC = kReduceTC;
  const int ST = p.stages;
  extern __shared__ __align__(16) uint8_t smem[];
  bf16 (*Us)[TC][S::kUP] = reinterpret_cast<bf16 (*)[TC][S::kUP]>(smem);
  bf16 (*Vs)[TC][S::kVP] = reinterpret_cast<bf16 (*)[TC][S::kVP]>(smem + ST * S::kUStage);
  bf16 (*Vs2)[TC][S::kVP] =
      reinterpret_cast<bf16 (*)[TC][S::kVP]>(smem + ST * (S::kUStage + S::kVStage));
  float (*Cs)[QT + 1] = reinterpret_cast<float (*)[QT + 1]>(smem);
  bf16 (*Ct)[PT + 8] = reinterpret_cast<bf16 (*)[PT + 8]>(smem + S::kCBytes);
  __shared__ int s_last;

  const int tile = blockIdx.x, ts = blockIdx.y;
  const int gi = find_group(p, tile);
  const ReduceGroup& gr = p.groups[gi];
  const int p0 = (tile - gr.tile_begin) * PT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int chunks = (p.T + TC - 1) / TC;
  const int per = (chunks + p.tsplit - 1) / p.tsplit;
  const int ch_lo = ts * per, ch_hi = min(chunks, ch_lo + per);
  const int n_ch = max(0, ch_hi - ch_lo);

  // per-thread copy geometry, hoisted out of the chunk loop: U chunk = TC x PT (2 16-byte vectors
  // per thread), V chunk = TC x QT (<= 1 vector per thread)
  const bf16* u_base = gr.U + gr.u_off + p0;
  const bf16* v_base = gr.V + gr.v_off;
  const bool has_v2 = gr.V2 != nullptr;  // CTA-uniform
  const long long v2_delta = has_v2 ? (long long)(gr.V2 - gr.V) : 0;  // V2 = V + delta
  const size_t ldu = gr.ldu, ldv = gr.ldv;
  const int T = p.T;
  static_assert(TC * (PT / 8) == 2 * kReduceThreads, "U chunk: two vectors per thread");
  static_assert(TC * (QT / 8) <= kReduceThreads, "V chunk: at most one vector per thread");
  const int u_r = threadIdx.x / (PT / 8), u_c = (threadIdx.x % (PT / 8)) * 8;
  const bool u_col_ok = p0 + u_c < gr.P;
  const bool v_on = threadIdx.x < TC * (QT / 8);
  const int v_r = threadIdx.x / (QT / 8), v_c = (threadIdx.x % (QT / 8)) * 8;
  const bool v_col_ok = v_on && v_c < gr.Q;
  auto load_chunk = [&](int stage, int ch) {
    const int t0 = ch * TC;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int r = u_r + k * (TC / 2), t = t0 + r;
      const bool ok = t < T && u_col_ok;
      cp_async_16(&Us[stage][r][u_c], ok ? u_base + (size_t)t * ldu + u_c : gr.U, ok);
    }
    if (v_on) {
      const int t = t0 + v_r;
      const bool ok = t < T && v_col_ok;
      cp_async_16(&Vs[stage][v_r][v_c], ok ? v_base + (size_t)t * ldv + v_c : gr.V, ok);
      if (has_v2)
        cp_async_16(&Vs2[stage][v_r][v_c], ok ? v_base + v2_delta + (size_t)t * ldv + v_c : gr.V, ok);
    }
  };

  float d[QT / 8][4];
#pragma unroll
  for (int j = 0; j < QT / 8; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.f;

  for (int i = 0; i < ST - 1; ++i) {
    if (i < n_ch) load_chunk(i, ch_lo + i);
    cp_async_commit();
  }
  int stage = 0, fill = ST - 1;  // ring slots of the chunk consumed / refilled (no divisions)
  for (int i = 0; i < n_ch; ++i) {
    cp_async_wait_dyn(ST - 2);
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TC; kk += 16) {
      uint32_t a0, a1, a2, a3;
      {
        const int mat = lane >> 3, rr = lane & 7;
        ldsm_x4_trans(a0, a1, a2, a3,
                      &Us[stage][kk + rr + ((mat & 2) ? 8 : 0)][warp * 16 + ((mat & 1) ? 8 : 0)]);
      }
#pragma unroll
      for (int j = 0; j < QT / 8; j += 2) {
        uint32_t b0, b1, b2, b3;
        if (j + 1 < QT / 8) {
          const int mat = lane >> 3, rr = lane & 7;
          ldsm_x4_trans(b0, b1, b2, b3,
                        &Vs[stage][kk + rr + ((mat & 1) ? 8 : 0)][(j + ((mat & 2) ? 1 : 0)) * 8]);
          mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
          mma_m16n8k16_bf16(d[j + 1], a0, a1, a2, a3, b2, b3);
          if (has_v2) {
            ldsm_x4_trans(b0, b1, b2, b3,
                          &Vs2[stage][kk + rr + ((mat & 1) ? 8 : 0)][(j + ((mat & 2) ? 1 : 0)) * 8]);
            mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
            mma_m16n8k16_bf16(d[j + 1], a0, a1, a2, a3, b2, b3);
          }
        } else {
          const int rr = lane & 7, mat = (lane >> 3) & 1;
          ldsm_x2_trans(b0, b1, &Vs[stage][kk + rr + mat * 8][j * 8]);
          mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
          if (has_v2) {
            ldsm_x2_trans(b0, b1, &Vs2[stage][kk + rr + mat * 8][j * 8]);
            mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
          }
        }
      }
    }
    if (i + ST - 1 < n_ch) load_chunk(fill, ch_lo + i + ST - 1);
    cp_async_commit();
    if (++stage == ST) stage = 0;
    if (++fill == ST) fill = 0;
  }
  cp_async_wait<0>();
  __syncthreads();

  // fragments -> smem tile (reuses the pipeline buffers)
  {
    const int g = lane >> 2, c = lane & 3;
#pragma unroll
    for (int j = 0; j < QT / 8; ++j) {
      Cs[warp * 16 + g][8 * j + 2 * c] = d[j][0];
      Cs[warp * 16 + g][8 * j + 2 * c + 1] = d[j][1];
      Cs[warp * 16 + g + 8][8 * j + 2 * c] = d[j][2];
      Cs[warp * 16 + g + 8][8 * j + 2 * c + 1] = d[j][3];
    }
  }
  __syncthreads();

  const int prow = min(PT, gr.P - p0);
  const int Q = gr.Q;
  const int n_el = prow * Q;
  const bool trans = gr.out_trans && p.mode != kModeStoreGrad;
  if (p.tsplit > 1) {
    float* mine = p.partials + ((size_t)ts * p.n_tiles + tile) * (PT * 64);
    for (int e = threadIdx.x; e < n_el; e += kReduceThreads) mine[e] = Cs[e / Q][e % Q];
    __syncthreads();  // CTA-scope: all partial stores happen-before thread 0's cumulative fence
    if (threadIdx.x == 0) {
      __threadfence();
      const int prev = atomicAdd(p.counters + tile, 1);
      s_last = (prev == p.tsplit - 1);
      if (s_last) p.counters[tile] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) __threadfence();  // acquire side of the arrival counter
    __syncthreads();
    finalize_tile<QT>(p, gr, p0, prow, nullptr, p.partials + (size_t)tile * (PT * 64),
                      (size_t)p.n_tiles * (PT * 64), Ct, trans);
  } else {
    finalize_tile<QT>(p, gr, p0, prow, Cs, nullptr, 0, Ct, trans);
  }
  if (trans) {  // coalesced transposed write-out: rows of the [Q, P] copy
    __syncthreads();
    for (int e = threadIdx.x; e < n_el; e += kReduceThreads) {
      const int q = e / prow, pp = e % prow;
      gr.out_trans[(size_t)(gr.t_row_off + q) * gr.ld_trans + gr.t_col_off + p0 + pp] = Ct[q][pp];
    }
  }
}

// Elementwise variant over the same group table with no reduction: used after a cross-replica
// gradient allreduce (mode AdamW from the grad buffer) and after a parameter average (copy-only).
__global__ void lora_apply_kernel(const ReduceParams p, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long base = 0;
    int gi = 0;
    for (; gi < p.n_groups - 1; ++gi) {
      const long long n = (long long)p.groups[gi].P * p.groups[gi].Q;
      if (e < base + n) break;
      base += n;
    }
    const ReduceGroup& gr = p.groups[gi];
    const long long off = e - base;
    const int pp = (int)(off / gr.Q), q = (int)(off % gr.Q);
    const bf16 wb = finalize_elem(p, gr, pp, q, 0.f, false);
    if (gr.out_trans && p.mode != kModeStoreGrad)
      gr.out_trans[(size_t)(gr.t_row_off + q) * gr.ld_trans + gr.t_col_off + pp] = wb;
  }
}

}  // namespace collm
