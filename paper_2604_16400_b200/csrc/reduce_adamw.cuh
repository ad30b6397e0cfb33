// reduce_adamw.cuh — K5: LoRA weight gradients as deterministic T-reductions, with the AdamW
// step fused into the final reduction stage.
//
//   C[p, q] = sum_t U[t, u_off + p] * V[t, v_off + q]        (fp32 accumulation)
//
//   dB_s   = dY[:, n-range of sub s]^T . H16[:, s*r : (s+1)*r]     (P = N_s, Q = r)
//   dA^T   = X^T . dH16                                            (P = K,   Q = R)
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

constexpr int kReduceMaxGroups = 16;

enum ReduceMode : int {
  kModeStoreGrad = 0,  // grad = C (* grad_scale) [+ grad]
  kModeAdamW = 1,      // g = C (* grad_scale) [+ grad]; AdamW on master/m/v; write bf16 copies
  kModeCopyOnly = 2,   // (apply kernel only) master -> bf16 copies
};

struct ReduceGroup {
  int u_off, P, v_off, Q;
  int c_row_off, c_col_off;  // placement in the fp32 (grad/master/m/v) layout, ld = ldc
  int t_row_off, t_col_off;  // placement of the transposed bf16 copy, ld = ld_trans
  int tile_begin;            // first CTA tile of this group (64-row P tiles)
};

// AdamW hyper-parameters live in DEVICE memory ({lr, beta1, beta2, eps, weight_decay,
// 1-beta1^step, 1-beta2^step}) so a captured CUDA graph can be replayed step after step with the
// host updating only this 28-byte block.

struct ReduceParams {
  const bf16* U;
  int ldu;
  const bf16* V;
  int ldv;
  int T;
  int n_groups;
  ReduceGroup groups[kReduceMaxGroups];
  int n_tiles;
  int tsplit;
  int mode;
  int accum_in;      // add the existing grad buffer contents
  float grad_scale;  // applied to the freshly reduced C
  float* grad;
  int ldc;
  float* master;
  float* m;
  float* v;
  bf16* out_same;
  bf16* out_trans;
  int ld_trans;
  const float* opt;  // device [7]
  float* partials;  // [tsplit][n_tiles][64*64]
  int32_t* counters;
};

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, bool pred) {
  const uint32_t s = smem_u32(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
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
// (decoupled weight decay; step_size = lr / bc1; denom = sqrt(v)/sqrt(bc2) + eps).
__device__ __forceinline__ void finalize_elem(const ReduceParams& p, const ReduceGroup& gr, int pp,
                                              int q, float c, bool have_c) {
  const size_t idx = (size_t)(gr.c_row_off + pp) * p.ldc + gr.c_col_off + q;
  if (p.mode == kModeCopyOnly) {
    const bf16 wb = __float2bfloat16_rn(p.master[idx]);
    if (p.out_same) p.out_same[idx] = wb;
    if (p.out_trans)
      p.out_trans[(size_t)(gr.t_row_off + q) * p.ld_trans + gr.t_col_off + pp] = wb;
    return;
  }
  float g = have_c ? c * p.grad_scale : 0.f;
  if (!have_c || p.accum_in) g += p.grad[idx];
  if (p.mode == kModeStoreGrad) {
    p.grad[idx] = g;
    return;
  }
  float w = p.master[idx];
  if (p.mode == kModeAdamW) {
    const float lr = __ldg(p.opt + 0), beta1 = __ldg(p.opt + 1), beta2 = __ldg(p.opt + 2);
    const float eps = __ldg(p.opt + 3), wd = __ldg(p.opt + 4);
    const float bc1 = __ldg(p.opt + 5), bc2 = __ldg(p.opt + 6);
    w -= lr * wd * w;
    const float m = beta1 * p.m[idx] + (1.f - beta1) * g;
    const float v = beta2 * p.v[idx] + (1.f - beta2) * g * g;
    p.m[idx] = m;
    p.v[idx] = v;
    const float denom = sqrtf(v) / sqrtf(bc2) + eps;
    w -= (lr / bc1) * (m / denom);
    p.master[idx] = w;
  }
  const bf16 wb = __float2bfloat16_rn(w);
  if (p.out_same) p.out_same[idx] = wb;
  if (p.out_trans)
    p.out_trans[(size_t)(gr.t_row_off + q) * p.ld_trans + gr.t_col_off + pp] = wb;
}

__device__ __forceinline__ int find_group(const ReduceParams& p, int tile) {
  int gi = 0;
  for (int i = 1; i < p.n_groups; ++i)
    if (tile >= p.groups[i].tile_begin) gi = i;
  return gi;
}

template <int QT>
__global__ void __launch_bounds__(128) lora_reduce_kernel(const ReduceParams p) {
  constexpr int PT = 64, TC = 32;
  constexpr int UP = PT + 8, VP = QT + 8;  // padded rows: conflict-free ldmatrix
  __shared__ __align__(16) bf16 Us[2][TC][UP];
  __shared__ __align__(16) bf16 Vs[2][TC][VP];
  __shared__ float Cs[PT][QT + 1];
  __shared__ int s_last;

  const int tile = blockIdx.x, ts = blockIdx.y;
  const int gi = find_group(p, tile);
  const ReduceGroup gr = p.groups[gi];
  const int p0 = (tile - gr.tile_begin) * PT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int chunks = (p.T + TC - 1) / TC;
  const int per = (chunks + p.tsplit - 1) / p.tsplit;
  const int ch_lo = ts * per, ch_hi = min(chunks, ch_lo + per);

  auto load_chunk = [&](int buf, int ch) {
    const int t0 = ch * TC;
    // U: 32 rows x 64 cols = 256 x 16B
    for (int i = threadIdx.x; i < TC * (PT / 8); i += 128) {
      const int r = i / (PT / 8), cc = (i % (PT / 8)) * 8;
      const int t = t0 + r, pp = p0 + cc;
      const bool ok = t < p.T && pp < gr.P;
      cp_async_16(&Us[buf][r][cc], ok ? p.U + (size_t)t * p.ldu + gr.u_off + pp : p.U, ok);
    }
    for (int i = threadIdx.x; i < TC * (QT / 8); i += 128) {
      const int r = i / (QT / 8), cc = (i % (QT / 8)) * 8;
      const int t = t0 + r;
      const bool ok = t < p.T && cc < gr.Q;
      cp_async_16(&Vs[buf][r][cc], ok ? p.V + (size_t)t * p.ldv + gr.v_off + cc : p.V, ok);
    }
  };

  float d[QT / 8][4];
#pragma unroll
  for (int j = 0; j < QT / 8; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.f;

  if (ch_lo < ch_hi) {
    load_chunk(0, ch_lo);
    cp_async_commit();
    for (int ch = ch_lo; ch < ch_hi; ++ch) {
      const int buf = (ch - ch_lo) & 1;
      if (ch + 1 < ch_hi) load_chunk(buf ^ 1, ch + 1);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TC; kk += 16) {
        // A fragment (m = p, k = t) from Us[t][p] via .trans
        uint32_t a0, a1, a2, a3;
        {
          const int mat = lane >> 3, rr = lane & 7;
          const int krow = kk + rr + ((mat & 2) ? 8 : 0);
          const int pcol = warp * 16 + ((mat & 1) ? 8 : 0);
          ldsm_x4_trans(a0, a1, a2, a3, &Us[buf][krow][pcol]);
        }
#pragma unroll
        for (int j = 0; j < QT / 8; j += 2) {
          uint32_t b0, b1, b2, b3;
          if (j + 1 < QT / 8) {
            const int mat = lane >> 3, rr = lane & 7;
            const int krow = kk + rr + ((mat & 1) ? 8 : 0);
            const int qcol = (j + ((mat & 2) ? 1 : 0)) * 8;
            ldsm_x4_trans(b0, b1, b2, b3, &Vs[buf][krow][qcol]);
            mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
            mma_m16n8k16_bf16(d[j + 1], a0, a1, a2, a3, b2, b3);
          } else {
            const int rr = lane & 7, mat = (lane >> 3) & 1;
            ldsm_x2_trans(b0, b1, &Vs[buf][kk + rr + mat * 8][j * 8]);
            mma_m16n8k16_bf16(d[j], a0, a1, a2, a3, b0, b1);
          }
        }
      }
      __syncthreads();
    }
  }

  // fragments -> smem tile
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
  const int n_el = prow * gr.Q;
  if (p.tsplit > 1) {
    float* mine = p.partials + ((size_t)ts * p.n_tiles + tile) * (64 * 64);
    for (int e = threadIdx.x; e < n_el; e += 128) mine[e] = Cs[e / gr.Q][e % gr.Q];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int prev = atomicAdd(p.counters + tile, 1);
      s_last = (prev == p.tsplit - 1);
      if (s_last) p.counters[tile] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int e = threadIdx.x; e < n_el; e += 128) {
      float acc = 0.f;
      for (int s = 0; s < p.tsplit; ++s)
        acc += __ldcg(p.partials + ((size_t)s * p.n_tiles + tile) * (64 * 64) + e);
      finalize_elem(p, gr, p0 + e / gr.Q, e % gr.Q, acc, true);
    }
  } else {
    for (int e = threadIdx.x; e < n_el; e += 128)
      finalize_elem(p, gr, p0 + e / gr.Q, e % gr.Q, Cs[e / gr.Q][e % gr.Q], true);
  }
}

// Elementwise variant over the same group table with no reduction: used after a cross-replica
// gradient allreduce (mode AdamW from the grad buffer) and after a parameter average (copy-only).
__global__ void lora_apply_kernel(const ReduceParams p, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long base = 0;
    int gi = 0;
    for (; gi < p.n_groups; ++gi) {
      const long long n = (long long)p.groups[gi].P * p.groups[gi].Q;
      if (e < base + n) break;
      base += n;
    }
    const ReduceGroup& gr = p.groups[gi];
    const long long off = e - base;
    finalize_elem(p, gr, (int)(off / gr.Q), (int)(off % gr.Q), 0.f, false);
  }
}

}  // namespace collm
