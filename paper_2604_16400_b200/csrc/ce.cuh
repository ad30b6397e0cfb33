// ce.cuh — K7: fused softmax cross-entropy forward + backward over the LM-head logits of the
// training rows (HBM-bound, one CTA per row).
//
//   lse_t = log sum_v exp(z[t, v]);  loss_t = lse_t - z[t, y_t]          (y_t < 0: ignored, 0)
//   mean  = sum_{valid t} loss_t / #valid                                 (fixed order)
//   dz[t, v] = grad_scale * (exp(z[t, v] - lse_t) - [v == y_t])           (0 for ignored rows)
//
// Replaces the reference's convergence stand-in `perf.train_step` (perf.py:111-126): the training
// loss the coordinator / TrainState consume becomes the real next-token cross-entropy of the
// co-batched training rows, and dz feeds the LM-head dX GEMM (the top of the LoRA backward).
//
// Pass 1 streams the row once with 16-byte loads keeping a per-thread online (max, sum of exp);
// the CTA combines the pairs in a fixed shuffle/shared-memory tree.  Pass 2 writes dz from the
// row kept in registers (V <= 32768: every logit read from HBM once), or re-reads it (it is
// L2-resident: the GEMM just wrote it and pass 1 just read it) for larger vocabularies.  Logits are
// bf16 (the GEMM output), all softmax arithmetic fp32.  The batch mean is taken by the last CTA
// to finish (arrival counter, restored to 0) summing the per-row losses in row order — bitwise
// deterministic, no atomics on floats.
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kCeUnroll = 4;  // 16-byte loads in flight per thread (two-pass variant)

struct CeParams {
  const bf16* logits;
  int ld;
  int T, V;
  const int32_t* labels;  // [T]; < 0 = ignored row
  float* loss_rows;       // [T]
  float* loss_mean;       // [1] (may be null)
  int32_t* counter;       // [1] arrival counter, 0 on entry and restored (needed with loss_mean)
  bf16* dlogits;          // [T, ld_d] (may be null: forward only)
  int ld_d;
  float grad_scale;
};

__device__ __forceinline__ float ex2_ftz(float x) {  // one MUFU.EX2 (no denormal fix-up code)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void ce_combine(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  // exp2 of (-inf) - finite = 0; both -inf (empty) stays (−inf, 0)
  const float a = (m == -INFINITY) ? 0.f : s * exp2f((m - mm) * 1.4426950408889634f);
  const float b = (m2 == -INFINITY) ? 0.f : s2 * exp2f((m2 - mm) * 1.4426950408889634f);
  m = mm;
  s = a + b;
}

// NV > 0: the whole row stays in registers (NV 16-byte vectors per thread, V <= 8*NV*kCeThreads):
// one HBM read per logit.  NV == 0: two passes over the row (the second from L2).
template <int NV, int NT>
__global__ void __launch_bounds__(NT) cross_entropy_kernel(const CeParams p) {
  constexpr int kCeThreads = NT;
  constexpr float kLog2e = 1.4426950408889634f;
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bf16* row = p.logits + (size_t)t * p.ld;
  const int nvec = p.V >> 3;  // 8 bf16 per 16-byte vector (V % 8 == 0)
  __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32];
  __shared__ float s_lse;

  // pass 1: online max / sum of exp per thread; kCeUnroll 16-byte loads in flight per thread
  float m = -INFINITY, s = 0.f;
  uint4 keep[NV > 0 ? NV : 1];
  if constexpr (NV > 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int i = threadIdx.x + j * kCeThreads;
      keep[j] = i < nvec ? ld_global_nc_v4(row + 8 * i) : make_uint4(0, 0, 0, 0);
    }
    // registers hold the row: a plain max, then a sum of exp against the row max — no serial
    // online-rescaling chain (the kernel is issue/latency-bound, not HBM-bound, otherwise)
    auto lo = [](uint32_t w) { return __uint_as_float(w << 16); };
    auto hi = [](uint32_t w) { return __uint_as_float(w & 0xffff0000u); };
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if (threadIdx.x + j * kCeThreads >= nvec) break;
      const uint32_t w[4] = {keep[j].x, keep[j].y, keep[j].z, keep[j].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) mx[k] = fmaxf(mx[k], fmaxf(lo(w[k]), hi(w[k])));
    }
    float M = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (lane == 0) sm[warp] = M;
    __syncthreads();
    M = sm[0];
#pragma unroll
    for (int w = 1; w < kCeThreads / 32; ++w) M = fmaxf(M, sm[w]);
    const float Mk = M * kLog2e;
    float sx[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      if (threadIdx.x + j * kCeThreads >= nvec) break;
      const uint32_t w[4] = {keep[j].x, keep[j].y, keep[j].z, keep[j].w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        sx[k] += ex2_ftz(fmaf(lo(w[k]), kLog2e, -Mk)) + ex2_ftz(fmaf(hi(w[k]), kLog2e, -Mk));
    }
    m = M;  // every thread: (M, its partial sum) — combined below exactly like the online path
    s = (sx[0] + sx[1]) + (sx[2] + sx[3]);
  }
  for (int i0 = threadIdx.x; NV == 0 && i0 < nvec; i0 += kCeThreads * kCeUnroll) {
    uint4 u[kCeUnroll];
#pragma unroll
    for (int j = 0; j < kCeUnroll; ++j) {
      const int i = i0 + j * kCeThreads;
      u[j] = i < nvec ? ld_global_nc_v4(row + 8 * i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kCeUnroll; ++j) {
      if (i0 + j * kCeThreads >= nvec) break;
      const uint32_t w[4] = {u[j].x, u[j].y, u[j].z, u[j].w};
      float x[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x[2 * k] = __uint_as_float(w[k] << 16);
        x[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
      }
      float vm = x[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) vm = fmaxf(vm, x[k]);
      float vs = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) vs += exp2f((x[k] - vm) * kLog2e);
      ce_combine(m, s, vm, vs);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    ce_combine(m, s, m2, s2);
  }
  if constexpr (NV > 0) __syncthreads();  // every warp has read sm[] (the row max) above
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    for (int w = 1; w < kCeThreads / 32; ++w) ce_combine(M, S, sm[w], ss[w]);
    const float lse = M + logf(S);
    s_lse = lse;
    const int y = p.labels[t];
    float loss = 0.f;
    if (y >= 0 && y < p.V) loss = lse - __bfloat162float(row[y]);
    p.loss_rows[t] = loss;
  }
  __syncthreads();
  const float lse = s_lse;
  const int y = p.labels[t];
  const bool valid = y >= 0 && y < p.V;

  // pass 2: dz = grad_scale * (softmax - onehot), bf16
  if (p.dlogits) {
    bf16* drow = p.dlogits + (size_t)t * p.ld_d;
    const float g = valid ? p.grad_scale : 0.f;
    // g * exp(z - lse) = 2^(z log2e - (lse log2e - log2 g)): one FFMA + one MUFU per logit
    const float off = valid && g > 0.f ? lse * kLog2e - log2f(g) : INFINITY;
    const int iy = valid ? y >> 3 : -1;  // the one vector holding the label
    auto emit = [&](int i, const uint4& u) {
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
      float e[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        e[2 * k] = ex2_ftz(fmaf(__uint_as_float(w[k] << 16), kLog2e, -off));
        e[2 * k + 1] = ex2_ftz(fmaf(__uint_as_float(w[k] & 0xffff0000u), kLog2e, -off));
      }
      if (i == iy) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == (y & 7)) e[k] -= g;
      }
      *reinterpret_cast<uint4*>(drow + 8 * i) =
          make_uint4(pack_bf16x2(e[0], e[1]), pack_bf16x2(e[2], e[3]), pack_bf16x2(e[4], e[5]),
                     pack_bf16x2(e[6], e[7]));
    };
    if constexpr (NV > 0) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const int i = threadIdx.x + j * kCeThreads;
        if (i < nvec) emit(i, keep[j]);
      }
    }
    for (int i0 = threadIdx.x; NV == 0 && i0 < nvec; i0 += kCeThreads * kCeUnroll) {
      uint4 u[kCeUnroll];
#pragma unroll
      for (int j = 0; j < kCeUnroll; ++j) {
        const int i = i0 + j * kCeThreads;
        u[j] = i < nvec ? ld_global_nc_v4(row + 8 * i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < kCeUnroll; ++j) {
        const int i = i0 + j * kCeThreads;
        if (i >= nvec) break;
        emit(i, u[j]);
      }
    }
  }

  // batch mean: the last CTA to arrive sums the per-row losses in row order
  if (p.loss_mean) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(p.counter, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && warp == 0) {
      __threadfence();
      float acc = 0.f;
      int cnt = 0;
      for (int i = lane; i < p.T; i += 32) {
        const int yi = p.labels[i];
        if (yi >= 0 && yi < p.V) {
          acc += __ldcg(p.loss_rows + i);
          ++cnt;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      }
      if (lane == 0) {
        *p.loss_mean = cnt ? acc / (float)cnt : 0.f;
        *p.counter = 0;
      }
    }
  }
}

}  // namespace collm
