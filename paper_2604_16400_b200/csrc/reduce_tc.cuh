// reduce_tc.cuh — K5 on the tensor core: the LoRA weight-gradient reductions of reduce_adamw.cuh
// (C[p, q] = sum_t U[t, u_off + p] (V + V2)[t, v_off + q], fp32) as a persistent, warp-specialised
// TMA -> tcgen05.mma -> TMEM pipeline, with the same fused AdamW finalize.
//
// The reduction is HBM-bound (U = dY or X_tr is read once; V = H16 / dH is small and L2-resident),
// so the design is a stream: one CTA per SM walks its share of the units (unit = 128-column P tile
// x a contiguous range of 128-row T chunks) through a 3-stage ring of 64 KB stages (U 32 KB as two
// [128 t][64 p] SWIZZLE_128B boxes, V and V2 16 KB boxes [128 t][64 q]) without draining between
// units.  Both operands are t-major in HBM, i.e. MN-major for the MMA: A = U^T (M = 128 P rows,
// LBO = the 16 KB distance of the two 64-column boxes), B = V (N = Q rounded to 16), K = 16 t per
// instruction.  The accumulator (128 lanes x 64 fp32 columns) is double-buffered in TMEM, so the
// epilogue warps finalize unit i (split partials / AdamW / bf16 copies) while unit i+1 streams.
//
// Roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-7
// epilogue (thread = one P row of the tile).  T splits: parts of a tile write fp32 partials; the
// last to arrive sums them in part order (bitwise reproducible, no float atomics).
#pragma once
#include "common.cuh"
#include "reduce_adamw.cuh"

namespace collm {

constexpr int kRtcRows = 128;                // T rows per chunk (K of 8 MMAs)
constexpr int kRtcStages = 3;
constexpr uint32_t kRtcBox = 128 * 128;      // one [128 t][64 cols] bf16 box = 16 KB
constexpr uint32_t kRtcStage = 4 * kRtcBox;  // U (2 boxes) | V | V2
constexpr int kRtcMaxMaps = 40;

struct ReduceTcSmem {
  static constexpr uint32_t kRing = 0;
  static constexpr uint32_t kBar = kRtcStages * kRtcStage;
  static constexpr uint32_t kTotal = kBar + 256 + 1024;
};

struct ReduceTcMaps {
  CUtensorMap m[kRtcMaxMaps];  // 2-D bf16 views [T rows][ld cols], boxes of [64 cols x 128 rows]
};

struct ReduceTcParams {
  ReduceParams r;
  int8_t map_u[kReduceMaxInner], map_v[kReduceMaxInner], map_v2[kReduceMaxInner];  // -1: none
  int n_units;   // n_tiles * tsplit (tile-major)
  int per;       // T chunks per part
  int n_chunks;  // ceil(T / 128)
  int n_maps;
  int debug_no_mma;  // timing experiments only: stream the operands, skip the MMAs
};

struct RtcUnit {
  int tile, part, gi, p0, ch_lo, n_ch;
};

__device__ __forceinline__ RtcUnit rtc_unit(const ReduceTcParams& tp, int u) {
  RtcUnit x;
  x.tile = u / tp.r.tsplit;
  x.part = u - x.tile * tp.r.tsplit;
  x.gi = find_group(tp.r, x.tile);
  x.p0 = (x.tile - tp.r.groups[x.gi].tile_begin) * kReducePT;
  x.ch_lo = x.part * tp.per;
  x.n_ch = min(tp.per, tp.n_chunks - x.ch_lo);
  return x;
}

__global__ void __launch_bounds__(256, 1)
    lora_reduce_tc_kernel(const __grid_constant__ ReduceTcMaps maps,
                          const __grid_constant__ ReduceTcParams tp) {
  using L = ReduceTcSmem;
  const ReduceParams& p = tp.r;
  extern __shared__ uint8_t rraw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* full = bar;                // [3] stage loaded
  uint64_t* empty = bar + 3;           // [3] stage consumed by the MMAs
  uint64_t* acc_full = bar + 6;        // [2] accumulator b complete
  uint64_t* acc_empty = bar + 8;       // [2] accumulator b read out by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 10);
  volatile int* s_last = reinterpret_cast<volatile int*>(bar + 11);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<128, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // columns [0,64): accumulator 0, [64,128): accumulator 1

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      for (int i = 0; i < tp.n_maps; ++i) tma_prefetch_desc(&maps.m[i]);
      int it = 0;
      for (int u = blockIdx.x; u < tp.n_units; u += gridDim.x) {
        const RtcUnit x = rtc_unit(tp, u);
        const ReduceGroup& gr = p.groups[x.gi];
        const CUtensorMap* mu = &maps.m[tp.map_u[x.gi]];
        const CUtensorMap* mv = &maps.m[tp.map_v[x.gi]];
        const bool v2 = tp.map_v2[x.gi] >= 0;
        const CUtensorMap* mv2 = &maps.m[v2 ? tp.map_v2[x.gi] : 0];
        const uint32_t bytes = (v2 ? 4 : 3) * kRtcBox;
        for (int c = 0; c < x.n_ch; ++c, ++it) {
          const int s = it % kRtcStages;
          if (it >= kRtcStages) mbar_wait(&empty[s], ((it / kRtcStages) - 1) & 1);
          uint8_t* st = smem + L::kRing + s * kRtcStage;
          const int t0 = (x.ch_lo + c) * kRtcRows;
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_2d(st, mu, &full[s], gr.u_off + x.p0, t0);
          tma_load_2d(st + kRtcBox, mu, &full[s], gr.u_off + x.p0 + 64, t0);
          tma_load_2d(st + 2 * kRtcBox, mv, &full[s], gr.v_off, t0);
          if (v2) tma_load_2d(st + 3 * kRtcBox, mv2, &full[s], gr.v_off, t0);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    int it = 0, k = 0;
    for (int u = blockIdx.x; u < tp.n_units; u += gridDim.x, ++k) {
      const RtcUnit x = rtc_unit(tp, u);
      const ReduceGroup& gr = p.groups[x.gi];
      const bool v2 = tp.map_v2[x.gi] >= 0;
      const uint32_t n16 = (uint32_t)((gr.Q + 15) & ~15);
      // A = U^T and B = V both MN-major (transpose bits 15 / 16)
      const uint32_t idesc = umma_idesc_bf16(128, n16) | (1u << 15) | (1u << 16);
      const int acc = k & 1;
      if (k >= 2) mbar_wait(&acc_empty[acc], ((k >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * 64;
      for (int c = 0; c < x.n_ch; ++c, ++it) {
        const int s = it % kRtcStages;
        mbar_wait(&full[s], (it / kRtcStages) & 1);
        tc_fence_after();
        const uint32_t su = smem_u32(smem + L::kRing + s * kRtcStage);
        if (elect_one()) {
          if (!tp.debug_no_mma)
#pragma unroll
          for (int kk = 0; kk < kRtcRows / 16; ++kk) {
            const uint64_t a = umma_desc_mnmajor(su + kk * 2048, kRtcBox);
            umma_bf16(d, a, umma_desc_mnmajor(su + 2 * kRtcBox + kk * 2048, kRtcBox), idesc,
                      (c | kk) ? 1u : 0u);
            if (v2) umma_bf16(d, a, umma_desc_mnmajor(su + 3 * kRtcBox + kk * 2048, kRtcBox), idesc, 1u);
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(&acc_full[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== epilogue: thread = one P row =====================
    const int ew = warp & 3, r = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const bool adam = p.mode == kModeAdamW, store = p.mode == kModeStoreGrad;
    const bool read_grad = store ? (p.accum_in != 0) : (adam && p.accum_in);
    float lr = 0.f, beta1 = 0.f, beta2 = 0.f, eps = 0.f, wd = 0.f, bc1 = 1.f, bc2 = 1.f;
    if (adam) {
      lr = __ldg(p.opt + 0); beta1 = __ldg(p.opt + 1); beta2 = __ldg(p.opt + 2);
      eps = __ldg(p.opt + 3); wd = __ldg(p.opt + 4); bc1 = __ldg(p.opt + 5); bc2 = __ldg(p.opt + 6);
    }
    const float step_size = lr / bc1, inv_sqrt_bc2 = rsqrtf(bc2);
    auto epi_sync = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    int k = 0;
    for (int u = blockIdx.x; u < tp.n_units; u += gridDim.x, ++k) {
      const RtcUnit x = rtc_unit(tp, u);
      const ReduceGroup& gr = p.groups[x.gi];
      const int acc = k & 1;
      mbar_wait(&acc_full[acc], (k >> 1) & 1);
      tc_fence_after();
      float c[64];
      {
        uint32_t v[2][32];
        tmem_ld_32x32b_x32(tmem + lane_base + acc * 64, v[0]);
        tmem_ld_32x32b_x32(tmem + lane_base + acc * 64 + 32, v[1]);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 64; ++e) c[e] = __uint_as_float(v[e >> 5][e & 31]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      const int Q = gr.Q;
      if (p.tsplit > 1) {
        float* mine = p.partials + ((size_t)(x.part * p.n_tiles + x.tile) * kReducePT + r) * 64;
#pragma unroll
        for (int q4 = 0; q4 < 16; ++q4)
          if (q4 * 4 < Q)
            __stcg(reinterpret_cast<float4*>(mine + q4 * 4),
                   make_float4(c[q4 * 4], c[q4 * 4 + 1], c[q4 * 4 + 2], c[q4 * 4 + 3]));
        epi_sync();  // all partial rows stored before the release below
        if (threadIdx.x == 128) {
          __threadfence();
          const int prev = atomicAdd(p.counters + x.tile, 1);
          const int last = prev == p.tsplit - 1;
          if (last) p.counters[x.tile] = 0;
          *s_last = last;
          if (last) __threadfence();  // acquire side of the arrival counter
        }
        epi_sync();
        const int last = *s_last;
        epi_sync();  // everyone read the flag before the next unit may rewrite it
        if (!last) continue;
        // sum the parts in part order; each pass issues all 16 vector loads of one part
        const float* base = p.partials + ((size_t)x.tile * kReducePT + r) * 64;
        const size_t part_stride = (size_t)p.n_tiles * kReducePT * 64;
#pragma unroll
        for (int e = 0; e < 64; ++e) c[e] = 0.f;
        for (int t = 0; t < p.tsplit; ++t) {
          float4 o[16];
#pragma unroll
          for (int q4 = 0; q4 < 16; ++q4)
            if (q4 * 4 < Q) o[q4] = __ldcg(reinterpret_cast<const float4*>(base + t * part_stride + q4 * 4));
#pragma unroll
          for (int q4 = 0; q4 < 16; ++q4)
            if (q4 * 4 < Q) {
              c[q4 * 4] += o[q4].x; c[q4 * 4 + 1] += o[q4].y;
              c[q4 * 4 + 2] += o[q4].z; c[q4 * 4 + 3] += o[q4].w;
            }
        }
      }
      // finalize this thread's row (same element math as finalize_tile), 4 vectors per batch
      // with every load of a batch issued before any is used
      if (x.p0 + r >= gr.P) continue;
      const size_t row = (size_t)(gr.c_row_off + x.p0 + r) * gr.ldc + gr.c_col_off;
      const bool trans = gr.out_trans && !store;
#pragma unroll
      for (int qb = 0; qb < 16; qb += 4) {
        if (qb * 4 >= Q) break;
        float4 gv[4], mv[4], vv[4], wv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q4 = qb + j;
          if (q4 * 4 >= Q) continue;
          const size_t idx = row + q4 * 4;
          if (read_grad) gv[j] = *reinterpret_cast<const float4*>(gr.grad + idx);
          if (adam) {
            mv[j] = *reinterpret_cast<const float4*>(gr.m + idx);
            vv[j] = *reinterpret_cast<const float4*>(gr.v + idx);
            wv[j] = *reinterpret_cast<const float4*>(gr.master + idx);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q4 = qb + j;
          if (q4 * 4 >= Q) continue;
          const size_t idx = row + q4 * 4;
          float g[4] = {c[q4 * 4] * p.grad_scale, c[q4 * 4 + 1] * p.grad_scale,
                        c[q4 * 4 + 2] * p.grad_scale, c[q4 * 4 + 3] * p.grad_scale};
          if (read_grad) { g[0] += gv[j].x; g[1] += gv[j].y; g[2] += gv[j].z; g[3] += gv[j].w; }
          if (store) {
            *reinterpret_cast<float4*>(gr.grad + idx) = make_float4(g[0], g[1], g[2], g[3]);
            continue;
          }
          float m[4] = {mv[j].x, mv[j].y, mv[j].z, mv[j].w};
          float v[4] = {vv[j].x, vv[j].y, vv[j].z, vv[j].w};
          float w[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
          bf16 wb[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            w[e] -= lr * wd * w[e];
            m[e] = beta1 * m[e] + (1.f - beta1) * g[e];
            v[e] = beta2 * v[e] + (1.f - beta2) * g[e] * g[e];
            w[e] -= step_size * (m[e] / (sqrtf(v[e]) * inv_sqrt_bc2 + eps));
            wb[e] = __float2bfloat16_rn(w[e]);
          }
          *reinterpret_cast<float4*>(gr.m + idx) = make_float4(m[0], m[1], m[2], m[3]);
          *reinterpret_cast<float4*>(gr.v + idx) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(gr.master + idx) = make_float4(w[0], w[1], w[2], w[3]);
          if (gr.out_same) {
            __nv_bfloat162 lo = __halves2bfloat162(wb[0], wb[1]), hi = __halves2bfloat162(wb[2], wb[3]);
            *reinterpret_cast<uint2*>(gr.out_same + idx) =
                make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
          }
          if (trans) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              gr.out_trans[(size_t)(gr.t_row_off + q4 * 4 + e) * gr.ld_trans + gr.t_col_off + x.p0 + r] = wb[e];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<128, 1>(tmem);
  }
}

}  // namespace collm
