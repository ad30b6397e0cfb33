// shrink_tc.cuh — K1 on reserved SMs: the LoRA shrink (SGMV) as a TMA-fed tcgen05 kernel that
// streams at ~150-190 GB/s per SM, so a handful of SMs (a "rank-space partition", whole TPCs)
// delivers the step's rank-space bandwidth while every other SM runs the base GEMM.
//
//   H[t, g.rank_off + j] = scale[a] * sum_{k in [g.k_lo, g.k_hi)} X[t, k] * Amat[a][g.rank_off + j, k]
//
// Same contract as lora_shrink_kernel (shrink.cuh): forward (X = mixed rows, Amat = adapters' A
// [R, K]) and backward dH (X = dY of the training rows, Amat = B_t^T [R, N], one rank group per
// sub-projection over its own N range); outputs H32 / H16 / H16lo / Hslots (the GEMM's slot blocks,
// own slot = value, other slots of the row's 256-row tile = 0).
//
// Why a second shrink: the register-fed kernel needs ~400 CTAs of latency hiding, i.e. the whole
// GPU, and its CTAs then hold SMs the GEMM it overlaps wants (measured: ~2 ms of a 7B step).  Here
// a work unit is a WINDOW of 128 consecutive rows and a run of up to 2^c consecutive adapter ids
// present in it (host-planned, LPT-assigned to the grid's W CTAs): per stage ONE 3-D TMA box of
// the window's X rows [kb k-blocks][128 rows][64] and ONE 4-D box of the adapters' rank rows
// [kb][2^c adapters][nr][64] (SWIZZLE_128B, k-block-major: per k-block exactly the K-major UMMA
// operand layouts), so a stage is two large copies (per-SM HBM bandwidth is set by copies in
// flight, tools/sm_bw.py).  One tcgen05.mma M = 128 rows x N = 2^c * nr x K = 16 serves all the
// window's rows of those adapters at once (block-diagonal: a row keeps its own adapter's nr
// columns) — each MMA costs ~25 ns nearly whatever its N, so stacking adapters in N cuts the MMA
// count ~2^c-fold versus one MMA per adapter (measured, profiles/r02_rank_partition.md).  TMEM
// accumulators double-buffered (2 x 256 columns); 4 epilogue warps scale, round and store while
// the next unit streams.
//
// Roles (256 threads, 1 CTA/SM, clusters of 2 so the grid holds whole TPCs):
//   warp 0: TMA producer;  warp 1: MMA issuer;  warp 2: TMEM allocator;  warps 4-7: epilogue.
// Deterministic: fixed item order per CTA, fixed-order accumulation in the tensor core, no atomics.
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kShrinkTcStages = 3;
constexpr uint32_t kShrinkTcStageBytes = 64 * 1024;
constexpr int kShrinkTcMaxGroups = 8;
constexpr int kShrinkTcClasses = 5;  // adapters stacked per MMA: 1, 2, 4, 8, 16
constexpr int kShrinkTcWindow = 128; // rows per work unit (the MMA's M)

struct ShrinkTcGroup {
  int rank_off;  // first rank row of Amat (and H column)
  int k_lo, k_hi;  // K range (multiples of 64)
};

struct ShrinkTcParams {
  int n_groups;
  int nr;  // ranks per adapter in a group (multiple of 16)
  ShrinkTcGroup groups[kShrinkTcMaxGroups];
  int kb[kShrinkTcClasses];  // k-blocks per stage of each class
  // work chunks: [n][8] = row0, n_rows (<= 128), a_lo (-1: base rows only), class c (adapters
  // a_lo .. a_lo + 2^c - 1 stacked as the MMA's N = 2^c * nr columns), S (the unit's K range is
  // split into S parts), part (this chunk's part), first chunk id of the unit, unit id
  const int32_t* items;
  float* partials;           // [chunk][group][128][256] fp32 (units with S > 1)
  int32_t* counters;         // [unit] arrivals (zero on entry, restored by the last part)
  const int32_t* cta_ptr;    // [gridDim.x + 1] unit range of each CTA
  const int32_t* row_adapter;  // [T] adapter of each row (-1: none)
  int a_single;              // A holds ONE adapter (B_t^T of the dH shrink): adapter coordinate 0
  const float* scale;        // [n_adapters]
  float* H32;
  bf16* H16;
  bf16* H16lo;
  int ldh;
  bf16* Hslots;
  const int32_t* slot_of_row;
  const int32_t* tile_slot_ptr;
};

// 32 lanes x 16 consecutive fp32 columns of TMEM per thread (32x32b shape, x16)
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

struct ShrinkTcSmem {
  static constexpr uint32_t kRing = kShrinkTcStages * kShrinkTcStageBytes;
  static constexpr uint32_t kBarOffset = kRing;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;  // + alignment pad
};

// X maps: [64 cols][rows][k-blocks] boxes of 128 rows x kb(c) k-blocks; A maps: [64][rank rows]
// [adapters][k-blocks] boxes of nr ranks x 2^c adapters x kb(c) k-blocks (class c)
struct ShrinkTcMaps {
  CUtensorMap x[kShrinkTcClasses];
  CUtensorMap a[kShrinkTcClasses];
};

__global__ void __launch_bounds__(256, 1)
    lora_shrink_tc_kernel(const __grid_constant__ ShrinkTcMaps maps, const ShrinkTcParams p) {
  using L = ShrinkTcSmem;
  // a GEMM launched programmatically dependent on this grid may start at once: its main loop runs
  // on the other SMs while this grid streams; its LoRA stages wait for our completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kShrinkTcStages;
  uint64_t* tfull = empty + kShrinkTcStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it_lo = p.cta_ptr[blockIdx.x], it_hi = p.cta_ptr[blockIdx.x + 1];
  const int nr = p.nr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kShrinkTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto nkb_of = [&](const ShrinkTcGroup& g) { return (g.k_hi - g.k_lo) / 64; };

  if (warp == 0) {
    // ===================== TMA producer: per stage one X box + one stacked-adapter A box ====
    if (elect_one()) {
      for (int c = 0; c < kShrinkTcClasses; ++c) {
        tma_prefetch_desc(&maps.x[c]);
        tma_prefetch_desc(&maps.a[c]);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int it = it_lo; it < it_hi; ++it) {
        const int row0 = p.items[8 * it], a_lo = p.items[8 * it + 2], cls = p.items[8 * it + 3];
        const int S = p.items[8 * it + 4], part = p.items[8 * it + 5];
        if (a_lo < 0) continue;
        const int kb = p.kb[cls], na = 1 << cls;
        const uint32_t bytes = (uint32_t)kb * (kShrinkTcWindow + na * nr) * 128;
        for (int gi = 0; gi < p.n_groups; ++gi) {
          const ShrinkTcGroup g = p.groups[gi];
          const int nkb = nkb_of(g);
          const int k_lo = nkb * part / S, k_hi = nkb * (part + 1) / S;
          for (int k0 = k_lo; k0 < k_hi; k0 += kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sb = smem + stage * kShrinkTcStageBytes;
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_3d(sb, &maps.x[cls], &full[stage], 0, row0, g.k_lo / 64 + k0);
            tma_load_4d(sb + (uint32_t)kb * kShrinkTcWindow * 128, &maps.a[cls], &full[stage], 0,
                        g.rank_off, p.a_single ? 0 : a_lo, g.k_lo / 64 + k0);
            if (++stage == kShrinkTcStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer: M = 128 rows, N = 2^c adapters x nr ranks =====
    const uint32_t sbase = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0, acc = 0, acc_phase = 0;
    for (int it = it_lo; it < it_hi; ++it) {
      const int a_lo = p.items[8 * it + 2], cls = p.items[8 * it + 3];
      const int S = p.items[8 * it + 4], part = p.items[8 * it + 5];
      if (a_lo < 0) continue;
      const int kb = p.kb[cls], ncols = (1 << cls) * nr;
      const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)ncols);
      for (int gi = 0; gi < p.n_groups; ++gi) {
        const int nkb = nkb_of(p.groups[gi]);
        const int k_lo = nkb * part / S, k_hi = nkb * (part + 1) / S;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * 256;
        for (int k0 = k_lo; k0 < k_hi; k0 += kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sx = sbase + stage * kShrinkTcStageBytes;
          const uint32_t sa = sx + (uint32_t)kb * kShrinkTcWindow * 128;
          const int n_here = min(kb, k_hi - k0);
          if (elect_one()) {
            // descriptors advanced by adding to the start-address field (addr >> 4)
            uint64_t dx = umma_desc_kmajor(sx, 128), da = umma_desc_kmajor(sa, 128);
            const uint64_t xstep = (uint64_t)(kShrinkTcWindow * 128) >> 4;
            const uint64_t astep = (uint64_t)(ncols * 128) >> 4;
            for (int j = 0; j < n_here; ++j) {
              umma_bf16(d, dx, da, idesc, (k0 != k_lo || j) ? 1u : 0u);
              umma_bf16(d, dx + 2, da + 2, idesc, 1u);
              umma_bf16(d, dx + 4, da + 4, idesc, 1u);
              umma_bf16(d, dx + 6, da + 6, idesc, 1u);
              dx += xstep;
              da += astep;
            }
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kShrinkTcStages) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> scale -> bf16 -> H16 / H16lo / H32 / Hslots =====
    // row i of the unit = TMEM lane i; its adapter's nr columns sit at (a - a_lo) * nr.  The
    // warp loads every 16-column chunk (tcgen05.ld addresses are warp-uniform) and each lane
    // keeps the chunks of its own adapter.
    const int ew = warp - 4;
    const int i = ew * 32 + lane;
    uint32_t acc = 0, acc_phase = 0;
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    for (int it = it_lo; it < it_hi; ++it) {
      const int row0 = p.items[8 * it], n_rows = p.items[8 * it + 1];
      const int a_lo = p.items[8 * it + 2], cls = p.items[8 * it + 3];
      const int S = p.items[8 * it + 4], part = p.items[8 * it + 5];
      const int chunk0 = p.items[8 * it + 6], unit = p.items[8 * it + 7];
      const int t = row0 + i;
      const int a = i < n_rows ? p.row_adapter[t] : -2;
      int mine = -1, sbeg = 0, send = 0;
      if (i < n_rows && p.Hslots) {
        const int m = t / kSlotTileM;
        mine = a >= 0 ? p.slot_of_row[t] : -1;
        sbeg = p.tile_slot_ptr[m];
        send = p.tile_slot_ptr[m + 1];
      }
      if (a_lo < 0) {  // base-only rows of the window: zeros in every slot of the row's tile
        if (a == -1)
          for (int gi = 0; gi < p.n_groups; ++gi)
            for (int c = 0; c < nr; c += 8)
              for (int s = sbeg; s < send; ++s)
                *reinterpret_cast<uint4*>(p.Hslots + ((size_t)s * kSlotTileM + (t % kSlotTileM)) * p.ldh +
                                          p.groups[gi].rank_off + c) = z4;
        continue;
      }
      const int na = 1 << cls, ncols = na * nr;
      const bool mine_unit = a >= a_lo && a < a_lo + na;
      const int cbase = mine_unit ? (a - a_lo) * nr : -100000;
      const float sc = mine_unit ? __ldg(p.scale + a) : 0.f;
      // the row's 16 values of rank columns [lc, lc+16) of group gi -> every output
      auto emit = [&](int gi, int lc, const float (&v)[16]) {
        const int col0 = p.groups[gi].rank_off;
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float v0 = v[2 * j] * sc, v1 = v[2 * j + 1] * sc;
          hw[j] = pack_bf16x2(v0, v1);
          const float f0 = __uint_as_float(hw[j] << 16), f1 = __uint_as_float(hw[j] & 0xffff0000u);
          lw[j] = pack_bf16x2(v0 - f0, v1 - f1);
        }
        const uint4 h0 = make_uint4(hw[0], hw[1], hw[2], hw[3]), h1 = make_uint4(hw[4], hw[5], hw[6], hw[7]);
        const size_t o = (size_t)t * p.ldh + col0 + lc;
        if (p.H16) {
          reinterpret_cast<uint4*>(p.H16 + o)[0] = h0;
          reinterpret_cast<uint4*>(p.H16 + o)[1] = h1;
        }
        if (p.H16lo) {
          reinterpret_cast<uint4*>(p.H16lo + o)[0] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
          reinterpret_cast<uint4*>(p.H16lo + o)[1] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
        }
        if (p.H32) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<float4*>(p.H32 + o)[j] =
                make_float4(v[4 * j] * sc, v[4 * j + 1] * sc, v[4 * j + 2] * sc, v[4 * j + 3] * sc);
        }
        if (p.Hslots) {
          for (int s = sbeg; s < send; ++s) {
            uint4* dst = reinterpret_cast<uint4*>(
                p.Hslots + ((size_t)s * kSlotTileM + (t % kSlotTileM)) * p.ldh + col0 + lc);
            dst[0] = s == mine ? h0 : z4;
            dst[1] = s == mine ? h1 : z4;
          }
        }
      };
      for (int gi = 0; gi < p.n_groups; ++gi) {
        const int nkb = (p.groups[gi].k_hi - p.groups[gi].k_lo) / 64;
        const bool has_k = nkb * (part + 1) / S > nkb * part / S;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        float* mypart = S > 1 ? p.partials + (((size_t)(chunk0 + part) * p.n_groups + gi) * 128 + i) * 256
                              : nullptr;
        for (int c = 0; c < ncols; c += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 256 + c, r);
          tmem_wait_ld();
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = has_k ? __uint_as_float(r[j]) : 0.f;
          if (S > 1) {  // this part's fp32 partial of the whole [128 x ncols] tile
#pragma unroll
            for (int j = 0; j < 4; ++j)
              __stcg(reinterpret_cast<float4*>(mypart + c) + j,
                     make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
            continue;
          }
          const int lc = c - cbase;  // this lane's rank offset of the chunk
          if (lc < 0 || lc >= nr) continue;
          emit(gi, lc, v);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (S > 1) {
        // the last part of the unit to arrive sums the S partials IN PART ORDER (deterministic)
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ew == 0 && lane == 0) {
          const int prev = atomicAdd(p.counters + unit, 1);
          s_last = prev == S - 1;
          if (s_last) p.counters[unit] = 0;
          __threadfence();
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (!s_last) continue;
        if (!mine_unit) continue;
        for (int gi = 0; gi < p.n_groups; ++gi) {
          for (int lc = 0; lc < nr; lc += 16) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            for (int q = 0; q < S; ++q) {
              const float4* src = reinterpret_cast<const float4*>(
                  p.partials + (((size_t)(chunk0 + q) * p.n_groups + gi) * 128 + i) * 256 + cbase + lc);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 f = __ldcg(src + j);
                v[4 * j] += f.x; v[4 * j + 1] += f.y; v[4 * j + 2] += f.z; v[4 * j + 3] += f.w;
              }
            }
            emit(gi, lc, v);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem_base);
  }
}

}  // namespace collm
