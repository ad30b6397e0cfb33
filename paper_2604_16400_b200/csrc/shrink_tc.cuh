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
// a work item (<= 128 consecutive rows of ONE adapter, host-planned and LPT-assigned to the grid's
// W CTAs, tools/sm_bw.py) streams through a 3-stage ring of ~64 KB stages: one 3-D TMA box of X
// rows [kb k-blocks][nb rows][64] and one of the adapter's rank rows [kb][nr][64] per stage
// (SWIZZLE_128B, k-block-major — exactly the K-major UMMA operand layout per k-block), so each
// stage is two large copies (per-SM HBM bandwidth is set by copies in flight, not bytes).
// tcgen05.mma M = 128 rows x N = nr ranks x K = 16 accumulates the item in TMEM (double-buffered,
// 2 x 256 columns); 4 epilogue warps scale, round and store while the next item streams.  Rows of
// the 128-row MMA beyond the item (nb < 128) read whatever follows in shared memory and land in
// accumulator rows that are never stored.
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
constexpr int kShrinkTcClasses = 4;  // X box heights 16 / 32 / 64 / 128 rows

struct ShrinkTcGroup {
  int rank_off;  // first rank row of Amat (and H column)
  int k_lo, k_hi;  // K range (multiples of 64)
};

struct ShrinkTcParams {
  int n_groups;
  int nr;  // ranks per group (multiple of 16, <= 256): the MMA N
  ShrinkTcGroup groups[kShrinkTcMaxGroups];
  int nb[kShrinkTcClasses];  // X box rows of each item class
  int kb[kShrinkTcClasses];  // k-blocks per stage of each class
  const int32_t* items;      // [n_items][4] = row_start, n_rows (<= 128), adapter (-1: none), class
  const int32_t* cta_ptr;    // [gridDim.x + 1] item range of each CTA
  int a_rows_per_adapter;    // Amat row of (adapter a, rank j) = a * this + j
  const float* scale;        // [n_adapters]
  float* H32;
  bf16* H16;
  bf16* H16lo;
  int ldh;
  bf16* Hslots;
  const int32_t* slot_of_row;
  const int32_t* tile_slot_ptr;
  int debug_no_mma;  // timing experiments only: skip the MMAs (results undefined)
};

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 16 lanes x 16 consecutive fp32 columns of TMEM per thread (32x32b shape, x16)
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
  static constexpr uint32_t kSlack = 16 * 1024;  // a 128-row UMMA read past the last stage
  static constexpr uint32_t kBarOffset = kRing + kSlack;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;  // + alignment pad
};

__global__ void __launch_bounds__(256, 1)
    lora_shrink_tc_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
                          const __grid_constant__ CUtensorMap tmX2, const __grid_constant__ CUtensorMap tmX3,
                          const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                          const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmA3,
                          const ShrinkTcParams p) {
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
    // ===================== TMA producer =====================
    if (elect_one()) {
      const CUtensorMap* mx[4] = {&tmX0, &tmX1, &tmX2, &tmX3};
      const CUtensorMap* ma[4] = {&tmA0, &tmA1, &tmA2, &tmA3};
      for (int c = 0; c < kShrinkTcClasses; ++c) {
        tma_prefetch_desc(mx[c]);
        tma_prefetch_desc(ma[c]);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int it = it_lo; it < it_hi; ++it) {
        const int row0 = p.items[4 * it], adapter = p.items[4 * it + 2], cls = p.items[4 * it + 3];
        if (adapter < 0) continue;
        const int nb = p.nb[cls], kb = p.kb[cls];
        const uint32_t bytes = (uint32_t)kb * (nb + nr) * 128;
        for (int gi = 0; gi < p.n_groups; ++gi) {
          const ShrinkTcGroup g = p.groups[gi];
          const int nkb = nkb_of(g);
          const int arow = adapter * p.a_rows_per_adapter + g.rank_off;
          for (int k0 = 0; k0 < nkb; k0 += kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sb = smem + stage * kShrinkTcStageBytes;
            mbar_arrive_expect_tx(&full[stage], bytes);
            tma_load_3d(sb, mx[cls], &full[stage], 0, row0, g.k_lo / 64 + k0);
            tma_load_3d(sb + (uint32_t)kb * nb * 128, ma[cls], &full[stage], 0, arow, g.k_lo / 64 + k0);
            if (++stage == kShrinkTcStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    const uint32_t idesc = umma_idesc_bf16(128, (uint32_t)nr);
    const uint32_t sbase = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0, acc = 0, acc_phase = 0;
    for (int it = it_lo; it < it_hi; ++it) {
      const int adapter = p.items[4 * it + 2], cls = p.items[4 * it + 3];
      if (adapter < 0) continue;
      const int nb = p.nb[cls], kb = p.kb[cls];
      for (int gi = 0; gi < p.n_groups; ++gi) {
        const int nkb = nkb_of(p.groups[gi]);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * 256;
        for (int k0 = 0; k0 < nkb; k0 += kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sx = sbase + stage * kShrinkTcStageBytes;
          const uint32_t sa = sx + (uint32_t)kb * nb * 128;
          const int n_here = min(kb, nkb - k0);
          if (elect_one()) {
            // descriptors advanced by adding to the start-address field (addr >> 4): one 64-bit
            // add per UMMA instead of rebuilding them (the issue loop bounds small-N UMMAs)
            const uint64_t dx0 = umma_desc_kmajor(sx, 128), da0 = umma_desc_kmajor(sa, 128);
            const uint64_t xstep = (uint64_t)(nb * 128) >> 4, astep = (uint64_t)(nr * 128) >> 4;
            if (p.debug_no_mma != 1) {
              uint64_t dx = dx0, da = da0;
              for (int j = 0; j < n_here; ++j) {
                umma_bf16(d, dx, da, idesc, (k0 | j) ? 1u : 0u);
                umma_bf16(d, dx + 2, da + 2, idesc, 1u);
                umma_bf16(d, dx + 4, da + 4, idesc, 1u);
                umma_bf16(d, dx + 6, da + 6, idesc, 1u);
                dx += xstep;
                da += astep;
              }
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
    const int ew = warp - 4;
    const int i = ew * 32 + lane;  // accumulator row = item row
    uint32_t acc = 0, acc_phase = 0;
    const uint4 z4 = make_uint4(0, 0, 0, 0);
    for (int it = it_lo; it < it_hi; ++it) {
      const int row0 = p.items[4 * it], n_rows = p.items[4 * it + 1], adapter = p.items[4 * it + 2];
      const bool row_ok = i < n_rows;
      const int t = row0 + i;
      int mine = -1, sbeg = 0, send = 0;
      if (row_ok && p.Hslots) {
        const int m = t / kSlotTileM;
        mine = adapter >= 0 ? p.slot_of_row[t] : -1;
        sbeg = p.tile_slot_ptr[m];
        send = p.tile_slot_ptr[m + 1];
      }
      if (adapter < 0) {  // base-only rows: zeros in every slot of the row's tile
        if (row_ok)
          for (int gi = 0; gi < p.n_groups; ++gi)
            for (int c = 0; c < nr; c += 8)
              for (int s = sbeg; s < send; ++s)
                *reinterpret_cast<uint4*>(p.Hslots + ((size_t)s * kSlotTileM + (t % kSlotTileM)) * p.ldh +
                                          p.groups[gi].rank_off + c) = z4;
        continue;
      }
      const float sc = __ldg(p.scale + adapter);
      for (int gi = 0; gi < p.n_groups; ++gi) {
        const int col0 = p.groups[gi].rank_off;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        for (int c = 0; c < nr; c += 16) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * 256 + c, r);
          tmem_wait_ld();
          if (!row_ok) continue;
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]) * sc;
          uint4 hv[2], lv[2];
          uint32_t* hp = reinterpret_cast<uint32_t*>(hv);
          uint32_t* lp = reinterpret_cast<uint32_t*>(lv);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            hp[j] = *reinterpret_cast<const uint32_t*>(&h2);
            const float2 hf = __bfloat1622float2(h2);
            lp[j] = pack_bf16x2(v[2 * j] - hf.x, v[2 * j + 1] - hf.y);
          }
          const size_t o = (size_t)t * p.ldh + col0 + c;
          if (p.H16) {
            reinterpret_cast<uint4*>(p.H16 + o)[0] = hv[0];
            reinterpret_cast<uint4*>(p.H16 + o)[1] = hv[1];
          }
          if (p.H16lo) {
            reinterpret_cast<uint4*>(p.H16lo + o)[0] = lv[0];
            reinterpret_cast<uint4*>(p.H16lo + o)[1] = lv[1];
          }
          if (p.H32) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              reinterpret_cast<float4*>(p.H32 + o)[j] =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          if (p.Hslots) {
            for (int s = sbeg; s < send; ++s) {
              uint4* dst = reinterpret_cast<uint4*>(
                  p.Hslots + ((size_t)s * kSlotTileM + (t % kSlotTileM)) * p.ldh + col0 + c);
              dst[0] = s == mine ? hv[0] : z4;
              dst[1] = s == mine ? hv[1] : z4;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
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
