// flash_tc.cuh — K9 forward on tcgen05/TMEM: causal attention of the packed sequences with the
// two matmuls on the 5th-generation tensor cores.
//
//   S = Q K^T   : tcgen05.mma M = 128 query rows x N = 128 keys x K = 128 dims (8 MMAs), Q and K
//                 K-major SWIZZLE_128B tiles loaded by TMA, S in TMEM (double-buffered);
//   softmax     : 4 warps, one query row per thread (tcgen05.ld of the row's 128 scores), base-2
//                 online softmax with a LAZY rescale (the running max is only moved when a tile's
//                 max exceeds it by more than 8 in log2 units: P <= 2^8, no overflow), P written as
//                 bf16 into a K-major swizzled shared tile;
//   O += P V    : tcgen05.mma M = 128 x N = 128 dims x K = 128 keys (8 MMAs), A = P from shared
//                 memory, B = V MN-major (V's [key][dim] rows as TMA loads them), O in TMEM for
//                 the whole key loop; a rescale multiplies the row of O in TMEM (ld / st).
// Same contract as flash_fwd_kernel (flash_attn.cuh): packed 128-row tiles of the batch (keys from
// the first row's sequence start to the tile's last row, masked same-sequence + causal), head dim
// 128, GQA, out bf16 and the base-2 LSE for the backward.  Deterministic (fixed MMA order).
//
// Roles (384 threads, 1 CTA/SM): warp 0 TMA producer (Q once, then K/V tiles through a 2-stage
// ring), warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-11 softmax + output (two threads per
// query row, one per 64-column half).  S and P are
// double-buffered, so a tile's softmax overlaps the next tile's Q K^T and the previous tile's P V.
#pragma once
#include "common.cuh"
#include "flash_attn.cuh"

namespace collm {

constexpr int kFtcRows = 128;
constexpr uint32_t kFtcTile = 128 * 128 * 2;  // 32 KB: [2 halves of 64 dims or keys][128][128 B]
constexpr int kFtcStages = 2;

struct FlashTcSmem {
  static constexpr uint32_t kQ = 0;
  static constexpr uint32_t kKV = kFtcTile;                       // [stage] K tile, V tile
  static constexpr uint32_t kP = kKV + kFtcStages * 2 * kFtcTile;  // [2] P tiles
  static constexpr uint32_t kBar = kP + 2 * kFtcTile;
  static constexpr uint32_t kTotal = kBar + 256 + 2 * 128 * 4 + 1024;  // barriers, pair exchange, align
};

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// mbarrier wait that names the barrier when it times out (a deadlock is a bug: trap after ~10 s)
__device__ __forceinline__ void ftc_wait(uint64_t* bar, uint32_t parity, int tag, int j) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  const unsigned long long t0 = clock64();
  while (!mbar_try_wait(a, parity)) {
    if (clock64() - t0 > COLLM_MBAR_TIMEOUT_CYCLES) {
      printf("collm: flash_tc barrier %d timeout at tile %d (block %d,%d thread %d)\n", tag, j,
             blockIdx.x, blockIdx.y, threadIdx.x);
      __trap();
    }
  }
}

struct FlashTcMaps {
  CUtensorMap q, k, v;  // 2-D maps, boxes of [64 columns x 128 rows], SWIZZLE_128B
};

__global__ void __launch_bounds__(384, 1)
    flash_fwd_tc_kernel(const __grid_constant__ FlashTcMaps maps, const FlashParams p) {
  using L = FlashTcSmem;
  extern __shared__ uint8_t fraw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bar;                      // Q loaded
  uint64_t* k_full = bar + 1;                  // [2] K tile of stage s loaded
  uint64_t* k_empty = bar + 3;                 // [2] Q K^T of stage s done (K free)
  uint64_t* s_full = bar + 5;                  // [2] S tile in TMEM buffer b
  uint64_t* s_free = bar + 7;                  // [2] softmax done reading S buffer b
  uint64_t* p_full = bar + 9;                  // [2] P tile b written
  uint64_t* pv_done = bar + 11;                // [2] O += P V from P tile b completed (V free)
  uint64_t* v_full = bar + 13;                 // [2] V tile of stage s loaded
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int h = blockIdx.y;
  const int q0 = (gridDim.x - 1 - blockIdx.x) * kFtcRows;  // late (long) query tiles first
  if (q0 >= p.T) return;
  const int hk = h / (p.n_heads / p.n_kv_heads);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = min(kFtcRows, p.T - q0);
  const int kstart = p.row_start[q0], kend = q0 + nq;
  const int n_kt = (kend - kstart + kFtcRows - 1) / kFtcRows;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&p_full[b], 8);
      mbar_init(&pv_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // columns [0,256): S buffers, [256,384): O

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
      mbar_arrive_expect_tx(q_full, kFtcTile);
      tma_load_2d(smem + L::kQ, &maps.q, q_full, h * kFaD, q0);
      tma_load_2d(smem + L::kQ + kFtcTile / 2, &maps.q, q_full, h * kFaD + 64, q0);
      for (int j = 0; j < n_kt; ++j) {
        const int s = j & 1;
        uint8_t* kb = smem + L::kKV + s * 2 * kFtcTile;
        uint8_t* vb = kb + kFtcTile;
        const int k0 = kstart + j * kFtcRows;
        // K of tile j+2 streams in as soon as Q K^T of tile j is done; V waits for P V of tile j
        if (j >= 2) ftc_wait(&k_empty[s], ((j >> 1) - 1) & 1, 1, j);
        mbar_arrive_expect_tx(&k_full[s], kFtcTile);
        tma_load_2d(kb, &maps.k, &k_full[s], hk * kFaD, k0);
        tma_load_2d(kb + kFtcTile / 2, &maps.k, &k_full[s], hk * kFaD + 64, k0);
        if (j >= 2) ftc_wait(&pv_done[s], ((j >> 1) - 1) & 1, 10, j);
        mbar_arrive_expect_tx(&v_full[s], kFtcTile);
        tma_load_2d(vb, &maps.v, &v_full[s], hk * kFaD, k0);
        tma_load_2d(vb + kFtcTile / 2, &maps.v, &v_full[s], hk * kFaD + 64, k0);
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    const uint32_t idesc_s = umma_idesc_bf16(128, 128);
    const uint32_t idesc_o = umma_idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
    const uint32_t sq = smem_u32(smem + L::kQ), sp = smem_u32(smem + L::kP);
    ftc_wait(q_full, 0, 2, 0);
    auto issue_s = [&](int j) {
      const int s = j & 1;
      ftc_wait(&k_full[s], (j >> 1) & 1, 3, j);
      if (j >= 2) ftc_wait(&s_free[s], ((j >> 1) - 1) & 1, 4, j);
      tc_fence_after();
      const uint32_t sk = smem_u32(smem + L::kKV + s * 2 * kFtcTile);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * (kFtcTile / 2) + (kk & 3) * 32;
          umma_bf16(tmem + s * 128, umma_desc_kmajor(sq + off, 128), umma_desc_kmajor(sk + off, 128),
                    idesc_s, kk ? 1u : 0u);
        }
        umma_commit(&s_full[s]);
        umma_commit(&k_empty[s]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < n_kt; ++j) {
      if (j + 1 < n_kt) issue_s(j + 1);  // the next scores overlap this tile's softmax
      const int s = j & 1;
      ftc_wait(&p_full[s], (j >> 1) & 1, 5, j);
      ftc_wait(&v_full[s], (j >> 1) & 1, 11, j);
      tc_fence_after();
      const uint32_t sv = smem_u32(smem + L::kKV + s * 2 * kFtcTile + kFtcTile);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per MMA: P columns / V rows
          const uint32_t pa = sp + s * kFtcTile + (kk >> 2) * (kFtcTile / 2) + (kk & 3) * 32;
          const uint32_t vb = sv + kk * 16 * 128;
          umma_bf16(tmem + 256, umma_desc_kmajor(pa, 128), umma_desc_mnmajor(vb, kFtcTile / 2),
                    idesc_o, (j | kk) ? 1u : 0u);
        }
        umma_commit(&pv_done[s]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== softmax + output: 8 warps, two threads per query row ==========
    // warps 4-7 and 8-11 read the same TMEM lane quarter (warp % 4); the first group owns columns
    // 0-63 of its rows, the second 64-127.  The pair exchanges the tile max and, at the end, the
    // row sum through shared memory (named barrier per row group, 64 threads).
    const int ew = warp & 3, cw = (warp - 4) >> 2;
    const int r = ew * 32 + lane;
    const int qr = q0 + r;
    const bool row_ok = qr < p.T;
    const int qs = row_ok ? p.row_start[qr] : 0x7fffffff;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const uint32_t col0 = (uint32_t)cw * 64;
    uint8_t* ps0 = smem + L::kP;
    float* xchg = reinterpret_cast<float*>(smem + L::kBar + 256);  // [2 halves][128 rows]
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + ew) : "memory"); };
    const int qs_last = p.row_start[q0 + nq - 1];  // row starts are nondecreasing
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int s = j & 1;
      ftc_wait(&s_full[s], (j >> 1) & 1, 6, j);
      tc_fence_after();
      const int key0 = kstart + j * kFtcRows + (int)col0;
      uint32_t sr[2][32];
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) tmem_ld_32x32b_x32(tmem + lane_base + s * 128 + col0 + ch * 32, sr[ch]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[s]);
      // raw scores; the causal / sequence mask only on tiles some row of the CTA cannot fully see
      const bool interior = key0 + 63 <= q0 && key0 >= qs_last && nq == kFtcRows;
      float hmax = -INFINITY;
      if (interior) {
#pragma unroll
        for (int ch = 0; ch < 2; ++ch)
#pragma unroll
          for (int e = 0; e < 32; ++e) hmax = fmaxf(hmax, __uint_as_float(sr[ch][e]));
      } else {
#pragma unroll
        for (int ch = 0; ch < 2; ++ch)
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int key = key0 + ch * 32 + e;
            const bool ok = row_ok & (key <= qr) & (key >= qs);  // branch-free
            const float v = ok ? __uint_as_float(sr[ch][e]) : -INFINITY;
            sr[ch][e] = __float_as_uint(v);
            hmax = fmaxf(hmax, v);
          }
      }
      xchg[cw * 128 + r] = hmax;
      pair_sync();
      const float tmax = fmaxf(xchg[r], xchg[128 + r]) * p.scale_log2;  // scale_log2 > 0
      pair_sync();  // both read before the next tile overwrites
      // P tile s is free once P V of tile j-2 is done (double-buffered P)
      if (j >= 2) ftc_wait(&pv_done[s], ((j >> 1) - 1) & 1, 7, j);
      tc_fence_after();
      // lazy rescale (the reference max moves only on a large increase); tcgen05.ld / st are
      // warp-collective: the warp rescales together when any lane needs it (others by 1)
      const bool bump = tmax > m + 8.f;
      const bool scale_o = bump && j > 0 && m != -INFINITY;
      if (__any_sync(0xffffffffu, scale_o)) {
        ftc_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1, 9, j);
        tc_fence_after();
        const float corr = scale_o ? exp2f(m - tmax) : 1.f;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tmem + lane_base + 256 + col0 + ch * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tmem_st_32x32b_x32(tmem + lane_base + 256 + col0 + ch * 32, o);
        }
        tmem_wait_st();
        l *= corr;
      }
      if (bump) m = tmax;
      // P = exp2(s * scale - m) as bf16 into this half of the K-major swizzled P tile
      const float mneg = m == -INFINITY ? 0.f : -m, c = p.scale_log2;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          float pv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float v = __uint_as_float(sr[ch][q8 * 8 + e]);
            pv[e] = ex2_approx(fmaf(v, c, mneg));
            l += pv[e];
          }
          const int q = ch * 4 + q8;  // 16-byte piece within this half's 128-byte row
          *reinterpret_cast<uint4*>(ps0 + s * kFtcTile + cw * (kFtcTile / 2) + r * 128 + ((q ^ (r & 7)) << 4)) =
              make_uint4(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                         pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[s]);
    }
    ftc_wait(&pv_done[(n_kt - 1) & 1], ((n_kt - 1) >> 1) & 1, 8, n_kt);
    tc_fence_after();
    // row sum of the two halves, in a fixed order
    xchg[cw * 128 + r] = l;
    pair_sync();
    const float lt = xchg[r] + xchg[128 + r];
    const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tmem + lane_base + 256 + col0 + ch * 32, o);
      tmem_wait_ld();
      if (row_ok) {
        bf16* dst = p.out + (size_t)qr * p.ldo + h * kFaD + col0 + ch * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 8)
          *reinterpret_cast<uint4*>(dst + e) =
              make_uint4(pack_bf16x2(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv),
                         pack_bf16x2(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv),
                         pack_bf16x2(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv),
                         pack_bf16x2(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv));
      }
    }
    if (row_ok && cw == 0) p.lse[(size_t)h * p.stat_ld + qr] = m + log2f(lt);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

}  // namespace collm
