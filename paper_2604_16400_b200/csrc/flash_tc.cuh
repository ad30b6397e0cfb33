// flash_tc.cuh — K9 forward on tcgen05/TMEM: causal attention of the packed sequences with the
// two matmuls on the 5th-generation tensor cores.
//
//   S = Q K^T   : tcgen05.mma M = 128 query rows x N = 128 keys x K = 128 dims (8 MMAs), Q and K
//                 K-major SWIZZLE_128B tiles loaded by TMA, S in TMEM (double-buffered);
//   softmax     : 8 warps, two threads per query row (64 of its 128 scores each, tcgen05.ld),
//                 base-2 online softmax with a LAZY rescale (the running max only moves when a
//                 tile's max exceeds it by more than 8 in log2 units: P <= 2^8, no overflow); P
//                 is packed as bf16 pairs back into TMEM over the S columns the thread read;
//   O += P V    : tcgen05.mma M = 128 x N = 128 dims x K = 128 keys (8 MMAs), A = P FROM TMEM,
//                 B = V MN-major (V's [key][dim] rows as TMA loads them), O in TMEM for the whole
//                 key loop; a rescale multiplies the row of O in TMEM (ld / st).
// Same contract as flash_fwd_kernel (flash_attn.cuh): packed 128-row tiles of the batch (keys from
// the first row's sequence start to the tile's last row, masked same-sequence + causal), head dim
// 128, GQA, out bf16 and the base-2 LSE for the backward.  Deterministic (fixed MMA order).
//
// Persistent (one CTA per SM walking (query tile, head) items): Q and O are double-buffered per
// item (smem / TMEM), so the next item's Q load, first Q K^T and the previous item's output
// epilogue all overlap the current item's work — short prefill sequences (2-3 key tiles per
// item) no longer pay a CTA launch, TMEM allocation and pipeline fill each.
//
// Roles (384 threads): warp 0 TMA producer (Q per item, K/V tiles through a 2-stage ring with
// separate K and V barriers), warp 1 MMA issuer, warp 2 TMEM allocator, warps 4-11 softmax +
// output.
#pragma once
#include "common.cuh"
#include "flash_attn.cuh"

namespace collm {

constexpr int kFtcRows = 128;
constexpr uint32_t kFtcTile = 128 * 128 * 2;  // 32 KB: [2 halves of 64 dims or keys][128][128 B]
constexpr int kFtcStages = 2;

struct FlashTcSmem {
  static constexpr uint32_t kQ = 0;                                // [2] Q tiles (per item)
  static constexpr uint32_t kKV = 2 * kFtcTile;                    // [stage] K tile, V tile
  static constexpr uint32_t kBar = kKV + kFtcStages * 2 * kFtcTile;
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

// One work item = (128-row query tile, head).  Items are walked persistently, tiles in reverse
// order (long sequences' late tiles first) with the heads fastest; every role derives the same
// sequence.
struct FtcItem {
  int h, q0, nq, kstart, n_kt;
};
__device__ __forceinline__ bool ftc_item(const FlashParams& p, int i, FtcItem& it) {
  const int n_qt = (p.T + kFtcRows - 1) / kFtcRows;
  if (i >= n_qt * p.n_heads) return false;
  it.h = i % p.n_heads;
  it.q0 = (n_qt - 1 - i / p.n_heads) * kFtcRows;
  it.nq = min(kFtcRows, p.T - it.q0);
  it.kstart = p.row_start[it.q0];
  it.n_kt = (it.q0 + it.nq - it.kstart + kFtcRows - 1) / kFtcRows;
  return true;
}

__global__ void __launch_bounds__(384, 1)
    flash_fwd_tc_kernel(const __grid_constant__ FlashTcMaps maps, const FlashParams p) {
  using L = FlashTcSmem;
  extern __shared__ uint8_t fraw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bar;        // [2] Q of item k in buffer k & 1
  uint64_t* q_empty = bar + 2;   // [2] the item's last Q K^T done (Q buffer free)
  uint64_t* k_full = bar + 4;    // [2] K tile of stage s loaded
  uint64_t* k_empty = bar + 6;   // [2] Q K^T of stage s done (K free)
  uint64_t* v_full = bar + 8;    // [2] V tile of stage s loaded
  uint64_t* s_full = bar + 10;   // [2] S tile in TMEM buffer b
  uint64_t* s_free = bar + 12;   // [2] softmax done reading S buffer b
  uint64_t* p_full = bar + 14;   // [2] P (packed bf16, in S buffer b) written
  uint64_t* pv_done = bar + 16;  // [2] O += P V of the tile in buffer b completed (V free)
  uint64_t* o_full = bar + 18;   // [2] the item's O (TMEM buffer k & 1) complete
  uint64_t* o_empty = bar + 20;  // [2] O buffer read out by the softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 22);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, G_heads = p.n_heads / p.n_kv_heads;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
      mbar_init(&k_full[b], 1);
      mbar_init(&k_empty[b], 1);
      mbar_init(&v_full[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 8);
      mbar_init(&p_full[b], 8);
      mbar_init(&pv_done[b], 1);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // [0,256): S buffers (P packed in place), [256,512): O buffers

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
      FtcItem it;
      int g = 0;
      for (int k = 0; ftc_item(p, blockIdx.x + k * G, it); ++k) {
        const int qb = k & 1, hk = it.h / G_heads;
        if (k >= 2) ftc_wait(&q_empty[qb], ((k >> 1) - 1) & 1, 0, k);
        mbar_arrive_expect_tx(&q_full[qb], kFtcTile);
        tma_load_2d(smem + L::kQ + qb * kFtcTile, &maps.q, &q_full[qb], it.h * kFaD, it.q0);
        tma_load_2d(smem + L::kQ + qb * kFtcTile + kFtcTile / 2, &maps.q, &q_full[qb], it.h * kFaD + 64, it.q0);
        for (int j = 0; j < it.n_kt; ++j, ++g) {
          const int s = g & 1;
          uint8_t* kb = smem + L::kKV + s * 2 * kFtcTile;
          uint8_t* vb = kb + kFtcTile;
          const int k0 = it.kstart + j * kFtcRows;
          // K of tile g+2 streams in as soon as Q K^T of tile g is done; V after P V of tile g
          if (g >= 2) ftc_wait(&k_empty[s], ((g >> 1) - 1) & 1, 1, g);
          mbar_arrive_expect_tx(&k_full[s], kFtcTile);
          tma_load_2d(kb, &maps.k, &k_full[s], hk * kFaD, k0);
          tma_load_2d(kb + kFtcTile / 2, &maps.k, &k_full[s], hk * kFaD + 64, k0);
          if (g >= 2) ftc_wait(&pv_done[s], ((g >> 1) - 1) & 1, 10, g);
          mbar_arrive_expect_tx(&v_full[s], kFtcTile);
          tma_load_2d(vb, &maps.v, &v_full[s], hk * kFaD, k0);
          tma_load_2d(vb + kFtcTile / 2, &maps.v, &v_full[s], hk * kFaD + 64, k0);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    const uint32_t idesc_s = umma_idesc_bf16(128, 128);
    const uint32_t idesc_o = umma_idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
    // S = Q K^T of item k's tile j (global tile g); the last one of an item frees its Q buffer
    auto issue_s = [&](int k, const FtcItem& it, int j, int g) {
      const int s = g & 1, qb = k & 1;
      if (j == 0) ftc_wait(&q_full[qb], (k >> 1) & 1, 2, k);
      ftc_wait(&k_full[s], (g >> 1) & 1, 3, g);
      if (g >= 2) ftc_wait(&s_free[s], ((g >> 1) - 1) & 1, 4, g);
      tc_fence_after();
      const uint32_t sq = smem_u32(smem + L::kQ + qb * kFtcTile);
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
        if (j == it.n_kt - 1) umma_commit(&q_empty[qb]);
      }
      __syncwarp();
    };
    FtcItem it, nx;
    if (ftc_item(p, blockIdx.x, it)) {
      issue_s(0, it, 0, 0);
      int g = 0;
      for (int k = 0;; ++k) {
        const bool has_next = ftc_item(p, blockIdx.x + (k + 1) * G, nx);
        const int ob = k & 1;
        for (int j = 0; j < it.n_kt; ++j, ++g) {
          // the next scores (this item's next tile, or the next item's first) overlap this
          // tile's softmax
          if (j + 1 < it.n_kt) issue_s(k, it, j + 1, g + 1);
          else if (has_next) issue_s(k + 1, nx, 0, g + 1);
          const int s = g & 1;
          ftc_wait(&p_full[s], (g >> 1) & 1, 5, g);
          ftc_wait(&v_full[s], (g >> 1) & 1, 11, g);
          if (j == 0 && k >= 2) ftc_wait(&o_empty[ob], ((k >> 1) - 1) & 1, 12, k);
          tc_fence_after();
          const uint32_t sv = smem_u32(smem + L::kKV + s * 2 * kFtcTile + kFtcTile);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {  // 16 keys per MMA: P (TMEM) columns / V rows
              const uint32_t pa = tmem + s * 128 + (kk >> 2) * 64 + (kk & 3) * 8;
              umma_bf16_ta(tmem + 256 + ob * 128, pa, umma_desc_mnmajor(sv + kk * 16 * 128, kFtcTile / 2),
                           idesc_o, (j | kk) ? 1u : 0u);
            }
            umma_commit(&pv_done[s]);
            if (j == it.n_kt - 1) umma_commit(&o_full[ob]);
          }
          __syncwarp();
        }
        if (!has_next) break;
        it = nx;
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax + output: 8 warps, two threads per query row ==========
    // warps 4-7 and 8-11 read the same TMEM lane quarter (warp % 4); the first group owns columns
    // 0-63 of its rows, the second 64-127.  The pair exchanges the tile max and, at the end, the
    // row sum through shared memory (named barrier per row group, 64 threads).
    const int ew = warp & 3, cw = (warp - 4) >> 2;
    const int r = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const uint32_t col0 = (uint32_t)cw * 64;
    float* xchg = reinterpret_cast<float*>(smem + L::kBar + 256);  // [2 halves][128 rows]
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + ew) : "memory"); };
    const float c = p.scale_log2;
    FtcItem it;
    int g = 0;
    for (int k = 0; ftc_item(p, blockIdx.x + k * G, it); ++k) {
      const int ob = k & 1;
      const uint32_t o_col = 256 + ob * 128 + col0;
      const int qr = it.q0 + r;
      const bool row_ok = qr < p.T;
      const int qs = row_ok ? p.row_start[qr] : 0x7fffffff;
      const int qs_last = p.row_start[it.q0 + it.nq - 1];  // row starts are nondecreasing
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < it.n_kt; ++j, ++g) {
        const int s = g & 1;
        ftc_wait(&s_full[s], (g >> 1) & 1, 6, g);
        tc_fence_after();
        const int key0 = it.kstart + j * kFtcRows + (int)col0;
        uint32_t sr[2][32];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) tmem_ld_32x32b_x32(tmem + lane_base + s * 128 + col0 + ch * 32, sr[ch]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[s]);
        // raw scores; the causal / sequence mask only on tiles some row of the CTA cannot see
        const bool interior = key0 + 63 <= it.q0 && key0 >= qs_last && it.nq == kFtcRows;
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
        const float tmax = fmaxf(xchg[r], xchg[128 + r]) * c;  // scale_log2 > 0
        pair_sync();  // both read before the next tile overwrites
        // lazy rescale (the reference max moves only on a large increase); tcgen05.ld / st are
        // warp-collective: the warp rescales together when any lane needs it (others by 1)
        const bool bump = tmax > m + 8.f;
        const bool scale_o = bump && j > 0 && m != -INFINITY;
        if (__any_sync(0xffffffffu, scale_o)) {
          ftc_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 9, g);
          tc_fence_after();
          const float corr = scale_o ? exp2f(m - tmax) : 1.f;
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tmem + lane_base + o_col + ch * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tmem + lane_base + o_col + ch * 32, o);
          }
          tmem_wait_st();
          l *= corr;
        }
        if (bump) m = tmax;
        // P = exp2(s * scale - m), packed bf16 pairs into the first 32 of the 64 S columns this
        // thread read (the P V that read the previous P in this buffer completed before S did)
        const float mneg = m == -INFINITY ? 0.f : -m;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float p0 = ex2_approx(fmaf(__uint_as_float(sr[ch][e]), c, mneg));
            const float p1 = ex2_approx(fmaf(__uint_as_float(sr[ch][e + 1]), c, mneg));
            l += p0 + p1;
            pk[e / 2] = pack_bf16x2(p0, p1);
          }
          tmem_st_32x32b_x16(tmem + lane_base + s * 128 + col0 + ch * 16, pk);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[s]);
      }
      ftc_wait(&o_full[ob], (k >> 1) & 1, 8, k);
      tc_fence_after();
      // row sum of the two halves, in a fixed order
      xchg[cw * 128 + r] = l;
      pair_sync();
      const float lt = xchg[r] + xchg[128 + r];
      pair_sync();  // both read before the next item's first tile overwrites
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tmem + lane_base + o_col + ch * 32, o);
        tmem_wait_ld();
        if (row_ok) {
          bf16* dst = p.out + (size_t)qr * p.ldo + it.h * kFaD + col0 + ch * 32;
#pragma unroll
          for (int e = 0; e < 32; e += 8)
            *reinterpret_cast<uint4*>(dst + e) =
                make_uint4(pack_bf16x2(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv),
                           pack_bf16x2(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv),
                           pack_bf16x2(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv),
                           pack_bf16x2(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ob]);
      if (row_ok && cw == 0) p.lse[(size_t)it.h * p.stat_ld + qr] = m + log2f(lt);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

}  // namespace collm
