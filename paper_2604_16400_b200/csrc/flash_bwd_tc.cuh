// flash_bwd_tc.cuh — K9 backward on tcgen05/TMEM (the training sequences' attention gradients).
//
// Same contract and math as flash_bwd_dkdv_kernel / flash_bwd_dq_kernel (flash_attn.cuh): P is
// recomputed from the forward's base-2 LSE, delta = rowsum(dO o O) (flash_delta_kernel),
// dS = P (dP - delta), dV = P^T dO, dK = scale dS^T Q, dQ = scale dS K; every output element is
// owned by one CTA and accumulated in a fixed order (no atomics: bitwise repeatable).
//
// dK/dV kernel — CTA = 128 keys x one kv head; loops over the G query heads of the group and the
// 64-query steps from the first key to the last key's sequence end.  Per step:
//   S^T  = K Q^T    tcgen05.mma M = 128 keys x N = 64 queries x K = 128 dims (A = K, B = Q, K-major)
//   dP^T = V dO^T   same shape (A = V, B = dO)            -> TMEM, double-buffered (next step's
//                                                            MMAs overlap this step's elementwise)
//   8 elementwise warps (thread = 32 queries of one key row): P^T = exp2(S^T c - lse[q]) masked
//   (k <= q < row_end[k]), dS^T = P^T (dP^T - delta[q]), both packed bf16 back into TMEM in
//   place of the S^T / dP^T columns the thread read (tcgen05.st);
//   dV  += P^T dO   M = 128 keys x N = 128 dims x K = 64 queries, A = P^T FROM TMEM, B = dO
//                   (MN-major smem)
//   dK  += dS^T Q   same (A = dS^T from TMEM, B = Q)     -> TMEM accumulators for the whole loop.
// Q / dO steps stream through a 4-stage TMA ring; warp 3 stages the step's lse / delta.  (dQ:
// K / V steps through a 3-stage ring; dS from TMEM as the A operand of dQ += dS K; persistent.)
// Measured limits (13B, `COLLM_DEBUG_FB`): the Q / dO (dQ: K / V) re-reads per tile are L2-bound
// (~6 TB/s L2 -> SM), then the N = 64 MMAs (~34 ns each, smem operand bandwidth), then the
// elementwise work; a CTA pair multicasting the steps would halve the first.
//
// dQ kernel — CTA = 128 queries x one head; loops over 64-key steps from the first row's
// sequence start to the tile's last row:
//   S = Q K^T, dP = dO V^T (M = 128 queries x N = 64 keys), dS = P (dP - delta) per query row,
//   dQ += dS K (N = 128 dims, B = K MN-major) in TMEM.
//
// Roles (384 threads, 1 CTA/SM): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
// warp 3 statistics (dK/dV), warps 4-11 elementwise + epilogue (warps w and w+4 share a TMEM
// lane quarter and take the two 32-column halves of a step).
#pragma once
#include "common.cuh"
#include "flash_attn.cuh"
#include "flash_tc.cuh"

namespace collm {

constexpr uint32_t kFbBox64 = 64 * 128;    // [64 rows][64 dims] bf16 TMA box, 8 KB
constexpr uint32_t kFbBox128 = 128 * 128;  // [128 rows][64 dims] bf16 TMA box, 16 KB
constexpr int kFbQStages = 4;   // dK/dV: Q / dO step ring depth
constexpr int kFbKVStages = 3;  // dQ: K / V step ring depth
// timing experiments only (COLLM_DEBUG_FB): 1 = skip the MMAs (commit only), 2 = skip the
// elementwise math (barriers only)
__device__ int g_fb_debug;

struct FlashBwdTcMaps {
  // dK/dV kernel: Q / dO steps of 64 rows as ONE 3-D box each ([2 dim blocks][64 rows][64 dims],
  // k-block view), K / V tiles of 128 rows (2-D boxes)
  CUtensorMap q64, o64, k128, v128;
  // dQ kernel: Q / dO tiles of 128 rows (2-D), K / V steps of 64 rows (3-D, one box each)
  CUtensorMap q128, o128, k64, v64;
};

struct FbDkdvSmem {
  static constexpr uint32_t kK = 0;                   // 2 boxes [128 keys][64 dims]
  static constexpr uint32_t kV = 2 * kFbBox128;
  static constexpr uint32_t kQO = 4 * kFbBox128;      // [stages] Q (2 boxes), dO (2 boxes)
  static constexpr uint32_t kStat = kQO + kFbQStages * 4 * kFbBox64;  // [stages][lse | delta]
  static constexpr uint32_t kBar = kStat + kFbQStages * 128 * 4;
  static constexpr uint32_t kTotal = kBar + 256 + 1024;
};

struct FbDqSmem {
  static constexpr uint32_t kQO = 0;                   // [2 items] Q (2 boxes [128][64]), dO
  static constexpr uint32_t kKV = 2 * 4 * kFbBox128;   // [stages] K (2 boxes [64][64]), V
  static constexpr uint32_t kBar = kKV + kFbKVStages * 4 * kFbBox64;
  static constexpr uint32_t kTotal = kBar + 256 + 1024;
};

// this thread's 32 values as 16 packed bf16 pairs at TMEM row `taddr` (the first half of the
// 32 fp32 columns the thread read them from: no other thread touches those columns)
__device__ __forceinline__ void fb_store_tmem32(uint32_t taddr, const float* v) {
  uint32_t pk[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
  tmem_st_32x32b_x16(taddr, pk);
}

// write 64 fp32 accumulator columns [c0, c0+64) of TMEM row `lane_base` to bf16 dst, times mul
__device__ __forceinline__ void fb_store_acc64(uint32_t taddr, bf16* dst, float mul, bool ok) {
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {
    uint32_t o[32];
    tmem_ld_32x32b_x32(taddr + ch * 32, o);
    tmem_wait_ld();
    if (ok) {
#pragma unroll
      for (int e = 0; e < 32; e += 8)
        *reinterpret_cast<uint4*>(dst + ch * 32 + e) =
            make_uint4(pack_bf16x2(__uint_as_float(o[e]) * mul, __uint_as_float(o[e + 1]) * mul),
                       pack_bf16x2(__uint_as_float(o[e + 2]) * mul, __uint_as_float(o[e + 3]) * mul),
                       pack_bf16x2(__uint_as_float(o[e + 4]) * mul, __uint_as_float(o[e + 5]) * mul),
                       pack_bf16x2(__uint_as_float(o[e + 6]) * mul, __uint_as_float(o[e + 7]) * mul));
    }
  }
}

// ================================================================== dK / dV
__global__ void __launch_bounds__(384, 1)
    flash_bwd_dkdv_tc_kernel(const __grid_constant__ FlashBwdTcMaps maps, const FlashParams p) {
  using L = FbDkdvSmem;
  extern __shared__ uint8_t fbraw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fbraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* kv_full = bar;        // K, V tiles loaded
  uint64_t* s_full = bar + 1;     // [2] S^T, dP^T of the step in TMEM buffer b
  uint64_t* s_free = bar + 3;     // [2] elementwise warps done reading TMEM buffer b
  uint64_t* p_full = bar + 5;     // [2] P^T / dS^T tiles b written
  uint64_t* mm_done = bar + 7;    // [2] dV / dK MMAs of the step done (tiles b free)
  uint64_t* qd_full = bar + 9;    // [stages] Q / dO step + its lse / delta staged
  uint64_t* qd_empty = bar + 9 + kFbQStages;  // [stages] the step's MMAs done (stage free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 9 + 2 * kFbQStages);

  const int hk = blockIdx.y;
  const int k0 = blockIdx.x * 128;  // early keys (the most queries) first
  if (k0 >= p.T) return;
  const int G = p.n_heads / p.n_kv_heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = min(128, p.T - k0);
  const int qend = p.row_end[k0 + nk - 1];  // queries that see these keys: [k0, qend)
  const int per_head = (qend - k0 + 63) / 64, total = G * per_head;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int b = 0; b < kFbQStages; ++b) {
      mbar_init(&qd_full[b], 2);
      mbar_init(&qd_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 8);
      mbar_init(&p_full[b], 8);
      mbar_init(&mm_done[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S^T [0,128), dP^T [128,256), dV [256,384), dK [384,512)

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&maps.q64);
      tma_prefetch_desc(&maps.o64);
      mbar_arrive_expect_tx(kv_full, 4 * kFbBox128);
      tma_load_2d(smem + L::kK, &maps.k128, kv_full, hk * kFaD, k0);
      tma_load_2d(smem + L::kK + kFbBox128, &maps.k128, kv_full, hk * kFaD + 64, k0);
      tma_load_2d(smem + L::kV, &maps.v128, kv_full, hk * kFaD, k0);
      tma_load_2d(smem + L::kV + kFbBox128, &maps.v128, kv_full, hk * kFaD + 64, k0);
      for (int it = 0; it < total; ++it) {
        const int s = it % kFbQStages, u = it / kFbQStages;
        if (it >= kFbQStages) ftc_wait(&qd_empty[s], (u - 1) & 1, 21, it);
        const int hq = hk * G + it / per_head, qr = k0 + (it % per_head) * 64;
        uint8_t* st = smem + L::kQO + s * 4 * kFbBox64;
        mbar_arrive_expect_tx(&qd_full[s], 4 * kFbBox64);
        tma_load_3d(st, &maps.q64, &qd_full[s], 0, qr, hq * 2);
        tma_load_3d(st + 2 * kFbBox64, &maps.o64, &qd_full[s], 0, qr, hq * 2);
      }
    }
  } else if (warp == 3) {
    // ===================== statistics of each step: lse, delta of its 64 queries =====================
    // 8 steps' loads in flight at once (a load round trip per step would pace the whole kernel)
    constexpr int D = 8;
    for (int base = 0; base < total; base += D) {
      float v[D][4];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int it = base + d;
        if (it >= total) break;
        const int hq = hk * G + it / per_head, qr = k0 + (it % per_head) * 64;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int q = qr + h2 * 32 + lane;
          const bool ok = q < qend;
          v[d][h2] = ok ? p.lse[(size_t)hq * p.stat_ld + q] : 0.f;
          v[d][2 + h2] = ok ? p.delta[(size_t)hq * p.stat_ld + q] : 0.f;
        }
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int it = base + d;
        if (it >= total) break;
        const int s = it % kFbQStages, u = it / kFbQStages;
        if (it >= kFbQStages) ftc_wait(&qd_empty[s], (u - 1) & 1, 22, it);
        float* stat = reinterpret_cast<float*>(smem + L::kStat) + s * 128;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          stat[h2 * 32 + lane] = v[d][h2];
          stat[64 + h2 * 32 + lane] = v[d][2 + h2];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&qd_full[s]);
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    const uint32_t idesc_s = umma_idesc_bf16(128, 64);
    const uint32_t idesc_g = umma_idesc_bf16(128, 128) | (1u << 16);  // B (dO / Q) MN-major
    const uint32_t sk = smem_u32(smem + L::kK), sv = smem_u32(smem + L::kV);
    ftc_wait(kv_full, 0, 23, 0);
    auto issue_s = [&](int j) {
      const int s = j & 1, qs = j % kFbQStages;
      ftc_wait(&qd_full[qs], (j / kFbQStages) & 1, 24, j);
      if (j >= 2) ftc_wait(&s_free[s], ((j >> 1) - 1) & 1, 25, j);
      tc_fence_after();
      const uint32_t sq = smem_u32(smem + L::kQO + qs * 4 * kFbBox64), so = sq + 2 * kFbBox64;
      if (elect_one()) {
        if (!(g_fb_debug & 1))
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offa = (kk >> 2) * kFbBox128 + (kk & 3) * 32;
          const uint32_t offb = (kk >> 2) * kFbBox64 + (kk & 3) * 32;
          umma_bf16(tmem + s * 64, umma_desc_kmajor(sk + offa, 128), umma_desc_kmajor(sq + offb, 128),
                    idesc_s, kk ? 1u : 0u);
          umma_bf16(tmem + 128 + s * 64, umma_desc_kmajor(sv + offa, 128),
                    umma_desc_kmajor(so + offb, 128), idesc_s, kk ? 1u : 0u);
        }
        umma_commit(&s_full[s]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < total; ++j) {
      if (j + 1 < total) issue_s(j + 1);  // the next step's scores overlap this step's elementwise
      const int s = j & 1;
      ftc_wait(&p_full[s], (j >> 1) & 1, 26, j);
      tc_fence_after();
      const int qs = j % kFbQStages;
      const uint32_t sq = smem_u32(smem + L::kQO + qs * 4 * kFbBox64), so = sq + 2 * kFbBox64;
      if (elect_one()) {
        if (!(g_fb_debug & 1))
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // 16 queries per MMA
          const uint32_t acc = (j | kk) ? 1u : 0u;
          // P^T / dS^T packed in TMEM: queries 32h..32h+31 at columns 32h..32h+15 of buffer s
          const uint32_t col = s * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
          umma_bf16_ta(tmem + 256, tmem + col, umma_desc_mnmajor(so + kk * 2048, kFbBox64), idesc_g, acc);
          umma_bf16_ta(tmem + 384, tmem + 128 + col, umma_desc_mnmajor(sq + kk * 2048, kFbBox64),
                       idesc_g, acc);
        }
        umma_commit(&mm_done[s]);
        umma_commit(&qd_empty[qs]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== elementwise: thread = 32 queries of one key row =====================
    const int ew = warp & 3, half = (warp - 4) >> 2;
    const int r = ew * 32 + lane, key = k0 + r;
    const bool key_ok = key < p.T;
    const int kend = key_ok ? p.row_end[key] : 0;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const bool tile_full = nk == 128;
    const int kend0 = p.row_end[k0];  // the smallest sequence end of the tile's keys
    const float c = p.scale_log2;
    for (int j = 0; j < total; ++j) {
      const int s = j & 1;
      const int qr = k0 + (j % per_head) * 64;
      const int q0 = qr + half * 32;
      ftc_wait(&s_full[s], (j >> 1) & 1, 27, j);
      tc_fence_after();
      if (g_fb_debug & 2) {
        __syncwarp();
        if (lane == 0) { mbar_arrive(&s_free[s]); mbar_arrive(&p_full[s]); }
        continue;
      }
      uint32_t sr[32], dp[32];
      tmem_ld_32x32b_x32(tmem + lane_base + s * 64 + half * 32, sr);
      tmem_ld_32x32b_x32(tmem + lane_base + 128 + s * 64 + half * 32, dp);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[s]);
      const int qs = j % kFbQStages;
      ftc_wait(&qd_full[qs], (j / kFbQStages) & 1, 28, j);  // the step's lse / delta (warp 3)
      const float* stat = reinterpret_cast<const float*>(smem + L::kStat) + qs * 128 + half * 32;
      float pv[32], dsv[32];
      const bool interior = tile_full && q0 >= k0 + 127 && q0 + 31 < kend0;
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        const float4 ls = *reinterpret_cast<const float4*>(stat + e4 * 4);
        const float4 dl = *reinterpret_cast<const float4*>(stat + 64 + e4 * 4);
        const float lsv[4] = {ls.x, ls.y, ls.z, ls.w}, dlv[4] = {dl.x, dl.y, dl.z, dl.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = e4 * 4 + i, q = q0 + e;
          // branch-free mask (select before the exp: ex2(-inf) = 0)
          const bool ok = interior | (key_ok & (q >= key) & (q < kend));
          const float pe = ex2_approx(ok ? fmaf(__uint_as_float(sr[e]), c, -lsv[i]) : -INFINITY);
          pv[e] = pe;
          dsv[e] = pe * (__uint_as_float(dp[e]) - dlv[i]);
        }
      }
      // P^T and dS^T packed in place of the S^T / dP^T columns this thread read (the MMAs that
      // read the previous step's P^T in this buffer completed before S^T(j) did: in order)
      fb_store_tmem32(tmem + lane_base + s * 64 + half * 32, pv);
      fb_store_tmem32(tmem + lane_base + 128 + s * 64 + half * 32, dsv);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[s]);
    }
    ftc_wait(&mm_done[(total - 1) & 1], ((total - 1) >> 1) & 1, 30, total);
    tc_fence_after();
    fb_store_acc64(tmem + lane_base + 256 + half * 64,
                   p.dv + (size_t)key * p.lddv + hk * kFaD + half * 64, 1.f, key_ok);
    fb_store_acc64(tmem + lane_base + 384 + half * 64,
                   p.dk + (size_t)key * p.lddk + hk * kFaD + half * 64, p.scale, key_ok);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

// ================================================================== dQ
// Persistent: one CTA per SM walks (query tile, head) items (late tiles first, heads fastest);
// Q / dO double-buffered per item in smem, dQ double-buffered in TMEM, so the next item's loads
// and first scores overlap this item's last steps and the previous item's dQ write-out.
struct FbDqItem {
  int h, q0, nq, kstart, n_steps;
};
__device__ __forceinline__ bool fb_dq_item(const FlashParams& p, int i, FbDqItem& it) {
  const int n_qt = (p.T + 127) / 128;
  if (i >= n_qt * p.n_heads) return false;
  it.h = i % p.n_heads;
  it.q0 = (n_qt - 1 - i / p.n_heads) * 128;
  it.nq = min(128, p.T - it.q0);
  it.kstart = p.row_start[it.q0];
  it.n_steps = (it.q0 + it.nq - it.kstart + 63) / 64;
  return true;
}

__global__ void __launch_bounds__(384, 1)
    flash_bwd_dq_tc_kernel(const __grid_constant__ FlashBwdTcMaps maps, const FlashParams p) {
  using L = FbDqSmem;
  extern __shared__ uint8_t fbraw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fbraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bar;          // [2] Q, dO of item k in buffer k & 1
  uint64_t* q_empty = bar + 2;     // [2] the item's last S / dP MMAs done (buffer free)
  uint64_t* s_full = bar + 4;      // [2]
  uint64_t* s_free = bar + 6;      // [2]
  uint64_t* p_full = bar + 8;      // [2] dS (packed into the dP buffer) written
  uint64_t* dq_full = bar + 10;    // [2] the item's dQ (TMEM buffer k & 1) complete
  uint64_t* dq_empty = bar + 12;   // [2] dQ buffer read out
  uint64_t* kv_full = bar + 14;    // [stages] K / V step loaded
  uint64_t* kv_empty = bar + 14 + kFbKVStages;  // [stages] the step's MMAs done (stage free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14 + 2 * kFbKVStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, Gh = p.n_heads / p.n_kv_heads;

  if (threadIdx.x == 0) {
    for (int b = 0; b < kFbKVStages; ++b) {
      mbar_init(&kv_full[b], 1);
      mbar_init(&kv_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 8);
      mbar_init(&p_full[b], 8);
      mbar_init(&dq_full[b], 1);
      mbar_init(&dq_empty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512, 1>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S [0,128), dP / dS [128,256), dQ [256,512) (2 buffers)

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch_desc(&maps.k64);
      tma_prefetch_desc(&maps.v64);
      FbDqItem it;
      int g = 0;
      for (int k = 0; fb_dq_item(p, blockIdx.x + k * G, it); ++k) {
        const int qb = k & 1, hk = it.h / Gh;
        if (k >= 2) ftc_wait(&q_empty[qb], ((k >> 1) - 1) & 1, 40, k);
        uint8_t* qo = smem + L::kQO + qb * 4 * kFbBox128;
        mbar_arrive_expect_tx(&q_full[qb], 4 * kFbBox128);
        tma_load_2d(qo, &maps.q128, &q_full[qb], it.h * kFaD, it.q0);
        tma_load_2d(qo + kFbBox128, &maps.q128, &q_full[qb], it.h * kFaD + 64, it.q0);
        tma_load_2d(qo + 2 * kFbBox128, &maps.o128, &q_full[qb], it.h * kFaD, it.q0);
        tma_load_2d(qo + 3 * kFbBox128, &maps.o128, &q_full[qb], it.h * kFaD + 64, it.q0);
        for (int j = 0; j < it.n_steps; ++j, ++g) {
          const int s = g % kFbKVStages, u = g / kFbKVStages;
          if (g >= kFbKVStages) ftc_wait(&kv_empty[s], (u - 1) & 1, 41, g);
          const int kr = it.kstart + j * 64;
          uint8_t* st = smem + L::kKV + s * 4 * kFbBox64;
          mbar_arrive_expect_tx(&kv_full[s], 4 * kFbBox64);
          tma_load_3d(st, &maps.k64, &kv_full[s], 0, kr, hk * 2);
          tma_load_3d(st + 2 * kFbBox64, &maps.v64, &kv_full[s], 0, kr, hk * 2);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc_s = umma_idesc_bf16(128, 64);
    const uint32_t idesc_g = umma_idesc_bf16(128, 128) | (1u << 16);  // B (K) MN-major
    // S = Q K^T, dP = dO V^T of item k's step j (global step g)
    auto issue_s = [&](int k, const FbDqItem& it, int j, int g) {
      const int s = g & 1, ks = g % kFbKVStages, qb = k & 1;
      if (j == 0) ftc_wait(&q_full[qb], (k >> 1) & 1, 42, k);
      ftc_wait(&kv_full[ks], (g / kFbKVStages) & 1, 43, g);
      if (g >= 2) ftc_wait(&s_free[s], ((g >> 1) - 1) & 1, 44, g);
      tc_fence_after();
      const uint32_t sq = smem_u32(smem + L::kQO + qb * 4 * kFbBox128), so = sq + 2 * kFbBox128;
      const uint32_t sk = smem_u32(smem + L::kKV + ks * 4 * kFbBox64), sv = sk + 2 * kFbBox64;
      if (elect_one()) {
        if (!(g_fb_debug & 1))
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offa = (kk >> 2) * kFbBox128 + (kk & 3) * 32;
          const uint32_t offb = (kk >> 2) * kFbBox64 + (kk & 3) * 32;
          umma_bf16(tmem + s * 64, umma_desc_kmajor(sq + offa, 128), umma_desc_kmajor(sk + offb, 128),
                    idesc_s, kk ? 1u : 0u);
          umma_bf16(tmem + 128 + s * 64, umma_desc_kmajor(so + offa, 128),
                    umma_desc_kmajor(sv + offb, 128), idesc_s, kk ? 1u : 0u);
        }
        umma_commit(&s_full[s]);
        if (j == it.n_steps - 1) umma_commit(&q_empty[qb]);
      }
      __syncwarp();
    };
    FbDqItem it, nx;
    if (fb_dq_item(p, blockIdx.x, it)) {
      issue_s(0, it, 0, 0);
      int g = 0;
      for (int k = 0;; ++k) {
        const bool has_next = fb_dq_item(p, blockIdx.x + (k + 1) * G, nx);
        const int ob = k & 1;
        for (int j = 0; j < it.n_steps; ++j, ++g) {
          if (j + 1 < it.n_steps) issue_s(k, it, j + 1, g + 1);
          else if (has_next) issue_s(k + 1, nx, 0, g + 1);
          const int s = g & 1, ks = g % kFbKVStages;
          ftc_wait(&p_full[s], (g >> 1) & 1, 45, g);
          if (j == 0 && k >= 2) ftc_wait(&dq_empty[ob], ((k >> 1) - 1) & 1, 49, k);
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + L::kKV + ks * 4 * kFbBox64);
          if (elect_one()) {
            if (!(g_fb_debug & 1))
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // 16 keys per MMA; dS packed in TMEM (dP buffer s)
              umma_bf16_ta(tmem + 256 + ob * 128, tmem + 128 + s * 64 + (kk >> 1) * 32 + (kk & 1) * 8,
                           umma_desc_mnmajor(sk + kk * 2048, kFbBox64), idesc_g, (j | kk) ? 1u : 0u);
            umma_commit(&kv_empty[ks]);
            if (j == it.n_steps - 1) umma_commit(&dq_full[ob]);
          }
          __syncwarp();
        }
        if (!has_next) break;
        it = nx;
      }
    }
  } else if (warp >= 4) {
    // ===================== elementwise: thread = 32 keys of one query row =====================
    const int ew = warp & 3, half = (warp - 4) >> 2;
    const int r = ew * 32 + lane;
    const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
    const float c = p.scale_log2;
    FbDqItem it;
    int g = 0;
    for (int k = 0; fb_dq_item(p, blockIdx.x + k * G, it); ++k) {
      const int ob = k & 1;
      const int qr = it.q0 + r;
      const bool row_ok = qr < p.T;
      const int qs = row_ok ? p.row_start[qr] : 0x7fffffff;
      const float lse = row_ok ? p.lse[(size_t)it.h * p.stat_ld + qr] : 0.f;
      const float dl = row_ok ? p.delta[(size_t)it.h * p.stat_ld + qr] : 0.f;
      const int qs_last = p.row_start[it.q0 + it.nq - 1];
      for (int j = 0; j < it.n_steps; ++j, ++g) {
        const int s = g & 1;
        const int key0 = it.kstart + j * 64 + half * 32;
        ftc_wait(&s_full[s], (g >> 1) & 1, 46, g);
        tc_fence_after();
        if (g_fb_debug & 2) {
          __syncwarp();
          if (lane == 0) { mbar_arrive(&s_free[s]); mbar_arrive(&p_full[s]); }
          continue;
        }
        uint32_t sr[32], dp[32];
        tmem_ld_32x32b_x32(tmem + lane_base + s * 64 + half * 32, sr);
        tmem_ld_32x32b_x32(tmem + lane_base + 128 + s * 64 + half * 32, dp);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[s]);
        const bool interior = it.nq == 128 && key0 + 31 <= it.q0 && key0 >= qs_last;
        float dsv[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int key = key0 + e;
          const bool ok = interior | (row_ok & (key <= qr) & (key >= qs));  // branch-free
          const float pe = ex2_approx(ok ? fmaf(__uint_as_float(sr[e]), c, -lse) : -INFINITY);
          dsv[e] = pe * (__uint_as_float(dp[e]) - dl);
        }
        fb_store_tmem32(tmem + lane_base + 128 + s * 64 + half * 32, dsv);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[s]);
      }
      ftc_wait(&dq_full[ob], (k >> 1) & 1, 48, k);
      tc_fence_after();
      fb_store_acc64(tmem + lane_base + 256 + ob * 128 + half * 64,
                     p.dq + (size_t)qr * p.lddq + it.h * kFaD + half * 64, p.scale, row_ok);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_empty[ob]);
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
