// gemm_lora.cuh — K2/K3: persistent tcgen05/TMEM GEMM fed by TMA, with the multi-adapter LoRA
// expand folded into the same TMEM accumulator as extra K-steps ("tensor-core SGMV expand").
//
//   Y[M,N] = A[M,K] . B[N,K]^T  +  sum_{slots s of the M-tile}  Hs[s][128, r] . LB_{a(s)}[N, r]^T
//
// Forward (K2):  A = X (all mixed rows), B = W (frozen base, [N,K] = nn.Linear layout),
//                Hs[s] = the tile's rows of s_a*X.A_a^T with rows of other adapters zeroed (the
//                shrink kernel writes these "slot blocks"), LB = the adapters' B matrices [N, r].
// Backward (K3): A = dY (training rows), B = W^T (frozen, [K_in, N]), one slot per tile holding
//                s*dY.B_t, LB = A_t^T [K_in, R] — i.e. dX = dY.W + s*dH.A_t in one pass.
//
// Replaces the reference's latency stand-ins `perf.true_infer_latency` / `true_train_latency`
// (/root/reference/pkg/src/coserve/perf.py:62-89) with the real projection arithmetic.
//
// Roles (256 threads, 1 CTA/SM, persistent over tiles, m-fastest raster so W tiles are shared
// through L2 by the CTAs that run concurrently):
//   warp 0 lane 0 : TMA producer (ring of STAGES smem stages, full/empty mbarriers)
//   warp 1 lane 0 : tcgen05.mma issuer into a double-buffered TMEM accumulator (2 x BN columns)
//   warp 2        : TMEM allocator
//   warps 4..7    : epilogue — tcgen05.ld 32x32b -> bf16 -> st.global, overlapped with the next
//                   tile's main loop through the second accumulator buffer.
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kMaxSub = 4;

struct GemmLoraParams {
  int M, N, K;
  bf16* Y;
  int ldy;  // elements
  // ---- LoRA K-extension (tile_slot_ptr == nullptr -> plain GEMM)
  const int32_t* tile_slot_ptr;  // [num_m_tiles + 1] slot range of each 128-row tile
  const int32_t* slot_adapter;   // [n_slots] adapter id of each slot
  int lora_rc;                   // columns per LoRA chunk: 16 / 32 / 64 (one TMA box each)
  int lora_chunks;               // chunks per slot (= lora width / rc)
  int lb_rows_per_adapter;       // LB row coordinate = adapter * this + n0
  int n_sub;                     // sub-projections along N (fused q|k|v, gate|up); >= 1
  int sub_n_start[kMaxSub + 1];  // N boundaries of the sub-projections (multiples of BN)
  int sub_h_col[kMaxSub];        // first H column used by each sub-projection
  int num_m_tiles, num_n_tiles;
};

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;  // 16 KB
  static constexpr uint32_t kBBytes = BN * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kBarOffset = STAGES * kStageBytes;
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;  // barriers + alignment slack
  static constexpr uint32_t kTmemCols = 2 * BN;               // double-buffered fp32 accumulator
};

__device__ __forceinline__ int sub_of_n0(const GemmLoraParams& p, int n0) {
  int s = 0;
#pragma unroll
  for (int i = 1; i < kMaxSub; ++i)
    if (i < p.n_sub && n0 >= p.sub_n_start[i]) s = i;
  return s;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    gemm_lora_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmLB,
                     const GemmLoraParams p) {
  using L = GemmSmem<BN, STAGES>;
  constexpr uint32_t BM = kGemmBM, BK = kGemmBK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_lora = p.tile_slot_ptr != nullptr;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (has_lora) {
      tma_prefetch_desc(&tmH);
      tma_prefetch_desc(&tmLB);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.num_m_tiles * p.num_n_tiles;
  const int nk = (p.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    // ===================== TMA producer =====================
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % p.num_m_tiles, n_blk = tile / p.num_m_tiles;
      const int m0 = m_blk * BM, n0 = n_blk * BN;
      if (has_lora) {
        const int s_beg = p.tile_slot_ptr[m_blk], s_end = p.tile_slot_ptr[m_blk + 1];
        const int hcol = p.sub_h_col[sub_of_n0(p, n0)];
        const uint32_t rc = p.lora_rc;
        for (int s = s_beg; s < s_end; ++s) {
          const int lb_row = p.slot_adapter[s] * p.lb_rows_per_adapter + n0;
          for (int c = 0; c < p.lora_chunks; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStageBytes;
            mbar_arrive_expect_tx(&full[stage], (BM + BN) * rc * 2);
            tma_load_2d(sa, &tmH, &full[stage], hcol + c * rc, s * BM);
            tma_load_2d(sa + L::kABytes, &tmLB, &full[stage], c * rc, lb_row);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * L::kStageBytes;
        mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
        tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
        tma_load_2d(sa + L::kABytes, &tmB, &full[stage], kb * BK, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ===================== tcgen05.mma issuer =====================
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, acc_phase = 0;
    const uint32_t smem_base = smem_u32(smem);
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % p.num_m_tiles;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      uint32_t accumulate = 0;
      if (has_lora) {
        const int n_lora = (p.tile_slot_ptr[m_blk + 1] - p.tile_slot_ptr[m_blk]) * p.lora_chunks;
        const uint32_t row_bytes = p.lora_rc * 2;
        const uint32_t ksteps = p.lora_rc / 16;
        for (int i = 0; i < n_lora; ++i) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_base + stage * L::kStageBytes;
          for (uint32_t k = 0; k < ksteps; ++k) {
            umma_bf16(d_tmem, umma_desc_kmajor(sa + k * 32, row_bytes),
                      umma_desc_kmajor(sa + L::kABytes + k * 32, row_bytes), idesc, accumulate);
            accumulate = 1;
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_base + stage * L::kStageBytes;
#pragma unroll
        for (uint32_t k = 0; k < BK / 16; ++k) {
          umma_bf16(d_tmem, umma_desc_kmajor(sa + k * 32, 128),
                    umma_desc_kmajor(sa + L::kABytes + k * 32, 128), idesc, accumulate);
          accumulate = 1;
        }
        umma_commit(&empty[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      umma_commit(&tfull[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // TMEM lanes [32*ew, 32*ew+32)
    uint32_t acc = 0, acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int m_blk = tile % p.num_m_tiles, n_blk = tile / p.num_m_tiles;
      const int row = m_blk * BM + ew * 32 + lane;
      const int n0 = n_blk * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      bf16* yrow = p.Y + (size_t)row * p.ldy;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c, r);
        tmem_wait_ld();
        if (row < p.M) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int col = n0 + c + j * 8;
            if (col + 8 <= p.N) {
              st_global_v4(yrow + col,
                           pack_bf16x2(__uint_as_float(r[8 * j + 0]), __uint_as_float(r[8 * j + 1])),
                           pack_bf16x2(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3])),
                           pack_bf16x2(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5])),
                           pack_bf16x2(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7])));
            }
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

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}

}  // namespace collm
