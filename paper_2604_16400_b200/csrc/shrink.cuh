// shrink.cuh — K1: segmented-gather LoRA shrink (SGMV), HBM-bound.
//
//   H[t, rank_off + j] = scale[a(t)] * sum_{k in [k_lo,k_hi)} X[t, k] * Amat_{a(t)}[rank_off + j, k]
//
// Forward:  X = the mixed rows, Amat = the adapters' A matrices [R, K] (q|k|v stacked along R).
// Backward: X = dY of the training rows, Amat = B_t^T [R, N] with one rank group per
//           sub-projection (its own N range) -> dH = s * dY . B_t.
//
// Work unit = one "row tile" (<= 16 consecutive rows of ONE adapter, planned on the host from the
// segment table) x one rank group.  A thread-block cluster of C CTAs (C = 1..8, chosen so the
// grid fills the SMs) covers the unit's K range, each CTA a contiguous 1/C of it with its 8 warps
// interleaving 32-wide K steps.  Each warp streams X and the adapter's rank rows with 128-bit
// loads straight into mma.sync m16n8k16: the reduction index k is permuted identically for both
// operands so each lane's 16-byte vector IS its fragment (no shared-memory staging, no ldmatrix).
// Loads for UNR K steps are issued before any MMA, so every lane keeps (2 + NT) * UNR 16-byte
// requests in flight.  Warp partials reduce through shared memory, the C CTA partials through
// distributed shared memory (rank 0 sums ranks 0..C-1 in order): deterministic, no atomics, no
// global workspace.  CUDA-core FMAs cannot keep up with HBM here: X at 6.5 TB/s is 3.3 G
// elements/s and every element needs R >= 16 FMAs, i.e. > 50 TFMA/s.
//
// The Hslots output (the GEMM's LoRA slot blocks) is written completely by this kernel: each row
// writes its value into its own adapter's slot and zeros into the other slots of its 128-row tile
// (rows of base-only segments, adapter -1, write zeros everywhere), so no memset is needed.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace collm {

constexpr int kShrinkMaxGroups = 8;
constexpr int kShrinkWarps = 8;

struct ShrinkGroup {
  int rank_off;  // first rank row (and H column) of the group
  int n_ranks;   // multiple of 8, <= 64
  int k_lo, k_hi;
};

struct ShrinkParams {
  const bf16* X;
  int ldx;
  const bf16* Amat;
  long long a_stride;    // elements between adapters
  int lda;               // elements between rank rows
  const int32_t* tiles;  // [n_tiles][3] = (row_start, n_rows, adapter or -1)
  int n_tiles;
  const float* scale;  // [n_adapters]
  int n_groups;
  ShrinkGroup groups[kShrinkMaxGroups];
  // outputs (any may be null)
  float* H32;
  bf16* H16;
  bf16* H16lo;  // residual v - bf16(v) (with H16: a bf16 hi+lo pair carrying ~16 mantissa bits)
  int ldh;
  bf16* Hslots;  // [n_slots*256, ldh] — row (slot*256 + t%256)
  const int32_t* slot_of_row;
  const int32_t* tile_slot_ptr;  // slot range of each 256-row slot tile (for the zero fill)
  int csize;                     // CTAs per cluster splitting the K range (1, 2, 4, 8)
  // completion signal for a consumer running concurrently on another stream (optional):
  // signal[0] = arrival counter (0 on entry, restored), signal[1] <- *gen once all is written
  int32_t* signal;
  const int32_t* gen;
  unsigned long long* dbg;  // debug only: [CTA][2] globaltimer at start / end
};

// Every CTA arrives once its outputs are written; the last one publishes *gen in signal[1]
// (release, gpu scope) for the GEMM waiting on it (wait_lora_flag in gemm_lora.cuh).
__device__ __forceinline__ void shrink_signal_done(const ShrinkParams& p) {
  if (p.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.dbg[2 * (blockIdx.y * gridDim.x + blockIdx.x) + 1] = t;
  }
  if (!p.signal) return;
  __syncthreads();  // this CTA's stores happen-before thread 0's cumulative fence
  if (threadIdx.x == 0) {
    __threadfence();
    const int total = (int)(gridDim.x * gridDim.y);
    if (atomicAdd(p.signal, 1) == total - 1) {
      __threadfence();
      p.signal[0] = 0;
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p.signal + 1), "r"(*p.gen) : "memory");
    }
  }
}

// Per-row output bookkeeping staged in shared memory once per CTA (no dependent global loads in
// the store loop): own slot and the slot range of the row's 128-row tile.
struct RowSlots {
  int mine[16], beg[16], end[16];
};

__device__ __forceinline__ void load_row_slots(const ShrinkParams& p, RowSlots& rs, int row_start,
                                               int n_rows, bool has_adapter) {
  if (threadIdx.x < 16) {
    const int i = threadIdx.x;
    int mine = -1, beg = 0, end = 0;
    if (i < n_rows && p.Hslots) {
      const int t = row_start + i, m = t / kSlotTileM;
      mine = has_adapter ? p.slot_of_row[t] : -1;
      beg = p.tile_slot_ptr[m];
      end = p.tile_slot_ptr[m + 1];
    }
    rs.mine[i] = mine;
    rs.beg[i] = beg;
    rs.end[i] = end;
  }
}

__device__ __forceinline__ void shrink_store(const ShrinkParams& p, const RowSlots& rs, int i,
                                             int t, int col, float v, bool has_adapter) {
  const bf16 vb = __float2bfloat16_rn(v);
  if (has_adapter) {
    if (p.H32) p.H32[(size_t)t * p.ldh + col] = v;
    if (p.H16) p.H16[(size_t)t * p.ldh + col] = vb;
    if (p.H16lo) p.H16lo[(size_t)t * p.ldh + col] = __float2bfloat16_rn(v - __bfloat162float(vb));
  }
  if (p.Hslots) {
    const bf16 zero = __float2bfloat16_rn(0.f);
    for (int s = rs.beg[i]; s < rs.end[i]; ++s)
      p.Hslots[((size_t)s * kSlotTileM + (t % kSlotTileM)) * p.ldh + col] = (s == rs.mine[i]) ? vb : zero;
  }
}

template <int NT, int UNR>  // NT: n8 rank tiles per warp (n_ranks <= 8*NT); UNR: K steps in flight
__global__ void __launch_bounds__(kShrinkWarps * 32, 3)
    lora_shrink_kernel(const ShrinkParams p) {
  namespace cg = cooperative_groups;
  // a GEMM launched programmatically dependent on this shrink (same stream, pdl_mode 2) may
  // start right away: its main loop overlaps this grid, its LoRA stages wait for our completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.dbg[2 * (blockIdx.y * gridDim.x + blockIdx.x)] = t;
  }
  constexpr int W2 = kShrinkWarps / 2;
  constexpr int LD = 8 * NT + 1;
  __shared__ float red[W2][16][LD];
  __shared__ RowSlots rs;

  const int C = p.csize;
  const int tile = blockIdx.x / C, rank = blockIdx.x % C, gi = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int row_start = p.tiles[3 * tile + 0];
  const int n_rows = p.tiles[3 * tile + 1];
  const int adapter = p.tiles[3 * tile + 2];
  const ShrinkGroup grp = p.groups[gi];
  const int n_out = 16 * grp.n_ranks;
  const bool has_adapter = adapter >= 0;
  if (rank == 0) load_row_slots(p, rs, row_start, n_rows, has_adapter);

  float d[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.f;

  if (has_adapter) {
    const int klen = grp.k_hi - grp.k_lo;
    const int steps = (klen + 31) / 32;
    const int st_lo = (int)((long long)steps * rank / C);
    const int st_hi = (int)((long long)steps * (rank + 1) / C);
    const bool r0_ok = g < n_rows, r1_ok = (g + 8) < n_rows;
    const bf16* x0 = p.X + (size_t)(row_start + g) * p.ldx + grp.k_lo + 8 * c;
    const bf16* x1 = x0 + (size_t)8 * p.ldx;
    const bf16* a_base = p.Amat + (size_t)adapter * p.a_stride +
                         (size_t)(grp.rank_off + g) * p.lda + grp.k_lo + 8 * c;
    const int nt_used = grp.n_ranks >> 3;
    const uint4 zero4 = make_uint4(0, 0, 0, 0);
    for (int st0 = st_lo + warp; st0 < st_hi; st0 += kShrinkWarps * UNR) {
      uint4 xa[UNR], xb[UNR], av[UNR][NT];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int st = st0 + u * kShrinkWarps;
        const int koff = st * 32;
        const bool k_ok = st < st_hi && (koff + 8 * c + 8) <= klen;  // K multiple of 8 (host)
        xa[u] = (r0_ok && k_ok) ? ld_global_nc_v4(x0 + koff) : zero4;
        xb[u] = (r1_ok && k_ok) ? ld_global_nc_v4(x1 + koff) : zero4;
#pragma unroll
        for (int j = 0; j < NT; ++j)
          av[u][j] = (j < nt_used && k_ok)
                         ? __ldg(reinterpret_cast<const uint4*>(a_base + (size_t)(8 * j) * p.lda + koff))
                         : zero4;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          mma_m16n8k16_bf16(d[j], xa[u].x, xb[u].x, xa[u].y, xb[u].y, av[u][j].x, av[u][j].y);
          mma_m16n8k16_bf16(d[j], xa[u].z, xb[u].z, xa[u].w, xb[u].w, av[u][j].z, av[u][j].w);
        }
      }
    }
  }

  // fixed-order reduction: warps (two levels through smem), then CTAs of the cluster (DSMEM)
  if (warp >= W2) {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      red[warp - W2][g][8 * j + 2 * c] = d[j][0];
      red[warp - W2][g][8 * j + 2 * c + 1] = d[j][1];
      red[warp - W2][g + 8][8 * j + 2 * c] = d[j][2];
      red[warp - W2][g + 8][8 * j + 2 * c + 1] = d[j][3];
    }
  }
  __syncthreads();
  if (warp < W2) {
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      red[warp][g][8 * j + 2 * c] += d[j][0];
      red[warp][g][8 * j + 2 * c + 1] += d[j][1];
      red[warp][g + 8][8 * j + 2 * c] += d[j][2];
      red[warp][g + 8][8 * j + 2 * c + 1] += d[j][3];
    }
  }
  __syncthreads();
  // red[0] <- sum of the W2 partials (in order)
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
    const int i = e / grp.n_ranks, j = e % grp.n_ranks;
    float v = red[0][i][j];
#pragma unroll
    for (int w = 1; w < W2; ++w) v += red[w][i][j];
    red[0][i][j] = v;
  }
  if (C > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // every CTA's red[0] complete and visible cluster-wide
    if (rank == 0) {
      const float sc = has_adapter ? p.scale[adapter] : 0.f;
      for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
        const int i = e / grp.n_ranks, j = e % grp.n_ranks;
        float v = red[0][i][j];
        for (int r = 1; r < C; ++r) v += cl.map_shared_rank(&red[0][i][j], r)[0];
        if (i < n_rows) shrink_store(p, rs, i, row_start + i, grp.rank_off + j, v * sc, has_adapter);
      }
    }
    cl.sync();  // peers keep their shared memory alive until rank 0 has read it
    shrink_signal_done(p);
    return;
  }
  __syncthreads();
  const float sc = has_adapter ? p.scale[adapter] : 0.f;
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
    const int i = e / grp.n_ranks, j = e % grp.n_ranks;
    if (i < n_rows)
      shrink_store(p, rs, i, row_start + i, grp.rank_off + j, red[0][i][j] * sc, has_adapter);
  }
  shrink_signal_done(p);
}

}  // namespace collm
