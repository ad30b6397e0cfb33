// shrink.cuh — K1: segmented-gather LoRA shrink (SGMV), HBM-bound.
//
//   H[t, rank_off + j] = scale[a(t)] * sum_{k in [k_lo,k_hi)} X[t, k] * Amat_{a(t)}[rank_off + j, k]
//
// Forward:  X = the mixed rows, Amat = the adapters' A matrices [R, K] (q|k|v stacked along R).
// Backward: X = dY of the training rows, Amat = B_t^T [R, N] with one rank group per
//           sub-projection (its own N range) -> dH = s * dY . B_t.
//
// Work unit = one "row tile" (<= 16 consecutive rows of ONE adapter, planned on the host from the
// segment table) x one rank group x one K split.  Each warp streams X and the adapter's rank rows
// with 128-bit loads and feeds them straight into mma.sync m16n8k16: the reduction index k is
// permuted identically for both operands so that each lane's 16-byte vector IS its fragment
// (no shared-memory staging, no ldmatrix).  The 4 warps of a CTA interleave 32-wide K steps; their
// partial sums are reduced through shared memory, CTAs of the same tile reduce through a
// workspace in a fixed order (last-arriving CTA sums splits 0..ks-1), so results are bitwise
// deterministic.  CUDA-core FMAs cannot keep up with HBM here: X at 6.5 TB/s is 3.3 G rows.K/s
// and every element needs R >= 16 FMAs, i.e. > 50 TFMA/s — more than the FP32 pipe has.
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kShrinkMaxGroups = 8;
constexpr int kShrinkWarps = 4;

struct ShrinkGroup {
  int rank_off;  // first rank row (and H column) of the group
  int n_ranks;   // multiple of 8, <= 64
  int k_lo, k_hi;
};

struct ShrinkParams {
  const bf16* X;
  int ldx;
  const bf16* Amat;
  long long a_stride;  // elements between adapters
  int lda;             // elements between rank rows
  const int32_t* tiles;  // [n_tiles][3] = (row_start, n_rows, adapter)
  int n_tiles;
  const float* scale;  // [n_adapters]
  int n_groups;
  ShrinkGroup groups[kShrinkMaxGroups];
  int ksplit;
  // outputs (any may be null)
  float* H32;
  bf16* H16;
  int ldh;
  bf16* Hslots;  // [n_slots*128, ldh] — row (slot_of_row[t]*128 + t%128)
  const int32_t* slot_of_row;
  // workspace
  float* partials;    // [ksplit][n_groups][n_tiles][16][64]
  int32_t* counters;  // [n_groups][n_tiles], zero on entry, restored to zero on exit
};

template <int NT>  // n8 tiles of ranks per warp (n_ranks <= 8*NT)
__global__ void __launch_bounds__(kShrinkWarps * 32)
    lora_shrink_kernel(const ShrinkParams p) {
  __shared__ float red[kShrinkWarps][16][8 * NT + 1];
  __shared__ int s_last;

  const int tile = blockIdx.x, gi = blockIdx.y, ks = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int row_start = p.tiles[3 * tile + 0];
  const int n_rows = p.tiles[3 * tile + 1];
  const int adapter = p.tiles[3 * tile + 2];
  const ShrinkGroup grp = p.groups[gi];

  // K range of this split, in 32-element steps
  const int klen = grp.k_hi - grp.k_lo;
  const int steps_total = (klen + 31) / 32;
  const int steps_per = (steps_total + p.ksplit - 1) / p.ksplit;
  const int st_lo = ks * steps_per;
  const int st_hi = min(steps_total, st_lo + steps_per);

  const bool r0_ok = g < n_rows, r1_ok = (g + 8) < n_rows;
  const bf16* x0 = p.X + (size_t)(row_start + g) * p.ldx + grp.k_lo + 8 * c;
  const bf16* x1 = x0 + (size_t)8 * p.ldx;
  const bf16* a_base = p.Amat + (size_t)adapter * p.a_stride +
                       (size_t)(grp.rank_off + g) * p.lda + grp.k_lo + 8 * c;
  const int nt_used = grp.n_ranks >> 3;

  float d[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.f;

  const uint4 zero4 = make_uint4(0, 0, 0, 0);
  for (int st = st_lo + warp; st < st_hi; st += kShrinkWarps) {
    const int koff = st * 32;
    const bool k_ok = (koff + 8 * c + 8) <= klen;  // K multiple of 8 (checked on host)
    const uint4 xa = (r0_ok && k_ok) ? ld_global_nc_v4(x0 + koff) : zero4;
    const uint4 xb = (r1_ok && k_ok) ? ld_global_nc_v4(x1 + koff) : zero4;
    uint4 av[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j)
      av[j] = (j < nt_used && k_ok) ? __ldg(reinterpret_cast<const uint4*>(
                                          a_base + (size_t)(8 * j) * p.lda + koff))
                                    : zero4;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < nt_used) {
        mma_m16n8k16_bf16(d[j], xa.x, xb.x, xa.y, xb.y, av[j].x, av[j].y);
        mma_m16n8k16_bf16(d[j], xa.z, xb.z, xa.w, xb.w, av[j].z, av[j].w);
      }
    }
  }

  // warp partials -> smem: C fragment (row g / g+8, cols 2c, 2c+1 of each n8 tile)
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    red[warp][g][8 * j + 2 * c] = d[j][0];
    red[warp][g][8 * j + 2 * c + 1] = d[j][1];
    red[warp][g + 8][8 * j + 2 * c] = d[j][2];
    red[warp][g + 8][8 * j + 2 * c + 1] = d[j][3];
  }
  __syncthreads();

  const int n_out = 16 * grp.n_ranks;
  const float sc = p.scale[adapter];
  if (p.ksplit == 1) {
    for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
      const int i = e / grp.n_ranks, j = e % grp.n_ranks;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kShrinkWarps; ++w) v += red[w][i][j];
      if (i < n_rows) {
        const int t = row_start + i, col = grp.rank_off + j;
        v *= sc;
        if (p.H32) p.H32[(size_t)t * p.ldh + col] = v;
        if (p.H16) p.H16[(size_t)t * p.ldh + col] = __float2bfloat16_rn(v);
        if (p.Hslots)
          p.Hslots[((size_t)p.slot_of_row[t] * 128 + (t & 127)) * p.ldh + col] =
              __float2bfloat16_rn(v);
      }
    }
    return;
  }

  // split-K: publish this CTA's partial, the last CTA of the (group, tile) reduces in order
  float* my_part = p.partials + (((size_t)ks * p.n_groups + gi) * p.n_tiles + tile) * 16 * 64;
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
    const int i = e / grp.n_ranks, j = e % grp.n_ranks;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kShrinkWarps; ++w) v += red[w][i][j];
    my_part[i * 64 + j] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* ctr = p.counters + gi * p.n_tiles + tile;
    const int prev = atomicAdd(ctr, 1);
    s_last = (prev == p.ksplit - 1);
    if (s_last) *ctr = 0;  // restore for the next launch / graph replay
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int e = threadIdx.x; e < n_out; e += blockDim.x) {
    const int i = e / grp.n_ranks, j = e % grp.n_ranks;
    float v = 0.f;
    for (int s = 0; s < p.ksplit; ++s)
      v += __ldcg(p.partials + (((size_t)s * p.n_groups + gi) * p.n_tiles + tile) * 16 * 64 +
                  i * 64 + j);
    if (i < n_rows) {
      const int t = row_start + i, col = grp.rank_off + j;
      v *= sc;
      if (p.H32) p.H32[(size_t)t * p.ldh + col] = v;
      if (p.H16) p.H16[(size_t)t * p.ldh + col] = __float2bfloat16_rn(v);
      if (p.Hslots)
        p.Hslots[((size_t)p.slot_of_row[t] * 128 + (t & 127)) * p.ldh + col] =
            __float2bfloat16_rn(v);
    }
  }
}

}  // namespace collm
