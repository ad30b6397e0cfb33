// expand_rows.cuh — the LoRA expand of many-adapter row tiles, one row at a time (BGMV-style).
//
//   Y[t, n] += sum_j H16[t, hcol(n) + j] * B_{a(t)}[n, j]        (t in the flagged 256-row tiles)
//
// The GEMM folds a tile's expand into its accumulator as (slots x r / 64) extra k-stages
// (gemm_lora.cuh).  A 256-row tile whose rows carry many DIFFERENT adapters (multi-tenant decode:
// up to 256 slots) would multiply the GEMM's MMA work by up to 1 + 256 r / K while only 1/slots of
// those MMAs are useful; such tiles skip the fused expand (GemmLoraParams.tile_skip) and get this
// HBM-bound pass instead, which reads each row's adapter's B rows once (the unavoidable bytes:
// distinct adapters x N x r x 2) and Y once more (coalesced reads of the contiguous B rows, fixed
// shuffle reduction order: deterministic).
#pragma once
#include "common.cuh"

namespace collm {

struct ExpandRowsParams {
  bf16* Y;
  int ldy, N;
  const bf16* H;  // H16 [T, ldh]: s_a * X . A_a^T (the scale is already in)
  int ldh;
  const bf16* B;  // [n_adapters, N, r_pad]
  int r_pad;
  const int32_t* row_adapter;  // [T]
  const int32_t* tiles;        // flagged 256-row slot tiles
  int n_tiles, T;
  int n_sub;
  int sub_n_start[5];
  int sub_h_col[4];
};

__global__ void __launch_bounds__(256) lora_expand_rows_kernel(const ExpandRowsParams p) {
  // one warp = one row t x 128 output columns n0..n0+127 (sub-projection boundaries are
  // multiples of 128, so the chunk has one H slice).  The adapter's B rows n0..n0+127 are
  // 128 x r_pad bf16 CONTIGUOUS: lanes read consecutive 16-byte pieces (8 ranks of one B row
  // each, cpr = r_pad/8 lanes per row), multiply by the matching 8 H values, reduce the cpr
  // partials by shuffles, park the row sums in shared memory, then each lane rewrites 4
  // consecutive outputs of Y (coalesced).
  __shared__ float rs[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_i = blockIdx.x / 32;                    // 32 CTAs x 8 warps = 256 rows
  const int t = p.tiles[tile_i] * kSlotTileM + (blockIdx.x % 32) * 8 + warp;
  if (t >= p.T) return;
  const int a = p.row_adapter[t];
  const int n0 = blockIdx.y * 128;
  if (a < 0 || n0 >= p.N) return;
  int sub = 0;
#pragma unroll
  for (int i = 1; i < 4; ++i)
    if (i < p.n_sub && n0 >= p.sub_n_start[i]) sub = i;
  const int cpr = p.r_pad >> 3;          // 16-byte pieces per B row (2..8)
  const int part = lane % cpr;           // this lane's 8 ranks
  auto lo = [](uint32_t u) { return __uint_as_float(u << 16); };
  auto hi = [](uint32_t u) { return __uint_as_float(u & 0xffff0000u); };
  const uint4 hv = *reinterpret_cast<const uint4*>(p.H + (size_t)t * p.ldh + p.sub_h_col[sub] + part * 8);
  const float h0 = lo(hv.x), h1 = hi(hv.x), h2 = lo(hv.y), h3 = hi(hv.y);
  const float h4 = lo(hv.z), h5 = hi(hv.z), h6 = lo(hv.w), h7 = hi(hv.w);
  const int rows = min(128, p.N - n0);
  const uint4* base = reinterpret_cast<const uint4*>(p.B + ((size_t)a * p.N + n0) * p.r_pad);
  const int n_pieces = rows * cpr;        // 16-byte pieces of this chunk
  for (int q0 = 0; q0 < n_pieces; q0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u * 32 + lane;
      v[u] = q < n_pieces ? ld_global_nc_v4(base + q) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float sum = h0 * lo(v[u].x) + h1 * hi(v[u].x) + h2 * lo(v[u].y) + h3 * hi(v[u].y) +
                  h4 * lo(v[u].z) + h5 * hi(v[u].z) + h6 * lo(v[u].w) + h7 * hi(v[u].w);
      for (int o = 1; o < cpr; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const int q = q0 + u * 32 + lane;
      if (part == 0 && q < n_pieces) rs[warp][q / cpr] = sum;
    }
  }
  __syncwarp();
  const int r0 = lane * 4;
  if (r0 >= rows) return;
  bf16* y = p.Y + (size_t)t * p.ldy + n0 + r0;
  if (r0 + 4 <= rows) {
    const uint2 yv = *reinterpret_cast<const uint2*>(y);
    const uint32_t a0 = pack_bf16x2(lo(yv.x) + rs[warp][r0], hi(yv.x) + rs[warp][r0 + 1]);
    const uint32_t a1 = pack_bf16x2(lo(yv.y) + rs[warp][r0 + 2], hi(yv.y) + rs[warp][r0 + 3]);
    *reinterpret_cast<uint2*>(y) = make_uint2(a0, a1);
  } else {
    for (int c = 0; r0 + c < rows; ++c) y[c] = __float2bfloat16_rn(__bfloat162float(y[c]) + rs[warp][r0 + c]);
  }
}

}  // namespace collm
