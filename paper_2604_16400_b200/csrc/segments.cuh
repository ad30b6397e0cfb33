// segments.cuh — K0 device side: expand the host-built segment table into per-row indices.
//
// The mixed batch is a row table: [training rows of adapter t] ++ [inference rows sorted by
// (adapter slot, request id, position)], described by seg_start[S+1] / seg_adapter[S].  This is
// the B200 replacement of the reference's batch composition (`domain.Batch`,
// /root/reference/pkg/src/coserve/domain.py:64-86; `StreamQueue.pop_up_to`, dispatcher.py:66-82),
// which cannot mix streams — the unified layer mixes adapters by design.
//
//   row_adapter[t] = seg_adapter[s] for seg_start[s] <= t < seg_start[s+1]
//   slot_of_row[t] = index (into slot_adapter) of row t's adapter within its 256-row slot tile, or -1
#pragma once
#include "common.cuh"

namespace collm {

__global__ void expand_segments_kernel(const int32_t* __restrict__ seg_start,
                                       const int32_t* __restrict__ seg_adapter, int n_seg,
                                       int n_rows, const int32_t* __restrict__ tile_slot_ptr,
                                       const int32_t* __restrict__ slot_adapter,
                                       int32_t* __restrict__ row_adapter,
                                       int32_t* __restrict__ slot_of_row) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rows) return;
  // largest s with seg_start[s] <= t
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int a = seg_adapter[lo];
  if (row_adapter) row_adapter[t] = a;
  if (slot_of_row) {
    int slot = -1;
    if (a >= 0) {
      const int m = t / kSlotTileM;
      for (int s = tile_slot_ptr[m]; s < tile_slot_ptr[m + 1]; ++s)
        if (slot_adapter[s] == a) { slot = s; break; }
    }
    slot_of_row[t] = slot;
  }
}

}  // namespace collm
