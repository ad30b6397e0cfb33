// gemm_lora.cuh — K2/K3: persistent stream-K tcgen05/TMEM GEMM fed by TMA, with the multi-adapter
// LoRA expand folded into the same TMEM accumulator as extra K-steps ("tensor-core SGMV expand").
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
// CG = 1: one CTA per 128-row tile (tcgen05.mma.cta_group::1, 128 x BN per CTA).
// CG = 2: a thread-block cluster of 2 CTAs per 256-row tile (tcgen05.mma.cta_group::2 issued by
//         the leader, M = 256 across the pair): each CTA loads its own 128 rows of A and HALF of
//         the BN rows of B, so the per-SM shared-memory operand traffic per MMA drops from
//         (128 + BN) x 16 to (128 + BN/2) x 16 elements; both CTAs' TMA loads complete on the
//         leader's mbarriers, the leader's commits multicast to both CTAs, both epilogues arrive
//         on the leader's TMEM-empty barrier.
//
// Roles (256 threads per CTA, 1 CTA/SM, persistent):
//   warp 0        : TMA producer (ring of STAGES smem stages, full/empty mbarriers; one
//                   elected lane issues)
//   warp 1        : tcgen05.mma issuer into a double-buffered TMEM accumulator (2 x BN columns;
//                   the whole warp runs the loop on uniform registers, one elected lane issues
//                   each stage's group of MMAs and its commit)
//   warp 2        : TMEM allocator
//   warps 4..7    : epilogue — tcgen05.ld 32x32b -> bf16 -> st.global, overlapped with the next
//                   segment's main loop through the second accumulator buffer.
//
// Hybrid data-parallel + stream-K schedule (computed on the device, identically by every role).
// Tiles are rastered m-fastest, so the CTAs of one data-parallel wave share each W tile through
// L2.  A tile's work is its k-stages: the K/64 main blocks, then the LoRA slot chunks — so the
// shrink producing the LoRA operand can run concurrently with this GEMM's main loop (another
// stream); the producer waits on its readiness flag only before the first LoRA stage.  All
// full waves but the last are data-parallel (CTA c takes tiles c, c+G, ...); the remaining tiles
// (between one and two waves' worth, or all of them when there is less than one wave) are cut into
// gridDim.x equal contiguous k-stage ranges ("stream-K"), which removes the wave-quantization
// tail.  A tile split across CTAs is finished by the CTA holding its last k-stage, which adds the
// other parts' fp32 partials (written to `partials[cta]`, published with a release flag) in CTA
// order — bitwise deterministic.  Each CTA walks its stream-K segments in REVERSE order, so the
// partial it produces is its first stream-K segment and the partials it waits for were produced
// first by the previous CTAs: no wait chain, no deadlock (all CTAs are co-resident: grid <= #SMs,
// one CTA per SM).
#pragma once
#include "common.cuh"

namespace collm {

constexpr int kGemmBM = 128;
constexpr int kGemmBK = 64;
constexpr int kMaxSub = 4;
constexpr int kMaxMTiles = 512;   // rows <= 512 * 128 * CG per launch

struct GemmLoraParams {
  int M, N, K;
  bf16* Y;
  int ldy;  // elements
  // ---- LoRA K-extension (tile_slot_ptr == nullptr -> plain GEMM)
  const int32_t* tile_slot_ptr;  // [num_m_tiles + 1] slot range of each 128-row tile
  const int32_t* tile_skip;      // optional [slot tiles]: 1 = no fused expand (expand_rows.cuh)
  const int32_t* slot_adapter;   // [n_slots] adapter id of each slot
  int lora_rc;                   // columns per LoRA chunk: 16 / 32 / 64 (one TMA box each)
  int lora_chunks;               // chunks per slot (= lora width / rc)
  int lora_per_stage;            // (slot, chunk) items packed into one LoRA k-stage (= 64 / rc)
  int lb_rows_per_adapter;       // LB row coordinate = adapter * this + n0
  int n_sub;                     // sub-projections along N (fused q|k|v, gate|up); >= 1
  int sub_n_start[kMaxSub + 1];  // N boundaries of the sub-projections (multiples of BN)
  int sub_h_col[kMaxSub];        // first H column used by each sub-projection
  int num_m_tiles, num_n_tiles;  // in units of (128 * CG) rows x BN columns
  // readiness of the LoRA operand written by a shrink running concurrently on another stream:
  // before its first LoRA k-stage the producer waits for *lora_flag == *gen (null: no wait)
  const int32_t* lora_flag;
  const int32_t* gen;
  // programmatic dependent launch: 1 = the whole kernel waits for the previous grid after its
  // prologue (GEMM after GEMM); 2 = only the LoRA stages wait (the previous grid is the shrink
  // producing the LoRA operand, launched just before on the same stream)
  int pdl_mode;
  int debug_no_wait;  // timing experiments only: skip that wait (results undefined)
  int sched;  // 0 = data-parallel (round-robin tiles), 1 = hybrid data-parallel + stream-K,
              // 2 = debug: stream-K split without fix-up (timing experiments only)
  int raster_gn;  // data-parallel raster: groups of this many N tiles (<= 1: m-fastest columns)
  // ---- stream-K
  float* partials;  // [gridDim.x][BM*BN] fp32 partial tiles
  int32_t* flags;   // [gridDim.x] partial-ready flags (0 on entry; consumers reset them)
  unsigned long long* dbg;  // optional timeline [gridDim.x][16] (globaltimer ns), debug only
};



// Wait until the concurrently running shrink has published the LoRA operand of this launch
// (*lora_flag == *gen, release/acquire at gpu scope), then order the TMA (async proxy) reads of it
// after that acquire.  A shrink that never runs traps after the timeout instead of hanging.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// debug counters (collm_gemm_wait_stats): total ns producers spent waiting for the flag, waits
__device__ unsigned long long g_lora_wait_ns = 0, g_lora_waits = 0;

__device__ __forceinline__ void wait_lora_flag(const GemmLoraParams& p) {
  const int32_t want = *p.gen;
  int32_t v;
  const unsigned long long t0 = clock64();
  const unsigned long long g0 = gtimer();
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p.lora_flag) : "memory");
    if (v == want) break;
    if (clock64() - t0 > COLLM_MBAR_TIMEOUT_CYCLES) {
      printf("collm: LoRA operand flag timeout (block %d: %d != %d)\n", blockIdx.x, v, want);
      __trap();
    }
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (p.dbg) {
    atomicAdd(&g_lora_wait_ns, gtimer() - g0);
    atomicAdd(&g_lora_waits, 1ull);
  }
}

template <int BN, int STAGES, int CG>
struct GemmSmem {
  static constexpr uint32_t kABytes = kGemmBM * kGemmBK * 2;  // 16 KB: this CTA's 128 rows
  static constexpr uint32_t kBRows = BN / CG;                  // this CTA's share of the N tile
  static constexpr uint32_t kBBytes = kBRows * kGemmBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kBarOffset = STAGES * kStageBytes;
  static constexpr uint32_t kPrefixOffset = kBarOffset + 512;
  // stream-K fix-up: earlier parts of a split tile stream into the idle pipeline stages as
  // 32-column pieces (16 KB) through a ring of kFixSlots slots
  static constexpr uint32_t kFixPiece = kGemmBM * 32 * 4;
  static constexpr int kFixSlots = (STAGES * kStageBytes / kFixPiece) < 16 ? (STAGES * kStageBytes / kFixPiece) : 16;
  // epilogue staging for the TMA stores: per epilogue warp 2 buffers of [32 rows x 32 cols] bf16
  static constexpr uint32_t kEpiBuf = 32 * 32 * 2;
  static constexpr uint32_t kEpiOffset = (kPrefixOffset + (kMaxMTiles + 1) * 4 + 1023) & ~1023u;
  static constexpr uint32_t kTotal = kEpiOffset + 4 * 2 * kEpiBuf + 1024;
  static constexpr uint32_t kTmemCols = 2 * BN;  // double-buffered fp32 accumulator
};

__device__ __forceinline__ int sub_of_n0(const GemmLoraParams& p, int n0) {
  int s = 0;
#pragma unroll
  for (int i = 1; i < kMaxSub; ++i)
    if (i < p.n_sub && n0 >= p.sub_n_start[i]) s = i;
  return s;
}

// One contiguous piece of a tile's k-stage list processed by one CTA.
struct Segment {
  int m_blk, n_blk;
  int k0, k1;     // stage range [k0, k1) within the tile
  int mode;       // 0 = whole tile, 1 = partial (write partials[cta]), 2 = finish (add parts),
                  // 3 = split-2 half (the two halves exchange each other's columns)
  int c_first;    // mode 2: the CTAs [c_first, this CTA) hold the earlier parts
};

struct StreamK {
  const int32_t* prefix;  // smem: stage prefix over m-tiles (num_m_tiles + 1)
  int num_m, sum_s;
  int G;
  int dp_tiles;           // tiles [0, dp_tiles) are data-parallel
  int gn, full_cols;      // grouped raster over the dp region's first full_cols N columns
  long long W_lo, W;      // stream-K region [W_lo, W_lo + W) of the global stage line
  bool split2;            // sched 4: unit u computes half (u & 1) of tile (u >> 1)
  int n_tiles;

  __device__ void init(const int32_t* pre, int nm, int nn, int grid, int sched, int raster_gn = 1) {
    prefix = pre;
    num_m = nm;
    sum_s = pre[nm];
    G = grid;
    split2 = sched == 4;
    n_tiles = nm * nn;
    const int tiles = nm * nn;
    const int waves = tiles / grid;
    dp_tiles = sched == 0 ? tiles : (waves >= 1 ? (waves - 1) * grid : 0);
    W_lo = pos_of_tile(dp_tiles);
    W = (long long)sum_s * nn - W_lo;
    gn = raster_gn > 1 ? raster_gn : 1;
    full_cols = dp_tiles / nm;
  }
  // Data-parallel tile t -> (m, n).  The dp region is the first dp_tiles tiles of the m-fastest
  // order (the stream-K tail is the rest of it); inside its first full_cols whole N columns the
  // tiles are visited in groups of gn columns, n-fastest within a group, so one wave touches
  // ~sqrt(G) A row-blocks and ~sqrt(G) W column-blocks instead of every A row-block of one
  // column: at large M (A >> L2) A then streams from DRAM num_n / gn times instead of num_n.
  __device__ void dp_tile(int t, int& m, int& n) const {
    if (gn > 1 && t < full_cols * num_m) {
      const int g = t / (gn * num_m);
      const int cols = min(gn, full_cols - g * gn);
      const int local = t - g * gn * num_m;
      m = local / cols;
      n = g * gn + local % cols;
    } else {
      m = t % num_m;
      n = t / num_m;
    }
  }
  __device__ long long pos_of_tile(int t) const {
    return (long long)(t / num_m) * sum_s + prefix[t % num_m];
  }
  __device__ int stages_of_m(int m) const { return prefix[m + 1] - prefix[m]; }
  __device__ long long bound(int c) const { return W_lo + (long long)c * W / G; }
  __device__ int cta_of(long long x) const {
    int c = (int)(((x - W_lo) * G) / W);
    while (c + 1 < G && bound(c + 1) <= x) ++c;
    while (c > 0 && bound(c) > x) --c;
    return c;
  }
  // The stream-K segment of CTA c that ends at global position x_end (exclusive).
  __device__ Segment seg_ending_at(long long x_end, long long range_lo, int c) const {
    const long long x = x_end - 1;
    const int n = (int)(x / sum_s);
    const int r = (int)(x % sum_s);
    int lo = 0, hi = num_m - 1;  // largest m with prefix[m] <= r
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (prefix[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const int m = lo;
    const long long t0 = (long long)n * sum_s + prefix[m];
    const long long t1 = t0 + stages_of_m(m);
    const long long s0 = t0 > range_lo ? t0 : range_lo;
    Segment sg;
    sg.m_blk = m;
    sg.n_blk = n;
    sg.k0 = (int)(s0 - t0);
    sg.k1 = (int)(x_end - t0);
    const bool first = s0 == t0, last = x_end == t1;
    sg.mode = (first && last) ? 0 : (last ? 2 : 1);
    sg.c_first = (sg.mode == 2) ? cta_of(t0) : c;
    return sg;
  }
  // Visit this CTA's work: its data-parallel tiles, then its stream-K segments in reverse.
  template <class F>
  __device__ void for_each(int c, F&& f) const {
    if (split2) {  // one half-tile per unit, halves of a tile in adjacent units
      const int t = c >> 1;
      if (t >= n_tiles) return;
      Segment sg;
      sg.m_blk = t % num_m;
      sg.n_blk = t / num_m;
      const int S = stages_of_m(sg.m_blk);
      sg.k0 = (c & 1) ? S / 2 : 0;  // the LoRA stages (last) fall in half 1
      sg.k1 = (c & 1) ? S : S / 2;
      sg.mode = 3;
      sg.c_first = c ^ 1;
      f(sg);
      return;
    }
    for (int t = c; t < dp_tiles; t += G) {
      Segment sg;
      dp_tile(t, sg.m_blk, sg.n_blk);
      sg.k0 = 0;
      sg.k1 = stages_of_m(sg.m_blk);
      sg.mode = 0;
      sg.c_first = c;
        f(sg);
    }
    const long long lo = bound(c);
    for (long long x_end = bound(c + 1); x_end > lo;) {
      const Segment sg = seg_ending_at(x_end, lo, c);
      x_end -= sg.k1 - sg.k0;
      f(sg);
    }
  }
};

template <int BN, int STAGES, int CG, int MC>
__global__ void __launch_bounds__(256, 2)  // <= 128 registers: a LoRA CTA can co-reside
    gemm_lora_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmLB,
                     const __grid_constant__ CUtensorMap tmY, const GemmLoraParams p) {
  using L = GemmSmem<BN, STAGES, CG>;
  constexpr uint32_t BM = kGemmBM, BK = kGemmBK;
  constexpr uint32_t UNIT_M = BM * CG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* fixbar = tempty + 2;  // stream-K fix-up ring: one barrier per 16 KB slot
  uint64_t* xfree = fixbar + 16;  // cluster split-2: the partner's smem may receive ours
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixbar + 17);
  int32_t* s_prefix = reinterpret_cast<int32_t*>(smem + L::kPrefixOffset);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool has_lora = p.tile_slot_ptr != nullptr;
  const int nk = (p.K + BK - 1) / BK;
  // MC == 2 (split-2 only): a cluster of the two CTA pairs computing the two K halves of one
  // tile, which swap their half-tile partials through distributed shared memory
  // MC == 3 (data-parallel only): a cluster of two CTA pairs on adjacent N tiles of the same rows;
  // each CTA loads half of its A box and multicasts it to the CTA at the same position of the
  // other pair (25 % less L2 -> SM operand traffic — energy, under the power cap)
  constexpr bool AMC = MC == 3;
  constexpr int CL = CG * (MC == 1 ? 1 : 2);  // CTAs per cluster
  static_assert(MC == 1 || CG == 2, "clusters of pairs are built from CTA pairs");
  const uint32_t crank = (CL > 1) ? cluster_ctarank() : 0;
  const uint32_t rank = (CG == 2) ? (crank & 1u) : 0;  // position in the pair
  const uint32_t q = crank >> 1;                        // pair within the cluster (MC == 2)
  const uint32_t leader_rank = crank & ~1u;             // this pair's MMA issuer
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * q));
  const bool leader = rank == 0;

  // LoRA stages of a (128*CG)-row unit: the slot list of the 256-row slot tile containing it
  // (slot, chunk) items of a unit; 64/rc of them share one k-stage (one barrier round trip):
  // the stage's A half holds their Hslots boxes side by side, its B half their adapters' B boxes
  auto lora_items = [&](int m) {
    if (!has_lora) return 0;
    const int st = (m * (int)UNIT_M) / kSlotTileM;
    if (p.tile_skip && p.tile_skip[st]) return 0;
    return (p.tile_slot_ptr[st + 1] - p.tile_slot_ptr[st]) * p.lora_chunks;
  };
  auto lora_stages = [&](int m) {
    return has_lora ? (lora_items(m) + p.lora_per_stage - 1) / p.lora_per_stage : 0;
  };

  // per-unit stage counts (all threads, independent global loads in flight) -> prefix (warp 0,
  // shuffle scan): every role needs it for the schedule.  A serial loop here cost one dependent
  // L2/DRAM round trip per m-tile (~50 us at the 8B/13B row counts).
  for (int m = threadIdx.x; m < p.num_m_tiles; m += blockDim.x) s_prefix[m + 1] = lora_stages(m) + nk;
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < p.num_m_tiles; base += 32) {
      const int m = base + lane;
      int v = m < p.num_m_tiles ? s_prefix[m + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (m < p.num_m_tiles) s_prefix[m + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) s_prefix[0] = 0;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmY);
    if (has_lora) {
      tma_prefetch_desc(&tmH);
      tma_prefetch_desc(&tmLB);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], AMC ? 2 : 1);  // AMC: both pairs' MMAs read each stage's A halves
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * CG);
    }
    for (int k = 0; k < 17; ++k) mbar_init(&fixbar[k], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<L::kTmemCols, CG>(tmem_slot);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch (GEMM after GEMM on one stream): everything above — barrier
  // init, TMEM allocation, descriptor prefetch, the schedule prefix — overlapped the previous
  // grid's tail; no global memory the previous grid may still write is touched before this wait.
  // The next grid may launch as SMs free up (its own prologue then waits here in turn).
  if (p.pdl_mode == 1) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  StreamK sk;
  sk.init(s_prefix, p.num_m_tiles, AMC ? (p.num_n_tiles + 1) / 2 : p.num_n_tiles,
          gridDim.x / (AMC ? CL : CG), p.sched, p.raster_gn);
  const int unit = blockIdx.x / (AMC ? CL : CG);  // CTA pair / CTA (AMC: cluster) in the schedule

  if (warp == 0) {
    // ===================== TMA producer (both CTAs of a pair; one elected lane issues) =====
    const bool issuer = elect_one();
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t rc = p.lora_rc;
    bool lora_ready = p.lora_flag == nullptr && p.pdl_mode != 2;
    sk.for_each(unit, [&](const Segment& sg) {
      const int m0 = sg.m_blk * UNIT_M + rank * BM;  // this CTA's rows
      const int n0 = (AMC ? sg.n_blk * 2 + (int)q : sg.n_blk) * BN;
      const int nb0 = n0 + rank * (int)L::kBRows;   // this CTA's share of the N tile
      const int st_tile = m0 / kSlotTileM;
      const int hrow0 = m0 % kSlotTileM;
      const int hcol = has_lora ? p.sub_h_col[sub_of_n0(p, n0)] : 0;
      for (int i = sg.k0; i < sg.k1; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (!issuer) {
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        uint8_t* sa = smem + stage * L::kStageBytes;
        const bool lora_stage = i >= nk;  // the tile's LoRA k-stages follow its K/64 main blocks
        if (lora_stage && !lora_ready) {
          if (p.pdl_mode == 2) {  // the shrink grid (launched just before) completed + visible
            if (!p.debug_no_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            if (p.dbg) p.dbg[(size_t)blockIdx.x * 32 + 20] = gtimer();
          } else {
            wait_lora_flag(p);
          }
          lora_ready = true;
        }
        int it0 = 0, n_it = 0;  // this LoRA stage's (slot, chunk) items
        if (lora_stage) {
          it0 = (i - nk) * p.lora_per_stage;
          n_it = min(p.lora_per_stage, lora_items(sg.m_blk) - it0);
        }
        const uint32_t bytes = lora_stage ? n_it * (BM + L::kBRows) * rc * 2 : L::kStageBytes;
        if (p.sched == 3) {  // debug: no operand loads (measures the MMA issue rate alone)
          if (leader) mbar_arrive(&full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
        }
        if (leader) mbar_arrive_expect_tx(&full[stage], bytes * CG);
        if (p.dbg && i == sg.k0 && p.dbg[(size_t)blockIdx.x * 32 + 15] == 0)
          p.dbg[(size_t)blockIdx.x * 32 + 15] = gtimer();
        if (lora_stage) {
          for (int j = 0; j < n_it; ++j) {
            const int s = p.tile_slot_ptr[st_tile] + (it0 + j) / p.lora_chunks;
            const int c = (it0 + j) % p.lora_chunks;
            const int lb_row = p.slot_adapter[s] * p.lb_rows_per_adapter + nb0;
            uint8_t* da = sa + j * (BM * rc * 2);
            uint8_t* db = sa + L::kABytes + j * (L::kBRows * rc * 2);
            if constexpr (CG == 2) {
              const uint32_t fb = mapa_shared(&full[stage], leader_rank);
              tma_load_2d_pair(da, &tmH, fb, hcol + c * rc, s * kSlotTileM + hrow0);
              tma_load_2d_pair(db, &tmLB, fb, c * rc, lb_row);
            } else {
              tma_load_2d(da, &tmH, &full[stage], hcol + c * rc, s * kSlotTileM + hrow0);
              tma_load_2d(db, &tmLB, &full[stage], c * rc, lb_row);
            }
          }
        } else {
          const int kb = i;
          if constexpr (AMC) {
            tma_load_2d_pair_mc(sa + q * (L::kABytes / 2), &tmA, &full[stage],
                                (uint16_t)(0x5u << rank), kb * BK, m0 + (int)q * (int)(BM / 2));
            tma_load_2d_pair(sa + L::kABytes, &tmB, mapa_shared(&full[stage], leader_rank),
                             kb * BK, nb0);
          } else if constexpr (CG == 2) {
            const uint32_t fb = mapa_shared(&full[stage], leader_rank);
            tma_load_2d_pair(sa, &tmA, fb, kb * BK, m0);
            tma_load_2d_pair(sa + L::kABytes, &tmB, fb, kb * BK, nb0);
          } else {
            tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
            tma_load_2d(sa + L::kABytes, &tmB, &full[stage], kb * BK, nb0);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    });
  } else if (warp == 1 && leader) {
    // ===================== tcgen05.mma issuer (the pair's leader; the whole warp runs the loop,
    // one elected lane issues each stage's group of MMAs + its commit) =====================
    constexpr uint32_t idesc = umma_idesc_bf16(UNIT_M, BN);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, acc_phase = 0;
    const uint32_t smem_base = smem_u32(smem);
    const uint32_t lrow = p.lora_rc * 2, lsteps = p.lora_rc / 16;
    // debug timeline (COLLM_GEMM_DEBUG): [4] first stage ready, [8] 32nd stage, [12] last issue
    unsigned long long* mdbg = p.dbg ? p.dbg + (size_t)blockIdx.x * 32 : nullptr;
    int kbi = 0;
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
      if constexpr (CG == 2) umma_bf16_pair(d, a, b, idesc, accumulate);
      else umma_bf16(d, a, b, idesc, accumulate);
    };
    auto commit = [&](uint64_t* bar) {  // both CTAs of this pair
      if constexpr (MC != 1) umma_commit_pair_mask(bar, pair_mask);
      else if constexpr (CG == 2) umma_commit_pair(bar);
      else umma_commit(bar);
    };
    auto release = [&](uint64_t* bar) {  // a stage: every CTA whose loads fed it
      if constexpr (AMC) umma_commit_pair_mask(bar, 0xF);
      else commit(bar);
    };
    sk.for_each(unit, [&](const Segment& sg) {
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      uint32_t accumulate = 0;
      for (int i = sg.k0; i < sg.k1; ++i) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (mdbg && lane == 0) {
          if (kbi == 0) mdbg[4] = gtimer();
          else if (kbi == 32) mdbg[8] = gtimer();
        }
        ++kbi;
        const uint32_t sa = smem_base + stage * L::kStageBytes;
        if (i >= nk) {  // LoRA expand k-stage: (Hslots chunk x adapter B chunk) per item
          const int it0 = (i - nk) * p.lora_per_stage;
          const int n_it = min(p.lora_per_stage, lora_items(sg.m_blk) - it0);
          if (elect_one()) {
            for (int j = 0; j < n_it; ++j)
              for (uint32_t k = 0; k < lsteps; ++k)
                mma(d_tmem, umma_desc_kmajor(sa + j * (BM * lrow) + k * 32, lrow),
                    umma_desc_kmajor(sa + L::kABytes + j * (L::kBRows * lrow) + k * 32, lrow),
                    (accumulate | j | k) ? 1u : 0u);
            release(&empty[stage]);
          }
        } else {
          if (elect_one()) {
#pragma unroll
            for (uint32_t k = 0; k < BK / 16; ++k)
              mma(d_tmem, umma_desc_kmajor(sa + k * 32, 128),
                  umma_desc_kmajor(sa + L::kABytes + k * 32, 128), accumulate | k);
            release(&empty[stage]);
          }
        }
        __syncwarp();
        accumulate = 1;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (mdbg && lane == 0) mdbg[12] = gtimer();
      if (elect_one()) commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    });
  } else if (warp >= 4) {
    // ===================== epilogue (both CTAs: each its own 128 rows) =====================
    const int ew = warp - 4;  // TMEM lanes [32*ew, 32*ew+32)
    const int tid = threadIdx.x - 128;
    uint32_t acc = 0, acc_phase = 0;
    int seg_i = 0;
    uint32_t epi_i = 0;  // TMA-store buffer toggle
    uint8_t* epi_buf = smem + L::kEpiOffset;
    const int cta = blockIdx.x;
    unsigned long long* dbg = p.dbg ? p.dbg + (size_t)cta * 32 : nullptr;
    if (dbg && tid == 0) dbg[0] = gtimer();
    sk.for_each(unit, [&](const Segment& sg_in) {
      Segment sg = sg_in;
      if (p.sched == 2) sg.mode = 0;  // debug: stream-K split without the fix-up (timing only)
      const int lrow_i = ew * 32 + lane;
      const int row = sg.m_blk * UNIT_M + rank * BM + lrow_i;
      const int n0 = (AMC ? sg.n_blk * 2 + (int)q : sg.n_blk) * BN;
      if (dbg && tid == 0 && seg_i < 3) dbg[1 + 4 * seg_i] = gtimer() | ((unsigned long long)sg.mode << 60);
      if (sg.mode == 2) {  // wait for the earlier parts of this tile (produced first by their CTAs)
        if (tid == 0) {
          for (int c = sg.c_first; c < unit; ++c) {
            if (sk.bound(c) == sk.bound(c + 1)) continue;  // empty range: no part
            const int32_t* f = p.flags + c * CG + rank;
            uint32_t v;
            const unsigned long long t0 = clock64();
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
              if (clock64() - t0 > COLLM_MBAR_TIMEOUT_CYCLES) {
                printf("collm: stream-K flag timeout (block %d)\n", blockIdx.x);
                __trap();
              }
            } while (v == 0);
          }
          // the parts' generic-proxy stores, acquired above, are read below by bulk copies
          // (async proxy): order them
          asm volatile("fence.proxy.async.global;" ::: "memory");
          if (dbg) dbg[14] = gtimer();
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (dbg && tid == 0 && seg_i < 3) dbg[2 + 4 * seg_i] = gtimer();
      // Finishing segment = this CTA's last: the MMAs are done with the pipeline smem, so the
      // earlier parts of the tile stream into it as 32-column pieces (chunk-major, parts in CTA
      // order) through a ring of bulk copies issued ahead of their use.
      constexpr int RS = L::kFixSlots;
      int np = 0;
      if (sg.mode == 2)
        for (int pc = sg.c_first; pc < unit; ++pc) np += sk.bound(pc) != sk.bound(pc + 1);
      auto issue_piece = [&](int q) {  // one thread; the i-th non-empty earlier part, CTA order
        const int slot = q % RS, chunk = q / np;
        int i = q % np, pc = sg.c_first;
        for (;; ++pc)
          if (sk.bound(pc) != sk.bound(pc + 1) && i-- == 0) break;
        mbar_arrive_expect_tx(&fixbar[slot], L::kFixPiece);
        bulk_copy_g2s(smem + slot * L::kFixPiece,
                      p.partials + (size_t)(pc * CG + (int)rank) * (BM * BN) + (size_t)chunk * (BM * 32),
                      L::kFixPiece, &fixbar[slot]);
      };
      const int n_pieces = np * (BN / 32);
      if (np && tid == 0)
        for (int q = 0; q < RS && q < n_pieces; ++q) issue_piece(q);
      // partial tiles are stored in the epilogue's own thread order — float4 index
      // ((chunk * 8 + j) * 128 + tid) — so writes and reads are 512 B-coalesced per warp
      float4* part_mine = reinterpret_cast<float4*>(p.partials + (size_t)cta * (BM * BN)) + tid;
      // bf16 row chunk -> this warp's staging buffer (64-byte TMA swizzle: 16-byte chunk j of
      // row r at j ^ ((r >> 1) & 3)), then one TMA store of the [32 rows x 32 cols] box; the
      // tensor map clips rows >= M and columns >= N
      auto store_chunk = [&](const uint32_t (&r)[32], int c) {
        uint8_t* buf = epi_buf + (ew * 2 + (epi_i & 1)) * L::kEpiBuf;
        if (lane == 0) bulk_wait_group_read<1>();  // the store that last used it has read it
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(r[8 * j + 0]), __uint_as_float(r[8 * j + 1]));
          v.y = pack_bf16x2(__uint_as_float(r[8 * j + 2]), __uint_as_float(r[8 * j + 3]));
          v.z = pack_bf16x2(__uint_as_float(r[8 * j + 4]), __uint_as_float(r[8 * j + 5]));
          v.w = pack_bf16x2(__uint_as_float(r[8 * j + 6]), __uint_as_float(r[8 * j + 7]));
          *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmY, buf, n0 + c, row - lane);
          bulk_commit_group();
        }
        ++epi_i;
      };
      if (sg.mode == 3) {
        // split-2 tile: both halves finish together; each writes the fp32 partial of the OTHER
        // half's columns, then adds the partner's partial of its own columns (streamed into the
        // idle pipeline smem) and stores them.  acc_0 + acc_1 is commutative: bitwise the same
        // whichever half adds.
        constexpr int NCH = BN / 32;
        const int half = unit & 1;
        const int own_lo = half ? NCH / 2 : 0, own_hi = half ? NCH : NCH / 2;
        if constexpr (MC == 2) {
          // cluster split-2: the two halves are the two pairs of this cluster.  Each of the other
          // half's 32-column chunks goes TMEM -> this CTA's idle pipeline smem (16 KB piece,
          // float4 index j * 128 + tid) -> a DSMEM bulk copy into the partner CTA (same position,
          // other pair; once it reports its smem idle), completing on the partner's piece
          // barrier; the partner adds piece i to its own chunk i as soon as it lands.  No global
          // memory, no gpu-scope fences.
          constexpr uint32_t kPiece = BM * 32 * 4, kX = kPiece * (NCH / 2);
          static_assert(2 * kX <= STAGES * L::kStageBytes, "split-2 exchange exceeds the pipeline smem");
          uint64_t* xr = fixbar;  // one barrier per incoming piece (the stream-K ring is unused)
          const uint32_t peer = crank ^ 2u;
          if (tid == 0) {
            for (int i = 0; i < NCH / 2; ++i) mbar_arrive_expect_tx(&xr[i], kPiece);
            mbar_arrive_cluster(mapa_shared(xfree, peer));  // our pipeline smem is idle
          }
          int lc = 0;
#pragma unroll 1
          for (int chunk = 0; chunk < NCH; ++chunk) {
            if (chunk >= own_lo && chunk < own_hi) continue;
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + chunk * 32, r);
            tmem_wait_ld();
            float4* s_out = reinterpret_cast<float4*>(smem + lc * kPiece) + tid;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              s_out[j * 128] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                           __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            fence_proxy_async_smem();  // generic smem writes -> the bulk copy (async proxy)
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (tid == 0) {
              if (lc == 0) {
                if (dbg) dbg[16] = gtimer();
                mbar_wait(xfree, 0);
                if (dbg) dbg[17] = gtimer();
              }
              bulk_copy_s2cluster(mapa_shared(smem + kX + lc * kPiece, peer), smem + lc * kPiece,
                                  kPiece, mapa_shared(&xr[lc], peer));
            }
            ++lc;
          }
#pragma unroll 1
          for (int chunk = own_lo; chunk < own_hi; ++chunk) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + chunk * 32, r);
            tmem_wait_ld();
            mbar_wait(&xr[chunk - own_lo], 0);
            if (dbg && tid == 0 && chunk == own_lo) dbg[18] = gtimer();
            const float4* src = reinterpret_cast<const float4*>(smem + kX + (chunk - own_lo) * kPiece) + tid;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = src[j * 128];
              r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
              r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
              r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
              r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
            }
            store_chunk(r, chunk * 32);
          }
          if (dbg && tid == 0) dbg[19] = gtimer();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(&tempty[acc], leader_rank));
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
          ++seg_i;
          return;
        }
        const int partner = sg.c_first * CG + (int)rank;
#pragma unroll 1
        for (int chunk = 0; chunk < NCH; ++chunk) {
          if (chunk >= own_lo && chunk < own_hi) continue;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + chunk * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(part_mine + (chunk * 8 + j) * 128,
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
        }
        if (dbg && tid == 0) dbg[16] = gtimer();
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (dbg && tid == 0) dbg[17] = gtimer();
        if (tid == 0) {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.flags + cta), "r"(1u) : "memory");
          const int32_t* f = p.flags + partner;
          uint32_t v;
          const unsigned long long t0 = clock64();
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if (clock64() - t0 > COLLM_MBAR_TIMEOUT_CYCLES) {
              printf("collm: split-2 flag timeout (block %d)\n", blockIdx.x);
              __trap();
            }
          } while (v == 0);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk reads
          if (dbg) dbg[18] = gtimer();
          for (int chunk = own_lo; chunk < own_hi; ++chunk) {  // one ring slot per own chunk
            const int slot = chunk - own_lo;
            mbar_arrive_expect_tx(&fixbar[slot], L::kFixPiece);
            bulk_copy_g2s(smem + slot * L::kFixPiece,
                          p.partials + (size_t)partner * (BM * BN) + (size_t)chunk * (BM * 32),
                          L::kFixPiece, &fixbar[slot]);
          }
        }
#pragma unroll 1
        for (int chunk = own_lo; chunk < own_hi; ++chunk) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + chunk * 32, r);
          tmem_wait_ld();
          const int slot = chunk - own_lo;
          mbar_wait(&fixbar[slot], 0);
          if (dbg && tid == 0) dbg[19 + slot] = gtimer();
          const float4* src = reinterpret_cast<const float4*>(smem + slot * L::kFixPiece) + tid;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 v = src[j * 128];
            r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
            r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
            r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
            r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
          }
          store_chunk(r, chunk * 32);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(&tempty[acc], leader_rank));
          else mbar_arrive(&tempty[acc]);
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the partner's partial is consumed
        if (tid == 0) p.flags[partner] = 0;                // ready for the next launch
        ++seg_i;
        return;
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c, r);
        tmem_wait_ld();
        const int chunk = c >> 5;
        if (dbg && tid == 0 && sg.mode == 2) dbg[24 + chunk] = gtimer();
        if (sg.mode == 1) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(part_mine + (chunk * 8 + j) * 128,
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
          continue;
        }
        if (sg.mode == 2 && np) {
          for (int i = 0; i < np; ++i) {
            const int q = chunk * np + i;
            mbar_wait(&fixbar[q % RS], (uint32_t)(q / RS) & 1u);
            const float4* src = reinterpret_cast<const float4*>(smem + (q % RS) * L::kFixPiece) + tid;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 v = src[j * 128];
              r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
              r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
              r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
              r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
            }
          }
          // every epilogue thread is done with this chunk's slots: refill them RS pieces ahead
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (dbg && tid == 0) dbg[16 + chunk] = gtimer();
          if (tid == 0) {
            fence_proxy_async_smem();
            for (int i = 0; i < np; ++i)
              if (chunk * np + i + RS < n_pieces) issue_piece(chunk * np + i + RS);
          }
        }
        store_chunk(r, c);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(&tempty[acc], leader_rank));
        else mbar_arrive(&tempty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      if (sg.mode == 1) {  // publish the partial
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 0)
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.flags + cta), "r"(1u)
                       : "memory");
      } else if (sg.mode == 2) {  // consumed: reset the producers' flags for the next launch
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 0)
          for (int c = sg.c_first; c < unit; ++c) p.flags[c * CG + rank] = 0;
      }
      if (dbg && tid == 0 && seg_i < 3) dbg[3 + 4 * seg_i] = gtimer();
      ++seg_i;
    });
    if (lane == 0) bulk_wait_group_read<0>();  // the TMA stores have read their smem (they
                                               // complete before the grid does)
    if (dbg && tid == 0) dbg[13] = gtimer();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols, CG>(tmem_base);
  }
}

}  // namespace collm
