// collm_abi.cu — the C ABI (include/collm.h): argument validation, host-side planning, TMA
// descriptor encoding and kernel launches.  Built with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/collm.h"
#include "common.cuh"
#include "gemm_lora.cuh"
#include "reduce_adamw.cuh"
#include "attn.cuh"
#include "ce.cuh"
#include "segments.cuh"
#include "shrink.cuh"
#include "shrink_tc.cuh"
#include "flash_attn.cuh"
#include "flash_tc.cuh"
#include "flash_bwd_tc.cuh"
#include "expand_rows.cuh"
#include "reduce_tc.cuh"

using namespace collm;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return fail(COLLM_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                  __FILE__, __LINE__);                                              \
  } while (0)

#define CHECK_ARG(cond, ...)                        \
  do {                                              \
    if (!(cond)) return fail(COLLM_EINVAL, __VA_ARGS__); \
  } while (0)

// Workspace layout shared by the split reductions: [kCounterCap int32 arrival counters][fp32
// partials].  Counters sit at a fixed prefix so that any launch (whatever its split factor or
// tile count) finds them zero — kernels restore them to zero, and partials never overlap them.
constexpr size_t kCounterCap = 1 << 16;
constexpr size_t kCounterBytes = kCounterCap * sizeof(int32_t);

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Per-device host state.  cudaFuncSetAttribute, SM counts and occupancy are properties of a
// device, so every cache below is indexed by the calling thread's current device and guarded by
// one mutex (the ABI functions are reentrant: any thread, any device).
constexpr int kMaxDevices = 64;
std::mutex g_state_mu;

int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) { cudaGetLastError(); d = 0; }
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

int num_sms_cached() {
  static int n[kMaxDevices] = {};  // 0: not queried yet
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_state_mu);
  if (n[dev] <= 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    n[dev] = v;
  }
  return n[dev];
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D bf16 tensor map over a row-major [rows, cols] matrix with leading dimension ld (elements).
int make_tmap(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t ld,
              uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMapSwizzle sw;
  switch (box_cols * 2) {
    case 128: sw = CU_TENSOR_MAP_SWIZZLE_128B; break;
    case 64: sw = CU_TENSOR_MAP_SWIZZLE_64B; break;
    case 32: sw = CU_TENSOR_MAP_SWIZZLE_32B; break;
    default: return fail(COLLM_EINTERNAL, "unsupported TMA box width %u", box_cols);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled failed (%d): cols=%llu rows=%llu ld=%llu",
                (int)r, (unsigned long long)cols, (unsigned long long)rows,
                (unsigned long long)ld);
  return COLLM_OK;
}

// 3-D bf16 tensor map viewing a row-major [rows, ld] matrix as [k-block][row][64 columns]:
// dims (64, rows, nkb) with strides (ld*2 B per row, 128 B per k-block); a box (64, box_rows,
// box_kb) lands in shared memory k-block-major, each k-block a [box_rows][128 B] SWIZZLE_128B
// tile — the K-major UMMA operand layout (lora_shrink_tc_kernel).
int make_tmap_kblocks(CUtensorMap* m, const void* base, uint64_t rows, uint64_t ld, uint64_t nkb,
                      uint32_t box_rows, uint32_t box_kb) {
  auto fn = encode_fn();
  if (!fn) return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {64, rows, nkb};
  cuuint64_t strides[2] = {ld * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_kb};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled (k-block view) failed (%d): rows=%llu ld=%llu nkb=%llu box=%ux%u",
                (int)r, (unsigned long long)rows, (unsigned long long)ld, (unsigned long long)nkb,
                box_rows, box_kb);
  return COLLM_OK;
}

template <int BN, int STAGES, int CG, int MC>
int configure_gemm() {
  using L = GemmSmem<BN, STAGES, CG>;
  static bool configured[kMaxDevices] = {};
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(g_state_mu);
  if (!configured[dev]) {
    CUDA_TRY(cudaFuncSetAttribute(gemm_lora_kernel<BN, STAGES, CG, MC>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal));
    // the whole unified L1/shared array as shared memory: the SM then has room for a rank-space
    // CTA next to this GEMM CTA (the two-stream overlap); the default carveout is the smallest
    // one that fits the GEMM alone.  (The rank-space kernels keep the default: alone on an SM
    // they profit from L1; next to a GEMM CTA the SM is already configured this way.)
    CUDA_TRY(cudaFuncSetAttribute(gemm_lora_kernel<BN, STAGES, CG, MC>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
    configured[dev] = true;
  }
  return COLLM_OK;
}

// Clusters of CG*MC CTAs of this variant that can be co-resident (the persistent schedule's
// flag waits need every CTA resident): 4-CTA clusters must fit inside one GPC.
template <int BN, int STAGES, int CG, int MC>
int max_gemm_clusters() {
  static int n[kMaxDevices] = {};  // 0: not computed yet (a device fits >= 1 cluster)
  const int dev = cur_device();
  if (n[dev] <= 0) {
    if (configure_gemm<BN, STAGES, CG, MC>()) return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(num_sms_cached() / (CG * (MC == 1 ? 1 : 2)) * (CG * (MC == 1 ? 1 : 2)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = GemmSmem<BN, STAGES, CG>::kTotal;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG * (MC == 1 ? 1 : 2);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, gemm_lora_kernel<BN, STAGES, CG, MC>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      c = num_sms_cached() / (CG * (MC == 1 ? 1 : 2));
    }
    std::lock_guard<std::mutex> lk(g_state_mu);
    n[dev] = c;
  }
  return n[dev];
}

template <int BN, int STAGES, int CG, int MC = 1>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& th,
                const CUtensorMap& tlb, const CUtensorMap& ty, const GemmLoraParams& p, int grid,
                cudaStream_t stream) {
  using L = GemmSmem<BN, STAGES, CG>;
  int rc = configure_gemm<BN, STAGES, CG, MC>();
  if (rc) return rc;
  if (MC > 1) {
    const int cap = (CG * (MC == 1 ? 1 : 2)) * max_gemm_clusters<BN, STAGES, CG, MC>();
    if (grid > cap)
      return fail(COLLM_EINVAL, "GEMM grid %d exceeds co-resident %d-CTA clusters (%d CTAs)", grid,
                  CG * (MC == 1 ? 1 : 2), cap);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = L::kTotal;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * (MC == 1 ? 1 : 2);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // PDL (opt-in, COLLM_GEMM_PDL=1): the prologue overlaps the previous grid of the stream (the
  // kernel waits for it with griddepcontrol.wait before touching global memory).  Measured: GEMM
  // chains -0.3 ms/step, but the full overlapped step no faster (early-resident GEMM CTAs hold SM
  // space the rank-space kernels want), so it is off by default.
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl_mode ? 2 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_lora_kernel<BN, STAGES, CG, MC>, ta, tb, th, tlb, ty, p));
  return COLLM_OK;
}

}  // namespace

extern "C" {

int collm_version(void) { return 1; }

const char* collm_last_error(void) { return g_err; }

int collm_device_info(int device, int* sm_major, int* sm_minor, int* num_sms) {
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (sm_major) *sm_major = prop.major;
  if (sm_minor) *sm_minor = prop.minor;
  if (num_sms) *num_sms = prop.multiProcessorCount;
  if (prop.major != 10)
    return fail(COLLM_EUNSUPPORTED, "collm is built for sm_100a; device %d is sm_%d%d", device,
                prop.major, prop.minor);
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K0 host
int collm_plan_segments(const int32_t* seg_start, const int32_t* seg_adapter, int n_seg,
                        int n_rows, int32_t* tile_slot_ptr, int32_t* slot_adapter, int slot_cap,
                        int32_t* n_slots, int32_t* shrink_tiles, int shrink_tile_cap,
                        int32_t* n_shrink_tiles) {
  CHECK_ARG(n_seg >= 1 && n_rows >= 1, "empty segment table (n_seg=%d, n_rows=%d)", n_seg, n_rows);
  CHECK_ARG(seg_start[0] == 0 && seg_start[n_seg] == n_rows,
            "segment table must cover rows [0, %d): starts at %d, ends at %d", n_rows,
            seg_start[0], seg_start[n_seg]);
  for (int s = 0; s < n_seg; ++s)
    CHECK_ARG(seg_start[s + 1] > seg_start[s], "segment %d is empty or unsorted", s);
  const int n_tiles = (n_rows + kSlotTileM - 1) / kSlotTileM;
  int ns = 0;
  int seg = 0;
  for (int m = 0; m < n_tiles; ++m) {
    if (tile_slot_ptr) tile_slot_ptr[m] = ns;
    const int r0 = m * kSlotTileM, r1 = std::min(n_rows, r0 + kSlotTileM);
    while (seg_start[seg + 1] <= r0) ++seg;
    const int first = ns;
    for (int s = seg; s < n_seg && seg_start[s] < r1; ++s) {
      const int a = seg_adapter[s];
      if (a < 0) continue;
      bool dup = false;
      for (int i = first; i < ns; ++i)
        if (slot_adapter[i] == a) { dup = true; break; }
      if (dup) continue;
      CHECK_ARG(ns < slot_cap, "slot capacity %d exceeded", slot_cap);
      slot_adapter[ns++] = a;
    }
  }
  if (tile_slot_ptr) tile_slot_ptr[n_tiles] = ns;
  if (n_slots) *n_slots = ns;
  // shrink work list: maximal runs of equal adapter (roles may differ: rows of one tenant's
  // prefill and decode requests share the adapter's A) cut into <= 16-row tiles; base-only runs
  // (adapter -1) are listed too so the shrink zero-fills their slot rows.
  int nt = 0;
  for (int s = 0; s < n_seg;) {
    int e = s + 1;
    while (e < n_seg && seg_adapter[e] == seg_adapter[s]) ++e;
    for (int r = seg_start[s]; r < seg_start[e]; r += 16) {
      CHECK_ARG(nt < shrink_tile_cap, "shrink tile capacity %d exceeded", shrink_tile_cap);
      if (shrink_tiles) {
        shrink_tiles[3 * nt + 0] = r;
        shrink_tiles[3 * nt + 1] = std::min(16, seg_start[e] - r);
        shrink_tiles[3 * nt + 2] = seg_adapter[s];
      }
      ++nt;
    }
    s = e;
  }
  if (n_shrink_tiles) *n_shrink_tiles = nt;
  return COLLM_OK;
}

int collm_expand_segments(const int32_t* seg_start, const int32_t* seg_adapter, int n_seg,
                          int n_rows, const int32_t* tile_slot_ptr, const int32_t* slot_adapter,
                          int32_t* row_adapter, int32_t* slot_of_row, void* stream) {
  CHECK_ARG(n_seg >= 1 && n_rows >= 1, "empty segment table");
  CHECK_ARG(!slot_of_row || (tile_slot_ptr && slot_adapter), "slot_of_row needs the tile slots");
  expand_segments_kernel<<<(n_rows + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      seg_start, seg_adapter, n_seg, n_rows, tile_slot_ptr, slot_adapter, row_adapter,
      slot_of_row);
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

// Overlap mode (collm_set_gemm_lean): GEMMs run "lean" pipelines and the rank-space kernels are
// sized and launched to fit next to a GEMM CTA on the same SM.
// per device (collm_set_gemm_lean applies to the caller's current device)
static std::atomic<bool> g_gemm_lean[kMaxDevices];
static unsigned long long* g_shrink_dbg = nullptr;  // debug only (COLLM_SHRINK_DEBUG)
// Shared-memory budget of the K5 reduction: lean = next to a GEMM CTA on the same SM (the
// two-stream overlap, collm_set_gemm_lean), else up to the full ring depth.
static std::atomic<bool> g_reduce_lean[kMaxDevices];
// Rank-space partition: SMs (whole TPCs) reserved for lora_shrink_tc_kernel; GEMM grids are capped
// at the rest so both are always co-resident (collm_set_rank_sms).
static std::atomic<int> g_rank_sms[kMaxDevices];

// ------------------------------------------------------------------------------------ K1


int collm_lora_shrink(const void* X, int ldx, const void* A, long long a_stride, int lda,
                      const int32_t* tiles, int n_tiles, const float* scale, const int32_t* groups,
                      int n_groups, float* H32, void* H16, void* H16lo, int ldh, void* Hslots,
                      const int32_t* slot_of_row, const int32_t* tile_slot_ptr, int32_t* signal,
                      const int32_t* gen, void* stream) {
  CHECK_ARG(X && A && tiles && scale && groups, "null input");
  CHECK_ARG(!H16lo || H16, "H16lo needs H16");
  CHECK_ARG(!signal == !gen, "signal and gen go together");
  CHECK_ARG(n_tiles >= 0, "n_tiles < 0");
  if (n_tiles == 0) return COLLM_OK;
  CHECK_ARG(n_groups >= 1 && n_groups <= kShrinkMaxGroups, "n_groups=%d out of [1,%d]", n_groups,
            kShrinkMaxGroups);
  CHECK_ARG(ldx % 8 == 0 && lda % 8 == 0 && a_stride % 8 == 0, "ldx/lda/a_stride must be x8");
  CHECK_ARG(aligned16(X) && aligned16(A), "X/A must be 16-byte aligned");
  CHECK_ARG(!Hslots || (slot_of_row && tile_slot_ptr), "Hslots needs slot_of_row, tile_slot_ptr");
  ShrinkParams p{};
  p.X = (const bf16*)X;
  p.ldx = ldx;
  p.Amat = (const bf16*)A;
  p.a_stride = a_stride;
  p.lda = lda;
  p.tiles = tiles;
  p.n_tiles = n_tiles;
  p.scale = scale;
  p.n_groups = n_groups;
  int max_ranks = 0;
  for (int g = 0; g < n_groups; ++g) {
    ShrinkGroup sg{groups[4 * g], groups[4 * g + 1], groups[4 * g + 2], groups[4 * g + 3]};
    CHECK_ARG(sg.n_ranks > 0 && sg.n_ranks <= 64 && sg.n_ranks % 8 == 0,
              "group %d: n_ranks=%d must be a multiple of 8 in [8,64]", g, sg.n_ranks);
    CHECK_ARG(sg.k_lo >= 0 && sg.k_hi > sg.k_lo && sg.k_lo % 8 == 0 && sg.k_hi % 8 == 0,
              "group %d: K range [%d,%d) must be non-empty and 8-aligned", g, sg.k_lo, sg.k_hi);
    CHECK_ARG(sg.rank_off >= 0 && sg.rank_off + sg.n_ranks <= ldh,
              "group %d: ranks [%d,%d) exceed ldh=%d", g, sg.rank_off, sg.rank_off + sg.n_ranks,
              ldh);
    p.groups[g] = sg;
    max_ranks = std::max(max_ranks, sg.n_ranks);
  }
  p.H32 = H32;
  p.H16 = (bf16*)H16;
  p.H16lo = (bf16*)H16lo;
  p.ldh = ldh;
  p.Hslots = (bf16*)Hslots;
  p.slot_of_row = slot_of_row;
  p.tile_slot_ptr = tile_slot_ptr;
  // cluster size: split K across up to 8 CTAs so the grid fills about three resident CTAs per SM
  int csize = 1;
  const int sms = num_sms_cached();
  while (csize < 8 && (long long)n_tiles * n_groups * csize * 2 <= 3LL * sms) csize *= 2;
  {
    const char* env = getenv("COLLM_SHRINK_CLUSTER");
    if (env) csize = std::max(1, std::min(8, atoi(env)));
  }
  p.csize = csize;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_tiles * csize, n_groups);
  cfg.blockDim = dim3(kShrinkWarps * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = (cudaStream_t)stream;
  p.signal = signal;
  p.gen = gen;
  {  // debug only: per-CTA start/end stamps (COLLM_SHRINK_DEBUG), read by collm_shrink_debug_copy
    static const bool dbg_on = getenv("COLLM_SHRINK_DEBUG") != nullptr;
    if (dbg_on && !g_shrink_dbg) cudaMalloc(&g_shrink_dbg, 4096 * 16);
    p.dbg = dbg_on ? g_shrink_dbg : nullptr;
  }
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (csize > 1) {  // no cluster launch unless the K range is split
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = csize;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  static const int carve_env = [] { const char* e = getenv("COLLM_SHRINK_CARVEOUT"); return e ? atoi(e) : 0; }();
  if (g_reduce_lean[cur_device()] || carve_env) {
    // next to a GEMM ask for the max-shared carveout: an SM this kernel reaches first must
    // still fit a GEMM CTA; alone, keep the default (more L1)
    attr[na].id = cudaLaunchAttributePreferredSharedMemoryCarveout;
    attr[na].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (max_ranks <= 16)
    CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_shrink_kernel<2, 4>, p));
  else if (max_ranks <= 32)
    CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_shrink_kernel<4, 3>, p));
  else if (max_ranks <= 48)
    CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_shrink_kernel<6, 2>, p));
  else
    CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_shrink_kernel<8, 2>, p));
  return COLLM_OK;
}


// ------------------------------------------------------------------------------------ K1 (tc)
int collm_set_rank_sms(int n) {
  CHECK_ARG(n >= 0 && n % 2 == 0 && n <= 64, "rank SMs %d must be even and in [0, 64]", n);
  g_rank_sms[cur_device()] = n;
  return COLLM_OK;
}
int collm_get_rank_sms(void) { return g_rank_sms[cur_device()].load(); }

// Host: work units of collm_lora_shrink_tc.  Rows go in windows of 128 consecutive rows; the
// distinct adapters of a window (from collm_plan_segments' shrink tiles) are cut into runs of
// consecutive ids whose span, rounded up to a power of two 2^c, keeps 2^c * nr <= 256 (the MMA's
// N; ids in the span without rows in the window are loaded and ignored).  Windows with base-only
// rows get one zero unit (a_lo = -1).  Units are assigned longest-first (cost ~ 128 + 2^c * nr
// rows streamed per k-block) to n_ctas CTAs.  units[4*i] = row0, n_rows, a_lo, c.
int collm_plan_shrink_windows(const int32_t* tiles, int n_tiles, int nr, int n_ctas,
                              int32_t* items, int item_cap, int32_t* n_items, int32_t* cta_ptr) {
  CHECK_ARG(n_tiles >= 0 && n_ctas >= 1, "n_tiles=%d n_ctas=%d", n_tiles, n_ctas);
  CHECK_ARG(nr >= 16 && nr % 16 == 0 && nr <= 256, "nr=%d must be a multiple of 16 <= 256", nr);
  int T = 0;
  for (int i = 0; i < n_tiles; ++i) T = std::max(T, tiles[3 * i] + tiles[3 * i + 1]);
  std::vector<int> row_ad(T, -1);
  for (int i = 0; i < n_tiles; ++i)
    for (int r = 0; r < tiles[3 * i + 1]; ++r) row_ad[tiles[3 * i] + r] = tiles[3 * i + 2];
  int max_span = 1;
  while (max_span * 2 <= 16 && max_span * 2 * nr <= 256) max_span *= 2;
  struct U { int r0, n, a, c; long long cost; };
  std::vector<U> v;
  for (int w = 0; w < T; w += kShrinkTcWindow) {
    const int n = std::min(kShrinkTcWindow, T - w);
    std::vector<int> ads;
    bool base = false;
    for (int r = w; r < w + n; ++r) {
      if (row_ad[r] < 0) base = true;
      else ads.push_back(row_ad[r]);
    }
    std::sort(ads.begin(), ads.end());
    ads.erase(std::unique(ads.begin(), ads.end()), ads.end());
    for (size_t k = 0; k < ads.size();) {
      const int a0 = ads[k];
      size_t e = k + 1;
      while (e < ads.size() && ads[e] - a0 + 1 <= max_span) ++e;
      const int span = ads[e - 1] - a0 + 1;
      int c = 0;
      while ((1 << c) < span) ++c;
      v.push_back({w, n, a0, c, (long long)kShrinkTcWindow + (1LL << c) * nr});
      k = e;
    }
    if (base) v.push_back({w, n, -1, 0, 1});
  }
  // split the K range of big units so there are about 2 chunks per CTA: S parts, the last part
  // to finish sums the fp32 partials in part order (deterministic)
  long long total = 0;
  int n_real = 0;
  for (const U& u : v) {
    total += u.a >= 0 ? u.cost : 0;
    n_real += u.a >= 0;
  }
  // measured (profiles/r02_rank_partition.md): splitting pays only when the units cannot fill
  // the CTAs at all (7B fwd down / dH gate|up: 8 units on 16 CTAs, 75 -> 38 us); with >= 3/4 of
  // a unit per CTA the partial round trip costs more than the imbalance (fwd q|k|v 25 -> 39 us)
  if (4 * n_real >= 3 * n_ctas) total = 0;
  struct Ch { int u, S, part, chunk0; long long cost; };
  std::vector<Ch> ch;
  for (size_t k = 0; k < v.size(); ++k) {
    int S = 1;
    if (v[k].a >= 0 && total > 0)
      S = (int)std::max(1LL, std::min(8LL, (2LL * n_ctas * v[k].cost + total / 2) / total));
    const int c0 = (int)ch.size();
    for (int j = 0; j < S; ++j) ch.push_back({(int)k, S, j, c0, v[k].cost / S + (S > 1 ? 8 : 0)});
  }
  CHECK_ARG((int)ch.size() <= item_cap, "shrink chunk capacity %d exceeded (%zu)", item_cap, ch.size());
  std::vector<int> order(ch.size());
  for (size_t i = 0; i < ch.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ch[x].cost > ch[y].cost; });
  std::vector<long long> load(n_ctas, 0);
  std::vector<std::vector<int>> per(n_ctas);
  for (int i : order) {
    int c = 0;
    for (int k = 1; k < n_ctas; ++k)
      if (load[k] < load[c]) c = k;
    load[c] += ch[i].cost;
    per[c].push_back(i);
  }
  int w = 0;
  for (int c = 0; c < n_ctas; ++c) {
    if (cta_ptr) cta_ptr[c] = w;
    for (int i : per[c]) {
      const U& u = v[ch[i].u];
      if (items) {
        int32_t* o = items + 8 * w;
        o[0] = u.r0; o[1] = u.n; o[2] = u.a; o[3] = u.c;
        o[4] = ch[i].S; o[5] = ch[i].part; o[6] = ch[i].chunk0; o[7] = ch[i].u;
      }
      ++w;
    }
  }
  if (cta_ptr) cta_ptr[n_ctas] = w;
  if (n_items) *n_items = w;
  return COLLM_OK;
}

size_t collm_shrink_tc_workspace_bytes(int n_chunks, int n_groups) {
  return kCounterBytes + (size_t)std::max(0, n_chunks) * std::max(1, n_groups) * 128 * 256 * sizeof(float);
}

int collm_lora_shrink_tc(const void* X, int ldx, int x_rows, const void* A, long long a_stride,
                         int lda, int a_rows, const int32_t* items, const int32_t* cta_ptr,
                         int n_ctas, int n_chunks, const int32_t* row_adapter, const float* scale,
                         const int32_t* groups, int n_groups, float* H32, void* H16, void* H16lo,
                         int ldh, void* Hslots, const int32_t* slot_of_row,
                         const int32_t* tile_slot_ptr, void* workspace, size_t ws_bytes,
                         void* stream) {
  CHECK_ARG(X && A && items && cta_ptr && scale && groups && row_adapter, "null input");
  CHECK_ARG(!H16lo || H16, "H16lo needs H16");
  CHECK_ARG(n_ctas >= 2 && n_ctas % 2 == 0, "n_ctas=%d must be even (TPC pairs)", n_ctas);
  CHECK_ARG(n_groups >= 1 && n_groups <= kShrinkTcMaxGroups, "n_groups=%d out of [1,%d]", n_groups,
            kShrinkTcMaxGroups);
  CHECK_ARG(ldx % 8 == 0 && lda % 8 == 0 && ldh % 16 == 0, "ldx/lda must be x8, ldh x16");
  CHECK_ARG(a_stride % lda == 0 && a_stride >= 0, "a_stride must be a multiple of lda");
  CHECK_ARG(aligned16(X) && aligned16(A), "X/A must be 16-byte aligned");
  CHECK_ARG(!Hslots || (slot_of_row && tile_slot_ptr), "Hslots needs slot_of_row, tile_slot_ptr");
  CHECK_ARG(x_rows >= 1 && a_rows >= 1, "empty X/A");
  ShrinkTcParams p{};
  p.n_groups = n_groups;
  p.nr = groups[1];
  int k_end = 0;
  for (int g = 0; g < n_groups; ++g) {
    const int ro = groups[4 * g], nr = groups[4 * g + 1], klo = groups[4 * g + 2], khi = groups[4 * g + 3];
    CHECK_ARG(nr == p.nr && nr % 16 == 0 && nr >= 16 && nr <= 256,
              "group %d: n_ranks=%d (all groups equal, multiple of 16 in [16,256])", g, nr);
    CHECK_ARG(klo >= 0 && khi > klo && klo % 64 == 0 && khi % 64 == 0,
              "group %d: K range [%d,%d) must be non-empty and 64-aligned", g, klo, khi);
    CHECK_ARG(ro >= 0 && ro + nr <= ldh, "group %d: ranks [%d,%d) exceed ldh=%d", g, ro, ro + nr, ldh);
    p.groups[g] = {ro, klo, khi};
    k_end = std::max(k_end, khi);
  }
  CHECK_ARG(k_end <= ldx && k_end <= lda, "K range %d exceeds ldx=%d / lda=%d", k_end, ldx, lda);
  CHECK_ARG(n_chunks >= 1 && n_chunks <= (int)kCounterCap, "n_chunks=%d", n_chunks);
  const size_t need = collm_shrink_tc_workspace_bytes(n_chunks, n_groups);
  CHECK_ARG(workspace && ws_bytes >= need, "shrink_tc workspace too small: %zu < %zu", ws_bytes, need);
  p.counters = (int32_t*)workspace;
  p.partials = (float*)((char*)workspace + kCounterBytes);
  p.items = items;
  p.cta_ptr = cta_ptr;
  p.row_adapter = row_adapter;
  p.a_single = a_stride == 0;
  p.scale = scale;
  p.H32 = H32;
  p.H16 = (bf16*)H16;
  p.H16lo = (bf16*)H16lo;
  p.ldh = ldh;
  p.Hslots = (bf16*)Hslots;
  p.slot_of_row = slot_of_row;
  p.tile_slot_ptr = tile_slot_ptr;
  // A viewed as [adapter][rank row][K]: rows per adapter = a_stride / lda (single adapter when
  // a_stride == 0: all a_rows rows)
  const long long rows_per_ad = a_stride > 0 ? a_stride / lda : a_rows;
  const long long n_ad = a_stride > 0 ? std::max(1LL, (long long)a_rows / rows_per_ad) : 1;
  auto fn = encode_fn();
  if (!fn) return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  ShrinkTcMaps maps;
  for (int c = 0; c < kShrinkTcClasses; ++c) {
    const int na = 1 << c;
    if (c > 0 && na * p.nr > 256) {  // class unusable at this width (the planner never emits it)
      maps.x[c] = maps.x[0];
      maps.a[c] = maps.a[0];
      p.kb[c] = p.kb[0];
      continue;
    }
    // k-blocks per stage: fill the ~64 KB stage (bigger copies stream faster per SM, sm_bw.py)
    int kb = (int)(kShrinkTcStageBytes / ((uint32_t)(kShrinkTcWindow + na * p.nr) * 128));
    kb = std::max(1, std::min(16, kb));
    p.kb[c] = kb;
    int rc = make_tmap_kblocks(&maps.x[c], X, x_rows, ldx, k_end / 64, kShrinkTcWindow, kb);
    if (rc) return rc;
    cuuint64_t dims[4] = {64, (cuuint64_t)rows_per_ad, (cuuint64_t)n_ad, (cuuint64_t)(k_end / 64)};
    cuuint64_t strides[3] = {(cuuint64_t)lda * 2,
                             (cuuint64_t)(a_stride > 0 ? a_stride * 2 : rows_per_ad * lda * 2), 128};
    cuuint32_t box[4] = {64, (cuuint32_t)p.nr, (cuuint32_t)na, (cuuint32_t)kb};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(&maps.a[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(A), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return fail(COLLM_ECUDA, "cuTensorMapEncodeTiled (stacked adapters) failed (%d)", (int)r);
  }
  {
    static bool configured[kMaxDevices] = {};
    const int dev = cur_device();
    std::lock_guard<std::mutex> lk(g_state_mu);
    if (!configured[dev]) {
      CUDA_TRY(cudaFuncSetAttribute(lora_shrink_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    ShrinkTcSmem::kTotal));
      configured[dev] = true;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_ctas);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = ShrinkTcSmem::kTotal;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // CTA pairs: the grid holds whole TPCs
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_shrink_tc_kernel, maps, p));
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K9
static int flash_setup(FlashParams& p, const void* q, int ldq, const void* k, int ldk, const void* v,
                       int ldv, int T, int n_heads, int n_kv_heads, int head_dim,
                       const int32_t* row_start, const int32_t* row_end, float scale) {
  CHECK_ARG(q && k && v && row_start && row_end, "null input");
  CHECK_ARG(head_dim == kFaD, "head_dim=%d (this build: %d)", head_dim, kFaD);
  CHECK_ARG(n_heads >= 1 && n_kv_heads >= 1 && n_heads % n_kv_heads == 0,
            "n_heads=%d must be a multiple of n_kv_heads=%d", n_heads, n_kv_heads);
  CHECK_ARG(T >= 1, "empty batch (T=%d)", T);
  CHECK_ARG(ldq % 8 == 0 && ldk % 8 == 0 && ldv % 8 == 0 && aligned16(q) && aligned16(k) && aligned16(v),
            "q/k/v must be 16-byte aligned with x8 leading dimensions");
  CHECK_ARG(ldq >= n_heads * kFaD && ldk >= n_kv_heads * kFaD && ldv >= n_kv_heads * kFaD,
            "leading dimensions too small for the heads");
  p = FlashParams{};
  p.q = (const bf16*)q; p.k = (const bf16*)k; p.v = (const bf16*)v;
  p.ldq = ldq; p.ldk = ldk; p.ldv = ldv;
  p.row_start = row_start;
  p.row_end = row_end;
  p.T = T; p.n_heads = n_heads; p.n_kv_heads = n_kv_heads;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.stat_ld = T;
  return COLLM_OK;
}

static int flash_launch(void (*kernel)(const FlashParams), int smem, dim3 grid, const FlashParams& p, cudaStream_t st) {
  static std::mutex mu;
  static bool done[kMaxDevices][4] = {};
  const int dev = cur_device();
  const int slot = smem == 81920 ? 0 : smem == 99840 ? 1 : smem == 49152 ? 3 : 2;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!done[dev][slot]) {
      CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      done[dev][slot] = true;
    }
  }
  kernel<<<grid, kFaThreads, smem, st>>>(p);
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

// Kernel selection per device (like the other mode switches): -1 = not set (the env default)
static std::atomic<int> g_flash_impl[kMaxDevices];
static std::atomic<int> g_reduce_impl[kMaxDevices];
static int impl_of(std::atomic<int>* per_dev, const char* env) {
  const int v = per_dev[cur_device()].load();
  if (v > 0) return v - 1;
  const char* e = getenv(env);
  return e ? (atoi(e) != 0) : 1;
}

int collm_set_flash_impl(int tc) {
  CHECK_ARG(tc == 0 || tc == 1, "flash impl %d (0 = mma.sync, 1 = tcgen05)", tc);
  g_flash_impl[cur_device()].store(tc + 1);
  return COLLM_OK;
}
int collm_get_flash_impl(void) { return impl_of(g_flash_impl, "COLLM_FA_TC"); }

int collm_flash_attention_fwd(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                              void* out, int ldo, float* lse, int T, int n_heads, int n_kv_heads,
                              int head_dim, const int32_t* row_start, const int32_t* row_end,
                              float scale, int stat_ld, void* stream) {
  FlashParams p;
  int rc = flash_setup(p, q, ldq, k, ldk, v, ldv, T, n_heads, n_kv_heads, head_dim, row_start, row_end, scale);
  if (rc) return rc;
  CHECK_ARG(out && lse && ldo % 8 == 0 && ldo >= n_heads * kFaD && aligned16(out), "bad out/lse");
  p.out = (bf16*)out; p.ldo = ldo; p.lse = lse;
  if (stat_ld > 0) p.stat_ld = stat_ld;
  CHECK_ARG(p.stat_ld >= T, "stat_ld=%d < T=%d", p.stat_ld, T);
  if (collm_get_flash_impl()) {  // the tcgen05/TMEM forward (flash_tc.cuh)
    CHECK_ARG(ldq % 8 == 0 && ldk % 8 == 0 && ldv % 8 == 0, "x8 leading dimensions");
    FlashTcMaps maps;
    int rc = make_tmap(&maps.q, q, ldq, T, ldq, 64, 128);
    if (!rc) rc = make_tmap(&maps.k, k, ldk, T, ldk, 64, 128);
    if (!rc) rc = make_tmap(&maps.v, v, ldv, T, ldv, 64, 128);
    if (rc) return rc;
    static bool configured[kMaxDevices] = {};
    const int dev = cur_device();
    {
      std::lock_guard<std::mutex> lk(g_state_mu);
      if (!configured[dev]) {
        CUDA_TRY(cudaFuncSetAttribute(flash_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      FlashTcSmem::kTotal));
        configured[dev] = true;
      }
    }
    // persistent: one CTA per SM walks (query tile, head) items
    const int n_items = (T + kFtcRows - 1) / kFtcRows * n_heads;
    flash_fwd_tc_kernel<<<std::min(n_items, num_sms_cached()), 384, FlashTcSmem::kTotal,
                          (cudaStream_t)stream>>>(maps, p);
    CUDA_TRY(cudaGetLastError());
    return COLLM_OK;
  }
  static const int st_env = [] { const char* e = getenv("COLLM_FA_STAGES"); return e ? atoi(e) : 1; }();
  if (st_env == 2)
    return flash_launch(flash_fwd_kernel<2>, 81920, dim3((T + kFaBM - 1) / kFaBM, n_heads), p,
                        (cudaStream_t)stream);
  return flash_launch(flash_fwd_kernel<1>, 49152, dim3((T + kFaBM - 1) / kFaBM, n_heads), p,
                      (cudaStream_t)stream);
}

int collm_flash_attention_bwd(const void* q, int ldq, const void* k, int ldk, const void* v, int ldv,
                              const void* out, int ldo, const void* dout, int lddo, const float* lse,
                              float* delta, void* dq, int lddq, void* dk, int lddk, void* dv, int lddv,
                              int T, int n_heads, int n_kv_heads, int head_dim,
                              const int32_t* row_start, const int32_t* row_end, float scale,
                              int stat_ld, void* stream) {
  FlashParams p;
  int rc = flash_setup(p, q, ldq, k, ldk, v, ldv, T, n_heads, n_kv_heads, head_dim, row_start, row_end, scale);
  if (rc) return rc;
  CHECK_ARG(out && dout && lse && delta && dq && dk && dv, "null backward operand");
  CHECK_ARG(ldo % 8 == 0 && lddo % 8 == 0 && lddq % 2 == 0 && lddk % 2 == 0 && lddv % 2 == 0 &&
                aligned16(dout) && aligned16(out),
            "bad backward leading dimensions / alignment");
  p.out = (bf16*)out; p.ldo = ldo; p.lse = const_cast<float*>(lse);
  p.dout = (const bf16*)dout; p.lddo = lddo; p.delta = delta;
  p.dq = (bf16*)dq; p.dk = (bf16*)dk; p.dv = (bf16*)dv;
  p.lddq = lddq; p.lddk = lddk; p.lddv = lddv;
  if (stat_ld > 0) p.stat_ld = stat_ld;
  CHECK_ARG(p.stat_ld >= T, "stat_ld=%d < T=%d", p.stat_ld, T);
  cudaStream_t st = (cudaStream_t)stream;
  const int warps = T * n_heads;
  flash_delta_kernel<<<(warps + 7) / 8, 256, 0, st>>>(p);
  CUDA_TRY(cudaGetLastError());
  if (collm_get_flash_impl() && lddq % 8 == 0 && lddk % 8 == 0 && lddv % 8 == 0 && aligned16(dq) &&
      aligned16(dk) && aligned16(dv)) {
    // tcgen05/TMEM backward (flash_bwd_tc.cuh)
    FlashBwdTcMaps maps;
    int rc2 = make_tmap_kblocks(&maps.q64, q, T, ldq, ldq / 64, 64, 2);
    if (!rc2) rc2 = make_tmap_kblocks(&maps.o64, dout, T, lddo, lddo / 64, 64, 2);
    if (!rc2) rc2 = make_tmap(&maps.k128, k, ldk, T, ldk, 64, 128);
    if (!rc2) rc2 = make_tmap(&maps.v128, v, ldv, T, ldv, 64, 128);
    if (!rc2) rc2 = make_tmap(&maps.q128, q, ldq, T, ldq, 64, 128);
    if (!rc2) rc2 = make_tmap(&maps.o128, dout, lddo, T, lddo, 64, 128);
    if (!rc2) rc2 = make_tmap_kblocks(&maps.k64, k, T, ldk, ldk / 64, 64, 2);
    if (!rc2) rc2 = make_tmap_kblocks(&maps.v64, v, T, ldv, ldv / 64, 64, 2);
    if (rc2) return rc2;
    static bool configured[kMaxDevices] = {};
    const int dev = cur_device();
    {
      std::lock_guard<std::mutex> lk(g_state_mu);
      if (!configured[dev]) {
        CUDA_TRY(cudaFuncSetAttribute(flash_bwd_dkdv_tc_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, FbDkdvSmem::kTotal));
        CUDA_TRY(cudaFuncSetAttribute(flash_bwd_dq_tc_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, FbDqSmem::kTotal));
        configured[dev] = true;
      }
    }
    static const int fb_debug = [] { const char* e = getenv("COLLM_DEBUG_FB"); return e ? atoi(e) : 0; }();
    if (fb_debug) CUDA_TRY(cudaMemcpyToSymbolAsync(g_fb_debug, &fb_debug, sizeof(int), 0, cudaMemcpyHostToDevice, st));
    const int t128 = (T + 127) / 128;
    flash_bwd_dkdv_tc_kernel<<<dim3(t128, n_kv_heads), 384, FbDkdvSmem::kTotal, st>>>(maps, p);
    CUDA_TRY(cudaGetLastError());
    flash_bwd_dq_tc_kernel<<<std::min(t128 * n_heads, num_sms_cached()), 384, FbDqSmem::kTotal, st>>>(maps, p);
    CUDA_TRY(cudaGetLastError());
    return COLLM_OK;
  }
  const int tiles = (T + kFaBM - 1) / kFaBM;
  rc = flash_launch(flash_bwd_dkdv_kernel, 99840, dim3(tiles, n_kv_heads), p, st);
  if (rc) return rc;
  return flash_launch(flash_bwd_dq_kernel, 98304, dim3(tiles, n_heads), p, st);
}


// ------------------------------------------------------------------------------------ expand rows
int collm_lora_expand_rows(void* Y, int ldy, int N, const void* H16, int ldh, const void* B,
                           int r_pad, const int32_t* row_adapter, const int32_t* tiles, int n_tiles,
                           int T, int n_sub, const int32_t* sub_n_start, const int32_t* sub_h_col,
                           void* stream) {
  CHECK_ARG(Y && H16 && B && row_adapter && tiles, "null input");
  CHECK_ARG(n_tiles >= 0 && T >= 1 && N >= 8 && N % 8 == 0, "n_tiles=%d T=%d N=%d", n_tiles, T, N);
  if (n_tiles == 0) return COLLM_OK;
  CHECK_ARG(r_pad == 16 || r_pad == 32 || r_pad == 64, "r_pad=%d must be 16, 32 or 64", r_pad);
  CHECK_ARG(ldy % 8 == 0 && ldh % 8 == 0 && aligned16(Y) && aligned16(H16) && aligned16(B),
            "Y/H16/B must be 16-byte aligned with x8 leading dimensions");
  CHECK_ARG(n_sub >= 1 && n_sub <= 4, "n_sub=%d", n_sub);
  ExpandRowsParams p{};
  p.Y = (bf16*)Y; p.ldy = ldy; p.N = N;
  p.H = (const bf16*)H16; p.ldh = ldh;
  p.B = (const bf16*)B; p.r_pad = r_pad;
  p.row_adapter = row_adapter; p.tiles = tiles; p.n_tiles = n_tiles; p.T = T;
  p.n_sub = n_sub;
  for (int i = 0; i <= 4; ++i) p.sub_n_start[i] = (i <= n_sub && sub_n_start) ? sub_n_start[i] : N;
  if (!sub_n_start) p.sub_n_start[0] = 0;
  for (int i = 0; i < 4; ++i) {
    p.sub_h_col[i] = (i < n_sub && sub_h_col) ? sub_h_col[i] : 0;
    CHECK_ARG(p.sub_h_col[i] % 8 == 0 && p.sub_h_col[i] + r_pad <= ldh, "sub %d: H columns exceed ldh", i);
  }
  for (int i = 1; i < n_sub; ++i)
    CHECK_ARG(p.sub_n_start[i] % 128 == 0, "sub boundaries must be multiples of 128");
  lora_expand_rows_kernel<<<dim3(n_tiles * 32, (N + 127) / 128), 256, 0, (cudaStream_t)stream>>>(p);
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K2/K3


int collm_shrink_debug_copy(void* host_dst, size_t bytes) {
  if (!g_shrink_dbg) return fail(COLLM_EINVAL, "no shrink debug timeline (COLLM_SHRINK_DEBUG)");
  CUDA_TRY(cudaMemcpy(host_dst, g_shrink_dbg, bytes, cudaMemcpyDeviceToHost));
  return COLLM_OK;
}
// debug-only: device pointer of the last GEMM's timeline (COLLM_GEMM_DEBUG set)
unsigned long long* collm_debug_timeline = nullptr;
// debug-only: total ns / count of LoRA-operand flag waits since the last call (COLLM_GEMM_DEBUG)
int collm_gemm_wait_stats(unsigned long long* ns, unsigned long long* waits) {
  CUDA_TRY(cudaMemcpyFromSymbol(ns, g_lora_wait_ns, sizeof(*ns)));
  CUDA_TRY(cudaMemcpyFromSymbol(waits, g_lora_waits, sizeof(*waits)));
  const unsigned long long z = 0;
  CUDA_TRY(cudaMemcpyToSymbol(g_lora_wait_ns, &z, sizeof(z)));
  CUDA_TRY(cudaMemcpyToSymbol(g_lora_waits, &z, sizeof(z)));
  return COLLM_OK;
}
int collm_gemm_debug_copy(void* host_dst, size_t bytes) {
  if (!collm_debug_timeline) return fail(COLLM_EINVAL, "no GEMM debug timeline (COLLM_GEMM_DEBUG)");
  CUDA_TRY(cudaMemcpy(host_dst, collm_debug_timeline, bytes, cudaMemcpyDeviceToHost));
  return COLLM_OK;
}

size_t collm_gemm_workspace_bytes(int bn) {
  const int b = bn == 128 ? 128 : 256;
  return kCounterBytes + (size_t)num_sms_cached() * kGemmBM * b * sizeof(float);
}

int collm_gemm_lora(const void* A, int lda, const void* B, int ldb, void* Y, int ldy, int M, int N,
                    int K, const void* Hslots, int ldh, int h_rows, const void* LB, int ld_lb,
                    int lb_rows, const int32_t* tile_slot_ptr, const int32_t* slot_adapter,
                    int lora_rank, int lb_rows_per_adapter, int n_sub, const int32_t* sub_n_start,
                    const int32_t* sub_h_col, int bn, void* workspace, size_t ws_bytes,
                    const int32_t* lora_flag, const int32_t* gen, int lora_pdl, void* stream) {
  return collm_gemm_lora_ex(A, lda, B, ldb, Y, ldy, M, N, K, Hslots, ldh, h_rows, LB, ld_lb,
                            lb_rows, tile_slot_ptr, slot_adapter, lora_rank, lb_rows_per_adapter,
                            n_sub, sub_n_start, sub_h_col, bn, workspace, ws_bytes, lora_flag, gen,
                            lora_pdl, nullptr, stream);
}

int collm_gemm_lora_ex(const void* A, int lda, const void* B, int ldb, void* Y, int ldy, int M,
                       int N, int K, const void* Hslots, int ldh, int h_rows, const void* LB,
                       int ld_lb, int lb_rows, const int32_t* tile_slot_ptr,
                       const int32_t* slot_adapter, int lora_rank, int lb_rows_per_adapter,
                       int n_sub, const int32_t* sub_n_start, const int32_t* sub_h_col, int bn,
                       void* workspace, size_t ws_bytes, const int32_t* lora_flag,
                       const int32_t* gen, int lora_pdl, const int32_t* tile_skip, void* stream) {
  CHECK_ARG(A && B && Y, "null operand");
  CHECK_ARG(!lora_flag == !gen, "lora_flag and gen go together");
  CHECK_ARG(M >= 1 && N >= 1 && K >= 1, "empty GEMM M=%d N=%d K=%d", M, N, K);
  CHECK_ARG(K % 8 == 0 && N % 8 == 0, "K=%d and N=%d must be multiples of 8", K, N);
  CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ldy % 8 == 0 && lda >= K && ldb >= K && ldy >= N,
            "bad leading dimensions lda=%d ldb=%d ldy=%d", lda, ldb, ldy);
  CHECK_ARG(aligned16(A) && aligned16(B) && aligned16(Y), "operands must be 16-byte aligned");
  const bool lora = tile_slot_ptr != nullptr;
  if (n_sub <= 0) n_sub = 1;
  CHECK_ARG(n_sub <= kMaxSub, "n_sub=%d > %d", n_sub, kMaxSub);

  // N tile: 256 unless the sub-projection boundaries (or a narrow N) call for 128; stream-K
  // removes the wave-quantization reason to prefer narrower tiles.
  static const int max_sms_env = [] { const char* e = getenv("COLLM_GEMM_MAX_SMS"); return e ? atoi(e) : 0; }();
  const int rank_sms = g_rank_sms[cur_device()].load();  // reserved for the rank-space kernels
  const int sms_avail = num_sms_cached() - rank_sms;
  const int sms = max_sms_env > 0 ? std::min(sms_avail, max_sms_env) : sms_avail;  // debug cap
  auto aligned_to = [&](int t) {
    if (!lora || !sub_n_start) return true;
    for (int i = 1; i < n_sub; ++i)
      if (sub_n_start[i] % t) return false;
    return true;
  };
  // Tile / schedule choice by a cost model calibrated on B200 (tools/gemm_bench.py, µs): time of
  // one 64-deep k-block of a unit tile — 1-CTA 128x256: 0.48, 1-CTA 128x128: 0.34, CTA-pair
  // 256x256: 0.43, CTA-pair 256x128: 0.34 — times the k-blocks on the critical path;
  // data-parallel: waves x k-blocks; hybrid stream-K: (full waves - 1) data-parallel + the rest
  // split evenly, plus a fix-up of ~12 + 8 x (parts per split tile) µs.
  // MC = 2: split-2 in 4-CTA clusters — the two pairs halving a tile's K swap their partials
  // through distributed shared memory (~1.5 us) instead of global memory + flags (~4 us); needs
  // every tile's cluster co-resident (tiles <= co-resident 4-CTA clusters, 33 on B200).
  struct Cand { int cg, mc, bn, sched; double cost; };
  auto env_int = [](const char* k, int d) { const char* e = getenv(k); return e ? atoi(e) : d; };
  const int force_cg = env_int("COLLM_GEMM_CG", 0), force_bn = env_int("COLLM_GEMM_BN", bn);
  const int force_mc = env_int("COLLM_GEMM_MC", 0);
  const char* sched_env = getenv("COLLM_GEMM_SCHED");
  const int force_sched = !sched_env ? -1 : strcmp(sched_env, "dp") == 0 ? 0
                          : strcmp(sched_env, "hybrid") == 0 ? 1 : strcmp(sched_env, "sknofix") == 0 ? 2
                          : strcmp(sched_env, "noload") == 0 ? 3
                          : strcmp(sched_env, "split2") == 0 ? 4 : -1;
  Cand best{0, 0, 0, 0, 1e30};
  const double nk = (K + kGemmBK - 1) / kGemmBK;
  int force_sched_eff = force_sched;
  for (int attempt = 0; attempt < 2 && best.cg == 0; ++attempt, force_sched_eff = -1)
  for (int cg : {2, 1})
  for (int mc : {1, 2, 3}) {
    if (force_cg && cg != force_cg) continue;
    if (mc != 1 && cg != 2) continue;
    if (mc == 3 && force_mc != 3) continue;  // A-multicast clusters: opt-in (COLLM_GEMM_MC=3)
    if (force_mc && mc != force_mc && attempt == 0) continue;  // retry: any, like the schedule
    const long long units = mc == 3 ? max_gemm_clusters<256, 6, 2, 3>() : sms / cg;
    const long long nmu = (M + kGemmBM * cg - 1) / (kGemmBM * cg);
    for (int b : {256, 128}) {
      if (force_bn && b != force_bn) continue;
      if (!aligned_to(b) || (b == 256 && N <= 128 && !force_bn)) continue;
      const double kb = cg == 2 ? (b == 256 ? 0.43 : 0.34) : (b == 256 ? 0.48 : 0.34);
      const long long tiles = nmu * (((N + b - 1) / b + (mc == 3 ? 1 : 0)) / (mc == 3 ? 2 : 1));
      if (mc == 3 && b != 256) continue;
      for (int sc : {0, 1, 4}) {
        if (mc == 3 && sc != 0) continue;  // data-parallel only
        if (force_sched_eff >= 0 && (force_sched_eff == 2 ? 1 : force_sched_eff == 3 ? 0 : force_sched_eff) != sc) continue;
        double cost;
        if (sc == 4) {
          // split-2: every tile's K halved over two units that swap half-tile partials (2-CTA
          // pairs only, needs 2 x tiles <= units); calibrated swap cost ~4 us
          if (cg != 2 || 2 * tiles > units || nk < 2) continue;  // both halves non-empty
          if (mc == 2 && tiles > (b == 256 ? max_gemm_clusters<256, 6, 2, 2>()
                                           : max_gemm_clusters<128, 8, 2, 2>()) - rank_sms / 2)
            continue;
          cost = std::ceil(nk / 2.0) * kb + (mc == 2 ? 1.5 : 4.0);
        } else if (mc == 2) {
          continue;  // 4-CTA clusters only for split-2
        } else if (sc == 0) {
          cost = (double)((tiles + units - 1) / units) * nk * kb;
        } else {
          const long long waves = tiles / units;
          const long long dp_waves = waves >= 1 ? waves - 1 : 0;
          const long long sk_tiles = tiles - dp_waves * units;
          const double parts = std::min(3.0, std::max(1.0, (double)units / sk_tiles));
          cost = dp_waves * nk * kb + (double)sk_tiles * nk * kb / units + 12.0 + 8.0 * parts;
        }
        if (cost < best.cost) best = {cg, mc, b, sc, cost};
      }
    }
  }
  if (best.cg == 0) return fail(COLLM_EINVAL, "no GEMM tile fits (sub-projection boundaries must be x128)");
  const int cg = best.cg, mc = best.mc;
  bn = best.bn;
  const int sched = (force_sched == 2 || force_sched == 3) ? force_sched : best.sched;
  const int nm = (M + kGemmBM * cg - 1) / (kGemmBM * cg);
  CHECK_ARG(nm <= kMaxMTiles, "M=%d exceeds %d rows", M, kMaxMTiles * kGemmBM);
  CHECK_ARG(bn == 128 || bn == 256, "bn must be 0, 128 or 256");
  CHECK_ARG(aligned_to(bn), "sub-projection boundaries are not multiples of bn=%d", bn);

  GemmLoraParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.Y = (bf16*)Y;
  p.ldy = ldy;
  p.num_m_tiles = nm;
  p.num_n_tiles = (N + bn - 1) / bn;
  p.n_sub = n_sub;
  p.sub_n_start[0] = 0;
  for (int i = 0; i <= kMaxSub; ++i) p.sub_n_start[i] = (i == 0) ? 0 : N;
  for (int i = 0; i < kMaxSub; ++i) p.sub_h_col[i] = 0;

  CUtensorMap ta, tb, th, tlb, ty;
  int rc = make_tmap(&ta, A, K, M, lda, kGemmBK, mc == 3 ? kGemmBM / 2 : kGemmBM);
  if (rc) return rc;
  rc = make_tmap(&ty, Y, N, M, ldy, 32, 32);  // epilogue TMA stores, [32 x 32] boxes
  if (rc) return rc;
  rc = make_tmap(&tb, B, K, N, ldb, kGemmBK, bn / cg);
  if (rc) return rc;
  if (lora) {
    CHECK_ARG(Hslots && LB && slot_adapter, "LoRA GEMM needs Hslots, LB and slot_adapter");
    CHECK_ARG(lora_rank > 0 && lora_rank % 16 == 0, "lora_rank=%d must be a multiple of 16",
              lora_rank);
    CHECK_ARG(ldh % 8 == 0 && ld_lb % 8 == 0 && aligned16(Hslots) && aligned16(LB),
              "Hslots/LB must be 16-byte aligned with x8 leading dimensions");
    CHECK_ARG(h_rows >= 1 && lb_rows >= 1, "empty Hslots/LB");
    // widest TMA/UMMA chunk (64/32/16 columns = 128/64/32-byte swizzle) dividing the LoRA width
    const int lrc = (lora_rank % 64 == 0) ? 64 : (lora_rank % 32 == 0) ? 32 : 16;
    p.tile_slot_ptr = tile_slot_ptr;
    p.tile_skip = tile_skip;
    p.slot_adapter = slot_adapter;
    p.lora_rc = lrc;
    p.lora_chunks = lora_rank / lrc;
    p.lora_per_stage = kGemmBK / lrc;
    p.lb_rows_per_adapter = lb_rows_per_adapter;
    if (sub_n_start) {
      CHECK_ARG(sub_n_start[0] == 0 && sub_n_start[n_sub] == N, "sub_n_start must span [0, N)");
      for (int i = 0; i <= n_sub; ++i) p.sub_n_start[i] = sub_n_start[i];
      for (int i = n_sub + 1; i <= kMaxSub; ++i) p.sub_n_start[i] = N;
    }
    for (int i = 0; i < n_sub; ++i) {
      p.sub_h_col[i] = sub_h_col ? sub_h_col[i] : 0;
      CHECK_ARG(p.sub_h_col[i] % 8 == 0 && p.sub_h_col[i] + lora_rank <= ldh,
                "sub %d: H columns [%d,%d) exceed ldh=%d", i, p.sub_h_col[i],
                p.sub_h_col[i] + lora_rank, ldh);
    }
    CHECK_ARG(lora_rank <= ld_lb, "lora_rank %d exceeds LB width %d", lora_rank, ld_lb);
    rc = make_tmap(&th, Hslots, ldh, h_rows, ldh, lrc, kGemmBM);
    if (rc) return rc;
    rc = make_tmap(&tlb, LB, ld_lb, lb_rows, ld_lb, lrc, bn / cg);
    if (rc) return rc;
  } else {
    th = ta;
    tlb = tb;
  }
  // persistent grid: one CTA (pair) per SM (pair), never more units than k-stages (every
  // stream-K range non-empty)
  const long long min_work = (long long)nm * p.num_n_tiles * ((K + kGemmBK - 1) / kGemmBK);
  const int grid = sched == 4 ? cg * 2 * nm * p.num_n_tiles
                   : mc == 3 ? 4 * (int)std::min<long long>(max_gemm_clusters<256, 6, 2, 3>(),
                                                            (long long)nm * ((p.num_n_tiles + 1) / 2))
                             : cg * (int)std::min<long long>(sms / cg, min_work);
  p.sched = sched;
  {
    // grouped raster when A does not stay L2-resident across an N column's wave (large M): the
    // data-parallel tiles go in groups of 8 N columns (measured: see DESIGN.md §GEMM raster)
    static const int gn_env = [] { const char* e = getenv("COLLM_GEMM_RASTER_GN"); return e ? atoi(e) : -1; }();
    const double a_bytes = 2.0 * M * K;
    p.raster_gn = gn_env >= 0 ? gn_env : (a_bytes > 32e6 ? 8 : 1);
  }
  p.lora_flag = lora ? lora_flag : nullptr;
  p.gen = gen;
  {
    static const bool prologue_pdl = [] { const char* e = getenv("COLLM_GEMM_PDL"); return e && atoi(e) != 0; }();
    p.pdl_mode = (lora && lora_pdl) ? 2 : (prologue_pdl ? 1 : 0);
    static const bool no_wait = getenv("COLLM_DEBUG_GEMM_NO_LORA_WAIT") != nullptr;
    p.debug_no_wait = no_wait ? 1 : 0;
  }
  const size_t need = collm_gemm_workspace_bytes(bn);
  CHECK_ARG(workspace && ws_bytes >= need, "gemm workspace too small: %zu < %zu", ws_bytes, need);
  p.flags = (int32_t*)workspace;
  {
    static unsigned long long* dbg_ptr = nullptr;
    const char* dbg_env = getenv("COLLM_GEMM_DEBUG");
    if (dbg_env && !dbg_ptr) {
      cudaMalloc(&dbg_ptr, 256 * 32 * 8);
      fprintf(stderr, "collm: co-resident GEMM clusters: pairs %d, 4-CTA %d (lean %d)\n",
              max_gemm_clusters<256, 6, 2, 1>(), max_gemm_clusters<256, 6, 2, 2>(),
              max_gemm_clusters<256, 5, 2, 2>());
    }
    // (COLLM_GEMM_DEBUG=2: no memset node, which would break a programmatic launch overlap)
    if (dbg_env && atoi(dbg_env) != 2) cudaMemsetAsync(dbg_ptr, 0, 256 * 32 * 8, (cudaStream_t)stream);
    p.dbg = dbg_env ? dbg_ptr : nullptr;
    collm_debug_timeline = p.dbg;
  }
  p.partials = (float*)((char*)workspace + kCounterBytes);
  cudaStream_t st = (cudaStream_t)stream;
  // "lean" pipelines (~128 KB smem, <= 128 registers) leave room on every SM for one CTA of the
  // LoRA kernels running concurrently on a second stream (collm_set_gemm_lean / COLLM_GEMM_LEAN)
  const char* lean_env = getenv("COLLM_GEMM_LEAN");
  const bool lean = lean_env ? atoi(lean_env) != 0 : g_gemm_lean[cur_device()].load();
  if (mc == 3) {
    if (lean) return launch_gemm<256, 5, 2, 3>(ta, tb, th, tlb, ty, p, grid, st);
    return launch_gemm<256, 6, 2, 3>(ta, tb, th, tlb, ty, p, grid, st);
  }
  if (mc == 2) {
    if (lean) {
      if (bn == 256) return launch_gemm<256, 5, 2, 2>(ta, tb, th, tlb, ty, p, grid, st);
      return launch_gemm<128, 6, 2, 2>(ta, tb, th, tlb, ty, p, grid, st);
    }
    if (bn == 256) return launch_gemm<256, 6, 2, 2>(ta, tb, th, tlb, ty, p, grid, st);
    return launch_gemm<128, 8, 2, 2>(ta, tb, th, tlb, ty, p, grid, st);
  }
  if (cg == 2) {
    if (lean) {
      static const int lean_stages = [] { const char* e = getenv("COLLM_GEMM_LEAN_STAGES"); return e ? atoi(e) : 5; }();
      if (bn == 256) {
        if (lean_stages == 5) return launch_gemm<256, 5, 2>(ta, tb, th, tlb, ty, p, grid, st);
        return launch_gemm<256, 4, 2>(ta, tb, th, tlb, ty, p, grid, st);
      }
      if (lean_stages == 5) return launch_gemm<128, 6, 2>(ta, tb, th, tlb, ty, p, grid, st);
      return launch_gemm<128, 5, 2>(ta, tb, th, tlb, ty, p, grid, st);
    }
    if (bn == 256) return launch_gemm<256, 6, 2>(ta, tb, th, tlb, ty, p, grid, st);
    return launch_gemm<128, 8, 2>(ta, tb, th, tlb, ty, p, grid, st);
  }
  if (lean) {
    if (bn == 256) return launch_gemm<256, 3, 1>(ta, tb, th, tlb, ty, p, grid, st);
    return launch_gemm<128, 4, 1>(ta, tb, th, tlb, ty, p, grid, st);
  }
  if (bn == 256) return launch_gemm<256, 4, 1>(ta, tb, th, tlb, ty, p, grid, st);
  return launch_gemm<128, 6, 1>(ta, tb, th, tlb, ty, p, grid, st);
}

// Force-load every kernel of the library now (CUDA lazy module loading would otherwise load a
// kernel at its first launch, which can implicitly synchronize the device — fatal when a GEMM is
// already running and waiting for the very shrink being launched on another stream).
int collm_preload(void) {
  cudaFuncAttributes a;
#define COLLM_PRELOAD(k) CUDA_TRY(cudaFuncGetAttributes(&a, k))
  COLLM_PRELOAD(expand_segments_kernel);
  COLLM_PRELOAD((lora_shrink_kernel<2, 4>));
  COLLM_PRELOAD((lora_shrink_kernel<4, 3>));
  COLLM_PRELOAD((lora_shrink_kernel<6, 2>));
  COLLM_PRELOAD((lora_shrink_kernel<8, 2>));
  COLLM_PRELOAD(lora_shrink_tc_kernel);
  COLLM_PRELOAD(flash_fwd_kernel<1>);
  COLLM_PRELOAD(flash_fwd_tc_kernel);
  COLLM_PRELOAD(flash_fwd_kernel<2>);
  COLLM_PRELOAD(lora_expand_rows_kernel);
  COLLM_PRELOAD(flash_delta_kernel);
  COLLM_PRELOAD(flash_bwd_dkdv_kernel);
  COLLM_PRELOAD(flash_bwd_dq_kernel);
  COLLM_PRELOAD((gemm_lora_kernel<256, 6, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 8, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 5, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 6, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 4, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 5, 2, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 6, 2, 2>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 8, 2, 2>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 5, 2, 2>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 6, 2, 2>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 6, 2, 3>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 5, 2, 3>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 4, 1, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 6, 1, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<256, 3, 1, 1>));
  COLLM_PRELOAD((gemm_lora_kernel<128, 4, 1, 1>));
  COLLM_PRELOAD((lora_reduce_kernel<16, 4>));
  COLLM_PRELOAD((lora_reduce_kernel<32, 4>));
  COLLM_PRELOAD((lora_reduce_kernel<48, 4>));
  COLLM_PRELOAD((lora_reduce_kernel<16, 3>));
  COLLM_PRELOAD((lora_reduce_kernel<32, 3>));
  COLLM_PRELOAD((lora_reduce_kernel<48, 3>));
  COLLM_PRELOAD((lora_reduce_kernel<64, 3>));
  COLLM_PRELOAD(lora_apply_kernel);
  COLLM_PRELOAD((cross_entropy_kernel<8, 512>));
  COLLM_PRELOAD(paged_attention_kernel<1>);
  COLLM_PRELOAD(paged_attention_kernel<2>);
  COLLM_PRELOAD(paged_attention_kernel<4>);
  COLLM_PRELOAD(paged_attention_kernel<8>);
  COLLM_PRELOAD(paged_attention_tc_kernel<1>);
  COLLM_PRELOAD(paged_attention_tc_kernel<2>);
  COLLM_PRELOAD(paged_attention_tc_kernel<4>);
  COLLM_PRELOAD(paged_attention_tc_kernel<8>);
  COLLM_PRELOAD((cross_entropy_kernel<0, 256>));
#undef COLLM_PRELOAD
  return COLLM_OK;
}

int collm_set_gemm_lean(int lean) {
  const int dev = cur_device();
  g_gemm_lean[dev] = (lean & 1) != 0;  // 1: lean GEMM pipelines too; 2: rank-space kernels only
  g_reduce_lean[dev] = lean != 0;
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K5
// ABI groups wider than kReduceMaxQ are reduced as several column chunks (same U, adjacent V
// columns, adjacent C columns / transposed rows), each <= kReduceMaxQ and a multiple of 8.
static int expand_reduce_groups(const collm_reduce_group* groups, int n_groups,
                                collm_reduce_group* out, int* n_out) {
  CHECK_ARG(groups && n_groups >= 1 && n_groups <= kReduceMaxGroups, "n_groups=%d out of [1,%d]",
            n_groups, kReduceMaxGroups);
  // One launch runs one tile width for all its groups (the MMAs of narrower groups are padded),
  // so 64-wide tiles pay only when every group is 64 wide (13B: r = 64 dB, 64-rank dA chunks —
  // each U then streams once per group instead of twice); otherwise groups are cut to <= 48.
  bool all64 = true;
  for (int g = 0; g < n_groups; ++g) all64 = all64 && groups[g].Q == 64;
  const int max_q = all64 ? 64 : 48;
  int n = 0;
  for (int g = 0; g < n_groups; ++g) {
    const collm_reduce_group& s = groups[g];
    CHECK_ARG(s.P > 0 && s.P % 8 == 0 && s.Q > 0 && s.Q % 8 == 0 && s.Q <= 64,
              "group %d: P=%d, Q=%d (need multiples of 8, Q <= 64)", g, s.P, s.Q);
    const int chunks = (s.Q + max_q - 1) / max_q;
    int off = 0;
    for (int c = 0; c < chunks; ++c) {
      const int q = ((s.Q / 8) * (c + 1) / chunks - (s.Q / 8) * c / chunks) * 8;
      CHECK_ARG(n < kReduceMaxInner, "too many reduction groups after splitting (%d)", n + 1);
      collm_reduce_group e = s;
      e.v_off = s.v_off + off;
      e.Q = q;
      e.c_col_off = s.c_col_off + off;
      e.t_row_off = s.t_row_off + off;
      out[n++] = e;
      off += q;
    }
  }
  *n_out = n;
  return COLLM_OK;
}

static int build_reduce_params(ReduceParams& p, const collm_reduce_group* abi_groups, int n_abi,
                               int& qmax, bool need_uv) {
  collm_reduce_group groups[kReduceMaxInner];
  int n_groups = 0;
  int rc = expand_reduce_groups(abi_groups, n_abi, groups, &n_groups);
  if (rc) return rc;
  p.n_groups = n_groups;
  int tiles = 0;
  qmax = 0;
  for (int g = 0; g < n_groups; ++g) {
    const collm_reduce_group& s = groups[g];
    ReduceGroup gr;
    gr.U = (const bf16*)s.U;
    gr.V = (const bf16*)s.V;
    gr.V2 = (const bf16*)s.V2;
    gr.grad = s.grad;
    gr.master = s.master;
    gr.m = s.m;
    gr.v = s.v;
    gr.out_same = (bf16*)s.out_same;
    gr.out_trans = (bf16*)s.out_trans;
    gr.ldu = s.ldu;
    gr.ldv = s.ldv;
    gr.u_off = s.u_off;
    gr.P = s.P;
    gr.v_off = s.v_off;
    gr.Q = s.Q;
    gr.ldc = s.ldc;
    gr.ld_trans = s.ld_trans;
    gr.c_row_off = s.c_row_off;
    gr.c_col_off = s.c_col_off;
    gr.t_row_off = s.t_row_off;
    gr.t_col_off = s.t_col_off;
    gr.tile_begin = tiles;
    if (need_uv) {
      CHECK_ARG(gr.U && gr.V, "group %d: null U/V", g);
      CHECK_ARG(gr.u_off % 8 == 0 && gr.v_off % 8 == 0 && gr.ldu % 8 == 0 && gr.ldv % 8 == 0 &&
                    aligned16(gr.U) && aligned16(gr.V) && (!gr.V2 || aligned16(gr.V2)),
                "group %d: U/V must be 16-byte aligned with x8 offsets/leading dimensions", g);
    }
    CHECK_ARG(gr.ldc >= gr.c_col_off + gr.Q, "group %d: ldc=%d too small", g, gr.ldc);
    CHECK_ARG(gr.ldc % 4 == 0 && gr.c_col_off % 4 == 0,
              "group %d: ldc and c_col_off must be multiples of 4 (vectorized finalize)", g);
    p.groups[g] = gr;
    tiles += (gr.P + kReducePT - 1) / kReducePT;
    qmax = std::max(qmax, gr.Q);
  }
  p.n_tiles = tiles;
  return COLLM_OK;
}

static int check_mode_targets(const ReduceParams& p, int mode, int accum_in) {
  for (int g = 0; g < p.n_groups; ++g) {
    const ReduceGroup& gr = p.groups[g];
    if (mode == COLLM_MODE_STORE_GRAD || accum_in)
      CHECK_ARG(gr.grad, "group %d: this mode needs grad", g);
    if (mode == COLLM_MODE_ADAMW) CHECK_ARG(gr.master && gr.m && gr.v, "group %d: ADAMW needs master/m/v", g);
    if (mode == COLLM_MODE_COPY_ONLY) CHECK_ARG(gr.master, "group %d: COPY_ONLY needs master", g);
  }
  return COLLM_OK;
}

size_t collm_reduce_workspace_bytes(const collm_reduce_group* groups, int n_groups, int tsplit) {
  if (tsplit <= 1 || !groups) return 0;
  collm_reduce_group ex[kReduceMaxInner];
  int n = 0;
  if (expand_reduce_groups(groups, n_groups, ex, &n) != COLLM_OK) return 0;
  int tiles = 0;
  for (int g = 0; g < n; ++g) tiles += (ex[g].P + kReducePT - 1) / kReducePT;
  return kCounterBytes + (size_t)tsplit * tiles * kReducePT * 64 * sizeof(float);
}

}  // extern "C"


template <int QT, int MINB>
static int launch_reduce(ReduceParams& p, cudaStream_t st) {
  static bool configured[kMaxDevices] = {};
  const int dev = cur_device();
  {
    std::lock_guard<std::mutex> lk(g_state_mu);
    if (!configured[dev]) {
      CUDA_TRY(cudaFuncSetAttribute(lora_reduce_kernel<QT, MINB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ReduceSmem<QT>::total(kReduceMaxStages)));
      configured[dev] = true;
    }
  }
  const bool reduce_lean = g_reduce_lean[dev];
  const size_t budget = reduce_lean ? 44u * 1024 : 100u * 1024;
  int stages = kReduceMaxStages;
  while (stages > 2 && ReduceSmem<QT>::total(stages) > budget) --stages;
  p.stages = stages;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.n_tiles, p.tsplit);
  cfg.blockDim = dim3(kReduceThreads);
  cfg.dynamicSmemBytes = ReduceSmem<QT>::total(stages);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePreferredSharedMemoryCarveout;  // see collm_lora_shrink
  attr[0].val.sharedMemCarveout = cudaSharedmemCarveoutMaxShared;
  cfg.attrs = attr;
  cfg.numAttrs = reduce_lean ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, lora_reduce_kernel<QT, MINB>, p));
  return COLLM_OK;
}

// K5 on the tensor core (reduce_tc.cuh), used when every operand can be viewed through a TMA map
// (<= kRtcMaxMaps distinct U / V / V2 tensors); returns 1 when the launch is not possible.
static int launch_reduce_tc(const ReduceParams& p, cudaStream_t st, bool* launched) {
  *launched = false;
  ReduceTcMaps maps;
  ReduceTcParams tp;
  const void* map_ptr[kRtcMaxMaps];
  int map_ld[kRtcMaxMaps];
  int n_maps = 0;
  auto map_of = [&](const void* ptr, int ld) -> int {
    for (int i = 0; i < n_maps; ++i)
      if (map_ptr[i] == ptr && map_ld[i] == ld) return i;
    if (n_maps == kRtcMaxMaps) return -1;
    if (make_tmap(&maps.m[n_maps], ptr, (uint64_t)ld, (uint64_t)p.T, (uint64_t)ld, 64, kRtcRows))
      return -2;
    map_ptr[n_maps] = ptr;
    map_ld[n_maps] = ld;
    return n_maps++;
  };
  for (int g = 0; g < p.n_groups; ++g) {
    const ReduceGroup& gr = p.groups[g];
    if (gr.Q > 64) return COLLM_OK;
    const int iu = map_of(gr.U, gr.ldu), iv = map_of(gr.V, gr.ldv);
    const int iv2 = gr.V2 ? map_of(gr.V2, gr.ldv) : -3;
    if (iu == -2 || iv == -2 || iv2 == -2) return COLLM_ECUDA;  // encode failure: error set
    if (iu < 0 || iv < 0 || iv2 == -1) return COLLM_OK;         // too many tensors: mma.sync path
    tp.map_u[g] = (int8_t)iu;
    tp.map_v[g] = (int8_t)iv;
    tp.map_v2[g] = (int8_t)(gr.V2 ? iv2 : -1);
  }
  tp.r = p;
  tp.n_maps = n_maps;
  static const int no_mma = [] { const char* e = getenv("COLLM_DEBUG_K5_NO_MMA"); return e ? atoi(e) : 0; }();
  tp.debug_no_mma = no_mma;
  tp.n_chunks = (p.T + kRtcRows - 1) / kRtcRows;
  const int ts = std::max(1, std::min(p.tsplit, tp.n_chunks));
  tp.per = (tp.n_chunks + ts - 1) / ts;
  tp.r.tsplit = (tp.n_chunks + tp.per - 1) / tp.per;  // no empty parts; <= the caller's split
  tp.n_units = p.n_tiles * tp.r.tsplit;
  static bool configured[kMaxDevices] = {};
  const int dev = cur_device();
  {
    std::lock_guard<std::mutex> lk(g_state_mu);
    if (!configured[dev]) {
      CUDA_TRY(cudaFuncSetAttribute(lora_reduce_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    ReduceTcSmem::kTotal));
      configured[dev] = true;
    }
  }
  const int grid = std::min(tp.n_units, num_sms_cached());
  lora_reduce_tc_kernel<<<grid, 256, ReduceTcSmem::kTotal, st>>>(maps, tp);
  CUDA_TRY(cudaGetLastError());
  *launched = true;
  return COLLM_OK;
}

extern "C" {

int collm_set_reduce_impl(int tc) {
  CHECK_ARG(tc == 0 || tc == 1, "reduce impl %d (0 = mma.sync, 1 = tcgen05)", tc);
  g_reduce_impl[cur_device()].store(tc + 1);
  return COLLM_OK;
}
int collm_get_reduce_impl(void) { return impl_of(g_reduce_impl, "COLLM_K5_TC"); }

int collm_lora_reduce(int T, const collm_reduce_group* groups, int n_groups, int mode,
                      int accum_in, float grad_scale, const float* adamw, int tsplit,
                      void* workspace, size_t ws_bytes, void* stream) {
  CHECK_ARG(T >= 1, "T=%d", T);
  CHECK_ARG(mode == COLLM_MODE_STORE_GRAD || mode == COLLM_MODE_ADAMW, "bad mode %d", mode);
  CHECK_ARG(mode != COLLM_MODE_ADAMW || adamw, "ADAMW needs the device argument block");
  CHECK_ARG(tsplit >= 1 && tsplit <= 256, "tsplit=%d", tsplit);
  ReduceParams p{};
  int qmax = 0;
  int rc = build_reduce_params(p, groups, n_groups, qmax, true);
  if (rc) return rc;
  rc = check_mode_targets(p, mode, accum_in);
  if (rc) return rc;
  p.T = T;
  p.tsplit = tsplit;
  p.mode = mode;
  p.accum_in = accum_in;
  p.grad_scale = grad_scale;
  p.opt = adamw;
  if (tsplit > 1) {
    const size_t need = collm_reduce_workspace_bytes(groups, n_groups, tsplit);
    CHECK_ARG(workspace && ws_bytes >= need, "reduce workspace too small: %zu < %zu", ws_bytes,
              need);
    CHECK_ARG((size_t)p.n_tiles <= kCounterCap, "too many reduce tiles (%d)", p.n_tiles);
    p.counters = (int32_t*)workspace;
    p.partials = (float*)((char*)workspace + kCounterBytes);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (collm_get_reduce_impl()) {
    bool launched = false;
    rc = launch_reduce_tc(p, st, &launched);
    if (rc || launched) return rc;
  }
  static const int minb = [] { const char* e = getenv("COLLM_K5_MINB"); return e ? atoi(e) : 4; }();
  // 64-wide tiles (r = 64 dB, 64-rank dA chunks: each U = dY / X_tr read once per ABI group
  // instead of twice) carry 32 accumulators per thread: 3 CTAs/SM register budget
  if (qmax > 48) return launch_reduce<64, 3>(p, st);
  if (minb == 3) {
    if (qmax <= 16) return launch_reduce<16, 3>(p, st);
    if (qmax <= 32) return launch_reduce<32, 3>(p, st);
    return launch_reduce<48, 3>(p, st);
  }
  if (qmax <= 16) return launch_reduce<16, 4>(p, st);
  if (qmax <= 32) return launch_reduce<32, 4>(p, st);
  return launch_reduce<48, 4>(p, st);
}

int collm_lora_apply(const collm_reduce_group* groups, int n_groups, int mode,
                     const float* adamw, void* stream) {
  CHECK_ARG(mode == COLLM_MODE_ADAMW || mode == COLLM_MODE_COPY_ONLY, "bad mode %d", mode);
  CHECK_ARG(mode != COLLM_MODE_ADAMW || adamw, "ADAMW needs the device argument block");
  ReduceParams p{};
  int qmax = 0;
  int rc = build_reduce_params(p, groups, n_groups, qmax, false);
  if (rc) return rc;
  rc = check_mode_targets(p, mode, mode == COLLM_MODE_ADAMW);
  if (rc) return rc;
  p.mode = mode;
  p.accum_in = 1;
  p.grad_scale = 1.f;
  p.opt = adamw;
  long long total = 0;
  for (int g = 0; g < n_groups; ++g) total += (long long)p.groups[g].P * p.groups[g].Q;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4LL * num_sms_cached());
  lora_apply_kernel<<<std::max(blocks, 1), 256, 0, (cudaStream_t)stream>>>(p, total);
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K8
size_t collm_attention_workspace_bytes(int T, int n_heads, int n_kv_heads, int max_ctx) {
  if (T <= 0 || n_kv_heads <= 0 || n_heads <= 0 || max_ctx <= 0) return 0;
  const size_t splits = (size_t)(max_ctx + kAttnSplit - 1) / kAttnSplit;
  const size_t counters = ((size_t)T * n_kv_heads * 4 + 255) & ~(size_t)255;
  return counters + (size_t)T * n_heads * splits * (kAttnD + 2) * 4;
}

int collm_paged_attention(const void* q, int ldq, int T, int n_heads, int n_kv_heads,
                          int head_dim, const void* k_cache, const void* v_cache, int page_size,
                          const int32_t* block_table, int bt_stride, const int32_t* row_seq,
                          const int32_t* row_pos, int max_ctx, float scale, void* out, int ldo,
                          void* workspace, size_t ws_bytes, void* stream) {
  CHECK_ARG(q && k_cache && v_cache && block_table && row_seq && row_pos && out, "null input");
  CHECK_ARG(T >= 0, "T=%d", T);
  if (T == 0) return COLLM_OK;
  CHECK_ARG(head_dim == kAttnD, "head_dim=%d (supported: %d)", head_dim, kAttnD);
  CHECK_ARG(n_kv_heads >= 1 && n_heads % n_kv_heads == 0 && n_heads / n_kv_heads <= kAttnMaxG,
            "n_heads=%d / n_kv_heads=%d (GQA group <= %d)", n_heads, n_kv_heads, kAttnMaxG);
  CHECK_ARG(page_size >= 1 && (page_size & (page_size - 1)) == 0, "page_size=%d must be 2^k",
            page_size);
  CHECK_ARG(max_ctx >= 1 && bt_stride * page_size >= max_ctx, "max_ctx=%d exceeds the block table",
            max_ctx);
  CHECK_ARG(ldq >= n_heads * head_dim && ldo >= n_heads * head_dim, "ldq/ldo too small");
  CHECK_ARG(aligned16(k_cache) && aligned16(v_cache), "KV caches must be 16-byte aligned");
  const size_t need = collm_attention_workspace_bytes(T, n_heads, n_kv_heads, max_ctx);
  CHECK_ARG(workspace && ws_bytes >= need, "attention workspace too small: %zu < %zu", ws_bytes,
            need);
  AttnParams p{};
  p.q = (const bf16*)q;
  p.ldq = ldq;
  p.k_cache = (const bf16*)k_cache;
  p.v_cache = (const bf16*)v_cache;
  int shift = 0;
  while ((1 << shift) < page_size) ++shift;
  p.page_shift = shift;
  p.n_heads = n_heads;
  p.n_kv_heads = n_kv_heads;
  p.block_table = block_table;
  p.bt_stride = bt_stride;
  p.row_seq = row_seq;
  p.row_pos = row_pos;
  p.out = (bf16*)out;
  p.ldo = ldo;
  p.scale = scale;
  p.max_splits = (max_ctx + kAttnSplit - 1) / kAttnSplit;
  p.counters = (int32_t*)workspace;
  p.part = (float*)((char*)workspace + (((size_t)T * n_kv_heads * 4 + 255) & ~(size_t)255));
  const dim3 grid(T, n_kv_heads, p.max_splits);
  cudaStream_t st = (cudaStream_t)stream;
  // the tensor-core variant (the G heads of a KV head are one MMA's rows; measured faster for
  // every G: 7B decode 0.81 of HBM vs 0.63, GQA G = 4 0.74 vs 0.22, tools/attn_bench.py);
  // COLLM_ATTN_TC=0 selects the CUDA-core half-warp streams
  static const int tc_env = [] { const char* e = getenv("COLLM_ATTN_TC"); return e ? atoi(e) : 1; }();
  const int G = n_heads / n_kv_heads;
  if (tc_env != 0) {
    static bool configured[kMaxDevices][4] = {};
    const int dev = cur_device(), gi = G == 1 ? 0 : G == 2 ? 1 : G == 4 ? 2 : 3;
    auto cfg_kernel = [&](auto kern) -> int {
      std::lock_guard<std::mutex> lk(g_state_mu);
      if (!configured[dev][gi]) {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnTcSmem));
        configured[dev][gi] = true;
      }
      return COLLM_OK;
    };
    int rc = COLLM_OK;
    switch (G) {
      case 1: rc = cfg_kernel(paged_attention_tc_kernel<1>); if (!rc) paged_attention_tc_kernel<1><<<grid, kAttnThreads, kAttnTcSmem, st>>>(p); break;
      case 2: rc = cfg_kernel(paged_attention_tc_kernel<2>); if (!rc) paged_attention_tc_kernel<2><<<grid, kAttnThreads, kAttnTcSmem, st>>>(p); break;
      case 4: rc = cfg_kernel(paged_attention_tc_kernel<4>); if (!rc) paged_attention_tc_kernel<4><<<grid, kAttnThreads, kAttnTcSmem, st>>>(p); break;
      case 8: rc = cfg_kernel(paged_attention_tc_kernel<8>); if (!rc) paged_attention_tc_kernel<8><<<grid, kAttnThreads, kAttnTcSmem, st>>>(p); break;
      default: return fail(COLLM_EINVAL, "GQA group %d not in {1, 2, 4, 8}", G);
    }
    if (rc) return rc;
    CUDA_TRY(cudaGetLastError());
    return COLLM_OK;
  }
  switch (n_heads / n_kv_heads) {
    case 1: paged_attention_kernel<1><<<grid, kAttnThreads, 0, st>>>(p); break;
    case 2: paged_attention_kernel<2><<<grid, kAttnThreads, 0, st>>>(p); break;
    case 4: paged_attention_kernel<4><<<grid, kAttnThreads, 0, st>>>(p); break;
    case 8: paged_attention_kernel<8><<<grid, kAttnThreads, 0, st>>>(p); break;
    default: return fail(COLLM_EINVAL, "GQA group %d not in {1, 2, 4, 8}", n_heads / n_kv_heads);
  }
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

// ------------------------------------------------------------------------------------ K7
int collm_cross_entropy(const void* logits, int ld, int T, int V, const int32_t* labels,
                        float* loss_rows, float* loss_mean, int32_t* counter, void* dlogits,
                        int ld_d, float grad_scale, void* stream) {
  CHECK_ARG(logits && labels && loss_rows, "null input");
  CHECK_ARG(T >= 0, "T=%d", T);
  if (T == 0) return COLLM_OK;
  CHECK_ARG(V >= 8 && V % 8 == 0 && ld % 8 == 0 && ld >= V, "V=%d / ld=%d must be multiples of 8",
            V, ld);
  CHECK_ARG(aligned16(logits), "logits must be 16-byte aligned");
  CHECK_ARG(!loss_mean || counter, "loss_mean needs the arrival counter");
  CHECK_ARG(!dlogits || (aligned16(dlogits) && ld_d % 8 == 0 && ld_d >= V),
            "dlogits must be 16-byte aligned with ld_d >= V, a multiple of 8");
  CeParams p{};
  p.logits = (const bf16*)logits;
  p.ld = ld;
  p.T = T;
  p.V = V;
  p.labels = labels;
  p.loss_rows = loss_rows;
  p.loss_mean = loss_mean;
  p.counter = counter;
  p.dlogits = (bf16*)dlogits;
  p.ld_d = ld_d;
  p.grad_scale = grad_scale;
  if (V <= 8 * 8 * 512)  // the row fits in registers: 8 vectors per thread x 512 threads
    cross_entropy_kernel<8, 512><<<T, 512, 0, (cudaStream_t)stream>>>(p);
  else
    cross_entropy_kernel<0, 256><<<T, 256, 0, (cudaStream_t)stream>>>(p);
  CUDA_TRY(cudaGetLastError());
  return COLLM_OK;
}

}  // extern "C"
