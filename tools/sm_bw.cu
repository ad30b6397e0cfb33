// Per-SM HBM streaming bandwidth probe: W CTAs (one per SM, optionally 2-CTA clusters so they
// hold whole TPCs) each stream a contiguous share of a buffer through a ring of S bulk-copy
// stages of C bytes (cp.async.bulk -> smem, mbarrier completion), consumers touch one word per
// stage.  Answers: how many bytes/s can W SMs pull from HBM, i.e. how many SMs a rank-space
// worker needs.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2604_16400_b200/csrc/common.cuh"
using namespace collm;
__device__ int g_wait_mode = 0;
__device__ __forceinline__ bool test_wait_p(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool try_wait_hint(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 20;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_m(uint64_t* bar, uint32_t parity, int mode) {
  const uint32_t a = smem_u32(bar);
  if (mode == 1) { while (!test_wait_p(a, parity)) {} return; }
  if (mode == 2) { while (!try_wait_hint(a, parity)) {} return; }
  mbar_wait(bar, parity);
}
__device__ __forceinline__ void tma_load_3d_probe(void* smem_dst, const CUtensorMap* m, uint64_t* bar,
                                                  int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__global__ void __launch_bounds__(160, 1)
bw_kernel(const uint8_t* __restrict__ src, long long bytes_per_cta, int stages, int chunk,
          unsigned long long* sink, int pieces, const __grid_constant__ CUtensorMap tmap, int box_rows, int box_kb) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 32;
  uint8_t* ring = smem + 1024;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    fence_mbar_init();
  }
  __syncthreads();
  const int wmode = g_wait_mode;
  const uint8_t* base = src + (long long)blockIdx.x * bytes_per_cta;
  const long long n = bytes_per_cta / chunk;
  unsigned long long acc = 0;
  if (tid == 128) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      const uint32_t ph = (uint32_t)((i / stages) & 1);
      if (i >= stages) wait_m(&empty[s], ph ^ 1, wmode);
      mbar_arrive_expect_tx(&full[s], chunk);
      if (box_kb > 0) {
        // 3-D k-block view (64, rows, 64 kblocks) of a [rows, 4096] matrix: one box = box_kb
        // k-blocks x box_rows rows; stage i walks (row group, k-block group), k fastest
        const long long rows_cta = bytes_per_cta / 8192;
        const int kgroups = 64 / box_kb;
        const int kg = (int)(i % kgroups);
        const long long rg = i / kgroups;
        tma_load_3d_probe(ring + (size_t)s * chunk, &tmap, &full[s], 0,
                          (int)(blockIdx.x * rows_cta + rg * box_rows), kg * box_kb);
      } else if (box_rows > 0) {
        // 2-D tensor boxes [64 cols x box_rows rows] of a [rows, 4096] bf16 matrix: this CTA's
        // rows, stage i covers one 64-col k block of chunk/(128*box_rows) row boxes
        const int boxes = chunk / (128 * box_rows);
        const long long rows_cta = bytes_per_cta / 8192;
        for (int b = 0; b < boxes; ++b) {
          const long long lin = i * boxes + b;  // (kblock, rowbox) order: k fastest
          const int kb = (int)(lin % 64);
          const long long rb = lin / 64;
          tma_load_2d(ring + (size_t)s * chunk + (size_t)b * 128 * box_rows, &tmap, &full[s],
                      kb * 64, (int)(blockIdx.x * rows_cta + rb * box_rows));
        }
      } else {
        const int pc = chunk / pieces;
        for (int q = 0; q < pieces; ++q)
          bulk_copy_g2s(ring + (size_t)s * chunk + q * pc, base + i * chunk + q * pc, pc, &full[s]);
      }
    }
  }
  if (tid < 128 && tid % 32 == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      wait_m(&full[s], (uint32_t)((i / stages) & 1), wmode);
      acc += ring[(size_t)s * chunk + tid];
      mbar_arrive(&empty[s]);
    }
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

// LDG.128 variant: every thread of `threads` keeps `unr` 16-byte loads in flight.
template <int UNR>
__global__ void ldg_kernel(const uint4* __restrict__ src, long long vec_per_cta, unsigned long long* sink) {
  const uint4* base = src + (long long)blockIdx.x * vec_per_cta;
  unsigned acc = 0;
  for (long long i = threadIdx.x; i < vec_per_cta; i += (long long)blockDim.x * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long long j = i + (long long)u * blockDim.x;
      v[u] = j < vec_per_cta ? __ldg(base + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

extern "C" int run_bw(const void* src, long long bytes_per_cta, int ctas, int cluster, int stages,
                      int chunk, void* sink, void* stream, int pieces, int box_rows, int box_kb) {
  CUtensorMap tm{};
  if (box_kb > 0) {
    cuuint64_t dims[3] = {64, (cuuint64_t)(bytes_per_cta * ctas / 8192), 64};
    cuuint64_t strides[2] = {8192, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)box_kb};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)src, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return 1000 + r;
  } else if (box_rows > 0) {
    cuuint64_t dims[2] = {4096, (cuuint64_t)(bytes_per_cta * ctas / 8192)};
    cuuint64_t strides[1] = {8192};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)src, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) return 1000 + r;
  }
  const int smem = 1024 + stages * chunk;
  cudaFuncSetAttribute(bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(160);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bw_kernel, (const uint8_t*)src, bytes_per_cta, stages, chunk,
                     (unsigned long long*)sink, pieces, tm, box_rows, box_kb);
  return (int)cudaGetLastError();
}

extern "C" int set_wait_mode(int m) { return (int)cudaMemcpyToSymbol(g_wait_mode, &m, sizeof(int)); }

extern "C" int run_ldg(const void* src, long long bytes_per_cta, int ctas, int threads, int unr,
                       void* sink, void* stream) {
  const long long v = bytes_per_cta / 16;
  if (unr == 4)
    ldg_kernel<4><<<ctas, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, v, (unsigned long long*)sink);
  else
    ldg_kernel<8><<<ctas, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, v, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}

// R independent rings per CTA (producer = lane 0 of warp 4+r, consumer = lane 0 of warp r), each
// streaming its own contiguous 1/R of the CTA's bytes: is the one-stage-in-flight behaviour per
// producer/ring or per SM?
__global__ void __launch_bounds__(256, 1)
rings_kernel(const uint8_t* __restrict__ src, long long bytes_per_cta, int stages, int chunk,
             int rings, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 64;
  uint8_t* ring0 = smem + 1024;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    for (int s = 0; s < stages * rings; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const long long per_ring = bytes_per_cta / rings;
  const long long n = per_ring / chunk;
  unsigned long long acc = 0;
  if (warp >= 4 && warp < 4 + rings && lane == 0) {
    const int r = warp - 4;
    const uint8_t* base = src + (long long)blockIdx.x * bytes_per_cta + r * per_ring;
    uint8_t* ring = ring0 + (size_t)r * stages * chunk;
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      const uint32_t ph = (uint32_t)((i / stages) & 1);
      if (i >= stages) mbar_wait(&empty[r * stages + s], ph ^ 1);
      mbar_arrive_expect_tx(&full[r * stages + s], chunk);
      bulk_copy_g2s(ring + (size_t)s * chunk, base + i * chunk, chunk, &full[r * stages + s]);
    }
  }
  if (warp < rings && lane == 0) {
    const int r = warp;
    uint8_t* ring = ring0 + (size_t)r * stages * chunk;
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      mbar_wait(&full[r * stages + s], (uint32_t)((i / stages) & 1));
      acc += ring[(size_t)s * chunk + 7];
      mbar_arrive(&empty[r * stages + s]);
    }
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

extern "C" int run_rings(const void* src, long long bytes_per_cta, int ctas, int stages, int chunk,
                         int rings, void* sink, void* stream) {
  const int smem = 1024 + rings * stages * chunk;
  cudaFuncSetAttribute(rings_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rings_kernel<<<ctas, 256, smem, (cudaStream_t)stream>>>((const uint8_t*)src, bytes_per_cta, stages,
                                                          chunk, rings, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}

// ONE ring (one consumer), P producer threads (lane 0 of warps 4..4+P-1) issuing stages
// round-robin (stage i by producer i % P): is the limit per issuing thread?
__global__ void __launch_bounds__(256, 1)
multiprod_kernel(const uint8_t* __restrict__ src, long long bytes_per_cta, int stages, int chunk,
                 int P, int cons_warps, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 64;
  uint8_t* ring = smem + 1024;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cons_warps); }
    fence_mbar_init();
  }
  __syncthreads();
  const long long n = bytes_per_cta / chunk;
  const uint8_t* base = src + (long long)blockIdx.x * bytes_per_cta;
  unsigned long long acc = 0;
  if (warp >= 4 && warp < 4 + P && lane == 0) {
    const int pr = warp - 4;
    for (long long i = pr; i < n; i += P) {
      const int s = (int)(i % stages);
      const uint32_t ph = (uint32_t)((i / stages) & 1);
      if (i >= stages) mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_copy_g2s(ring + (size_t)s * chunk, base + i * chunk, chunk, &full[s]);
    }
  }
  if (warp < cons_warps && lane == 0) {
    for (long long i = 0; i < n; ++i) {
      const int s = (int)(i % stages);
      mbar_wait(&full[s], (uint32_t)((i / stages) & 1));
      acc += ring[(size_t)s * chunk + 7 + warp];
      mbar_arrive(&empty[s]);
    }
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

extern "C" int run_multiprod(const void* src, long long bytes_per_cta, int ctas, int stages, int chunk,
                             int P, int cons_warps, void* sink, void* stream) {
  const int smem = 1024 + stages * chunk;
  cudaFuncSetAttribute(multiprod_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  multiprod_kernel<<<ctas, 256, smem, (cudaStream_t)stream>>>((const uint8_t*)src, bytes_per_cta, stages,
                                                              chunk, P, cons_warps, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}
