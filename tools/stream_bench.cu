// Microbenchmark: per-SM streaming bandwidth of TMA 2D tiles, 1D bulk copies
// and plain LDG.128 on B200 (one CTA per SM, ring of mbarrier stages).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_23914_b200/csrc
//        -I../include tools/stream_bench.cu -o stream_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace kvp::sm100;

constexpr int kStage = 16384;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* src,
                                                        long bytes_per_cta, int stages, unsigned long long* sink, int panels) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  const long n_items = bytes_per_cta / kStage;
  const char* base = src + blockIdx.x * bytes_per_cta;
  if (MODE == 3) {  // qdots pattern: block = 256-byte column slice (one head) of an [rows x 8 KB] matrix
    const int slice = blockIdx.x % 32, inst = blockIdx.x / 32;
    const long row_bytes = 8192, rows = bytes_per_cta / 256;  // same bytes per block as the other modes
    const char* mbase = src + static_cast<long>(inst) * rows * row_bytes + slice * 256;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned acc = 0;
    for (long r0 = (warp * 2 + lane / 16); r0 < rows; r0 += 2 * nw * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long r = r0 + u * 2 * nw;
        if (r < rows) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(mbase + r * row_bytes + (lane % 16) * 16));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345) sink[0] = acc;
    return;
  }
  if (MODE == 2) {  // LDG.128 streaming by all 128 threads, 8 loads in flight per thread
    const uint4* p = reinterpret_cast<const uint4*>(base);
    const long n16 = bytes_per_cta / 16;
    unsigned acc = 0;
    const int nt = blockDim.x;
    for (long i = threadIdx.x; i < n16; i += nt * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + u * nt < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * nt));
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345) sink[0] = acc;
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long rows_per_cta = bytes_per_cta / 128;  // 64-element boxes of 128 B
    const long row0 = blockIdx.x * rows_per_cta;
    for (long i = 0; i < n_items + stages; ++i) {
      if (i >= stages) {  // consume item i - stages
        const long j = i - stages;
        mbar_wait(&full[j % stages], (j / stages) & 1);
      }
      if (i < n_items) {
        const int s = i % stages;
        unsigned char* dst = smem + s * kStage;
        mbar_expect_tx(&full[s], kStage);
        if (MODE == 0) {  // walk the 64-column panels of consecutive 128-row tiles
          const long tile = i / panels, panel = i % panels;
          tma_load_2d(dst, &map, static_cast<int>(panel * 64), static_cast<int>((row0 / panels) + tile * 128), &full[s]);
        }
        else bulk_load(dst, base + i * kStage, kStage, &full[s]);
      }
    }
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int stages = argc > 2 ? atoi(argv[2]) : 8;
  const int row_elems = argc > 3 ? atoi(argv[3]) : 64;  // tensor row length (bf16); box reads 64 of them
  const int ldg_threads = argc > 4 ? atoi(argv[4]) : 128;
  const long per = 8l << 20;  // 8 MiB per CTA
  char* buf;
  cudaMalloc(&buf, per * ctas);
  cudaMemset(buf, 1, per * ctas);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), 12000, cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(row_elems), static_cast<cuuint64_t>(per * ctas / (2 * row_elems))};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_elems) * 2};
  const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = stages * kStage + 1024;
  cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"tma2d", "bulk1d", "ldg128", "slice"};
  const int mode0 = argc > 5 ? atoi(argv[5]) : 0;
  for (int mode = mode0; mode < 4; ++mode) {
    auto k = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : mode == 2 ? stream_kernel<2> : stream_kernel<3>;
    const dim3 grid(ctas);
    const int panels = row_elems / 64;
    const int nthr = mode >= 2 ? ldg_threads : 128;
    for (int rep = 0; rep < 2; ++rep) k<<<grid, nthr, smem>>>(map, buf, per, stages, sink, panels);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) k<<<grid, nthr, smem>>>(map, buf, per, stages, sink, panels);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 5.0 * per * ctas / (ms * 1e-3) / 1e9;
    printf("%-7s thr=%4d ctas=%3d stages=%2d  total %7.1f GB/s  per-CTA %6.1f GB/s  (%s)\n", names[mode], nthr, ctas, stages, gbs,
           gbs / ctas, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
