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
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* src,
                                                        long bytes_per_cta, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  const long n_items = bytes_per_cta / kStage;
  const char* base = src + blockIdx.x * bytes_per_cta;
  if (MODE == 2) {  // LDG.128 streaming by all 128 threads, 8 loads in flight per thread
    const uint4* p = reinterpret_cast<const uint4*>(base);
    const long n16 = bytes_per_cta / 16;
    unsigned acc = 0;
    for (long i = threadIdx.x; i < n16; i += 128 * 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (i + u * 128 < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * 128));
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
    const long row0 = blockIdx.x * (bytes_per_cta / 128);  // rows of 128 B (MODE 0 map: 64 bf16 x rows)
    for (long i = 0; i < n_items + stages; ++i) {
      if (i >= stages) {  // consume item i - stages
        const long j = i - stages;
        mbar_wait(&full[j % stages], (j / stages) & 1);
      }
      if (i < n_items) {
        const int s = i % stages;
        unsigned char* dst = smem + s * kStage;
        mbar_expect_tx(&full[s], kStage);
        if (MODE == 0) tma_load_2d(dst, &map, 0, static_cast<int>(row0 + i * 128), &full[s]);
        else bulk_load(dst, base + i * kStage, kStage, &full[s]);
      }
    }
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int stages = argc > 2 ? atoi(argv[2]) : 8;
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
  const cuuint64_t dims[2] = {64, static_cast<cuuint64_t>(per * ctas / 128)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = stages * kStage + 1024;
  cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"tma2d", "bulk1d", "ldg128"};
  for (int mode = 0; mode < 3; ++mode) {
    auto k = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : stream_kernel<2>;
    for (int rep = 0; rep < 2; ++rep) k<<<ctas, 128, smem>>>(map, buf, per, stages, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) k<<<ctas, 128, smem>>>(map, buf, per, stages, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 5.0 * per * ctas / (ms * 1e-3) / 1e9;
    printf("%-7s ctas=%3d stages=%2d  total %7.1f GB/s  per-CTA %6.1f GB/s  (%s)\n", names[mode], ctas, stages, gbs,
           gbs / ctas, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
