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
                                                        long bytes_per_cta, int stages, unsigned long long* sink, int panels,
                                                        int gap, int variant, int sb, long cta_stride) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);  // [stages] full (+ [stages] empty)
  const long n_items = bytes_per_cta / (kStage + gap);
  const char* base = src + blockIdx.x * (cta_stride ? cta_stride : bytes_per_cta);
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
  if (MODE == 4) {  // warp-specialised: warp 0 produces, warps 2.. consume
    const long n_items = bytes_per_cta / (sb + gap);
    full = reinterpret_cast<uint64_t*>(smem + stages * sb);
    uint64_t* empty = full + stages;
    const int nwarps = (blockDim.x - 64) / 32;
    if (threadIdx.x == 0) {
      for (int s = 0; s < stages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], variant == 0 ? 1 : nwarps);
      }
      fence_mbar_init();
    }
    __syncthreads();
    const int nthr = blockDim.x - 64;
    if (threadIdx.x == 0) {
      for (long i = 0; i < n_items; ++i) {
        const int s = i % stages;
        mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
        mbar_expect_tx(&full[s], sb);
        bulk_load(smem + s * sb, base + i * (sb + gap), sb, &full[s]);
      }
    } else if (threadIdx.x >= 64) {
      const int tid = threadIdx.x - 64;
      unsigned acc = 0;
      for (long i = 0; i < n_items; ++i) {
        const int s = i % stages;
        if (variant == 0) {
          if (tid == 0) mbar_wait(&full[s], (i / stages) & 1);
          named_bar(1, nthr);
          if (panels > 1) acc ^= reinterpret_cast<const unsigned*>(smem + s * kStage)[tid];
          named_bar(1, nthr);
          if (tid == 0) mbar_arrive(&empty[s]);
        } else {
          if (variant == 2 || (tid & 31) == 0) mbar_wait(&full[s], (i / stages) & 1);
          __syncwarp();
          if (panels > 1) acc ^= reinterpret_cast<const unsigned*>(smem + s * kStage)[tid];
          __syncwarp();
          if ((tid & 31) == 0) mbar_arrive(&empty[s]);
        }
      }
      if (acc == 0x12345) sink[0] = acc;
    }
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
        else bulk_load(dst, base + i * (kStage + gap), kStage, &full[s]);
      }
    }
  }
}

__global__ void fill_kernel(unsigned* p, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    unsigned x = static_cast<unsigned>(i) * 2654435761u + 0x9E3779B9u;
    x ^= x >> 15; x *= 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
    p[i] = x;
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
  if (getenv("RANDOM_FILL")) {  // incompressible contents
    fill_kernel<<<1024, 256>>>(reinterpret_cast<unsigned*>(buf), per * ctas / 4);
    cudaDeviceSynchronize();
  }
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
  const size_t smem = stages * (argc > 12 ? atoi(argv[12]) : kStage) + 1024 + (argc > 8 ? atoi(argv[8]) : 0);
  cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[5] = {"tma2d", "bulk1d", "ldg128", "slice", "wspec"};
  const int mode0 = argc > 5 ? atoi(argv[5]) : 0;
  const int mode1 = argc > 9 ? atoi(argv[9]) : 4;
  for (int mode = mode0; mode < mode1; ++mode) {
    auto k = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : mode == 2 ? stream_kernel<2> : mode == 3 ? stream_kernel<3> : stream_kernel<4>;
    const dim3 grid(ctas);
    const int panels = row_elems / 64;
    const int nthr = argc > 11 ? atoi(argv[11]) : mode == 4 ? 576 : mode >= 2 ? ldg_threads : 128;
    const int csz = argc > 6 ? atoi(argv[6]) : 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(nthr);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csz;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int gap = argc > 7 ? atoi(argv[7]) : 0;
    const int variant = argc > 10 ? atoi(argv[10]) : 0;
    const int sb = argc > 12 ? atoi(argv[12]) : kStage;
    const long cta_stride = argc > 13 ? atol(argv[13]) : 0;
    const long per_run = argc > 14 ? atol(argv[14]) : per;
    // ROTATE=1: every launch reads a different region (inputs never L2-resident)
    const bool rotate = getenv("ROTATE") != nullptr;
    int rot = 0;
    auto launch = [&] {
      const char* base = (const char*)buf + (rotate ? static_cast<long>(rot++ % 7) * ctas * per_run : 0);
      cudaLaunchKernelEx(&cfg, k, map, base, per_run, stages, sink, panels, gap, variant, sb, cta_stride);
    };
    for (int rep = 0; rep < 2; ++rep) launch();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double moved = mode == 4 ? static_cast<double>(per_run / (sb + gap)) * sb : static_cast<double>(per_run);
    const double gbs = 5.0 * moved * ctas / (ms * 1e-3) / 1e9;
    printf("csz=%d %-7s thr=%4d ctas=%3d stages=%2d  total %7.1f GB/s  per-CTA %6.1f GB/s  (%s)\n", csz, names[mode], nthr, ctas, stages, gbs,
           gbs / ctas, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
