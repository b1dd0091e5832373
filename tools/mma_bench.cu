// Tensor-pipe rate of the decode core's two MMA shapes on one SM per CTA:
//   mode 0: S-like  A K-major  (M=128 tokens x K=16 ranks), B K-major, N = n
//   mode 1: U-like  A MN-major (M=128 ranks  x K=16 tokens), B K-major, N = n
//   mode 2: U transposed: A = p K-major (M=64), B = left_v MN-major (N = n ranks)
// Cycles per MMA from the first issue to the commit's arrival (operands: whatever
// is in shared memory; only the rate matters).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_23914_b200/csrc -I../include
//        tools/mma_bench.cu -o tools/mma_bench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace kvp::sm100;

__global__ void __launch_bounds__(128, 1) mma_kernel(int mode, int n, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_addr(smem), b = smem_addr(smem + 65536);
    const uint32_t m = mode == 2 ? 64 : 128;
    const uint32_t idesc = idesc_bf16(m, static_cast<uint32_t>(n), mode == 1, mode == 2);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int j = 0; j < 8; ++j) {
        uint64_t ad, bd;
        if (mode == 0) {  // two 16 KB K-major panels, 4 K steps each
          ad = smem_desc(a + (j >> 2) * 16384 + (j & 3) * 32, 16, 1024, kSwizzle128B);
          bd = smem_desc(b + (j >> 2) * 8192 + (j & 3) * 32, 16, 1024, kSwizzle128B);
        } else if (mode == 1) {  // MN-major A: 2 panels (LBO 16 KB) along M, K step = 16 rows
          ad = smem_desc(a + j * 2048, 16384, 1024, kSwizzle128B);
          bd = smem_desc(b + (j >> 2) * 8192 + (j & 3) * 32, 16, 1024, kSwizzle128B);
        } else {  // A = p K-major (64 rows), B = left_v MN-major (n ranks along N, 64 per 16 KB panel)
          ad = smem_desc(b + (j >> 2) * 8192 + (j & 3) * 32, 16, 1024, kSwizzle128B);
          bd = smem_desc(a + j * 2048, 16384, 1024, kSwizzle128B);
        }
        mma_bf16(tmem, ad, bd, idesc, (r | j) != 0);
      }
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 256;
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int smem = 65536 + 16384 + 1024;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"S-like  A K-major  M=128", "U-like  A MN-major M=128", "U^T     B MN-major M=64 "};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {32, 64, 128, 256}) {
      if (mode < 2 && n > 64) continue;
      mma_kernel<<<148, 128, smem>>>(mode, n, reps, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per = static_cast<double>(mx) / (reps * 8.0);
      const double flop = 2.0 * (mode == 2 ? 64 : 128) * n * 16;
      printf("%s N=%3d: %7.1f cycles/MMA  %7.0f flop/cycle/SM  (%s)\n", names[mode], n, per, flop / per,
             cudaGetErrorString(e));
    }
  return 0;
}
