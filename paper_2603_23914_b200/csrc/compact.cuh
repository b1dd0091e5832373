// Prefill-time compaction (compact.cu): batched randomized truncated SVD.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace kvp {
// a: batch x (T x W) row-major fp32; left: batch x (T x rank), right: batch x (rank x W).
void randomized_svd_batched(cublasHandle_t blas, cudaStream_t stream, const float* a, int batch, int T, int W,
                            int rank, uint64_t seed, int oversampling, int power_iterations, float* left,
                            float* right);
}  // namespace kvp
