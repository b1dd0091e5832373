// Prefill-time compaction (compact.cu): batched randomized truncated SVD.
#pragma once

#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace kvp {
// a: batch x (T x W) row-major fp32; left: batch x (T x rank), right: batch x (rank x W).
void randomized_svd_batched(cublasHandle_t blas, cudaStream_t stream, const float* a, int batch, int T, int W,
                            int rank, uint64_t seed, int oversampling, int power_iterations, float* left,
                            float* right, bool precise = false, float* sv = nullptr);
// tcgen05 range-finder GEMM (compact_gemm.cu).  a: bf16 [batch][T][W];
// xt: bf16 [batch or 1][range_gemm_npad()][K] (X^T, zero rows beyond n);
// c: fp32 [batch][M][ldc] (ldc 0 = n) with M = trans_a ? W : T, K = trans_a ? T : W; accumulate: c += A X.
// Returns the compaction scratch pool's idle pages to the device.
void svd_pool_trim();
// Maps `bytes` into the compaction scratch pool ahead of a timed region.
void svd_pool_reserve(size_t bytes, cudaStream_t st);
int range_gemm_npad();
// bf16 [batch][rows][cols] row-major as a 3-D tensor map, box {64, box_rows, 1}, 128-byte swizzle,
// out-of-bounds rows zero-filled.
CUtensorMap encode_bf16_map(const void* base, int cols, int rows, int batch, int box_rows);
void range_gemm(const __nv_bfloat16* a, int T, int W, int batch, bool trans_a, const __nv_bfloat16* xt, bool x_batched,
                int n, float* c, cudaStream_t st, bool accumulate = false, int ldc = 0);
// fp32 [batch][rows][cols] (row stride ld, batch stride in_stride) -> bf16 [batch][npad][rows];
// The three-term hi/lo product a x + a x_lo + a_lo x in one launch (one GEMM with a 3x K loop).
void range_gemm3(const __nv_bfloat16* a, const __nv_bfloat16* a_lo, int T, int W, int batch, bool trans_a,
                 const __nv_bfloat16* xt, const __nv_bfloat16* xt_lo, bool x_batched, int n, float* c, cudaStream_t st,
                 bool accumulate = false, int ldc = 0);
// lo: the bf16 residual x - bf16(x) instead.
void transpose_to_bf16(const float* in, long in_stride, int rows, int cols, int ld, __nv_bfloat16* out, int batch,
                       cudaStream_t st, bool lo = false);
// Small dense factorisations of the randomized SVD (small_linalg.cu).
// g: [batch][k][k] fp64 symmetric (overwritten); lo: [batch][k][k] fp64 lower factor,
// g + shift_rel*trace/k*I = lo lo^T; lf (optional): fp32 copy with reciprocal diagonal (trsm_rows
// operand); perm: [batch][k] (identity).
void chol_batched(double* g, int k, int batch, double shift_rel, double* lo, float* lf, int* perm, cudaStream_t st);
// q (row-major [batch][n][k]) = y L^-T (columns in step order); q must not alias y.
void trsm_rows(const float* y, float* q, int n, int k, int batch, const float* lf, const int* perm, cudaStream_t st);
// The same with fp64 arithmetic against the fp64 factor lo (precise path).
void trsm_rows_f64(const float* y, float* q, int n, int k, int batch, const double* lo, const int* perm,
                   cudaStream_t st);
// Eigenvectors of C = lo lo^T by one-sided block Jacobi on the columns of lo (fp32 work matrix x:
// [batch][jacobi_kp(k)]^2, flags: [max_sweeps][batch] ints); us/ui: column-major k x R Ritz factors
// (U_R s_R, U_R / s_R), sv: descending singular values of the top R (optional).
int jacobi_kp(int k);
size_t jacobi_ws_ints(int k, int batch, int max_sweeps);  // ints of the flags workspace
void jacobi_eig(const double* lo, int k, int batch, int R, float* x, int* flags, int max_sweeps, float tol,
                double rank_tol, float* us, float* ui, float* sv, cudaStream_t st);
}  // namespace kvp
