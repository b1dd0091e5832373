// The small dense linear algebra of the batched randomized SVD, hand-written
// for sm_100a (replaces cuSOLVER potrfBatched / XsyevBatched and cuBLAS
// trsmBatched in compact.cu).
//
// Reference steps (linalg.cpp:68-105): thin_q = Eigen::HouseholderQR of the
// sketch (linalg.cpp:80-84) and the BDCSVD of B = Q^T A (linalg.cpp:93).  Here:
//
//   thin_q(Y)  -> shifted CholeskyQR:  G = Y^T Y,  G + shift = L L^T  (fp64, blocked right-looking:
//                 a panel launch and a tiled trailing-update launch per 32 columns),  Q = Y L^-T
//                 (trsm_rows_kernel: blocked forward substitution, 32 rows of Y
//                 per CTA, warp-shuffle triangular core).
//   SVD of B   -> C = B B^T (k x k, fp64); Cholesky C = X X^T (a round-off sized
//                 shift makes a semidefinite C factor); one-sided block Jacobi on the columns
//                 of X (jacobi_round_kernel: 16-column blocks, one launch per
//                 round of the circle tournament, every pair of the round in its
//                 own CTA, 32x32 inner Jacobi in shared memory); at convergence
//                 X = U diag(s), so U (eigenvectors of C = left singular vectors
//                 of B) and s come from the column norms (jacobi_finish_kernel:
//                 norms, descending sort, U_R s_R and U_R / s_R).
//
// No V is accumulated: X V = U diag(s) with X X^T = C gives C = U diag(s^2) U^T
// directly from the final columns.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "compact.cuh"

namespace kvp {
namespace {

// ---------------------------------------------------------------------------
// Batched Cholesky, fp64, blocked right-looking over 32-column panels, two launches per panel:
//   chol_panel_kernel  (64-row chunks of the panel per CTA): factor the 32 x 32 diagonal block in
//                      registers (one warp, lane = row, shuffles; every chunk's CTA redundantly),
//                      then its rows of the panel, L_iJ = S_iJ L_JJ^-T (one thread per row, forward
//                      substitution in registers against the reciprocal diagonal);
//   chol_update_kernel (one CTA per 64 x 64 tile of the trailing lower triangle, every matrix):
//                      S_im -= L_iJ L_mJ^T.
//   s    : [batch][k][k] symmetric input (lower triangle read), overwritten by the updates
//   lo   : [batch][k][k] lower factor L (zeros above), g + shift = L L^T
//   lf   : optional fp32 copy of L with the diagonal replaced by its reciprocal (trsm_rows operand)
//   perm : [batch][k] identity (the trsm_rows interface takes a column order)
// shift = shift_rel * trace/k (chol_prep_kernel): the shifted CholeskyQR of the range finder uses
// 1e-5 / 1e-7, the PSD factorisations a round-off sized 1e-13 (a semidefinite C then factors
// without pivoting; its null directions get columns of size sqrt(shift), far below the rank
// tolerance).  A non-positive pivot gives a zero column.
// ---------------------------------------------------------------------------
constexpr int kCp = 32;  // panel width

__global__ void chol_prep_kernel(double* __restrict__ s_all, int k, double shift_rel, int* __restrict__ perm_all) {
  __shared__ double red[32];
  const int b = blockIdx.x, tid = threadIdx.x;
  double* S = s_all + static_cast<size_t>(b) * k * k;
  double tr = 0.0;
  for (int i = tid; i < k; i += blockDim.x) {
    tr += S[static_cast<size_t>(i) * k + i];
    perm_all[static_cast<size_t>(b) * k + i] = i;
  }
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  if ((tid & 31) == 0) red[tid >> 5] = tr;
  __syncthreads();
  if (tid < 32) {
    double t = tid < static_cast<int>(blockDim.x >> 5) ? red[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (tid == 0) red[0] = t;
  }
  __syncthreads();
  const double shift = shift_rel * red[0] / k + 1e-300;
  for (int i = tid; i < k; i += blockDim.x) S[static_cast<size_t>(i) * k + i] += shift;
}

__global__ void __launch_bounds__(64)
    chol_panel_kernel(const double* __restrict__ s_all, int k, int j0, double* __restrict__ lo_all) {
  __shared__ double D[kCp][kCp + 1];
  __shared__ double dinv[kCp];
  const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const double* S = s_all + static_cast<size_t>(b) * k * k;
  double* lo = lo_all + static_cast<size_t>(b) * k * k;
  const int nb = min(kCp, k - j0);
  // rows of the panel below are split over gridDim.x CTAs; each factors the diagonal block itself
  const int rows_per = (k - j0 - nb + gridDim.x - 1) / gridDim.x;
  const int rbeg = j0 + nb + blockIdx.x * rows_per, rend = min(k, rbeg + rows_per);
  for (int e = tid; e < kCp * kCp; e += blockDim.x) {
    const int r = e / kCp, c = e % kCp;
    D[r][c] = (r < nb && c <= r) ? S[static_cast<size_t>(j0 + r) * k + j0 + c] : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    // lane = row r of the diagonal block, held in registers; column c: the pivot comes from lane c,
    // rows below scale their entry and take the rank-1 update with the other rows' column-c
    // entries by shuffle (fully unrolled: static register indices, no shared-memory round trips)
    double row[kCp];
#pragma unroll
    for (int q = 0; q < kCp; ++q) row[q] = D[lane][q];
#pragma unroll
    for (int c = 0; c < kCp; ++c) {
      if (c < nb) {
        const double piv = __shfl_sync(0xffffffffu, row[c], c);
        const double l = piv > 0.0 ? sqrt(piv) : 0.0;
        const double inv = piv > 0.0 ? 1.0 / l : 0.0;
        if (lane == c) row[c] = l;
        else if (lane > c) row[c] *= inv;
        const double lc = row[c];
#pragma unroll
        for (int q = c + 1; q < kCp; ++q) {
          const double lq = __shfl_sync(0xffffffffu, lc, q);  // L[q][c]
          if (lane >= q) row[q] = fma(-lc, lq, row[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kCp; ++q) D[lane][q] = (lane < nb && q <= lane) ? row[q] : 0.0;
    const double dl = D[lane][lane];  // this lane's own store above
    dinv[lane] = (lane < nb && dl > 0.0) ? 1.0 / dl : 0.0;
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int e = tid; e < nb * nb; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      if (c <= r) lo[static_cast<size_t>(j0 + r) * k + j0 + c] = D[r][c];
    }
  // panel below: row i solves x L_JJ^T = S[i][J]
  for (int i = rbeg + tid; i < rend; i += blockDim.x) {
    double x[kCp];
    const double* srow = S + static_cast<size_t>(i) * k + j0;
#pragma unroll
    for (int c = 0; c < kCp; ++c) x[c] = c < nb ? srow[c] : 0.0;
#pragma unroll
    for (int c = 0; c < kCp; ++c) {
      if (c < nb) {
        double v = x[c];
        for (int t = 0; t < c; ++t) v = fma(-x[t], D[c][t], v);
        x[c] = v * dinv[c];
      }
    }
    double* lrow = lo + static_cast<size_t>(i) * k + j0;
#pragma unroll
    for (int c = 0; c < kCp; ++c)
      if (c < nb) lrow[c] = x[c];
  }
}

// Trailing update of the lower triangle below panel j0: one CTA per 64 x 64 tile (ta >= tb),
// thread -> 4 x 4 register tile, L rows staged in shared memory.
constexpr int kCu = 64;
__global__ void __launch_bounds__(256)
    chol_update_kernel(double* __restrict__ s_all, int k, int j0, const double* __restrict__ lo_all) {
  __shared__ double La[kCu][kCp + 1], Lb[kCu][kCp + 1];
  const int b = blockIdx.y, tid = threadIdx.x;
  const int r0 = j0 + kCp;
  const int tt = blockIdx.x;
  int ta = static_cast<int>((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
  while ((ta + 1) * (ta + 2) / 2 <= tt) ++ta;
  while (ta * (ta + 1) / 2 > tt) --ta;
  const int tb = tt - ta * (ta + 1) / 2;
  const int i0 = r0 + ta * kCu, m0 = r0 + tb * kCu;
  double* S = s_all + static_cast<size_t>(b) * k * k;
  const double* lo = lo_all + static_cast<size_t>(b) * k * k;
  for (int e = tid; e < kCu * kCp; e += blockDim.x) {
    const int r = e / kCp, c = e % kCp;
    La[r][c] = i0 + r < k ? lo[static_cast<size_t>(i0 + r) * k + j0 + c] : 0.0;
    Lb[r][c] = m0 + r < k ? lo[static_cast<size_t>(m0 + r) * k + j0 + c] : 0.0;
  }
  __syncthreads();
  const int ri = (tid >> 4) * 4, ci = (tid & 15) * 4;
  double acc[4][4] = {};
#pragma unroll 4
  for (int t = 0; t < kCp; ++t) {
    double av[4], bv[4];
    for (int x = 0; x < 4; ++x) {
      av[x] = La[ri + x][t];
      bv[x] = Lb[ci + x][t];
    }
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
  }
  for (int x = 0; x < 4; ++x) {
    const int i = i0 + ri + x;
    if (i >= k) continue;
    for (int y = 0; y < 4; ++y) {
      const int m = m0 + ci + y;
      if (m < k && m <= i) S[static_cast<size_t>(i) * k + m] -= acc[x][y];
    }
  }
}

__global__ void chol_lf_kernel(const double* __restrict__ lo_all, int k, float* __restrict__ lf_all) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<long>(k) * k) return;
  const size_t off = static_cast<size_t>(blockIdx.y) * k * k;
  const int j = static_cast<int>(e / k), t = static_cast<int>(e % k);
  const double dd = lo_all[off + e];
  float v = 0.f;
  if (t < j) v = static_cast<float>(dd);
  else if (t == j) v = dd > 0.0 ? static_cast<float>(1.0 / dd) : 0.f;
  lf_all[off + e] = v;
}

// ---------------------------------------------------------------------------
// Q = Y L^-T for row-major Y [batch][n][k]: every row y solves L q = y[perm],
// (lf: the fp32 lower factor with reciprocal diagonal).  32 rows per CTA (one
// warp per 4 rows, lane = column inside a 32-column block); per block the
// off-diagonal part is a GEMM against the solved columns with L staged 128
// columns at a time, the 32 x 32 diagonal part a warp-shuffle forward substitution.
// ---------------------------------------------------------------------------
constexpr int kTrThreads = 256;
constexpr int kTrStage = 128;

// T = float: l is the fp32 factor with reciprocal diagonal (lf); T = double: l is the fp64
// factor itself (lo), for the precise path (fp64 arithmetic keeps the span of an
// ill-conditioned Y to fp32 rounding of the output).
template <typename T>
__global__ void __launch_bounds__(kTrThreads)
    trsm_rows_kernel(const float* __restrict__ y_all, float* __restrict__ q_all, int n, int k,
                     const T* __restrict__ l_all, const int* __restrict__ perm_all) {
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  T* tsm = reinterpret_cast<T*>(tsm_raw);
  const int kp = (k + 31) & ~31;
  const int kTrRows = (blockDim.x >> 5) * 4;  // 4 rows per warp
  const int ld = kp + 4;                      // 16-byte aligned rows
  T* qs = tsm;                                // [kTrRows][ld]
  T* ls = qs + static_cast<size_t>(kTrRows) * ld;  // [kTrStage (t)][33] staged L block^T
  const int b = blockIdx.y, r0 = blockIdx.x * kTrRows;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* y = y_all + static_cast<size_t>(b) * n * k;
  float* q = q_all + static_cast<size_t>(b) * n * k;
  const T* lf = l_all + static_cast<size_t>(b) * k * k;
  const int* perm = perm_all + static_cast<size_t>(b) * k;
  for (int e = tid; e < kTrRows * kp; e += blockDim.x) {
    const int r = e / kp, c = e % kp;
    T v = 0;
    if (r0 + r < n && c < k) v = y[static_cast<size_t>(r0 + r) * k + perm[c]];
    qs[r * ld + c] = v;
  }
  __syncthreads();
  for (int j0 = 0; j0 < kp; j0 += 32) {
    const int c = j0 + lane;  // this lane's column in the block
    T acc[4];
    for (int x = 0; x < 4; ++x) acc[x] = qs[(warp * 4 + x) * ld + c];
    // off-diagonal: acc -= sum_{t < j0} L[c][t] q[r][t]
    for (int t0 = 0; t0 < j0; t0 += kTrStage) {
      const int tw = min(kTrStage, j0 - t0);  // a multiple of 32
      __syncthreads();
      for (int e = tid; e < 32 * tw; e += blockDim.x) {
        const int cr = e / tw, tt = e % tw;  // row j0+cr of L, column t0+tt
        ls[tt * 33 + cr] = (j0 + cr < k) ? lf[static_cast<size_t>(j0 + cr) * k + t0 + tt] : T(0);
      }
      __syncthreads();
      for (int tt = 0; tt < tw; tt += 4) {
        const T l0 = ls[tt * 33 + lane], l1 = ls[(tt + 1) * 33 + lane], l2 = ls[(tt + 2) * 33 + lane],
                l3 = ls[(tt + 3) * 33 + lane];
        for (int x = 0; x < 4; ++x) {
          const T* qr = &qs[(warp * 4 + x) * ld + t0 + tt];
          T q0, q1, q2, q3;
          if constexpr (sizeof(T) == 4) {
            const float4 qv = *reinterpret_cast<const float4*>(qr);
            q0 = qv.x;
            q1 = qv.y;
            q2 = qv.z;
            q3 = qv.w;
          } else {
            const double2 qa = *reinterpret_cast<const double2*>(qr), qb = *reinterpret_cast<const double2*>(qr + 2);
            q0 = qa.x;
            q1 = qa.y;
            q2 = qb.x;
            q3 = qb.y;
          }
          acc[x] = fma(-l0, q0, acc[x]);
          acc[x] = fma(-l1, q1, acc[x]);
          acc[x] = fma(-l2, q2, acc[x]);
          acc[x] = fma(-l3, q3, acc[x]);
        }
      }
    }
    // diagonal block: stage L[j0.., j0..]
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
      const int cr = e / 32, tt = e % 32;
      ls[tt * 33 + cr] = (j0 + cr < k && j0 + tt < k) ? lf[static_cast<size_t>(j0 + cr) * k + j0 + tt] : T(0);
    }
    __syncthreads();
    T dinv = ls[lane * 33 + lane];
    if constexpr (sizeof(T) == 8) dinv = dinv > 0 ? 1.0 / dinv : 0.0;
    for (int jj = 0; jj < 32; ++jj) {
      const T l = ls[jj * 33 + lane];  // L[j0+lane][j0+jj]
      for (int x = 0; x < 4; ++x) {
        const T qv = __shfl_sync(0xffffffffu, acc[x] * dinv, jj);
        if (lane == jj) acc[x] = qv;
        else if (lane > jj) acc[x] = fma(-l, qv, acc[x]);
      }
    }
    for (int x = 0; x < 4; ++x) qs[(warp * 4 + x) * ld + c] = acc[x];
  }
  __syncthreads();
  for (int e = tid; e < kTrRows * k; e += blockDim.x) {
    const int r = e / k, c = e % k;
    if (r0 + r < n) q[static_cast<size_t>(r0 + r) * k + c] = static_cast<float>(qs[r * ld + c]);
  }
}

// ---------------------------------------------------------------------------
// One-sided block Jacobi.  X: [batch][kp][kp] fp32 column-major (column c at
// X + c*kp), kp a multiple of 64 (the row chunk); 16-column blocks, nb = kp/16 of them.  Round
// `rnd` of the circle tournament pairs block nb-1 with rnd and (rnd+p)%m with
// (rnd-p)%m (m = nb-1): every pair of blocks meets once per sweep.  Each CTA:
//   G = X_P^T X_P (32 x 32) streamed over 64-row chunks,
//   convergence test max |g_ij| / sqrt(g_ii g_jj) <= tol  -> no change,
//   one cyclic sweep of two-sided Jacobi on G accumulating J,
//   X_P <- X_P J.
// flags[sweep][b] = 1 when any pair of matrix b rotated in that sweep; a matrix
// whose previous sweep had no rotation is converged and its CTAs exit.
// ---------------------------------------------------------------------------
constexpr int kJb = 16;
constexpr int kJw = 2 * kJb;   // 32 columns per pair
constexpr int kJThreads = 256;
constexpr int kJChunk = 64;    // rows per streamed chunk

__global__ void __launch_bounds__(kJThreads, 4)
    jacobi_round_kernel(float* __restrict__ x_all, int kp, int rnd, int sweep, int* __restrict__ flags, int batch,
                        float tol, int max_sweeps) {
  __shared__ __align__(16) float xc[kJChunk][kJw + 4];
  __shared__ float gs[kJw][kJw + 1];
  __shared__ float gs2[kJw][kJw + 1];
  __shared__ __align__(16) float js[kJw][kJw + 4];
  __shared__ float red[kJThreads / 32];
  const int b = blockIdx.y, pi = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  if (sweep > 0 && flags[(sweep - 1) * batch + b] == 0) return;
  const int nb = kp / kJb, m = nb - 1;
  int P, Qb;
  if (pi == 0) {
    P = nb - 1;
    Qb = rnd;
  } else {
    P = (rnd + pi) % m;
    Qb = (rnd - pi + m) % m;
  }
  // A pair found converged stays converged until one of its blocks is rotated with another
  // partner: block stamps (round of the last rotation) and pair stamps (round found converged)
  // let it skip the Gram.
  int* bstamp = flags + max_sweeps * batch + b * nb;
  int* pstamp = flags + max_sweeps * batch + batch * nb + static_cast<size_t>(b) * nb * nb;
  const int now = sweep * m + rnd + 1;
  const int pq = min(P, Qb) * nb + max(P, Qb);
  {
    const int ps = pstamp[pq];
    if (ps > 0 && bstamp[P] < ps && bstamp[Qb] < ps) return;
  }
  float* x = x_all + static_cast<size_t>(b) * kp * kp;
  auto col_ptr = [&](int c) { return x + static_cast<size_t>(c < kJb ? P * kJb + c : Qb * kJb + c - kJb) * kp; };
  // Chunk staging, software-pipelined: the next 64-row chunk's global loads are issued into
  // registers before the current chunk is computed, so their latency hides behind the FMAs.
  // lane -> column, warp -> 8 consecutive rows (one 32-byte sector per lane; conflict-free stores)
  float4 pa, pb;
  auto fetch_chunk = [&](int r0) {
    const int c = tid & 31, rr = (tid >> 5) * 8;
    const float* src = col_ptr(c) + r0 + rr;
    pa = *reinterpret_cast<const float4*>(src);
    pb = *reinterpret_cast<const float4*>(src + 4);
  };
  auto store_chunk = [&]() {
    const int c = tid & 31, rr = (tid >> 5) * 8;
    xc[rr + 0][c] = pa.x;
    xc[rr + 1][c] = pa.y;
    xc[rr + 2][c] = pa.z;
    xc[rr + 3][c] = pa.w;
    xc[rr + 4][c] = pb.x;
    xc[rr + 5][c] = pb.y;
    xc[rr + 6][c] = pb.z;
    xc[rr + 7][c] = pb.w;
  };
  // ---- Gram G = X_P^T X_P: four row groups of 16 rows per 64-row chunk; inside a group
  // thread (ti, tj) owns the 4 x 4 tile G[4ti.., 4tj..] (two float4 shared loads per 16 FMA).
  // Chunk partials are summed in fp32, chunks and groups in fp64 (the convergence test
  // compares normalised |g_ij| against tol).
  const int rg = tid >> 6, ti = (tid >> 3) & 7, tj = tid & 7;
  double accd[4][4];
  for (int x = 0; x < 4; ++x)
    for (int y = 0; y < 4; ++y) accd[x][y] = 0.0;
  fetch_chunk(0);
  for (int r0 = 0; r0 < kp; r0 += kJChunk) {
    store_chunk();
    __syncthreads();
    if (r0 + kJChunk < kp) fetch_chunk(r0 + kJChunk);
    float acc[4][4] = {};
#pragma unroll 4
    for (int r = rg * 16; r < rg * 16 + 16; ++r) {
      const float4 va = *reinterpret_cast<const float4*>(&xc[r][4 * ti]);
      const float4 vb = *reinterpret_cast<const float4*>(&xc[r][4 * tj]);
      const float av[4] = {va.x, va.y, va.z, va.w}, bv[4] = {vb.x, vb.y, vb.z, vb.w};
      for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
    }
    for (int x = 0; x < 4; ++x)
      for (int y = 0; y < 4; ++y) accd[x][y] += acc[x][y];
    __syncthreads();
  }
  __shared__ double gd[kJw][kJw + 1];
  for (int g = 0; g < 4; ++g) {
    if (rg == g)
      for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) {
          double& e = gd[4 * ti + x][4 * tj + y];
          e = (g == 0 ? 0.0 : e) + accd[x][y];
        }
    __syncthreads();
  }
  float off = 0.f;
  for (int e = tid; e < kJw * kJw; e += kJThreads) {
    const int i = e / kJw, j = e % kJw;
    gs[i][j] = static_cast<float>(gd[i][j]);
    if (i == j) continue;
    const double nn = gd[i][i] * gd[j][j];
    if (nn > 0.0) off = fmaxf(off, static_cast<float>(fabs(gd[i][j]) * rsqrt(nn)));
  }
  for (int e = tid; e < kJw * kJw; e += kJThreads) js[e / kJw][e % kJw] = (e / kJw == e % kJw) ? 1.f : 0.f;
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) off = fmaxf(off, __shfl_xor_sync(0xffffffffu, off, o));
  if (lane == 0) red[warp] = off;
  __syncthreads();
  off = 0.f;
  for (int w = 0; w < kJThreads / 32; ++w) off = fmaxf(off, red[w]);
  if (!(off > tol)) {  // uniform across the CTA
    if (tid == 0) pstamp[pq] = now;
    return;
  }
  if (tid == 0) {
    flags[sweep * batch + b] = 1;
    bstamp[P] = now;
    bstamp[Qb] = now;
  }
  // ---- one cyclic sweep of two-sided Jacobi on G (31 rounds of 16 disjoint rotations).
  // Thread t owns the 2x2 block (pair p = t/16, pair q = t%16) of the round's pairing and
  // writes G'_pq = R_p^T G_pq R_q from the previous G (double buffer: one barrier per
  // round); both owners of a pair recompute its rotation from the same old entries.
  // J' = J R in place: rows 2(t/16), +1 of pair t%16.
  {
    float* gsrc = &gs[0][0];
    float* gdst = &gs2[0][0];
    constexpr int ld = kJw + 1;
    const int p = tid >> 4, q = tid & 15;
    const float thr = 0.25f * tol;
    // the inner circle schedule (31 rounds x 16 pairs, i < j) as a shared table
    __shared__ unsigned char sched[kJw - 1][kJb][2];
    for (int e = tid; e < (kJw - 1) * kJb; e += kJThreads) {
      const int ir = e / kJb, x = e % kJb;
      int i = ir, j = kJw - 1;
      if (x != 0) {
        i = (ir + x) % (kJw - 1);
        j = (ir - x + kJw - 1) % (kJw - 1);
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
      }
      sched[ir][x][0] = static_cast<unsigned char>(i);
      sched[ir][x][1] = static_cast<unsigned char>(j);
    }
    __syncthreads();
    auto pair_of = [&](int ir, int x, int& i, int& j) {
      i = sched[ir][x][0];
      j = sched[ir][x][1];
    };
    auto rot = [&](const float* g, int i, int j, float& c, float& s) {
      const float gii = g[i * ld + i], gjj = g[j * ld + j], gij = g[i * ld + j];
      c = 1.f;
      s = 0.f;
      if (gij * gij > thr * thr * fmaxf(gii * gjj, 0.f) && gij != 0.f) {
        const float zeta = __fdividef(gjj - gii, 2.f * gij);
        const float t = __fdividef(copysignf(1.f, zeta), fabsf(zeta) + sqrtf(fmaf(zeta, zeta, 1.f)));
        // c = (1 + t^2)^-1/2 with one Newton step on rsqrtf: c^2 + s^2 = 1 to rounding (a biased
        // rsqrtf alone compounds over the thousands of rotations a column sees)
        const float u = fmaf(t, t, 1.f);
        float r = rsqrtf(u);
        r = r * fmaf(-0.5f * u, r * r, 1.5f);
        c = r;
        s = r * t;
      }
    };
    for (int ir = 0; ir < kJw - 1; ++ir) {
      int ip, jp, iq, jq;
      pair_of(ir, p, ip, jp);
      pair_of(ir, q, iq, jq);
      // every warp computes the round's 16 rotations once (lane l: pair l % 16) and hands
      // them out by shuffle
      float cl, sl;
      {
        int il, jl;
        pair_of(ir, lane & 15, il, jl);
        rot(gsrc, il, jl, cl, sl);
      }
      const float cp = __shfl_sync(0xffffffffu, cl, p & 15), sp = __shfl_sync(0xffffffffu, sl, p & 15);
      const float cq = __shfl_sync(0xffffffffu, cl, q), sq = __shfl_sync(0xffffffffu, sl, q);
      const float a = gsrc[ip * ld + iq], bb = gsrc[ip * ld + jq], c = gsrc[jp * ld + iq], d = gsrc[jp * ld + jq];
      const float a1 = cp * a - sp * c, b1 = cp * bb - sp * d, c1 = sp * a + cp * c, d1 = sp * bb + cp * d;
      gdst[ip * ld + iq] = cq * a1 - sq * b1;
      gdst[ip * ld + jq] = sq * a1 + cq * b1;
      gdst[jp * ld + iq] = cq * c1 - sq * d1;
      gdst[jp * ld + jq] = sq * c1 + cq * d1;
      for (int mm = 2 * p; mm < 2 * p + 2; ++mm) {
        const float x0 = js[mm][iq], x1 = js[mm][jq];
        js[mm][iq] = cq * x0 - sq * x1;
        js[mm][jq] = sq * x0 + cq * x1;
      }
      __syncthreads();
      float* t = gsrc;
      gsrc = gdst;
      gdst = t;
    }
  }
  // ---- X_P <- X_P J, chunk by chunk (in place: a chunk is staged before it is overwritten).
  // Thread (rr = tid/8, cg = tid%8) computes rows 2rr, 2rr+1 x columns 4cg..4cg+3.
  {
    const int rr = tid >> 3, cg = tid & 7;
    fetch_chunk(0);
    for (int r0 = 0; r0 < kp; r0 += kJChunk) {
      store_chunk();
      __syncthreads();
      if (r0 + kJChunk < kp) fetch_chunk(r0 + kJChunk);
      float o[2][4] = {};
#pragma unroll 2
      for (int mm = 0; mm < kJw; mm += 4) {
        const float4 x0 = *reinterpret_cast<const float4*>(&xc[2 * rr][mm]);
        const float4 x1 = *reinterpret_cast<const float4*>(&xc[2 * rr + 1][mm]);
        const float a0[4] = {x0.x, x0.y, x0.z, x0.w}, a1[4] = {x1.x, x1.y, x1.z, x1.w};
        for (int u = 0; u < 4; ++u) {
          const float4 jv = *reinterpret_cast<const float4*>(&js[mm + u][4 * cg]);
          const float jj[4] = {jv.x, jv.y, jv.z, jv.w};
          for (int y = 0; y < 4; ++y) {
            o[0][y] = fmaf(a0[u], jj[y], o[0][y]);
            o[1][y] = fmaf(a1[u], jj[y], o[1][y]);
          }
        }
      }
      __syncthreads();
      *reinterpret_cast<float4*>(&xc[2 * rr][4 * cg]) = make_float4(o[0][0], o[0][1], o[0][2], o[0][3]);
      *reinterpret_cast<float4*>(&xc[2 * rr + 1][4 * cg]) = make_float4(o[1][0], o[1][1], o[1][2], o[1][3]);
      __syncthreads();
      {
        const int c = tid & 31, r8 = (tid >> 5) * 8;
        float* dst = col_ptr(c) + r0 + r8;
        *reinterpret_cast<float4*>(dst) = make_float4(xc[r8][c], xc[r8 + 1][c], xc[r8 + 2][c], xc[r8 + 3][c]);
        *reinterpret_cast<float4*>(dst + 4) =
            make_float4(xc[r8 + 4][c], xc[r8 + 5][c], xc[r8 + 6][c], xc[r8 + 7][c]);
      }
      __syncthreads();
    }
  }
}

// X (fp32 [batch][kp][kp] column-major, zero padded) from lo (fp64 [batch][k][k], rows original order).
__global__ void lo_to_x_kernel(const double* __restrict__ lo_all, int k, float* __restrict__ x_all, int kp) {
  const int b = blockIdx.y;
  const double* lo = lo_all + static_cast<size_t>(b) * k * k;
  float* x = x_all + static_cast<size_t>(b) * kp * kp;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < static_cast<long>(kp) * kp;
       e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(e / kp), i = static_cast<int>(e % kp);
    x[e] = (c < k && i < k) ? static_cast<float>(lo[static_cast<size_t>(i) * k + c]) : 0.f;
  }
}

// Column norms (fp64), descending order (ties: lower column first), then the
// Ritz factors of the top R: us[:, j] = u_j s_j = x_src, ui[:, j] = u_j / s_j =
// x_src / s_j^2 (column-major k x R), sv[j] = s_j.  Components at or below
// kTol * s_max are dead (zeros; compact.cu fills an orthonormal complement).
constexpr int kFinThreads = 1024;
__global__ void __launch_bounds__(kFinThreads)
    jacobi_finish_kernel(const float* __restrict__ x_all, int kp, int k, int R, float* __restrict__ us_all,
                         float* __restrict__ ui_all, float* __restrict__ sv_all, double rank_tol) {
  extern __shared__ double fsm[];
  const int ns = 2 * kFinThreads;  // sort slots (kp <= 2048)
  double* key = fsm;
  int* idx = reinterpret_cast<int*>(key + ns);
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* x = x_all + static_cast<size_t>(b) * kp * kp;
  // one warp per column norm
  for (int c = warp; c < ns; c += kFinThreads / 32) {
    double s = 0.0;
    if (c < k)
      for (int i = lane; i < k; i += 32) {
        const double v = x[static_cast<size_t>(c) * kp + i];
        s = fma(v, v, s);
      }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      key[c] = c < k ? sqrt(s) : -1.0;
      idx[c] = c;
    }
  }
  __syncthreads();
  // bitonic sort, descending key, ascending index on ties
  for (int size = 2; size <= ns; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < ns / 2; t += kFinThreads) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const double ka = key[lo], kb = key[hi];
        const int ia = idx[lo], ib = idx[hi];
        const bool a_first = ka > kb || (ka == kb && ia < ib);
        if (a_first != desc) {
          key[lo] = kb;
          key[hi] = ka;
          idx[lo] = ib;
          idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  const double top = key[0];
  float* us = us_all + static_cast<size_t>(b) * k * R;
  float* ui = ui_all + static_cast<size_t>(b) * k * R;
  for (int e = tid; e < k * R; e += kFinThreads) {
    const int j = e / k, i = e % k;
    const double s = key[j];
    const bool live = s > rank_tol * top && s > 0.0;
    const double v = x[static_cast<size_t>(idx[j]) * kp + i];
    us[e] = live ? static_cast<float>(v) : 0.f;
    ui[e] = live ? static_cast<float>(v / (s * s)) : 0.f;
  }
  if (sv_all)
    for (int j = tid; j < R; j += kFinThreads) sv_all[static_cast<size_t>(b) * R + j] = static_cast<float>(key[j]);
}


}  // namespace

void chol_batched(double* g, int k, int batch, double shift_rel, double* lo, float* lf, int* perm, cudaStream_t st) {
  require(k >= 1, KVP_ERR_PARAMETER, "chol: k out of range");
  KVP_CUDA(cudaMemsetAsync(lo, 0, sizeof(double) * batch * k * k, st));
  chol_prep_kernel<<<batch, 256, 0, st>>>(g, k, shift_rel, perm);
  KVP_LAUNCHED();
  for (int j0 = 0; j0 < k; j0 += kCp) {
    const int below = k - j0 - kCp;
    chol_panel_kernel<<<dim3(below > 0 ? cdiv(below, 64) : 1, batch), 64, 0, st>>>(g, k, j0, lo);
    KVP_LAUNCHED();
    const int n = k - j0 - kCp;
    if (n <= 0) break;
    const int nt = (n + kCu - 1) / kCu;
    chol_update_kernel<<<dim3(nt * (nt + 1) / 2, batch), 256, 0, st>>>(g, k, j0, lo);
    KVP_LAUNCHED();
  }
  if (lf) {
    chol_lf_kernel<<<dim3(cdiv(static_cast<long>(k) * k, 256), batch), 256, 0, st>>>(lo, k, lf);
    KVP_LAUNCHED();
  }
}

template <typename T>
void trsm_rows_t(const float* y, float* q, int n, int k, int batch, const T* l, const int* perm, cudaStream_t st) {
  const int kp = (k + 31) & ~31;
  // 32 rows per CTA (8 warps), 16 for very wide sketches
  const size_t stage = static_cast<size_t>(kTrStage) * 33 * sizeof(T);
  const int threads = 32 * (kp + 4) * sizeof(T) + stage <= 160 * 1024 ? kTrThreads : kTrThreads / 2;
  const int rows = (threads >> 5) * 4;
  const size_t smem = static_cast<size_t>(rows) * (kp + 4) * sizeof(T) + stage;
  require(smem <= 220 * 1024, KVP_ERR_PARAMETER, "trsm: k too large");
  KVP_CUDA(cudaFuncSetAttribute(trsm_rows_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(cdiv(n, rows), batch);
  trsm_rows_kernel<T><<<grid, threads, smem, st>>>(y, q, n, k, l, perm);
  KVP_LAUNCHED();
}

void trsm_rows(const float* y, float* q, int n, int k, int batch, const float* lf, const int* perm, cudaStream_t st) {
  trsm_rows_t<float>(y, q, n, k, batch, lf, perm, st);
}

void trsm_rows_f64(const float* y, float* q, int n, int k, int batch, const double* lo, const int* perm,
                   cudaStream_t st) {
  trsm_rows_t<double>(y, q, n, k, batch, lo, perm, st);
}

int jacobi_kp(int k) { return (k + kJChunk - 1) / kJChunk * kJChunk; }
size_t jacobi_ws_ints(int k, int batch, int max_sweeps) {
  const size_t nb = static_cast<size_t>(jacobi_kp(k)) / kJb;
  return static_cast<size_t>(max_sweeps) * batch + batch * nb + batch * nb * nb;
}

void jacobi_eig(const double* lo, int k, int batch, int R, float* x, int* flags, int max_sweeps, float tol,
                double rank_tol, float* us, float* ui, float* sv, cudaStream_t st) {
  const int kp = jacobi_kp(k);
  require(kp <= 2 * kFinThreads, KVP_ERR_PARAMETER, "jacobi: k too large");
  lo_to_x_kernel<<<dim3(cdiv(static_cast<long>(kp) * kp, 256 * 8), batch), 256, 0, st>>>(lo, k, x, kp);
  KVP_LAUNCHED();
  KVP_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * jacobi_ws_ints(k, batch, max_sweeps), st));
  const int nb = kp / kJb;
  for (int s = 0; s < max_sweeps; ++s)
    for (int r = 0; r < nb - 1; ++r) {
      jacobi_round_kernel<<<dim3(nb / 2, batch), kJThreads, 0, st>>>(x, kp, r, s, flags, batch, tol, max_sweeps);
      KVP_LAUNCHED();
    }
  const size_t smem = 2 * kFinThreads * (sizeof(double) + sizeof(int));
  jacobi_finish_kernel<<<batch, kFinThreads, smem, st>>>(x, kp, k, R, us, ui, sv, rank_tol);
  KVP_LAUNCHED();
}

}  // namespace kvp
