// The range-finder products of the batched randomized SVD (linalg.cpp:86-92:
// a*omega, a.transpose()*q, a*q, q.transpose()*a) as a hand-written sm_100a
// GEMM: TMA (SWIZZLE_128B tensor maps) -> shared memory ring -> tcgen05.mma
// with the fp32 accumulator in TMEM -> tcgen05.ld epilogue.
//
//   trans_a = false:  C[b] (T x n) = A[b] (T x W) . X[b]        M = T, K = W, A K-major
//   trans_a = true :  C[b] (W x n) = A[b]^T (W x T) . X[b]      M = W, K = T, A MN-major
//
// A is the bf16 segment matrix [batch][T][W]; X is passed transposed, Xt[b] =
// X^T as bf16 [n_pad][K] (K-major B operand, n_pad = 384 >= n, zero rows
// beyond n).  One CTA computes a 128-row M tile for all n_pad columns (two
// N = 192 accumulators), so A is streamed from HBM exactly once per product and
// X (a few MB, shared by the batch's M tiles) is served from L2.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2..5 epilogue (TMEM lane quadrants).
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "compact.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {

using namespace sm100;

constexpr int kGThreads = 192;
constexpr int kGStages = 3;
constexpr int kNHalf = 192;                 // N of one MMA (two halves cover n_pad = 384)
constexpr int kNPad = 2 * kNHalf;
constexpr uint32_t kABytes = 128 * 64 * 2;  // A tile per K step (64): 16 KB
constexpr uint32_t kBBytes = kNPad * 128;   // X^T tile per K step: 384 rows x 128 B = 48 KB
constexpr uint32_t kGStage = kABytes + kBBytes;
constexpr uint32_t kGSmem = kGStages * kGStage + 1024;

// terms = 3: the three-term hi/lo product A_hi X_hi + A_hi X_lo + A_lo X_hi in one launch, as one
// GEMM with a 3x longer K loop (term t of k-step kt = kt / ksteps picks the operand maps), so the
// three terms share the ring, the TMEM accumulator and one epilogue.
template <bool TRANS_A>
__global__ void __launch_bounds__(kGThreads, 1)
    range_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_x,
                      const __grid_constant__ CUtensorMap map_a2, const __grid_constant__ CUtensorMap map_x2, int terms,
                      int M, int K, int n, int x_batched, float* __restrict__ c, long c_stride, int ldc, int accumulate) {
  extern __shared__ __align__(1024) unsigned char gsmem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(gsmem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kGStages], empty[kGStages], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, b = blockIdx.y;
  const int m0 = mt * 128;
  const int ksteps = (K + 63) / 64;  // a partial last step reads zeros (TMA out-of-bounds fill)
  const int ktotal = ksteps * terms;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_x);
    if (terms > 1) {
      prefetch_tmap(&map_a2);
      prefetch_tmap(&map_x2);
    }
  }
  if (warp == 1) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kt = 0; kt < ktotal; ++kt) {
        const int s = kt % kGStages;
        const int term = kt / ksteps, ks = kt - term * ksteps;
        const CUtensorMap* ma = term == 2 ? &map_a2 : &map_a;
        const CUtensorMap* mx = term == 1 ? &map_x2 : &map_x;
        if (kt >= kGStages) mbar_wait(&empty[s], ((kt / kGStages) - 1) & 1);
        unsigned char* sa = smem + s * kGStage;
        unsigned char* sb = sa + kABytes;
        mbar_expect_tx(&full[s], kGStage);
        if (!TRANS_A) {
          // A tile: rows m0..m0+127 (T), columns ks*64.. (W): one K-major SW128 panel
          tma_load_3d(sa, ma, ks * 64, m0, b, &full[s]);
        } else {
          // A^T tile (MN-major): K rows ks*64.. (T) x M columns m0..m0+127 (W), two 64-column panels
          tma_load_3d(sa, ma, m0, ks * 64, b, &full[s]);
          tma_load_3d(sa + kABytes / 2, ma, m0 + 64, ks * 64, b, &full[s]);
        }
        // X^T tile: rows 0..383 (n), columns ks*64.. (K): two 192-row K-major SW128 panels
        tma_load_3d(sb, mx, ks * 64, 0, x_batched ? b : 0, &full[s]);
        tma_load_3d(sb + kNHalf * 128, mx, ks * 64, kNHalf, x_batched ? b : 0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, kNHalf, TRANS_A, false);
      const uint32_t base = smem_addr(smem);
      for (int ks = 0; ks < ktotal; ++ks) {
        const int s = ks % kGStages;
        mbar_wait(&full[s], (ks / kGStages) & 1);
        tc_fence_after();
        const uint32_t sa = base + s * kGStage, sb = sa + kABytes;
        for (int kk = 0; kk < 4; ++kk) {
          // K-major A: 32 bytes per K=16 step inside the 128-byte swizzled row;
          // MN-major A: 16 K rows = 2 KB per step, the two M halves kABytes/2 apart
          const uint64_t ad = TRANS_A ? smem_desc(sa + kk * 2048, kABytes / 2, 1024, kSwizzle128B)
                                      : smem_desc(sa + kk * 32, 16, 1024, kSwizzle128B);
          for (int h = 0; h < 2; ++h) {
            const uint64_t bd = smem_desc(sb + h * kNHalf * 128 + kk * 32, 16, 1024, kSwizzle128B);
            mma_bf16(tmem + h * kNHalf, ad, bd, idesc, (ks | kk) != 0);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(&done);
    }
    __syncwarp();
  } else {
    // epilogue: warp (2..5) % 4 = TMEM lane quadrant; 32 rows x n columns each
    const int qd = warp & 3;
    mbar_wait(&done, 0);
    tc_fence_after();
    const int row = m0 + qd * 32 + lane;
    float* crow = c + static_cast<long>(b) * c_stride + static_cast<long>(row) * ldc;
    for (int c0 = 0; c0 < kNPad; c0 += 8) {
      if (c0 >= n) break;
      float v[8];
      tmem_ld8(tmem + (static_cast<uint32_t>(qd * 32) << 16) + static_cast<uint32_t>(c0), v);
      if (row < M) {
        if (accumulate)
          for (int e = 0; e < 8 && c0 + e < n; ++e) v[e] += crow[c0 + e];
        if (c0 + 8 <= n && (ldc & 3) == 0) {
          *reinterpret_cast<float4*>(crow + c0) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(crow + c0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
        } else {
          for (int e = 0; e < 8 && c0 + e < n; ++e) crow[c0 + e] = v[e];
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  require(fn != nullptr, KVP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// bf16 [batch][rows][cols] row-major as {cols, rows, batch}; box {64, box_rows, 1}, 128-byte swizzle.
CUtensorMap encode_bf16(const void* base, int cols, int rows, int batch, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2, static_cast<cuuint64_t>(cols) * 2 * rows};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, KVP_ERR_CUDA, "cuTensorMapEncodeTiled failed (compaction GEMM operand)");
  return m;
}

// fp32 [batch][rows][cols] (row stride ld) -> bf16 [batch][cols_pad][rows]: the
// transposed, K-major X operand; rows c >= cols are zero.
// lo: the residual bf16(x - bf16(x)) instead of bf16(x) (second term of a hi/lo split).
__global__ void transpose_bf16_kernel(const float* __restrict__ in, long in_stride, int rows, int cols, int ld,
                                      __nv_bfloat16* __restrict__ out, int cols_pad, int lo) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z;
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const float* src = in + static_cast<long>(b) * in_stride;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, cc = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && cc < cols) ? src[static_cast<long>(r) * ld + cc] : 0.f;
  }
  __syncthreads();
  __nv_bfloat16* dst = out + static_cast<long>(b) * cols_pad * rows;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int cc = c0 + i, r = r0 + threadIdx.x;
    if (cc < cols_pad && r < rows) {
      const float x = tile[threadIdx.x][i];
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      dst[static_cast<long>(cc) * rows + r] = lo ? __float2bfloat16_rn(x - __bfloat162float(h)) : h;
    }
  }
}

}  // namespace

CUtensorMap encode_bf16_map(const void* base, int cols, int rows, int batch, int box_rows) {
  return encode_bf16(base, cols, rows, batch, box_rows);
}

int range_gemm_npad() { return kNPad; }

void transpose_to_bf16(const float* in, long in_stride, int rows, int cols, int ld, __nv_bfloat16* out, int batch,
                       cudaStream_t st, bool lo) {
  const dim3 grid((rows + 31) / 32, (kNPad + 31) / 32, batch);
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, st>>>(in, in_stride, rows, cols, ld, out, kNPad, lo ? 1 : 0);
  KVP_LAUNCHED();
}

void range_gemm3(const __nv_bfloat16* a, const __nv_bfloat16* a_lo, int T, int W, int batch, bool trans_a,
                 const __nv_bfloat16* xt, const __nv_bfloat16* xt_lo, bool x_batched, int n, float* c, cudaStream_t st,
                 bool accumulate, int ldc) {
  if (ldc <= 0) ldc = n;
  require(n <= kNPad, KVP_ERR_PARAMETER, "compaction: sketch width above 384 (rank + oversampling)");
  require(T % 8 == 0 && W % 8 == 0, KVP_ERR_PARAMETER, "compaction GEMM: T and W must be multiples of 8");
  const int M = trans_a ? W : T, K = trans_a ? T : W;
  // A: trans_a=false -> box {64 cols (K), 128 rows (M)}; true -> box {64 cols (M), 64 rows (K)}
  const CUtensorMap ma = encode_bf16(a, W, T, batch, trans_a ? 64 : 128);
  const CUtensorMap mx = encode_bf16(xt, K, kNPad, x_batched ? batch : 1, kNHalf);
  const bool three = a_lo != nullptr && xt_lo != nullptr;
  const CUtensorMap ma2 = three ? encode_bf16(a_lo, W, T, batch, trans_a ? 64 : 128) : ma;
  const CUtensorMap mx2 = three ? encode_bf16(xt_lo, K, kNPad, x_batched ? batch : 1, kNHalf) : mx;
  auto kernel = trans_a ? range_gemm_kernel<true> : range_gemm_kernel<false>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[trans_a]) {
    KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGSmem)));
    attr_set[trans_a] = true;
  }
  const dim3 grid((M + 127) / 128, batch);
  kernel<<<grid, kGThreads, kGSmem, st>>>(ma, mx, ma2, mx2, three ? 3 : 1, M, K, n, x_batched ? 1 : 0, c,
                                          static_cast<long>(M) * ldc, ldc, accumulate ? 1 : 0);
  KVP_LAUNCHED();
}

void range_gemm(const __nv_bfloat16* a, int T, int W, int batch, bool trans_a, const __nv_bfloat16* xt,
                bool x_batched, int n, float* c, cudaStream_t st, bool accumulate, int ldc) {
  range_gemm3(a, nullptr, T, W, batch, trans_a, xt, nullptr, x_batched, n, c, st, accumulate, ldc);
}

}  // namespace kvp
