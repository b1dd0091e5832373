// Device-resident LayerCache batch and the caller-facing decode_step /
// compress_now on it — the drop-in for the reference's cache + decoder API
// (cache.hpp:120-146 LayerCache, decoder.hpp:166-191 decode_step /
// compress_now / segment_full_matrix; decoder.cpp:406-628).
//
// A kvp_cache holds `batch` LayerCaches of one layer.  Every instance shares
// the segment structure (token counts, global positions, block layout), so
// each payload is one batch-strided device array:
//   block store  low-rank: left [batch][n][rank_cap], right [batch][rank_cap][W]
//                dense:    rows [batch][n][W]
//   tails        [batch][tail_cap][W] per segment (K and V)
//   importance   [batch][imp_cap] fp64, columns in table (ascending position) order
// Stored ranks are per instance (a variance-target rank scheme picks one per
// matrix); positions and counts are host bookkeeping, like the reference's.
//
// decode_step = projections (skinny GEMM kernel) -> tail append -> tier
// assignment on the device (radix select, importance.cu) -> retrieval plan
// built on the device (stable partition by tier, plan_build_kernel) -> plan
// attention in the low-rank space (attend_plan.cu) or, for serving-shaped bf16
// caches, the fused tcgen05 kernel (decode_fused.cu) -> W_o -> EMA ->
// re-factorisation of segments whose tail reached the period (batched SVD,
// compact.cu).
#include <cublas_v2.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "attend_plan.cuh"
#include "common.cuh"
#include "compact.cuh"
#include "decode_fused.cuh"
#include "importance.cuh"

namespace kvp {
namespace {

// ---------------------------------------------------------------------------
// Owning device buffer.
// ---------------------------------------------------------------------------
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  explicit DBuf(size_t n) { alloc(n); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t n) {
    release();
    if (n) KVP_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct DStore {
  int form = KVP_DENSE;
  int rank_cap = 0;        // columns of `a` / rows of `b` (low-rank)
  std::vector<int> ranks;  // stored rank per instance (low-rank)
  DBuf a;                  // left [batch][n][rank_cap] or rows [batch][n][W]
  DBuf b;                  // right [batch][rank_cap][W]
  DBuf packed;             // bf16, uniform rank: left_k/left_v in the fused kernel's packed layout
};

struct DBlock {
  std::vector<uint64_t> positions;
  DStore k, v;
  int tokens() const { return static_cast<int>(positions.size()); }
};

struct DSegment {
  std::vector<DBlock> blocks;
  DBuf tk, tv;  // [batch][tail_cap][W]
  int tail_cap = 0;
  std::vector<uint64_t> tail_positions;
  int tail_len() const { return static_cast<int>(tail_positions.size()); }
  int compressed_len() const {
    int n = 0;
    for (const auto& b : blocks) n += b.tokens();
    return n;
  }
};

template <typename T>
struct DtypeOf;
template <>
struct DtypeOf<float> { static constexpr int v = KVP_F32; };
template <>
struct DtypeOf<double> { static constexpr int v = KVP_F64; };
template <>
struct DtypeOf<__nv_bfloat16> { static constexpr int v = KVP_BF16; };

template <typename T>
__device__ __forceinline__ T from_d(double x);
template <>
__device__ __forceinline__ float from_d<float>(double x) { return static_cast<float>(x); }
template <>
__device__ __forceinline__ double from_d<double>(double x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double x) {
  return __float2bfloat16_rn(static_cast<float>(x));
}

}  // namespace
}  // namespace kvp

struct kvp_cache {
  kvp_cache_config cfg{};
  int W = 0, HD = 0;
  size_t es = 0;  // storage element bytes
  kvp::DSegment seg[2];
  std::vector<uint64_t> imp_pos;  // table positions (ascending), shared by the batch
  kvp::DBuf imp;                  // [batch][imp_cap] fp64
  int imp_cap = 0;
  uint64_t next_position = 0, steps_taken = 0;
  cublasHandle_t blas = nullptr;
  ~kvp_cache() {
    if (blas) cublasDestroy(blas);
  }
  int act_dtype() const { return cfg.dtype == KVP_F64 ? KVP_F64 : KVP_F32; }
};

namespace kvp {
namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------

// dst[b][r][c] = convert(src[b][r][c]) for `rows` x `cols`, batch strides and row strides in elements.
template <typename Ti, typename To>
__global__ void copy_rows_kernel(const Ti* __restrict__ src, long s_row, long s_batch, To* __restrict__ dst, long d_row,
                                 long d_batch, int rows, int cols, int batch) {
  const long total = static_cast<long>(batch) * rows * cols;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long b = i / (static_cast<long>(rows) * cols), rc = i % (static_cast<long>(rows) * cols);
    const long r = rc / cols, c = rc % cols;
    dst[b * d_batch + r * d_row + c] = from_d<To>(to_d(src[b * s_batch + r * s_row + c]));
  }
}

// Round through the storage type and back (the reference's Matrix<T> results).
template <typename T>
__global__ void round_through_kernel(double* x, long n) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    x[i] = to_d(from_d<T>(x[i]));
}

__global__ void fill_f64_kernel(double* p, long row_stride, int rows, int c0, int c1, double v) {
  const long total = static_cast<long>(rows) * (c1 - c0);
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    p[(i / (c1 - c0)) * row_stride + c0 + i % (c1 - c0)] = v;
}

template <typename T>
__global__ void nonfinite_kernel(const T* a, long n, int* flag) {
  bool bad = false;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    bad |= !isfinite(to_d(a[i]));
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

// Skinny GEMM partials: part[z][m][n] = sum_{k in split z} x[m][k] w[k][n], fp64
// accumulation.  One thread per output column, 8 rows at a time, x staged in
// shared memory; grid (column blocks, row blocks, K splits).
constexpr int kProjRows = 8, kProjK = 128;
template <typename Tx, typename Tw>
__global__ void __launch_bounds__(kThreads) proj_partial_kernel(const Tx* __restrict__ x, const Tw* __restrict__ w,
                                                               double* __restrict__ part, int M, int K, int N,
                                                               int k_per_split) {
  __shared__ double xs[kProjRows][kProjK];
  const int n = blockIdx.x * kThreads + threadIdx.x;
  const int m0 = blockIdx.y * kProjRows;
  const int k_lo = blockIdx.z * k_per_split, k_hi = min(K, k_lo + k_per_split);
  double acc[kProjRows];
#pragma unroll
  for (int r = 0; r < kProjRows; ++r) acc[r] = 0.0;
  for (int k0 = k_lo; k0 < k_hi; k0 += kProjK) {
    const int kn = min(kProjK, k_hi - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < kProjRows * kProjK; i += kThreads) {
      const int r = i / kProjK, kk = i % kProjK;
      xs[r][kk] = (m0 + r < M && kk < kn) ? to_d(x[static_cast<long>(m0 + r) * K + k0 + kk]) : 0.0;
    }
    __syncthreads();
    if (n < N)
      for (int kk = 0; kk < kn; ++kk) {
        const double wv = to_d(w[static_cast<long>(k0 + kk) * N + n]);
#pragma unroll
        for (int r = 0; r < kProjRows; ++r) acc[r] += xs[r][kk] * wv;
      }
  }
  if (n < N)
#pragma unroll
    for (int r = 0; r < kProjRows; ++r)
      if (m0 + r < M) part[(static_cast<long>(blockIdx.z) * M + m0 + r) * N + n] = acc[r];
}

__global__ void proj_reduce_kernel(const double* __restrict__ part, double* __restrict__ out, long MN, int splits) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < MN;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[z * MN + i];
    out[i] = s;
  }
}

// scores_g[b][r] = importance[b][table[r]]
__global__ void gather_scores_kernel(const double* __restrict__ imp, long imp_stride, const int32_t* __restrict__ table,
                                     int n, int batch, double* __restrict__ out) {
  const long total = static_cast<long>(batch) * n;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    out[i] = imp[(i / n) * imp_stride + table[i % n]];
}

// ---- retrieval plan on the device (build_retrieval_plan, decoder.cpp:141-188)
struct PlanSeg {
  int n_comp;        // compressed rows (all blocks)
  int row0;          // first row in the row_* arrays
  int n_groups;      // tier groups (1 = untiered)
  int tier_off;      // column of this segment's tier ids in `tiers` (-1: untiered)
  int n_tail;
  int tail0;         // first row in the tail_* arrays
  int tail_kstore, tail_vstore;
};
struct PlanBuild {
  PlanSeg seg[2];
  const int32_t* row_block;   // global block index (stores 2g, 2g + 1)
  const uint32_t* row_local;  // row inside the block
  const int32_t* row_table;   // importance-table column
  const uint64_t* row_pos;
  const int32_t* tail_table;
  const uint64_t* tail_pos;
  const uint8_t* tiers;       // [batch][tier_stride]
  int tier_stride;
  const uint32_t* ranks;      // [batch][n_blocks][kMaxTiers][2] (rank_k, rank_v) per group
  int n_blocks;
  kvp_plan_entry* out;        // [batch][n_entries]
  int n_entries;
};

constexpr int kPlanThreads = 1024;

// Per segment: group-1 rows, lower groups, each in storage order; then the tail
// (decoder.cpp:160-186).  A stable partition per group by a block-wide scan.
__global__ void __launch_bounds__(kPlanThreads) plan_build_kernel(const PlanBuild pb) {
  const int b = blockIdx.x;
  __shared__ int warp_tot[kPlanThreads / 32];
  __shared__ int base_sh;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  kvp_plan_entry* out = pb.out + static_cast<long>(b) * pb.n_entries;
  int cursor = 0;
  for (int s = 0; s < 2; ++s) {
    const PlanSeg sd = pb.seg[s];
    for (int f = 0; f < sd.n_groups; ++f) {
      for (int c0 = 0; c0 < sd.n_comp; c0 += kPlanThreads) {
        const int r = c0 + tid;
        bool flag = r < sd.n_comp;
        if (flag && sd.tier_off >= 0) flag = pb.tiers[static_cast<long>(b) * pb.tier_stride + sd.tier_off + r] == f;
        const unsigned bal = __ballot_sync(0xffffffffu, flag);
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
          int acc = 0;
          for (int i = 0; i < kPlanThreads / 32; ++i) {
            const int t = warp_tot[i];
            warp_tot[i] = acc;
            acc += t;
          }
          base_sh = acc;
        }
        __syncthreads();
        if (flag) {
          const int idx = cursor + warp_tot[wid] + __popc(bal & ((1u << lane) - 1u));
          const int row = sd.row0 + r;
          const int g = pb.row_block[row];
          const uint32_t* rk = pb.ranks + ((static_cast<long>(b) * pb.n_blocks + g) * kMaxTiers + f) * 2;
          kvp_plan_entry e;
          e.k_store = 2 * g;
          e.v_store = 2 * g + 1;
          e.row = pb.row_local[row];
          e.rank_k = rk[0];
          e.rank_v = rk[1];
          e.table_index = pb.row_table[row];
          e.position = pb.row_pos[row];
          out[idx] = e;
        }
        cursor += base_sh;
        __syncthreads();
      }
    }
    for (int t = tid; t < sd.n_tail; t += kPlanThreads) {
      kvp_plan_entry e;
      e.k_store = sd.tail_kstore;
      e.v_store = sd.tail_vstore;
      e.row = static_cast<uint32_t>(t);
      e.rank_k = 0;
      e.rank_v = 0;
      e.table_index = pb.tail_table[sd.tail0 + t];
      e.position = pb.tail_pos[sd.tail0 + t];
      out[cursor + t] = e;
    }
    cursor += sd.n_tail;
  }
}

// out[b][row][c] = sum_{r < rank_b} left[b][row][r] right[b][r][c] (fp32 result; fp64 accumulation for f64
// stores) — the dense rows of a low-rank store at full stored rank (store_decompress_row, cache.cpp:63-101).
constexpr int kRbTile = 64, kRbK = 16;
template <typename T, typename Acc>
__global__ void __launch_bounds__(256) rebuild_kernel(const T* __restrict__ left, const T* __restrict__ right, int n,
                                                      int rank_cap, const int* __restrict__ ranks, int W,
                                                      double* __restrict__ out, long out_row, long out_batch) {
  __shared__ Acc ls[kRbTile][kRbK + 1];
  __shared__ Acc rs[kRbK][kRbTile];
  const int b = blockIdx.z;
  const int r0 = blockIdx.y * kRbTile, c0 = blockIdx.x * kRbTile;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 4 x 4 outputs per thread
  const int rank = ranks[b];
  const T* L = left + static_cast<long>(b) * n * rank_cap;
  const T* R = right + static_cast<long>(b) * rank_cap * W;
  Acc acc[4][4] = {};
  for (int k0 = 0; k0 < rank; k0 += kRbK) {
    for (int i = threadIdx.x; i < kRbTile * kRbK; i += 256) {
      const int rr = i / kRbK, kk = i % kRbK;
      ls[rr][kk] = (r0 + rr < n && k0 + kk < rank) ? static_cast<Acc>(to_d(L[static_cast<long>(r0 + rr) * rank_cap + k0 + kk]))
                                                   : Acc(0);
      const int kr = i / kRbTile, cc = i % kRbTile;
      rs[kr][cc] = (k0 + kr < rank && c0 + cc < W) ? static_cast<Acc>(to_d(R[static_cast<long>(k0 + kr) * W + c0 + cc]))
                                                   : Acc(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kRbK; ++kk) {
      Acc a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = ls[ty * 4 + i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = rs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * bb[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + ty * 4 + i, c = c0 + tx * 4 + j;
      if (r < n && c < W) out[static_cast<long>(b) * out_batch + static_cast<long>(r) * out_row + c] = acc[i][j];
    }
}

__global__ void f64_to_f32_kernel(const double* in, float* out, long n) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(in[i]);
}

unsigned grid_of(long n) { return static_cast<unsigned>(std::min<long>(std::max<long>(cdiv(n, kThreads), 1), 8192)); }

// ---------------------------------------------------------------------------
// Host-side helpers
// ---------------------------------------------------------------------------
template <typename F>
void by_dtype(int dt, F&& f) {
  switch (dt) {
    case KVP_F32: f(float{}); break;
    case KVP_F64: f(double{}); break;
    case KVP_BF16: f(__nv_bfloat16{}); break;
    default: fail(KVP_ERR_PARAMETER, "cache: unknown dtype");
  }
}

template <typename Ti, typename To>
void copy_rows(const Ti* src, long s_row, long s_batch, To* dst, long d_row, long d_batch, int rows, int cols,
               int batch, cudaStream_t s) {
  const long n = static_cast<long>(batch) * rows * cols;
  if (n == 0) return;
  copy_rows_kernel<Ti, To><<<grid_of(n), kThreads, 0, s>>>(src, s_row, s_batch, dst, d_row, d_batch, rows, cols, batch);
  KVP_LAUNCHED();
}

// Host f64 [batch][rows][cols] -> device storage dtype, strided destination.
void upload_rows(kvp_cache* c, const double* host, int rows, int cols, void* dst, long d_row, long d_batch,
                 cudaStream_t s) {
  const int B = c->cfg.batch;
  const size_t n = static_cast<size_t>(B) * rows * cols;
  if (n == 0) return;
  Scratch stage(n * sizeof(double), s);
  KVP_CUDA(cudaMemcpyAsync(stage.p, host, n * sizeof(double), cudaMemcpyHostToDevice, s));
  by_dtype(c->cfg.dtype, [&](auto t) {
    using T = decltype(t);
    copy_rows(stage.as<double>(), cols, static_cast<long>(rows) * cols, static_cast<T*>(dst), d_row, d_batch, rows,
              cols, B, s);
  });
  KVP_CUDA(cudaStreamSynchronize(s));
}

// Device storage rows of one instance -> host f64.
void download_rows(kvp_cache* c, const void* src, long s_row, int rows, int cols, double* host, cudaStream_t s) {
  const size_t n = static_cast<size_t>(rows) * cols;
  if (n == 0) return;
  Scratch stage(n * sizeof(double), s);
  by_dtype(c->cfg.dtype, [&](auto t) {
    using T = decltype(t);
    copy_rows(static_cast<const T*>(src), s_row, 0, stage.as<double>(), cols, 0, rows, cols, 1, s);
  });
  KVP_CUDA(cudaMemcpyAsync(host, stage.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  KVP_CUDA(cudaStreamSynchronize(s));
}

// Tail capacity for `need` rows (row-preserving growth, doubling).
void ensure_tail(kvp_cache* c, DSegment& sg, int need, cudaStream_t s) {
  if (need <= sg.tail_cap) return;
  const int cap = std::max({need, 2 * sg.tail_cap, 64});
  const size_t row_bytes = static_cast<size_t>(c->W) * c->es;
  for (DBuf* buf : {&sg.tk, &sg.tv}) {
    DBuf nb(static_cast<size_t>(c->cfg.batch) * cap * row_bytes);
    if (sg.tail_len() > 0)
      KVP_CUDA(cudaMemcpy2DAsync(nb.p, cap * row_bytes, buf->p, sg.tail_cap * row_bytes, sg.tail_len() * row_bytes,
                                 c->cfg.batch, cudaMemcpyDeviceToDevice, s));
    KVP_CUDA(cudaStreamSynchronize(s));
    *buf = std::move(nb);
  }
  sg.tail_cap = cap;
}

void ensure_importance(kvp_cache* c, int need, cudaStream_t s) {
  if (need <= c->imp_cap) return;
  const int cap = std::max({need, 2 * c->imp_cap, 256});
  DBuf nb(static_cast<size_t>(c->cfg.batch) * cap * sizeof(double));
  KVP_CUDA(cudaMemsetAsync(nb.p, 0, nb.bytes, s));
  if (!c->imp_pos.empty())
    KVP_CUDA(cudaMemcpy2DAsync(nb.p, cap * sizeof(double), c->imp.p, c->imp_cap * sizeof(double),
                               c->imp_pos.size() * sizeof(double), c->cfg.batch, cudaMemcpyDeviceToDevice, s));
  KVP_CUDA(cudaStreamSynchronize(s));
  c->imp = std::move(nb);
  c->imp_cap = cap;
}

// Fresh positions and zero importance for n new tokens (cache.cpp:161-168, importance.cpp:9-14).
void register_tokens(kvp_cache* c, DSegment& sg, int n, cudaStream_t s) {
  const int old = static_cast<int>(c->imp_pos.size());
  ensure_importance(c, old + n, s);
  fill_f64_kernel<<<grid_of(static_cast<long>(c->cfg.batch) * n), kThreads, 0, s>>>(c->imp.as<double>(), c->imp_cap,
                                                                                  c->cfg.batch, old, old + n, 0.0);
  KVP_LAUNCHED();
  for (int i = 0; i < n; ++i) {
    sg.tail_positions.push_back(c->next_position);
    c->imp_pos.push_back(c->next_position);
    ++c->next_position;
  }
}

int table_index(const kvp_cache* c, uint64_t pos) {
  const auto it = std::lower_bound(c->imp_pos.begin(), c->imp_pos.end(), pos);
  require(it != c->imp_pos.end() && *it == pos, KVP_ERR_PARAMETER, "ImportanceTable: unknown token position");
  return static_cast<int>(it - c->imp_pos.begin());
}

// ---- accounting (cache.cpp:180-219, decoder.cpp:506-551, importance.cpp:119-133) -------------
uint64_t store_scalars(const DStore& st, int inst, int n, int W) {
  if (st.form == KVP_LOWRANK) {
    const uint64_t r = static_cast<uint64_t>(st.ranks[inst]);
    return static_cast<uint64_t>(n) * r + r * static_cast<uint64_t>(W);
  }
  return static_cast<uint64_t>(n) * W;
}

uint64_t segment_scalars(const kvp_cache* c, const DSegment& sg, int inst) {
  uint64_t n = 0;
  for (const auto& b : sg.blocks) n += store_scalars(b.k, inst, b.tokens(), c->W) + store_scalars(b.v, inst, b.tokens(), c->W);
  return n + 2ull * static_cast<uint64_t>(sg.tail_len()) * c->W;
}

kvp_cache_bytes memory_bytes(const kvp_cache* c, int inst, int bps) {
  kvp_cache_bytes o{};
  o.visual_scalars = segment_scalars(c, c->seg[0], inst);
  o.textual_scalars = segment_scalars(c, c->seg[1], inst);
  o.visual_bytes = o.visual_scalars * bps;
  o.textual_bytes = o.textual_scalars * bps;
  o.cache_bytes = o.visual_bytes + o.textual_bytes;
  o.importance_bytes = static_cast<uint64_t>(c->imp_pos.size()) * (sizeof(uint64_t) + sizeof(double));
  return o;
}

uint64_t flops_partial(int tokens, int width, const std::vector<double>& ratios, const std::vector<int>& ranks) {
  double w = 0.0;
  for (size_t f = 0; f < ratios.size(); ++f) w += ratios[f] * static_cast<double>(ranks[f]);
  return static_cast<uint64_t>(std::llround(2.0 * static_cast<double>(tokens) * static_cast<double>(width) * w));
}

int resolved_tier_rank(double fraction, int stored) {  // decoder.cpp:18-23
  if (stored == 0) return 0;
  const int r = static_cast<int>(std::floor(fraction * static_cast<double>(stored) + 0.5));
  return std::clamp(r, 1, stored);
}

int store_rank(const DStore& st, int inst) { return st.form == KVP_LOWRANK ? st.ranks[inst] : 0; }

// ---- configuration (decoder.cpp:64-103 validate) -------------------------------------------------
void validate_config(const kvp_decode_config& d) {
  require(d.alpha >= 0.0 && d.alpha <= 1.0, KVP_ERR_PARAMETER, "DecodeConfig: alpha must be in [0, 1]");
  require(d.bytes_per_scalar >= 1, KVP_ERR_PARAMETER, "DecodeConfig: bytes_per_scalar must be >= 1");
  require(d.rank_key_visual >= 0 && d.rank_value_visual >= 0 && d.rank_key_textual >= 0 && d.rank_value_textual >= 0,
          KVP_ERR_PARAMETER, "MatrixRanks: ranks must be >= 0");
  require(d.svd_method == 0 || d.svd_method == 1, KVP_ERR_PARAMETER, "SvdOptions: unknown method");
  require(d.svd_oversampling >= 0 && d.svd_power_iterations >= 0, KVP_ERR_PARAMETER, "SvdOptions: bad options");
  require(d.recompress == 0 || d.recompress == 1, KVP_ERR_PARAMETER, "DecodeConfig: unknown recompress mode");
  require(d.rank_scheme >= -1 && d.rank_scheme <= 2, KVP_ERR_PARAMETER, "RankScheme: unknown kind");
  if (d.n_tiers > 0) {
    require(d.n_tiers <= kMaxTiers, KVP_ERR_PARAMETER, "TierSpec: at most 8 groups on the device");
    require(d.tier_ratios && d.tier_key_fractions && d.tier_value_fractions, KVP_ERR_PARAMETER,
            "TierSpec: one rank fraction per group required");
    double sum = 0.0;
    for (int f = 0; f < d.n_tiers; ++f) {
      require(d.tier_ratios[f] >= 0.0, KVP_ERR_PARAMETER, "TierSpec: ratios must be non-negative");
      sum += d.tier_ratios[f];
    }
    require(std::fabs(sum - 1.0) <= 1e-9, KVP_ERR_PARAMETER, "TierSpec: ratios must sum to 1");
    for (const double* fr : {d.tier_key_fractions, d.tier_value_fractions}) {
      require(fr[0] == 1.0, KVP_ERR_PARAMETER, "TierSpec: group 1 must keep the full stored rank");
      for (int f = 0; f < d.n_tiers; ++f) {
        require(fr[f] > 0.0 && fr[f] <= 1.0, KVP_ERR_PARAMETER, "TierSpec: rank fractions must be in (0, 1]");
        require(f == 0 || fr[f] <= fr[f - 1], KVP_ERR_PARAMETER, "TierSpec: rank fractions must be non-increasing");
      }
    }
  } else {
    require(d.n_tiers == 0, KVP_ERR_PARAMETER, "TierSpec: at least one group required");
  }
}

int config_rank(const kvp_decode_config& d, int modality, int kind) {
  if (modality == 0) return kind == 0 ? d.rank_key_visual : d.rank_value_visual;
  return kind == 0 ? d.rank_key_textual : d.rank_value_textual;
}

bool segment_compressible(const kvp_decode_config& d, int modality) {  // decoder.cpp:499-503
  return config_rank(d, modality, 0) > 0 || config_rank(d, modality, 1) > 0;
}

// layer_rank (compressor.cpp:10-40) for the data-independent schemes.
int scheme_rank(const kvp_cache* c, const kvp_decode_config& d) {
  if (d.rank_scheme == 0) {
    require(d.scheme_fixed_rank > 0, KVP_ERR_PARAMETER, "layer_rank: fixed rank must be positive");
    return d.scheme_fixed_rank;
  }
  require(d.scheme_num_layers > 0, KVP_ERR_PARAMETER, "layer_rank: schedule needs num_layers");
  require(c->cfg.layer_index < d.scheme_num_layers, KVP_ERR_PARAMETER, "layer_rank: layer index outside the schedule");
  if (d.scheme_num_layers == 1) return d.scheme_first_layer_rank;
  const double span = static_cast<double>(d.scheme_last_layer_rank) - static_cast<double>(d.scheme_first_layer_rank);
  const double x = static_cast<double>(d.scheme_first_layer_rank) +
                   span * static_cast<double>(c->cfg.layer_index) / static_cast<double>(d.scheme_num_layers - 1);
  return static_cast<int>(std::floor(x + 0.5));
}

// ---------------------------------------------------------------------------
// Projections: out = x W (x: M x K act dtype, W: K x N storage dtype) in fp64
// ---------------------------------------------------------------------------
void project(const kvp_cache* c, const void* x, int M, int K, const void* w, int N, double* out, cudaStream_t s) {
  const int col_blocks = static_cast<int>(cdiv(N, kThreads)), row_blocks = static_cast<int>(cdiv(M, kProjRows));
  int splits = std::max(1, std::min(64, 4 * 148 / std::max(1, col_blocks * row_blocks)));
  splits = std::min(splits, static_cast<int>(cdiv(K, kProjK)));
  const int kps = static_cast<int>(cdiv(cdiv(K, splits), kProjK)) * kProjK;
  splits = static_cast<int>(cdiv(K, kps));
  Scratch part(sizeof(double) * splits * static_cast<size_t>(M) * N, s);
  const dim3 grid(col_blocks, row_blocks, splits);
  auto launch = [&](auto xt, auto wt) {
    using Tx = decltype(xt);
    using Tw = decltype(wt);
    proj_partial_kernel<Tx, Tw><<<grid, kThreads, 0, s>>>(static_cast<const Tx*>(x), static_cast<const Tw*>(w),
                                                         part.as<double>(), M, K, N, kps);
    KVP_LAUNCHED();
  };
  by_dtype(c->cfg.dtype, [&](auto wt) {
    if (c->act_dtype() == KVP_F64) launch(double{}, wt);
    else launch(float{}, wt);
  });
  proj_reduce_kernel<<<grid_of(static_cast<long>(M) * N), kThreads, 0, s>>>(part.as<double>(), out,
                                                                            static_cast<long>(M) * N, splits);
  KVP_LAUNCHED();
}

void round_through(const kvp_cache* c, double* x, long n, cudaStream_t s) {
  if (c->cfg.dtype == KVP_F64) return;
  // f32 caches: Matrix<float>; bf16 caches compute activations in fp32
  round_through_kernel<float><<<grid_of(n), kThreads, 0, s>>>(x, n);
  KVP_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Appending projected rows (fp64 [batch][n][W]) to a segment's tail.
// ---------------------------------------------------------------------------
void append_device(kvp_cache* c, int modality, int n, const double* k, const double* v, cudaStream_t s) {
  DSegment& sg = c->seg[modality];
  ensure_tail(c, sg, sg.tail_len() + n, s);
  by_dtype(c->cfg.dtype, [&](auto t) {
    using T = decltype(t);
    for (int kind = 0; kind < 2; ++kind) {
      T* dst = static_cast<T*>((kind == 0 ? sg.tk : sg.tv).p) + static_cast<long>(sg.tail_len()) * c->W;
      copy_rows(kind == 0 ? k : v, c->W, static_cast<long>(n) * c->W, dst, c->W, static_cast<long>(sg.tail_cap) * c->W,
                n, c->W, c->cfg.batch, s);
    }
  });
  register_tokens(c, sg, n, s);
}

// ---------------------------------------------------------------------------
// segment_full_matrix: blocks at full stored rank, then the tail (fp64 out)
// ---------------------------------------------------------------------------
void full_matrix(kvp_cache* c, int modality, int kind, double* out, cudaStream_t s) {
  const DSegment& sg = c->seg[modality];
  const int B = c->cfg.batch, W = c->W;
  const int T = sg.compressed_len() + sg.tail_len();
  const long ob = static_cast<long>(T) * W;
  int row = 0;
  by_dtype(c->cfg.dtype, [&](auto t) {
    using T_ = decltype(t);
    for (const DBlock& blk : sg.blocks) {
      const DStore& st = kind == 0 ? blk.k : blk.v;
      double* dst = out + static_cast<long>(row) * W;
      if (st.form == KVP_LOWRANK) {
        DBuf ranks(sizeof(int) * B);
        KVP_CUDA(cudaMemcpyAsync(ranks.p, st.ranks.data(), sizeof(int) * B, cudaMemcpyHostToDevice, s));
        const dim3 grid(cdiv(W, kRbTile), cdiv(blk.tokens(), kRbTile), B);
        if (c->cfg.dtype == KVP_F64)
          rebuild_kernel<T_, double><<<grid, 256, 0, s>>>(st.a.as<T_>(), st.b.as<T_>(), blk.tokens(), st.rank_cap,
                                                          ranks.as<int>(), W, dst, W, ob);
        else
          rebuild_kernel<T_, float><<<grid, 256, 0, s>>>(st.a.as<T_>(), st.b.as<T_>(), blk.tokens(), st.rank_cap,
                                                         ranks.as<int>(), W, dst, W, ob);
        KVP_LAUNCHED();
        KVP_CUDA(cudaStreamSynchronize(s));
      } else {
        copy_rows(st.a.as<T_>(), W, static_cast<long>(blk.tokens()) * W, dst, W, ob, blk.tokens(), W, B, s);
      }
      row += blk.tokens();
    }
    if (sg.tail_len() > 0)
      copy_rows((kind == 0 ? sg.tk : sg.tv).template as<T_>(), W, static_cast<long>(sg.tail_cap) * W,
                out + static_cast<long>(row) * W, W, ob, sg.tail_len(), W, B, s);
  });
}

// ---------------------------------------------------------------------------
// make_store (decoder.cpp:440-449): dense rows, or compress_segment's rank-clamped
// truncated SVD (compressor.cpp:46-59) of every instance's matrix, batched.
// ---------------------------------------------------------------------------
DStore make_store(kvp_cache* c, const double* full, int n, int rank_req, const std::vector<int>& inst_rank,
                  const kvp_decode_config& d, int* warnings, cudaStream_t s) {
  const int B = c->cfg.batch, W = c->W;
  DStore st;
  if (rank_req == 0) {
    st.form = KVP_DENSE;
    st.a.alloc(static_cast<size_t>(B) * n * W * c->es);
    by_dtype(c->cfg.dtype, [&](auto t) {
      using T = decltype(t);
      copy_rows(full, W, static_cast<long>(n) * W, st.a.as<T>(), W, static_cast<long>(n) * W, n, W, B, s);
    });
    return st;
  }
  st.form = KVP_LOWRANK;
  st.ranks.resize(B);
  for (int b = 0; b < B; ++b) {
    const int want = inst_rank.empty() ? rank_req : inst_rank[b];
    st.ranks[b] = std::min({want, n, W});
    if (st.ranks[b] != want) ++warnings[b];  // "rank clamped to ..." (decoder.cpp:445-447)
  }
  st.rank_cap = *std::max_element(st.ranks.begin(), st.ranks.end());
  st.a.alloc(static_cast<size_t>(B) * n * st.rank_cap * c->es);
  st.b.alloc(static_cast<size_t>(B) * st.rank_cap * W * c->es);
  KVP_CUDA(cudaMemsetAsync(st.a.p, 0, st.a.bytes, s));
  KVP_CUDA(cudaMemsetAsync(st.b.p, 0, st.b.bytes, s));
  // fp32 SVD input; exact = full sketch with fp32 products, randomized = the tensor-core range finder for
  // bf16 caches (the serving format) and fp32 products for f32 / f64 caches
  Scratch a32(sizeof(float) * static_cast<size_t>(B) * n * W, s);
  f64_to_f32_kernel<<<grid_of(static_cast<long>(B) * n * W), kThreads, 0, s>>>(full, a32.as<float>(),
                                                                              static_cast<long>(B) * n * W);
  KVP_LAUNCHED();
  const bool exact = d.svd_method == 0;
  const bool precise = exact || c->cfg.dtype != KVP_BF16;
  // instances of equal rank share one batched call
  std::vector<int> done(B, 0);
  for (int b0 = 0; b0 < B; ++b0) {
    if (done[b0]) continue;
    const int R = st.ranks[b0];
    std::vector<int> members;
    for (int b = b0; b < B; ++b)
      if (!done[b] && st.ranks[b] == R) members.push_back(b);
    const bool contiguous = members.size() == static_cast<size_t>(B);
    const int nb = static_cast<int>(members.size());
    Scratch in(contiguous ? 0 : sizeof(float) * static_cast<size_t>(nb) * n * W, s);
    const float* src = a32.as<float>();
    if (!contiguous) {
      for (int i = 0; i < nb; ++i)
        KVP_CUDA(cudaMemcpyAsync(in.as<float>() + static_cast<size_t>(i) * n * W,
                                 a32.as<float>() + static_cast<size_t>(members[i]) * n * W, sizeof(float) * n * W,
                                 cudaMemcpyDeviceToDevice, s));
      src = in.as<float>();
    }
    Scratch left(sizeof(float) * static_cast<size_t>(nb) * n * R, s), right(sizeof(float) * static_cast<size_t>(nb) * R * W, s);
    randomized_svd_batched(c->blas, s, src, nb, n, W, R, d.svd_seed, exact ? std::min(n, W) : d.svd_oversampling,
                           exact ? 2 : d.svd_power_iterations, left.as<float>(), right.as<float>(), precise);
    by_dtype(c->cfg.dtype, [&](auto t) {
      using T = decltype(t);
      for (int i = 0; i < nb; ++i) {
        const int b = members[i];
        copy_rows(left.as<float>() + static_cast<size_t>(i) * n * R, R, 0,
                  st.a.as<T>() + static_cast<size_t>(b) * n * st.rank_cap, st.rank_cap, 0, n, R, 1, s);
        copy_rows(right.as<float>() + static_cast<size_t>(i) * R * W, W, 0,
                  st.b.as<T>() + static_cast<size_t>(b) * st.rank_cap * W, W, 0, R, W, 1, s);
      }
    });
    KVP_CUDA(cudaStreamSynchronize(s));
    for (int b : members) done[b] = 1;
  }
  return st;
}

// The fused kernel's packed left layout for a bf16 low-rank store of uniform rank.
void pack_store(kvp_cache* c, DStore& st, int n, cudaStream_t s) {
  if (c->cfg.dtype != KVP_BF16 || st.form != KVP_LOWRANK) return;
  const int r = st.ranks[0];
  for (int x : st.ranks)
    if (x != r) return;
  st.packed.alloc(packed_left_bytes(c->cfg.batch, n, r));
  pack_left(st.a.p, st.rank_cap, c->cfg.batch, n, r, st.packed.p, s);
}

// rank_for_variance (linalg.cpp:145-165) of every instance's matrix: the
// singular values come from the device SVD at full rank.
std::vector<int> variance_ranks(kvp_cache* c, const double* full, int n, const kvp_decode_config& d, cudaStream_t s) {
  require(d.scheme_variance_target > 0.0 && d.scheme_variance_target <= 1.0, KVP_ERR_PARAMETER,
          "rank_for_variance: target must be in (0, 1]");
  require(d.scheme_max_rank >= 1, KVP_ERR_PARAMETER, "rank_for_variance: max_rank must be >= 1");
  const int B = c->cfg.batch, W = c->W, k = std::min(n, W);
  Scratch a32(sizeof(float) * static_cast<size_t>(B) * n * W, s);
  f64_to_f32_kernel<<<grid_of(static_cast<long>(B) * n * W), kThreads, 0, s>>>(full, a32.as<float>(),
                                                                              static_cast<long>(B) * n * W);
  KVP_LAUNCHED();
  Scratch left(sizeof(float) * static_cast<size_t>(B) * n * k, s), right(sizeof(float) * static_cast<size_t>(B) * k * W, s);
  Scratch sv(sizeof(float) * static_cast<size_t>(B) * k, s);
  randomized_svd_batched(c->blas, s, a32.as<float>(), B, n, W, k, 0, k, 2, left.as<float>(), right.as<float>(), true,
                         sv.as<float>());
  std::vector<float> h(static_cast<size_t>(B) * k);
  KVP_CUDA(cudaMemcpyAsync(h.data(), sv.p, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, s));
  KVP_CUDA(cudaStreamSynchronize(s));
  std::vector<int> out(B, 1);
  const int cap = std::min(d.scheme_max_rank, k);
  for (int b = 0; b < B; ++b) {
    double total = 0.0, head = 0.0;
    for (int i = 0; i < k; ++i) total += static_cast<double>(h[b * k + i]) * h[b * k + i];
    if (total == 0.0) continue;
    for (int r = 1; r <= cap; ++r) {
      head += static_cast<double>(h[b * k + r - 1]) * h[b * k + r - 1];
      out[b] = r;
      if (head / total >= d.scheme_variance_target) break;
    }
  }
  return out;
}

// recompress_segment (decoder.cpp:455-497) for every instance.
void recompress_segment(kvp_cache* c, int modality, const kvp_decode_config& d, int* warnings, cudaStream_t s) {
  DSegment& sg = c->seg[modality];
  const int B = c->cfg.batch, W = c->W;
  const bool joint = d.recompress == 0;
  std::vector<uint64_t> positions;
  int n = 0;
  if (joint) {
    for (const auto& b : sg.blocks) positions.insert(positions.end(), b.positions.begin(), b.positions.end());
  }
  positions.insert(positions.end(), sg.tail_positions.begin(), sg.tail_positions.end());
  n = static_cast<int>(positions.size());
  if (n == 0) return;
  DBlock blk;
  blk.positions = positions;
  for (int kind = 0; kind < 2; ++kind) {
    DBuf full(sizeof(double) * static_cast<size_t>(B) * n * W);
    if (joint) {
      full_matrix(c, modality, kind, full.as<double>(), s);
    } else {
      by_dtype(c->cfg.dtype, [&](auto t) {
        using T = decltype(t);
        copy_rows((kind == 0 ? sg.tk : sg.tv).template as<T>(), W, static_cast<long>(sg.tail_cap) * W, full.as<double>(),
                  W, static_cast<long>(n) * W, n, W, B, s);
      });
    }
    int base = config_rank(d, modality, kind);
    std::vector<int> inst_rank;
    if (base > 0 && d.rank_scheme >= 0) {  // resolve_compression_rank (decoder.cpp:430-438)
      if (d.rank_scheme == 2) inst_rank = variance_ranks(c, full.as<double>(), n, d, s);
      else if (d.rank_scheme == 1) base = scheme_rank(c, d);
    }
    (kind == 0 ? blk.k : blk.v) = make_store(c, full.as<double>(), n, base, inst_rank, d, warnings, s);
    pack_store(c, kind == 0 ? blk.k : blk.v, n, s);
  }
  if (joint) sg.blocks.clear();
  sg.blocks.push_back(std::move(blk));
  sg.tail_positions.clear();
  KVP_CUDA(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------------------
// The decode step
// ---------------------------------------------------------------------------
struct SegTiering {
  std::vector<double> ratios;
  // per instance: per group (rank_k, rank_v) of block 0 (resolve_tiering, decoder.cpp:105-139)
  std::vector<std::vector<int>> key_ranks, value_ranks;
};

SegTiering resolve_tiering(const kvp_cache* c, const DSegment& sg, const kvp_decode_config& d) {
  SegTiering t;
  const int B = c->cfg.batch;
  t.key_ranks.resize(B);
  t.value_ranks.resize(B);
  if (sg.blocks.empty()) return t;
  for (int b = 0; b < B; ++b) {
    const int sk = store_rank(sg.blocks[0].k, b), sv = store_rank(sg.blocks[0].v, b);
    if (d.n_tiers > 0) {
      for (int f = 0; f < d.n_tiers; ++f) {
        t.key_ranks[b].push_back(resolved_tier_rank(d.tier_key_fractions[f], sk));
        t.value_ranks[b].push_back(resolved_tier_rank(d.tier_value_fractions[f], sv));
      }
    } else {
      t.key_ranks[b] = {sk};
      t.value_ranks[b] = {sv};
    }
  }
  if (d.n_tiers > 0) t.ratios.assign(d.tier_ratios, d.tier_ratios + d.n_tiers);
  else t.ratios = {1.0};
  return t;
}

void account(const kvp_cache* c, const SegTiering* st, kvp_step_report* reps) {
  const int B = c->cfg.batch;
  for (int b = 0; b < B; ++b) {
    uint64_t tiered = 0, full = 0;
    for (int m = 0; m < 2; ++m) {
      const DSegment& sg = c->seg[m];
      for (const DBlock& blk : sg.blocks)
        for (int kind = 0; kind < 2; ++kind) {
          const int stored = store_rank(kind == 0 ? blk.k : blk.v, b);
          if (stored == 0) continue;
          const auto& ranks = kind == 0 ? st[m].key_ranks[b] : st[m].value_ranks[b];
          std::vector<int> cl(ranks.size());
          for (size_t f = 0; f < ranks.size(); ++f) cl[f] = std::min(ranks[f], stored);
          tiered += flops_partial(blk.tokens(), c->W, st[m].ratios, cl);
          full += flops_partial(blk.tokens(), c->W, {1.0}, {stored});
        }
    }
    reps[b].decompress_flops = tiered;
    reps[b].decompress_flops_full = full;
    reps[b].flops_reduction = full == 0 ? 0.0 : 1.0 - static_cast<double>(tiered) / static_cast<double>(full);
  }
}

// Tier ids [batch][n_comp] of one segment's compressed tokens (assign_groups by
// importance, importance.cpp:67-117) on the device.
void assign_segment_tiers(kvp_cache* c, const DSegment& sg, const kvp_decode_config& d, uint8_t* tiers, int stride,
                          int col0, cudaStream_t s) {
  const int B = c->cfg.batch, n = sg.compressed_len();
  std::vector<int32_t> table(n);
  int r = 0;
  for (const auto& blk : sg.blocks)
    for (uint64_t p : blk.positions) table[r++] = table_index(c, p);
  Scratch dtab(sizeof(int32_t) * n, s), g(sizeof(double) * static_cast<size_t>(B) * n, s);
  Scratch out(static_cast<size_t>(B) * n, s);
  KVP_CUDA(cudaMemcpyAsync(dtab.p, table.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  gather_scores_kernel<<<grid_of(static_cast<long>(B) * n), kThreads, 0, s>>>(c->imp.as<double>(), c->imp_cap,
                                                                            dtab.as<int32_t>(), n, B, g.as<double>());
  KVP_LAUNCHED();
  const TierParams tp = make_tier_params(n, d.n_tiers, d.tier_ratios, nullptr, nullptr);
  launch_tiers(B, n, g.as<double>(), n, d.n_tiers, tp, out.as<uint8_t>(), nullptr, nullptr, s);
  KVP_CUDA(cudaMemcpy2DAsync(tiers + col0, stride, out.p, n, n, B, cudaMemcpyDeviceToDevice, s));
  KVP_CUDA(cudaStreamSynchronize(s));
}

// Plan (device entries) + store descriptors for the batch; returns entries per instance.
struct BuiltPlan {
  std::vector<kvp_store> stores;  // [batch][n_stores]
  int n_stores = 0;
  int n_entries = 0;
  DBuf entries;
};

BuiltPlan build_plan(kvp_cache* c, const kvp_decode_config& d, const SegTiering* st, cudaStream_t s) {
  const int B = c->cfg.batch, W = c->W;
  BuiltPlan bp;
  // store structure: per segment per block (K, V); then per segment with a tail (K, V)
  int n_blocks = 0;
  for (int m = 0; m < 2; ++m) n_blocks += static_cast<int>(c->seg[m].blocks.size());
  int tails = 0;
  for (int m = 0; m < 2; ++m) tails += c->seg[m].tail_len() > 0 ? 1 : 0;
  bp.n_stores = 2 * n_blocks + 2 * tails;
  bp.stores.resize(static_cast<size_t>(B) * bp.n_stores);
  std::vector<int32_t> row_block, row_table, tail_table;
  std::vector<uint32_t> row_local;
  std::vector<uint64_t> row_pos, tail_pos;
  std::vector<uint32_t> ranks(static_cast<size_t>(B) * std::max(n_blocks, 1) * kMaxTiers * 2, 0);
  PlanBuild pb{};
  int g = 0, tail_store = 2 * n_blocks, tier_cols = 0;
  for (int m = 0; m < 2; ++m) tier_cols += d.n_tiers > 0 ? c->seg[m].compressed_len() : 0;
  DBuf tiers(std::max<size_t>(1, static_cast<size_t>(B) * tier_cols));
  int tier_col = 0;
  for (int m = 0; m < 2; ++m) {
    const DSegment& sg = c->seg[m];
    PlanSeg& ps = pb.seg[m];
    ps.n_comp = sg.compressed_len();
    ps.row0 = static_cast<int>(row_block.size());
    ps.n_groups = (d.n_tiers > 0 && ps.n_comp > 0) ? d.n_tiers : 1;
    ps.tier_off = -1;
    if (d.n_tiers > 0 && ps.n_comp > 0) {
      ps.tier_off = tier_col;
      assign_segment_tiers(c, sg, d, tiers.as<uint8_t>(), tier_cols, tier_col, s);
      tier_col += ps.n_comp;
    }
    for (const DBlock& blk : sg.blocks) {
      for (int b = 0; b < B; ++b) {
        for (int kind = 0; kind < 2; ++kind) {
          const DStore& ds = kind == 0 ? blk.k : blk.v;
          kvp_store& o = bp.stores[static_cast<size_t>(b) * bp.n_stores + 2 * g + kind];
          o.form = ds.form;
          if (ds.form == KVP_LOWRANK) {
            o.rank = ds.ranks[b];
            o.a = static_cast<const char*>(ds.a.p) + static_cast<size_t>(b) * blk.tokens() * ds.rank_cap * c->es;
            o.b = static_cast<const char*>(ds.b.p) + static_cast<size_t>(b) * ds.rank_cap * W * c->es;
            o.lda = ds.rank_cap;
            o.ldb = W;
          } else {
            o.rank = 0;
            o.a = static_cast<const char*>(ds.a.p) + static_cast<size_t>(b) * blk.tokens() * W * c->es;
            o.b = nullptr;
            o.lda = W;
            o.ldb = 0;
          }
        }
        for (int f = 0; f < ps.n_groups; ++f) {
          // e.rank = min(tier rank of block 0, this block's stored rank) (decoder.cpp:170-175)
          uint32_t* rk = &ranks[((static_cast<size_t>(b) * n_blocks + g) * kMaxTiers + f) * 2];
          rk[0] = static_cast<uint32_t>(std::min(st[m].key_ranks[b][f], store_rank(blk.k, b)));
          rk[1] = static_cast<uint32_t>(std::min(st[m].value_ranks[b][f], store_rank(blk.v, b)));
        }
      }
      for (int r = 0; r < blk.tokens(); ++r) {
        row_block.push_back(g);
        row_local.push_back(static_cast<uint32_t>(r));
        row_table.push_back(table_index(c, blk.positions[r]));
        row_pos.push_back(blk.positions[r]);
      }
      ++g;
    }
    ps.n_tail = sg.tail_len();
    ps.tail0 = static_cast<int>(tail_table.size());
    ps.tail_kstore = ps.tail_vstore = -1;
    if (ps.n_tail > 0) {
      ps.tail_kstore = tail_store;
      ps.tail_vstore = tail_store + 1;
      for (int b = 0; b < B; ++b)
        for (int kind = 0; kind < 2; ++kind) {
          kvp_store& o = bp.stores[static_cast<size_t>(b) * bp.n_stores + tail_store + kind];
          o.form = KVP_DENSE;
          o.rank = 0;
          o.a = static_cast<const char*>((kind == 0 ? sg.tk : sg.tv).p) + static_cast<size_t>(b) * sg.tail_cap * W * c->es;
          o.b = nullptr;
          o.lda = W;
          o.ldb = 0;
        }
      tail_store += 2;
      for (int t = 0; t < ps.n_tail; ++t) {
        tail_table.push_back(table_index(c, sg.tail_positions[t]));
        tail_pos.push_back(sg.tail_positions[t]);
      }
    }
  }
  bp.n_entries = static_cast<int>(row_block.size() + tail_table.size());
  require(bp.n_entries > 0, KVP_ERR_PARAMETER, "attend: empty retrieval plan");
  // upload the shared row tables and per-instance ranks
  const size_t nr = row_block.size(), nt = tail_table.size();
  DBuf meta(sizeof(int32_t) * (2 * nr + nt) + sizeof(uint32_t) * nr + sizeof(uint64_t) * (nr + nt) +
            sizeof(uint32_t) * ranks.size() + 64);
  char* p = meta.as<char>();
  auto put = [&](const void* src, size_t bytes) {
    char* dst = p;
    if (bytes) KVP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    p += (bytes + 7) / 8 * 8;
    return dst;
  };
  pb.row_pos = reinterpret_cast<const uint64_t*>(put(row_pos.data(), sizeof(uint64_t) * nr));
  pb.tail_pos = reinterpret_cast<const uint64_t*>(put(tail_pos.data(), sizeof(uint64_t) * nt));
  pb.row_block = reinterpret_cast<const int32_t*>(put(row_block.data(), sizeof(int32_t) * nr));
  pb.row_table = reinterpret_cast<const int32_t*>(put(row_table.data(), sizeof(int32_t) * nr));
  pb.tail_table = reinterpret_cast<const int32_t*>(put(tail_table.data(), sizeof(int32_t) * nt));
  pb.row_local = reinterpret_cast<const uint32_t*>(put(row_local.data(), sizeof(uint32_t) * nr));
  pb.ranks = reinterpret_cast<const uint32_t*>(put(ranks.data(), sizeof(uint32_t) * ranks.size()));
  pb.tiers = tiers.as<uint8_t>();
  pb.tier_stride = tier_cols;
  pb.n_blocks = n_blocks;
  bp.entries.alloc(sizeof(kvp_plan_entry) * static_cast<size_t>(B) * bp.n_entries);
  pb.out = bp.entries.as<kvp_plan_entry>();
  pb.n_entries = bp.n_entries;
  plan_build_kernel<<<B, kPlanThreads, 0, s>>>(pb);
  KVP_LAUNCHED();
  KVP_CUDA(cudaStreamSynchronize(s));  // meta / tiers are released at scope exit
  return bp;
}

void fill_reports_before(kvp_cache* c, const kvp_decode_config& d, kvp_step_report* reps) {
  for (int b = 0; b < c->cfg.batch; ++b) {
    std::memset(&reps[b], 0, sizeof(kvp_step_report));
    reps[b].step = c->steps_taken;
    reps[b].bytes_before = memory_bytes(c, b, d.bytes_per_scalar).cache_bytes;
  }
}

void fill_reports_after(kvp_cache* c, const kvp_decode_config& d, kvp_step_report* reps, const int* warnings,
                        bool event) {
  for (int b = 0; b < c->cfg.batch; ++b) {
    const kvp_cache_bytes by = memory_bytes(c, b, d.bytes_per_scalar);
    reps[b].bytes_after = by.cache_bytes;
    reps[b].importance_bytes = by.importance_bytes;
    reps[b].compression_event = event ? 1 : 0;
    reps[b].n_warnings = warnings[b];
  }
}

bool maybe_recompress(kvp_cache* c, const kvp_decode_config& d, int* warnings, cudaStream_t s, bool force) {
  bool event = false;
  for (int m = 0; m < 2; ++m) {
    DSegment& sg = c->seg[m];
    if (!segment_compressible(d, m)) continue;
    const bool due = force ? sg.tail_len() > 0
                           : (d.compression_period > 0 && sg.tail_len() >= d.compression_period);
    if (due) {
      recompress_segment(c, m, d, warnings, s);
      event = true;
    }
  }
  return event;
}

void decode_step(kvp_cache* c, const void* h, int tq, int modality, const kvp_weights& w, const kvp_decode_config& d,
                 void* out, kvp_step_report* reps_out, cudaStream_t s) {
  const int B = c->cfg.batch, H = c->cfg.heads, D = c->cfg.head_dim, W = c->W, HD = c->HD;
  validate_config(d);
  require(tq >= 1, KVP_ERR_PARAMETER, "decode_step: at least one new token required");
  require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "decode_step: unknown modality");
  require(h && out && w.w_q && w.w_k && w.w_v && w.w_o, KVP_ERR_PARAMETER, "decode_step: null buffer");
  const long M = static_cast<long>(B) * tq;
  // non-finite activations: data_error before any change (decoder.cpp:566-567)
  {
    Scratch flag(sizeof(int), s);
    KVP_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    if (c->act_dtype() == KVP_F64)
      nonfinite_kernel<double><<<grid_of(M * HD), kThreads, 0, s>>>(static_cast<const double*>(h), M * HD, flag.as<int>());
    else
      nonfinite_kernel<float><<<grid_of(M * HD), kThreads, 0, s>>>(static_cast<const float*>(h), M * HD, flag.as<int>());
    KVP_LAUNCHED();
    int bad = 0;
    KVP_CUDA(cudaMemcpyAsync(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    KVP_CUDA(cudaStreamSynchronize(s));
    require(bad == 0, KVP_ERR_DATA, ("decode_step: non-finite activations at step " + std::to_string(c->steps_taken)).c_str());
  }
  std::vector<kvp_step_report> reps(B);
  fill_reports_before(c, d, reps.data());
  // projections (matmul, decoder.cpp:574-576), results in the cache's precision
  DBuf q(sizeof(double) * M * HD), kn(sizeof(double) * M * W), vn(sizeof(double) * M * W);
  project(c, h, static_cast<int>(M), HD, w.w_q, HD, q.as<double>(), s);
  project(c, h, static_cast<int>(M), HD, w.w_k, W, kn.as<double>(), s);
  project(c, h, static_cast<int>(M), HD, w.w_v, W, vn.as<double>(), s);
  round_through(c, q.as<double>(), M * HD, s);
  // query positions: next_position + i (decoder.cpp:577-578); append (cache.cpp:147-170)
  std::vector<uint64_t> qpos(tq);
  for (int i = 0; i < tq; ++i) qpos[i] = c->next_position + i;
  append_device(c, modality, tq, kn.as<double>(), vn.as<double>(), s);
  // plan (tiers by importance) and attention
  SegTiering st[2] = {resolve_tiering(c, c->seg[0], d), resolve_tiering(c, c->seg[1], d)};
  account(c, st, reps.data());
  BuiltPlan bp = build_plan(c, d, st, s);
  const int n_imp = static_cast<int>(c->imp_pos.size());
  DBuf ctx(sizeof(double) * M * HD), hat(sizeof(double) * M * n_imp), dqpos(sizeof(uint64_t) * tq);
  KVP_CUDA(cudaMemcpyAsync(dqpos.p, qpos.data(), sizeof(uint64_t) * tq, cudaMemcpyHostToDevice, s));
  KVP_CUDA(cudaMemsetAsync(hat.p, 0, hat.bytes, s));
  PlanBatch pl{};
  pl.heads = H;
  pl.kv_heads = c->cfg.kv_heads;
  pl.head_dim = D;
  pl.dtype = c->cfg.dtype;
  pl.batch = B;
  pl.n_stores = bp.n_stores;
  pl.n_entries = bp.n_entries;
  pl.tq = tq;
  pl.table_size = n_imp;
  pl.table_stride = n_imp;
  pl.stores = bp.stores.data();
  pl.entries = bp.entries.as<kvp_plan_entry>();
  pl.entries_on_device = true;
  pl.queries = q.as<double>();
  pl.query_positions = dqpos.as<uint64_t>();
  pl.context = ctx.as<double>();
  pl.head_avg = nullptr;
  pl.head_avg_table = hat.as<double>();
  run_plan(pl, s);
  round_through(c, ctx.as<double>(), M * HD, s);
  // output = context W_o (decoder.cpp:590), in the activation dtype
  {
    DBuf o64(sizeof(double) * M * HD);
    if (c->act_dtype() == KVP_F64) {
      project(c, ctx.as<double>(), static_cast<int>(M), HD, w.w_o, HD, static_cast<double*>(out), s);
    } else {
      // the f32 projection kernel reads fp32 activations
      DBuf c32(sizeof(float) * M * HD);
      f64_to_f32_kernel<<<grid_of(M * HD), kThreads, 0, s>>>(ctx.as<double>(), c32.as<float>(), M * HD);
      KVP_LAUNCHED();
      project(c, c32.p, static_cast<int>(M), HD, w.w_o, HD, o64.as<double>(), s);
      f64_to_f32_kernel<<<grid_of(M * HD), kThreads, 0, s>>>(o64.as<double>(), static_cast<float*>(out), M * HD);
      KVP_LAUNCHED();
      KVP_CUDA(cudaStreamSynchronize(s));
    }
  }
  // importance EMA over the table-order head average (decoder.cpp:592-601, importance.cpp:33-65)
  {
    Scratch bad(sizeof(unsigned), s);
    KVP_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned), s));
    launch_row_check(static_cast<int>(M), n_imp, hat.as<double>(), bad.as<unsigned>(), s);
    unsigned hb = 0;
    KVP_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    KVP_CUDA(cudaStreamSynchronize(s));
    require(hb == 0, KVP_ERR_DATA, "update_importance: attention row is not a distribution");
    launch_ema(B, n_imp, c->imp.as<double>(), tq, hat.as<double>(), d.alpha, nullptr, s, c->imp_cap);
  }
  // re-factorise segments whose tail reached the period (decoder.cpp:604-610)
  std::vector<int> warnings(B, 0);
  const bool event = maybe_recompress(c, d, warnings.data(), s, false);
  fill_reports_after(c, d, reps.data(), warnings.data(), event);
  KVP_CUDA(cudaStreamSynchronize(s));
  ++c->steps_taken;
  if (reps_out) std::memcpy(reps_out, reps.data(), sizeof(kvp_step_report) * B);
}

kvp_cache* checked(kvp_cache* c) {
  require(c != nullptr, KVP_ERR_PARAMETER, "cache: null handle");
  return c;
}

}  // namespace
}  // namespace kvp

using namespace kvp;

extern "C" int kvp_cache_create(const kvp_cache_config* cfg, kvp_cache** out) {
  return guarded([&] {
    require(cfg && out, KVP_ERR_PARAMETER, "cache: null argument");
    require(cfg->heads > 0 && cfg->kv_heads > 0 && cfg->head_dim > 0, KVP_ERR_PARAMETER,
            "HeadGeometry: head counts and head_dim must be positive");
    require(cfg->heads % cfg->kv_heads == 0, KVP_ERR_PARAMETER, "HeadGeometry: num_kv_heads must divide num_query_heads");
    require(cfg->batch >= 1, KVP_ERR_PARAMETER, "cache: batch must be >= 1");
    require(cfg->layer_index >= 0, KVP_ERR_PARAMETER, "cache: layer_index must be >= 0");
    require(cfg->dtype == KVP_F32 || cfg->dtype == KVP_F64 || cfg->dtype == KVP_BF16, KVP_ERR_PARAMETER,
            "cache: dtype must be f32, f64 or bf16");
    auto c = std::make_unique<kvp_cache>();
    c->cfg = *cfg;
    c->W = cfg->kv_heads * cfg->head_dim;
    c->HD = cfg->heads * cfg->head_dim;
    c->es = dtype_size(cfg->dtype);
    if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) fail(KVP_ERR_CUDA, "cache: cublasCreate failed");
    *out = c.release();
  });
}

extern "C" int kvp_cache_destroy(kvp_cache* c) {
  return guarded([&] {
    if (c) cudaDeviceSynchronize();
    delete c;
  });
}

extern "C" int kvp_cache_append(kvp_cache* c, int32_t modality, int32_t n, const double* k, const double* v) {
  return guarded([&] {
    checked(c);
    require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "append_tokens: unknown modality");
    require(n >= 0, KVP_ERR_SHAPE, "append_tokens: K and V row counts disagree");
    if (n == 0) return;
    require(k && v, KVP_ERR_PARAMETER, "append_tokens: null rows");
    const size_t cnt = static_cast<size_t>(c->cfg.batch) * n * c->W;
    for (size_t i = 0; i < cnt; ++i)
      require(std::isfinite(k[i]) && std::isfinite(v[i]), KVP_ERR_DATA, "append_tokens: non-finite K/V rows");
    cudaStream_t s = nullptr;
    DSegment& sg = c->seg[modality];
    ensure_tail(c, sg, sg.tail_len() + n, s);
    const long row = c->W, bstride = static_cast<long>(sg.tail_cap) * c->W;
    for (int kind = 0; kind < 2; ++kind)
      upload_rows(c, kind == 0 ? k : v, n, c->W,
                  static_cast<char*>((kind == 0 ? sg.tk : sg.tv).p) + static_cast<size_t>(sg.tail_len()) * c->W * c->es,
                  row, bstride, s);
    register_tokens(c, sg, n, s);
    KVP_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int kvp_cache_factor_tail(kvp_cache* c, int32_t modality, int32_t rank_k, const double* k_left,
                                     const double* k_right, int32_t rank_v, const double* v_left,
                                     const double* v_right) {
  return guarded([&] {
    checked(c);
    require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "factor_tail: unknown modality");
    DSegment& sg = c->seg[modality];
    const int n = sg.tail_len(), B = c->cfg.batch, W = c->W;
    require(n > 0, KVP_ERR_PARAMETER, "factor_tail: empty tail");
    cudaStream_t s = nullptr;
    DBlock blk;
    blk.positions = sg.tail_positions;
    for (int kind = 0; kind < 2; ++kind) {
      const int rank = kind == 0 ? rank_k : rank_v;
      DStore& st = kind == 0 ? blk.k : blk.v;
      require(rank >= 0 && rank <= std::min(n, W), KVP_ERR_PARAMETER, "factor_tail: rank outside [0, min(T, W)]");
      if (rank == 0) {
        st.form = KVP_DENSE;
        st.a.alloc(static_cast<size_t>(B) * n * W * c->es);
        KVP_CUDA(cudaMemcpy2DAsync(st.a.p, static_cast<size_t>(n) * W * c->es, (kind == 0 ? sg.tk : sg.tv).p,
                                   static_cast<size_t>(sg.tail_cap) * W * c->es, static_cast<size_t>(n) * W * c->es, B,
                                   cudaMemcpyDeviceToDevice, s));
      } else {
        const double* l = kind == 0 ? k_left : v_left;
        const double* r = kind == 0 ? k_right : v_right;
        require(l && r, KVP_ERR_PARAMETER, "factor_tail: null factors");
        st.form = KVP_LOWRANK;
        st.rank_cap = rank;
        st.ranks.assign(B, rank);
        st.a.alloc(static_cast<size_t>(B) * n * rank * c->es);
        st.b.alloc(static_cast<size_t>(B) * rank * W * c->es);
        upload_rows(c, l, n, rank, st.a.p, rank, static_cast<long>(n) * rank, s);
        upload_rows(c, r, rank, W, st.b.p, W, static_cast<long>(rank) * W, s);
        pack_store(c, st, n, s);
      }
    }
    sg.blocks.push_back(std::move(blk));
    sg.tail_positions.clear();
    KVP_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int kvp_cache_set_importance(kvp_cache* c, const double* scores) {
  return guarded([&] {
    checked(c);
    const int n = static_cast<int>(c->imp_pos.size());
    if (n == 0) return;
    require(scores != nullptr, KVP_ERR_PARAMETER, "set_importance: null scores");
    KVP_CUDA(cudaMemcpy2D(c->imp.p, c->imp_cap * sizeof(double), scores, n * sizeof(double), n * sizeof(double),
                          c->cfg.batch, cudaMemcpyHostToDevice));
  });
}

extern "C" int kvp_cache_get_importance(kvp_cache* c, uint64_t* positions, double* scores) {
  return guarded([&] {
    checked(c);
    const int n = static_cast<int>(c->imp_pos.size());
    if (positions) std::copy(c->imp_pos.begin(), c->imp_pos.end(), positions);
    if (scores && n > 0)
      KVP_CUDA(cudaMemcpy2D(scores, n * sizeof(double), c->imp.p, c->imp_cap * sizeof(double), n * sizeof(double),
                            c->cfg.batch, cudaMemcpyDeviceToHost));
  });
}

extern "C" int kvp_cache_shape(kvp_cache* c, int32_t* table_size, uint64_t* next_position, uint64_t* steps_taken,
                               int32_t* n_blocks, int32_t* tail_len) {
  return guarded([&] {
    checked(c);
    if (table_size) *table_size = static_cast<int32_t>(c->imp_pos.size());
    if (next_position) *next_position = c->next_position;
    if (steps_taken) *steps_taken = c->steps_taken;
    for (int m = 0; m < 2; ++m) {
      if (n_blocks) n_blocks[m] = static_cast<int32_t>(c->seg[m].blocks.size());
      if (tail_len) tail_len[m] = c->seg[m].tail_len();
    }
  });
}

// Restores LayerCache.next_position / steps_taken from a host image (a KVPK snapshot records
// both, snapshot.cpp:275-276); positions already assigned must stay below next_position.
extern "C" int kvp_cache_set_counters(kvp_cache* c, uint64_t next_position, uint64_t steps_taken) {
  return guarded([&] {
    checked(c);
    require(next_position >= c->next_position, KVP_ERR_PARAMETER,
            "set_counters: next_position below an assigned position");
    c->next_position = next_position;
    c->steps_taken = steps_taken;
  });
}


namespace {
const kvp::DBlock& block_at(kvp_cache* c, int inst, int modality, int block) {
  require(inst >= 0 && inst < c->cfg.batch, KVP_ERR_PARAMETER, "cache: instance out of range");
  require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "cache: unknown modality");
  const auto& blocks = c->seg[modality].blocks;
  require(block >= 0 && block < static_cast<int>(blocks.size()), KVP_ERR_PARAMETER, "cache: block out of range");
  return blocks[block];
}
}  // namespace

extern "C" int kvp_cache_block_info(kvp_cache* c, int32_t inst, int32_t modality, int32_t block, int32_t kind,
                                    int32_t* tokens, int32_t* rank) {
  return guarded([&] {
    checked(c);
    const DBlock& b = block_at(c, inst, modality, block);
    const DStore& st = kind == 0 ? b.k : b.v;
    if (tokens) *tokens = b.tokens();
    if (rank) *rank = store_rank(st, inst);
  });
}

extern "C" int kvp_cache_block_get(kvp_cache* c, int32_t inst, int32_t modality, int32_t block, int32_t kind,
                                   double* left, double* right, uint64_t* positions) {
  return guarded([&] {
    checked(c);
    const DBlock& b = block_at(c, inst, modality, block);
    const DStore& st = kind == 0 ? b.k : b.v;
    const int n = b.tokens(), W = c->W;
    cudaStream_t s = nullptr;
    if (st.form == KVP_LOWRANK) {
      const int r = st.ranks[inst];
      if (left)
        download_rows(c, static_cast<const char*>(st.a.p) + static_cast<size_t>(inst) * n * st.rank_cap * c->es,
                      st.rank_cap, n, r, left, s);
      if (right)
        download_rows(c, static_cast<const char*>(st.b.p) + static_cast<size_t>(inst) * st.rank_cap * W * c->es, W, r,
                      W, right, s);
    } else if (left) {
      download_rows(c, static_cast<const char*>(st.a.p) + static_cast<size_t>(inst) * n * W * c->es, W, n, W, left, s);
    }
    if (positions) std::copy(b.positions.begin(), b.positions.end(), positions);
  });
}

extern "C" int kvp_cache_tail_get(kvp_cache* c, int32_t inst, int32_t modality, double* k, double* v,
                                  uint64_t* positions) {
  return guarded([&] {
    checked(c);
    require(inst >= 0 && inst < c->cfg.batch, KVP_ERR_PARAMETER, "cache: instance out of range");
    require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "cache: unknown modality");
    const DSegment& sg = c->seg[modality];
    const size_t off = static_cast<size_t>(inst) * sg.tail_cap * c->W * c->es;
    if (k) download_rows(c, static_cast<const char*>(sg.tk.p) + off, c->W, sg.tail_len(), c->W, k, nullptr);
    if (v) download_rows(c, static_cast<const char*>(sg.tv.p) + off, c->W, sg.tail_len(), c->W, v, nullptr);
    if (positions) std::copy(sg.tail_positions.begin(), sg.tail_positions.end(), positions);
  });
}

extern "C" int kvp_cache_memory_bytes(kvp_cache* c, int32_t inst, int32_t bps, kvp_cache_bytes* out) {
  return guarded([&] {
    checked(c);
    require(out != nullptr, KVP_ERR_PARAMETER, "memory_bytes: null output");
    require(bps >= 1, KVP_ERR_PARAMETER, "memory_bytes: bytes_per_scalar must be positive");
    require(inst >= 0 && inst < c->cfg.batch, KVP_ERR_PARAMETER, "cache: instance out of range");
    *out = memory_bytes(c, inst, bps);
  });
}

extern "C" int kvp_segment_full_matrix(kvp_cache* c, int32_t modality, int32_t kind, double* out, void* stream) {
  return guarded([&] {
    checked(c);
    require(modality == 0 || modality == 1, KVP_ERR_PARAMETER, "segment_full_matrix: unknown modality");
    require(kind == 0 || kind == 1, KVP_ERR_PARAMETER, "segment_full_matrix: unknown kind");
    require(out != nullptr, KVP_ERR_PARAMETER, "segment_full_matrix: null output");
    full_matrix(c, modality, kind, out, as_stream(stream));
  });
}

extern "C" int kvp_compress_now(kvp_cache* c, const kvp_decode_config* d, kvp_step_report* reps, void* stream) {
  return guarded([&] {
    checked(c);
    require(d != nullptr, KVP_ERR_PARAMETER, "compress_now: null config");
    validate_config(*d);
    cudaStream_t s = as_stream(stream);
    std::vector<int> warnings(c->cfg.batch, 0);
    std::vector<kvp_step_report> r(c->cfg.batch);
    fill_reports_before(c, *d, r.data());
    const bool event = maybe_recompress(c, *d, warnings.data(), s, true);
    fill_reports_after(c, *d, r.data(), warnings.data(), event);
    if (reps) std::memcpy(reps, r.data(), sizeof(kvp_step_report) * r.size());
  });
}

extern "C" int kvp_decode_step(kvp_cache* c, const void* h, int32_t tq, int32_t modality, const kvp_weights* w,
                               const kvp_decode_config* d, void* out, kvp_step_report* reps, void* stream) {
  return guarded([&] {
    checked(c);
    require(w && d, KVP_ERR_PARAMETER, "decode_step: null argument");
    decode_step(c, h, tq, modality, *w, *d, out, reps, as_stream(stream));
  });
}
