// Importance tracking on the GPU: the Eq. 1 EMA (importance.cpp:33-65) and
// importance-ordered tier assignment (importance.cpp:67-117 assign_groups as
// used by resolve_tiering, decoder.cpp:105-139).  Both are bit-exact with the
// reference for identical inputs: the EMA is evaluated with explicit
// round-to-nearest multiplies/adds in the reference's operation order (no FMA
// contraction — g++ for x86-64 without -mfma never fuses), and the tier order
// is a total order on (score desc, index asc), so any correct sort yields the
// reference's std::sort + tie-break result.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "importance.cuh"

#include <cstdlib>

namespace kvp {

// s_j <- decay*s_j + blend*mean_t attn[t][j]; one thread per (table, j).
__global__ void ema_kernel(int n_tables, int n, double* __restrict__ scores, long stride, int tq,
                           const double* __restrict__ attn, double decay, double blend, double inv_tq) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)n_tables * n) return;
  const long tbl = idx / n, j = idx % n;
  const double* a = attn + tbl * tq * (long)n + j;
  double mean = 0.0;
  for (int t = 0; t < tq; ++t) mean = __dadd_rn(mean, a[(long)t * n]);
  mean = __dmul_rn(mean, inv_tq);
  double* sc = scores + tbl * stride + j;
  *sc = __dadd_rn(__dmul_rn(decay, *sc), __dmul_rn(blend, mean));
}

// |row sum - 1| > 1e-4 or non-finite -> count it (importance.cpp:45-54).
__global__ void row_check_kernel(int n, const double* __restrict__ attn, unsigned* bad) {
  const double* a = attn + (long)blockIdx.x * n;
  __shared__ double red[256];
  __shared__ int nonfinite;
  if (threadIdx.x == 0) nonfinite = 0;
  __syncthreads();
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double v = a[j];
    if (!isfinite(v)) nonfinite = 1;
    s += v;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0 && (nonfinite || fabs(red[0] - 1.0) > 1e-4)) atomicAdd(bad, 1u);
}

void launch_row_check(int rows, int n, const double* attn, unsigned* bad, cudaStream_t s) {
  row_check_kernel<<<rows, 256, 0, s>>>(n, attn, bad);
  KVP_LAUNCHED();
}

void launch_ema(int n_tables, int n, double* scores, int tq, const double* attn, double alpha,
                unsigned* bad_rows, cudaStream_t s, long score_stride) {
  // decay = alpha^tq with the same libm pow the reference calls
  // (importance.cpp:58); blend and 1/tq as in importance.cpp:59-60.
  const double decay = std::pow(alpha, static_cast<double>(tq));
  const double blend = 1.0 - decay;
  const double inv_tq = 1.0 / static_cast<double>(tq);
  if (bad_rows) {
    row_check_kernel<<<n_tables * tq, 256, 0, s>>>(n, attn, bad_rows);
    KVP_LAUNCHED();
  }
  const long total = (long)n_tables * n;
  ema_kernel<<<cdiv(total, 256), 256, 0, s>>>(n_tables, n, scores, score_stride < 0 ? n : score_stride, tq, attn,
                                               decay, blend, inv_tq);
  KVP_LAUNCHED();
}

// ---- tier assignment --------------------------------------------------------

// Order-preserving map of a double onto uint64 (ascending), then inverted so
// that an ascending sort yields descending scores.  -0.0 is canonicalised to
// +0.0 because the reference compares with `!=` (equal scores tie-break).
__device__ __forceinline__ uint64_t desc_key(double s) {
  if (s == 0.0) s = 0.0;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  return ~b;
}

// One CTA per table: bitonic sort of (key, index) pairs in shared memory,
// then the group of the token at sorted rank p is the f with
// bounds[f] <= p < bounds[f+1].
__global__ void tier_kernel(int n, int npow2, const double* __restrict__ scores, long stride, int n_groups,
                            TierParams tp, uint8_t* tier_out, uint16_t* rk_out, uint16_t* rv_out) {
  extern __shared__ unsigned char smem[];
  uint64_t* key = reinterpret_cast<uint64_t*>(smem);
  uint32_t* idx = reinterpret_cast<uint32_t*>(key + npow2);
  const double* sc = scores + (long)blockIdx.x * stride;
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    key[i] = i < n ? desc_key(sc[i]) : ~0ull;
    idx[i] = i < n ? i : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const uint64_t ki = key[i], kl = key[l];
          const uint32_t ii = idx[i], il = idx[l];
          const bool gt = ki > kl || (ki == kl && ii > il);
          if (gt == up) {
            key[i] = kl;
            key[l] = ki;
            idx[i] = il;
            idx[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  const long out = (long)blockIdx.x * n;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    int f = 0;
    while (f + 1 < n_groups && p >= tp.bounds[f + 1]) ++f;
    const uint32_t t = idx[p];
    if (tier_out) tier_out[out + t] = static_cast<uint8_t>(f);
    if (rk_out) rk_out[out + t] = static_cast<uint16_t>(tp.rank_k[f]);
    if (rv_out) rv_out[out + t] = static_cast<uint16_t>(tp.rank_v[f]);
  }
}

// One CTA per table, n <= kSelThreads * kSelPer: radix select instead of a sort.
// Rank order is (key ascending = score descending, index ascending).  For each
// group boundary b_f the b_f-th smallest key D* is found with eight 8-bit digit
// passes over the keys held in registers; a token is inside the boundary when
// its key is below D*, or equal to it and among the first (b_f - #below) such
// tokens by index (block-wide prefix count).  Its group is the number of
// boundaries it falls outside of.  Same result as the sort, bit for bit.
constexpr int kSelThreads = 512, kSelPer = 8;
__device__ __forceinline__ unsigned block_exclusive_scan(unsigned v, unsigned* wsum, unsigned* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    unsigned w = lane < nw ? wsum[lane] : 0u, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) wsum[lane] = wi - w;
    if (lane == nw - 1) *total = wi;
  }
  __syncthreads();
  const unsigned r = wsum[warp] + inc - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kSelThreads) tier_select_kernel(int n, const double* __restrict__ scores, long stride,
                                                                  int n_groups, TierParams tp, uint8_t* tier_out,
                                                                  uint16_t* rk_out, uint16_t* rv_out) {
  __shared__ unsigned hist[256];
  __shared__ unsigned sel[2];
  __shared__ unsigned wsum[32];
  __shared__ unsigned total;
  const double* sc = scores + (long)blockIdx.x * stride;
  const int base = threadIdx.x * kSelPer;  // a contiguous chunk of indices per thread
  const int lane = threadIdx.x & 31;
  uint64_t key[kSelPer];
  int grp[kSelPer];
#pragma unroll
  for (int j = 0; j < kSelPer; ++j) {
    key[j] = base + j < n ? desc_key(sc[base + j]) : 0ull;
    grp[j] = 0;
  }
  for (int f = 1; f < n_groups; ++f) {
    const int k = tp.bounds[f];
    if (k >= n) continue;  // everybody inside
    if (k <= 0) {
#pragma unroll
      for (int j = 0; j < kSelPer; ++j) grp[j] += 1;
      continue;
    }
    uint64_t prefix = 0, mask = 0;
    unsigned remaining = static_cast<unsigned>(k);
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kSelPer; ++j)
        if (base + j < n && (key[j] & mask) == prefix) atomicAdd(&hist[(key[j] >> shift) & 255u], 1u);
      __syncthreads();
      if (threadIdx.x < 32) {
        unsigned own = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) own += hist[lane * 8 + b];
        unsigned inc = own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const unsigned before = inc - own;
        if (before < remaining && remaining <= inc) {
          unsigned cum = before;
          for (int b = 0; b < 8; ++b) {
            const unsigned h = hist[lane * 8 + b];
            if (cum + h >= remaining) {
              sel[0] = static_cast<unsigned>(lane * 8 + b);
              sel[1] = remaining - cum;
              break;
            }
            cum += h;
          }
        }
      }
      __syncthreads();
      prefix |= static_cast<uint64_t>(sel[0]) << shift;
      mask |= 255ull << shift;
      remaining = sel[1];
      __syncthreads();
    }
    // ties with the boundary key: the first `remaining` of them by index are inside
    unsigned eq = 0;
#pragma unroll
    for (int j = 0; j < kSelPer; ++j) eq += (base + j < n && key[j] == prefix) ? 1u : 0u;
    unsigned order = block_exclusive_scan(eq, wsum, &total);
#pragma unroll
    for (int j = 0; j < kSelPer; ++j) {
      bool inside = key[j] < prefix;
      if (base + j < n && key[j] == prefix) inside = order++ < remaining;
      if (!inside) grp[j] += 1;
    }
  }
  const long out = (long)blockIdx.x * n;
#pragma unroll
  for (int j = 0; j < kSelPer; ++j) {
    const int t = base + j;
    if (t >= n) break;
    if (tier_out) tier_out[out + t] = static_cast<uint8_t>(grp[j]);
    if (rk_out) rk_out[out + t] = static_cast<uint16_t>(tp.rank_k[grp[j]]);
    if (rv_out) rv_out[out + t] = static_cast<uint16_t>(tp.rank_v[grp[j]]);
  }
}

TierParams make_tier_params(int n, int n_groups, const double* ratios, const int32_t* key_ranks,
                            const int32_t* value_ranks) {
  require(n_groups >= 1 && n_groups <= kMaxTiers, KVP_ERR_PARAMETER,
          "assign_groups: ratios and ranks must be non-empty and aligned");
  double sum = 0.0;
  for (int f = 0; f < n_groups; ++f) {
    require(ratios[f] >= 0.0, KVP_ERR_PARAMETER, "assign_groups: ratios must be non-negative");
    sum += ratios[f];
  }
  require(std::fabs(sum - 1.0) <= 1e-9, KVP_ERR_PARAMETER, "assign_groups: ratios must sum to 1");
  for (int f = 1; f < n_groups; ++f) {
    const int32_t* basis = value_ranks ? value_ranks : key_ranks;
    if (basis) require(basis[f] <= basis[f - 1], KVP_ERR_PARAMETER, "assign_groups: ranks must be non-increasing");
  }
  TierParams tp{};
  // Group sizes exactly as importance.cpp:98-110 (floor(r*n + 0.5), clamp,
  // last group absorbs the remainder).
  int cursor = 0;
  for (int f = 0; f < n_groups; ++f) {
    tp.bounds[f] = cursor;
    int take;
    if (f + 1 == n_groups) {
      take = n - cursor;
    } else {
      take = static_cast<int>(std::floor(ratios[f] * static_cast<double>(n) + 0.5));
      take = std::min(take, n - cursor);
    }
    cursor += take;
    tp.rank_k[f] = key_ranks ? key_ranks[f] : 0;
    tp.rank_v[f] = value_ranks ? value_ranks[f] : 0;
  }
  tp.bounds[n_groups] = n;
  return tp;
}

void launch_tiers(int n_tables, int n, const double* scores, long stride, int n_groups, const TierParams& tp,
                  uint8_t* tier_out, uint16_t* rk_out, uint16_t* rv_out, cudaStream_t s) {
  if (n == 0 || n_tables == 0) return;
  if (n <= kSelThreads * kSelPer) {
    tier_select_kernel<<<n_tables, kSelThreads, 0, s>>>(n, scores, stride, n_groups, tp, tier_out, rk_out, rv_out);
    KVP_LAUNCHED();
    return;
  }
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  const size_t smem = (size_t)npow2 * (sizeof(uint64_t) + sizeof(uint32_t));
  require(smem <= 200 * 1024, KVP_ERR_PARAMETER, "assign_tiers: more than 16384 compressed tokens per segment");
  static bool attr_set = false;
  if (!attr_set) {
    KVP_CUDA(cudaFuncSetAttribute(tier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  tier_kernel<<<n_tables, 1024, smem, s>>>(n, npow2, scores, stride, n_groups, tp, tier_out, rk_out, rv_out);
  KVP_LAUNCHED();
}

}  // namespace kvp

extern "C" int kvp_update_importance(int32_t n_tables, int32_t n, double* scores, int32_t tq, const double* attn,
                                     double alpha, int32_t check, void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(n_tables >= 0 && n >= 0 && tq >= 0, KVP_ERR_SHAPE, "update_importance: negative size");
    if (tq == 0 || n == 0 || n_tables == 0) return;
    require(alpha >= 0.0 && alpha <= 1.0, KVP_ERR_PARAMETER, "update_importance: alpha must be in [0, 1]");
    cudaStream_t s = as_stream(stream);
    if (check) {
      Scratch bad(sizeof(unsigned), s);
      KVP_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned), s));
      // Validate before mutating, like the reference (checks precede the update).
      row_check_kernel<<<n_tables * tq, 256, 0, s>>>(n, attn, bad.as<unsigned>());
      KVP_LAUNCHED();
      unsigned h_bad = 0;
      KVP_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      KVP_CUDA(cudaStreamSynchronize(s));
      require(h_bad == 0, KVP_ERR_DATA, "update_importance: attention row is not a distribution");
    }
    launch_ema(n_tables, n, scores, tq, attn, alpha, nullptr, s);
  });
}

extern "C" int kvp_assign_tiers(int32_t n_tables, int32_t n, const double* scores, int64_t score_stride,
                                int32_t n_groups, const double* ratios, const int32_t* key_ranks,
                                const int32_t* value_ranks, uint8_t* tier_out, uint16_t* rank_k_out,
                                uint16_t* rank_v_out, void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    const TierParams tp = make_tier_params(n, n_groups, ratios, key_ranks, value_ranks);
    launch_tiers(n_tables, n, scores, score_stride, n_groups, tp, tier_out, rank_k_out, rank_v_out,
                 as_stream(stream));
  });
}

extern "C" int kvp_update_importance_host(int32_t n, double* scores, int32_t tq, const double* attn, double alpha) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(n >= 0 && tq >= 0, KVP_ERR_SHAPE, "update_importance: negative size");
    if (tq == 0 || n == 0) return;
    cudaStream_t s = nullptr;
    Scratch buf(sizeof(double) * ((long)n + (long)tq * n), s);
    double* ds = buf.as<double>();
    double* da = ds + n;
    KVP_CUDA(cudaMemcpyAsync(ds, scores, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    KVP_CUDA(cudaMemcpyAsync(da, attn, sizeof(double) * tq * (long)n, cudaMemcpyHostToDevice, s));
    const int rc = kvp_update_importance(1, n, ds, tq, da, alpha, 1, s);
    if (rc != KVP_OK) fail(rc, kvp_last_error_message());
    KVP_CUDA(cudaMemcpyAsync(scores, ds, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    KVP_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int kvp_assign_groups_host(int32_t n, const double* scores, int32_t n_groups, const double* ratios,
                                      const int32_t* ranks, uint32_t* tier_out) {
  return kvp::guarded([&] {
    using namespace kvp;
    const TierParams tp = make_tier_params(n, n_groups, ratios, ranks, nullptr);
    if (n == 0) return;
    cudaStream_t s = nullptr;
    Scratch buf(sizeof(double) * n + n, s);
    double* ds = buf.as<double>();
    uint8_t* dt = reinterpret_cast<uint8_t*>(ds + n);
    KVP_CUDA(cudaMemcpyAsync(ds, scores, sizeof(double) * n, cudaMemcpyHostToDevice, s));
    launch_tiers(1, n, ds, n, n_groups, tp, dt, nullptr, nullptr, s);
    std::vector<uint8_t> h(n);
    KVP_CUDA(cudaMemcpyAsync(h.data(), dt, n, cudaMemcpyDeviceToHost, s));
    KVP_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) tier_out[i] = h[i];
  });
}
