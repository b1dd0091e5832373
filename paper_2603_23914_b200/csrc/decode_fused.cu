// Compressed-cache decode attention, bf16 storage, T_q = 1 — the serving hot
// path.  Replaces the reference's per-(instance, layer) decode loop
// (decoder.cpp:555-601: build plan -> attend_{materialized,fused} ->
// head-average -> update_importance), whose cost is ~100% row rebuilding in
// store_decompress_row (cache.cpp:63-101).  Nothing of width W = H_kv*D is
// rebuilt; every byte of the cache is read exactly once, in three launches:
//
//  1. qdots  (grid: kv-head x instance, CUDA cores, streaming)
//       P[h, r]      = right_k[r, g(h)-slice] . q_h / sqrt(D)     (project q into the key basis)
//       s_tail[h, t] = tail_k[t, g(h)-slice] . q_h / sqrt(D)     (dense-tail logits)
//  2. core   (one thread-block cluster per instance, tcgen05 + TMEM + TMA + DSMEM)
//       S[t, h]  = left_k[t, :] . P[h, :]        tcgen05 M=128 tokens, N=heads, K=rank; S stays in TMEM
//       m_h, z_h over S and s_tail, reduced across the cluster through DSMEM (no online rescaling)
//       p = exp(S - m);  importance EMA (importance.cpp:33-65) from the head average, fp64
//       U^T[r, h] += left_v[t, r] p[t, h]         tcgen05 M=128 ranks, N=heads, K=tokens
//       U (reduce-scattered over the cluster) / z_h -> workspace; p_tail / z_h -> workspace
//  3. vsum   (grid: kv-head x instance, CUDA cores, streaming)
//       out[h, :] = U[h, :] . right_v[:, g-slice] + p_tail[h, :] . tail_v[:, g-slice]
//
// bf16 operands: the cached factors are bf16 (the serving format); the
// on-the-fly operands P and p are split into hi+lo bf16 pairs (two MMAs into
// the same fp32 accumulator), so the only rounding vs an fp64 oracle fed the
// same bf16 factors is fp32 accumulation.
//
// core kernel warp roles (320 threads): warp 0 = TMA producer, warp 1 = MMA
// issuer + TMEM owner, warps 2..9 = TMEM epilogues / softmax / EMA / DSMEM.
// left_k / left_v stream through a 6-stage x 16 KB mbarrier ring in a fixed
// item order that producer and MMA issuer derive identically.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <tuple>
#include <string>

#include "common.cuh"
#include "decode_fused.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {

using namespace sm100;

constexpr int kMaxStages = 12;  // ring stages (even: V panel pairs never straddle the ring wrap)
constexpr uint32_t kStageBytes = 16384;
constexpr int kThreads = 576;         // warp 0 TMA, warp 1 MMA, warps 2..17 compute
constexpr int kComputeThreads = 512;
constexpr int kComputeWarps = 16;
constexpr uint32_t kBarCompute = 1;  // named barrier id for the compute warps
constexpr int kTailMax = 96;
constexpr int kStreamThreads = 256;  // qdots / vsum blocks

struct Smem {
  uint32_t ring, phi, plo, pt, stail, part, stats, imps, bars, tslot, total;
  uint32_t uloc;  // late-phase alias over [phi, ...), valid once the U MMAs completed
  int uloc_stride;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_layout(const FusedPlan& p) {
  Smem s{};
  const uint32_t np = p.np;
  s.ring = 0;
  s.phi = s.ring + p.stages * kStageBytes;
  s.plo = s.phi + p.kpk * np * 128;
  s.pt = align_up(s.plo + p.kpk * np * 128, 1024);  // 2 buffers x {hi, lo} x 2 panels
  const uint32_t pt_end = s.pt + 8 * np * 128;
  s.uloc_stride = static_cast<int>(align_up(p.s.rank_v, 4));
  s.uloc = s.phi;
  const uint32_t uloc_end = s.uloc + np * s.uloc_stride * 4;
  s.stail = align_up(pt_end > uloc_end ? pt_end : uloc_end, 16);
  s.part = s.stail + p.tail_max * np * 4;
  s.stats = s.part + 2 * kComputeWarps * np * 4 + 4 * 128 * 4;
  s.imps = align_up(s.stats + (5 + 8) * np * 4, 16);
  s.bars = align_up(s.imps + (p.chunk + p.tail_max) * 8, 8);
  s.tslot = s.bars + 40 * 8;
  s.total = align_up(s.tslot + 16, 1024);
  return s;
}

enum Bar : int {
  kFull = 0,                      // [kMaxStages]
  kEmpty = kMaxStages,            // [kMaxStages]
  kPopReady = 2 * kMaxStages,     // P operand image landed (producer bulk copy -> MMA)
  kSFull,                         // S MMAs complete (MMA -> compute)
  kPFull0, kPFull1,               // p tile buffer ready (compute -> MMA)
  kPEmpty0, kPEmpty1,             // p tile buffer consumed (MMA -> compute)
  kUFull,                         // U MMAs complete
  kTmemFree,                      // compute finished reading TMEM
  kSlices,                        // (unused)
  kStats,                         // cluster: all (m, z) published (count C)
  kUReady,                        // cluster: all U partials published (count C)
  kDone,                          // cluster: all peers finished reading my smem (count C)
  kNumBars
};

struct Items {
  int lk0, lv0, total;
  int n_tk, tiles, chunk_len, c_first, t_first;
};

__device__ __forceinline__ Items make_items(const FusedPlan& p, int c, int n_tail) {
  Items it{};
  const int C = p.s.cluster;
  const int tail_per = (n_tail + C - 1) / C;
  it.t_first = c * tail_per;
  it.n_tk = max(0, min(n_tail, it.t_first + tail_per) - it.t_first);
  it.c_first = c * p.chunk;
  it.chunk_len = max(0, min(p.s.n_comp, it.c_first + p.chunk) - it.c_first);
  it.tiles = (it.chunk_len + 127) / 128;
  // ring items (MMA operands only): left_k panels, even-pad, left_v panels
  it.lk0 = 0;
  const int after_lk = it.tiles * p.kpk;
  it.lv0 = after_lk + (after_lk & 1);  // V panel pairs must sit in adjacent stages
  it.total = it.lv0 + it.tiles * p.vpanels;
  return it;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// Streaming 16-byte global load that bypasses L1 (every byte is used once).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void unpack8(const uint4& raw, float (&v)[8]) {
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h2[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

// ============================================================================
// 1. qdots: one block per (kv head g, instance b).  Rows = right_k (rank_k)
//    then tail_k (n_tail); each lane owns 8 columns of the g-slice, D/8 lanes
//    span one row segment and reduce with shuffles.
// ============================================================================
template <int PER_KV, int D>
__global__ void __launch_bounds__(kStreamThreads) qdots_kernel(const FusedPlan p, const FusedArgs a) {
  constexpr int LPH = D / 8, RPI = 32 / LPH;
  const int g = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.s.H, W = p.s.Hkv * D;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const int rk = p.s.rank_k, rows = rk + n_tail;
  const int col8 = (lane % LPH) * 8, rsub = lane / LPH;
  const float scale = rsqrtf(static_cast<float>(D));
  float qv[PER_KV][8];
#pragma unroll
  for (int y = 0; y < PER_KV; ++y)
#pragma unroll
    for (int e = 0; e < 8; ++e) qv[y][e] = a.q[static_cast<long>(b) * H * D + (g * PER_KV + y) * D + col8 + e] * scale;
  const __nv_bfloat16* rkb = a.right_k + static_cast<long>(b) * rk * W + g * D + col8;
  const __nv_bfloat16* tkb = a.tail_k + static_cast<long>(b) * p.s.tail_cap * W + g * D + col8;
  const int NP = p.np;
  const uint32_t plane = static_cast<uint32_t>(p.kpk) * NP * 128;  // bytes of one (hi or lo) operand
  unsigned char* pimg = a.ws_pimg + static_cast<size_t>(b) * 2 * plane;
  float* tout = a.ws_tail + static_cast<long>(b) * H * p.s.tail_cap;
  // zero padding of the operand image: ranks >= rank_k of my heads; heads >= H (block g == 0)
  for (int i = threadIdx.x; i < PER_KV * (p.kpk * 64 - rk); i += kStreamThreads) {
    const int h = g * PER_KV + i / (p.kpk * 64 - rk), r = rk + i % (p.kpk * 64 - rk);
    const uint32_t off = (r >> 6) * NP * 128 + sw128_off(h, r & 63);
    *reinterpret_cast<__nv_bfloat16*>(pimg + off) = __float2bfloat16_rn(0.f);
    *reinterpret_cast<__nv_bfloat16*>(pimg + plane + off) = __float2bfloat16_rn(0.f);
  }
  if (g == 0)
    for (int i = threadIdx.x; i < (NP - H) * p.kpk * 64; i += kStreamThreads) {
      const int h = H + i / (p.kpk * 64), r = i % (p.kpk * 64);
      const uint32_t off = (r >> 6) * NP * 128 + sw128_off(h, r & 63);
      *reinterpret_cast<__nv_bfloat16*>(pimg + off) = __float2bfloat16_rn(0.f);
      *reinterpret_cast<__nv_bfloat16*>(pimg + plane + off) = __float2bfloat16_rn(0.f);
    }
  constexpr int U = 8;
  const int stride = 8 * RPI;  // rows advanced per warp-instruction round across the block
  for (int r0 = warp * RPI + rsub; r0 < rows; r0 += U * stride) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * stride;
      if (r < rows) raw[u] = ldg_stream(r < rk ? rkb + static_cast<long>(r) * W : tkb + static_cast<long>(r - rk) * W);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * stride;
      float v[8];
      unpack8(raw[u], v);
#pragma unroll
      for (int y = 0; y < PER_KV; ++y) {
        float acc = v[0] * qv[y][0];
#pragma unroll
        for (int e = 1; e < 8; ++e) acc = fmaf(v[e], qv[y][e], acc);
#pragma unroll
        for (int o = LPH / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((lane % LPH) == 0 && r < rows) {
          const int h = g * PER_KV + y;
          if (r < rk) {
            __nv_bfloat16 hi, lo;
            split_bf16(acc, hi, lo);
            const uint32_t off = (r >> 6) * NP * 128 + sw128_off(h, r & 63);
            *reinterpret_cast<__nv_bfloat16*>(pimg + off) = hi;
            *reinterpret_cast<__nv_bfloat16*>(pimg + plane + off) = lo;
          } else {
            tout[static_cast<long>(h) * p.s.tail_cap + (r - rk)] = acc;
          }
        }
      }
    }
  }
}

// ============================================================================
// 3. vsum: out[h, :] = sum_r U[h, r] right_v[r, g-slice] + sum_t p_tail[h, t] tail_v[t, g-slice]
// ============================================================================
template <int PER_KV, int D>
__global__ void __launch_bounds__(kStreamThreads) vsum_kernel(const FusedPlan p, const FusedArgs a) {
  constexpr int LPH = D / 8, RPI = 32 / LPH, NPART = 8 * RPI;
  extern __shared__ __align__(16) float vsm[];
  const int g = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.s.H, W = p.s.Hkv * D;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const int rv = p.s.rank_v, rows = rv + n_tail;
  const int col8 = (lane % LPH) * 8, rsub = lane / LPH;
  // weights for this block's query heads: [PER_KV][rows]
  float* wts = vsm;
  const int wstride = (rv + p.s.tail_cap + 3) & ~3;
  float* red = vsm + PER_KV * wstride;
  for (int i = threadIdx.x; i < PER_KV * rows; i += kStreamThreads) {
    const int y = i / rows, r = i % rows, h = g * PER_KV + y;
    wts[y * wstride + r] = r < rv ? a.ws_u[(static_cast<long>(b) * H + h) * rv + r]
                                  : a.ws_tail[(static_cast<long>(b) * H + h) * p.s.tail_cap + (r - rv)];
  }
  __syncthreads();
  const __nv_bfloat16* rvb = a.right_v + static_cast<long>(b) * rv * W + g * D + col8;
  const __nv_bfloat16* tvb = a.tail_v + static_cast<long>(b) * p.s.tail_cap * W + g * D + col8;
  float acc[PER_KV][8];
#pragma unroll
  for (int y = 0; y < PER_KV; ++y)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[y][e] = 0.f;
  constexpr int U = 8;
  const int stride = 8 * RPI;
  for (int r0 = warp * RPI + rsub; r0 < rows; r0 += U * stride) {
    uint4 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * stride;
      if (r < rows) raw[u] = ldg_stream(r < rv ? rvb + static_cast<long>(r) * W : tvb + static_cast<long>(r - rv) * W);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * stride;
      if (r >= rows) break;
      float v[8];
      unpack8(raw[u], v);
#pragma unroll
      for (int y = 0; y < PER_KV; ++y) {
        const float w = wts[y * wstride + r];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[y][e] = fmaf(w, v[e], acc[y][e]);
      }
    }
  }
  // reduce the NPART (warp, row-subset) partials of every column
#pragma unroll
  for (int y = 0; y < PER_KV; ++y) {
    float* dst = red + ((warp * RPI + rsub) * PER_KV + y) * D + col8;
    *reinterpret_cast<float4*>(dst) = make_float4(acc[y][0], acc[y][1], acc[y][2], acc[y][3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[y][4], acc[y][5], acc[y][6], acc[y][7]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < PER_KV * D; i += kStreamThreads) {
    const int y = i / D, col = i % D;
    float s = 0.f;
#pragma unroll 8
    for (int k = 0; k < NPART; ++k) s += red[(k * PER_KV + y) * D + col];
    const long oi = static_cast<long>(b) * H * D + static_cast<long>(g * PER_KV + y) * D + col;
    if (a.ctx_bf16)
      reinterpret_cast<__nv_bfloat16*>(a.ctx_out)[oi] = __float2bfloat16_rn(s);
    else
      reinterpret_cast<float*>(a.ctx_out)[oi] = s;
  }
}

// ============================================================================
// 2. core: one cluster of C CTAs per instance.
// ============================================================================
template <int NPT>
__global__ void __launch_bounds__(kThreads, 1)
    core_kernel(const FusedPlan p, const __grid_constant__ CUtensorMap map_lk,
                const __grid_constant__ CUtensorMap map_lv, const __grid_constant__ CUtensorMap map_lk32,
                const __grid_constant__ CUtensorMap map_lv32, const FusedArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const Smem L = smem_layout(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.s.cluster;
  const int c = static_cast<int>(cluster_rank());
  const int b = blockIdx.x / C;
  const int H = p.s.H;
  constexpr int NP = NPT;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const Items it = make_items(p, c, n_tail);
  const uint32_t s_cols = static_cast<uint32_t>(p.max_tiles * NP);
  const int NS = p.stages;

  // ---- prologue: zero ring + P operand, barriers, TMEM -------------------------
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = L.phi / 16;  // ring only (P arrives as a bulk copy)
    for (uint32_t i = threadIdx.x; i < n16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&bars[kFull + s], 1);
      mbar_init(&bars[kEmpty + s], 1);
    }
    for (int i = kPopReady; i <= kTmemFree; ++i) mbar_init(&bars[i], 1);  // kPopReady: producer's expect_tx
    for (int i = kSlices; i <= kDone; ++i) mbar_init(&bars[i], C);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, static_cast<uint32_t>(p.tmem_cols));
  fence_proxy_async();  // zeroed operand bytes visible to the async proxy
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ===================== producer: left_k / left_v panels =====================
    if (lane == 0) {
      prefetch_tmap(&map_lk);
      prefetch_tmap(&map_lv);
      prefetch_tmap(&map_lk32);
      prefetch_tmap(&map_lv32);
      {  // P operand image (bf16 hi/lo, already swizzled by qdots) -> smem in one bulk copy
        const uint32_t pbytes = 2u * p.kpk * NP * 128;
        mbar_expect_tx(&bars[kPopReady], pbytes);
        bulk_load(smem + L.phi, reinterpret_cast<const unsigned char*>(a.ws_pimg) + static_cast<size_t>(b) * pbytes,
                  pbytes, &bars[kPopReady]);
      }
      for (int i = 0; i < it.total; ++i) {
        const int s = i % NS;
        mbar_wait(&bars[kEmpty + s], ((i / NS) & 1) ^ 1);
        unsigned char* dst = smem + L.ring + s * kStageBytes;
        uint64_t* full = &bars[kFull + s];
        const bool is_v = i >= it.lv0;
        const int rel = is_v ? i - it.lv0 : i - it.lk0;
        const int per_tile = is_v ? p.vpanels : p.kpk;
        if (!is_v && rel >= it.tiles * p.kpk) {  // even-pad slot
          mbar_arrive(full);
          continue;
        }
        const int tile = rel / per_tile, panel = rel % per_tile;
        const int rank = is_v ? p.s.rank_v : p.s.rank_k;
        if (panel * 64 >= rank) {  // V pad panel: U rows >= rank_v are never read
          mbar_arrive(full);
          continue;
        }
        if (a.trace && i == it.lv0) a.trace[blockIdx.x * 16ull + 10] = global_ns();
        const int row0 = tile * 128;
        const int nbox = min(4, (it.chunk_len - row0 + 31) / 32);
        mbar_expect_tx(full, static_cast<uint32_t>(nbox) * 4096u);
        const int grow = b * p.s.n_comp + it.c_first + row0;
        if (nbox == 4 && !p.box32_only) {  // full 128-token tile: one 16 KB box
          tma_load_2d(dst, is_v ? &map_lv : &map_lk, panel * 64, grow, full);
        } else {
          for (int k = 0; k < nbox; ++k)
            tma_load_2d(dst + k * 4096, is_v ? &map_lv32 : &map_lk32, panel * 64, grow + 32 * k, full);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, NP, false, false);
      const uint32_t idesc_u = idesc_bf16(128, NP, true, false);
      const uint32_t ring = smem_addr(smem + L.ring);
      const uint32_t phi = smem_addr(smem + L.phi), plo = smem_addr(smem + L.plo);
      const uint32_t pt = smem_addr(smem + L.pt);
      mbar_wait(&bars[kPopReady], 0);
      tc_fence_after();
      if (a.trace) a.trace[blockIdx.x * 16ull + 8] = global_ns();
      for (int t = 0; t < it.tiles; ++t) {
        for (int kp = 0; kp < p.kpk; ++kp) {
          const int i = it.lk0 + t * p.kpk + kp, s = i % NS;
          mbar_wait(&bars[kFull + s], (i / NS) & 1);
          tc_fence_after();
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = smem_desc(ring + s * kStageBytes + kk * 32, 16, 1024, kSwizzle128B);
            const uint64_t bh = smem_desc(phi + kp * NP * 128 + kk * 32, 16, 1024, kSwizzle128B);
            const uint64_t bl = smem_desc(plo + kp * NP * 128 + kk * 32, 16, 1024, kSwizzle128B);
            const uint32_t d = tmem + static_cast<uint32_t>(t * NP);
            mma_bf16(d, ad, bh, idesc_s, (kp | kk) != 0);
            mma_bf16(d, ad, bl, idesc_s, 1);
          }
          mma_commit(&bars[kEmpty + s]);
        }
      }
      if (it.lv0 > it.tiles * p.kpk) {  // release the even-pad slot
        const int i = it.lv0 - 1, s = i % NS;
        mbar_wait(&bars[kFull + s], (i / NS) & 1);
        mbar_arrive(&bars[kEmpty + s]);
      }
      mma_commit(&bars[kSFull]);
      if (a.trace) a.trace[blockIdx.x * 16ull + 9] = global_ns();
      for (int t = 0; t < it.tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(&bars[kPFull0 + buf], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t pth = pt + buf * 4 * NP * 128, ptl = pth + 2 * NP * 128;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const int i0 = it.lv0 + t * p.vpanels + 2 * mt;
          const int s0 = i0 % NS, s1 = (i0 + 1) % NS;
          mbar_wait(&bars[kFull + s0], (i0 / NS) & 1);
          mbar_wait(&bars[kFull + s1], ((i0 + 1) / NS) & 1);
          tc_fence_after();
          const uint32_t d = tmem + s_cols + static_cast<uint32_t>(mt * NP);
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t ad = smem_desc(ring + s0 * kStageBytes + ks * 2048, kStageBytes, 1024, kSwizzle128B);
            const uint32_t boff = (ks >> 2) * NP * 128 + (ks & 3) * 32;
            const uint64_t bh = smem_desc(pth + boff, 16, 1024, kSwizzle128B);
            const uint64_t bl = smem_desc(ptl + boff, 16, 1024, kSwizzle128B);
            mma_bf16(d, ad, bh, idesc_u, (t | ks) != 0);
            mma_bf16(d, ad, bl, idesc_u, 1);
          }
          mma_commit(&bars[kEmpty + s0]);
          mma_commit(&bars[kEmpty + s1]);
        }
        mma_commit(&bars[kPEmpty0 + buf]);
      }
      mma_commit(&bars[kUFull]);
      mbar_wait(&bars[kTmemFree], 0);
    }
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, static_cast<uint32_t>(p.tmem_cols));
  } else {
    // ===================== compute warps =====================
    const int cw = warp - 2;                 // 0..15
    const int tid = threadIdx.x - 64;        // 0..511
    float* stail = reinterpret_cast<float*>(smem + L.stail);
    float* part = reinterpret_cast<float*>(smem + L.part);
    float* stats = reinterpret_cast<float*>(smem + L.stats);
    double* imps = reinterpret_cast<double*>(smem + L.imps);
    float* m_loc = stats;
    float* z_loc = stats + NP;
    float* m_g = stats + 2 * NP;
    float* f_me = stats + 3 * NP;  // exp(m_loc - m_g) / z_g   (my tokens' softmax correction)
    float* zi_g = stats + 4 * NP;  // 1 / z_g
    float* scale_c = stats + 5 * NP;  // [C][NP]: exp(m_c - m_g) per peer
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 0] = global_ns();

    // prefetch my importance scores and tail logits (latency off the critical path)
    const float* tg = a.ws_tail + static_cast<long>(b) * H * p.s.tail_cap;
    if (a.importance) {
      const double* ib = a.importance + static_cast<long>(b) * a.imp_stride;
      for (int i = tid; i < it.chunk_len; i += kComputeThreads) imps[i] = ib[it.c_first + i];
      for (int j = tid; j < it.n_tk; j += kComputeThreads) imps[p.chunk + j] = ib[p.s.n_comp + it.t_first + j];
    }
    for (int i = tid; i < it.n_tk * H; i += kComputeThreads) {
      const int j = i % it.n_tk, h = i / it.n_tk;
      stail[j * NP + h] = tg[static_cast<long>(h) * p.s.tail_cap + it.t_first + j];
    }

    // ---- local softmax: max over TMEM-resident S + my tail logits (no exponentials)
    const int qd = warp & 3;                 // TMEM lane quadrant this warp may access
    const int cg = cw >> 2;                  // column group 0..3
    constexpr int gcols = NP / 4;            // multiple of 4 columns
    const int gbase = cg * gcols;
    auto tmem_row = [&](uint32_t col) { return tmem + (static_cast<uint32_t>(qd * 32) << 16) + col; };
    mbar_wait(&bars[kSFull], 0);
    tc_fence_after();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 1] = global_ns();
    float* part_m = part;                         // [16 warps][NP]
    float* part_s = part + kComputeWarps * NP;    // [16 warps][NP]
    for (int c0 = 0; c0 < gcols; c0 += 4) {
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int t = 0; t < it.tiles; ++t) {
        float v[4];
        tmem_ld4(tmem_row(static_cast<uint32_t>(t * NP + gbase + c0)), v);
        if (t * 128 + qd * 32 + lane < it.chunk_len)
          for (int e = 0; e < 4; ++e) mx[e] = fmaxf(mx[e], v[e]);
      }
      for (int e = 0; e < 4; ++e) {
        const float m = warp_max(mx[e]);
        if (lane == 0) part_m[cw * NP + gbase + c0 + e] = m;
      }
    }
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 6] = global_ns();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < H) {
      const int h = tid, w0 = (h / gcols) * 4;
      float m = -INFINITY;
      for (int w = 0; w < 4; ++w) m = fmaxf(m, part_m[(w0 + w) * NP + h]);
      for (int j = 0; j < it.n_tk; ++j) m = fmaxf(m, stail[j * NP + h]);
      m_loc[h] = m;
    }
    named_bar(kBarCompute, kComputeThreads);
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 2] = global_ns();

    // ---- p tiles with the local max (bf16 hi/lo B operand, K-major over tokens); z from the same pass
    float zp[gcols];
#pragma unroll
    for (int e = 0; e < gcols; ++e) zp[e] = 0.f;
    for (int t = 0; t < it.tiles; ++t) {
      const int buf = t & 1;
      if (t >= 2) mbar_wait(&bars[kPEmpty0 + buf], ((t - 2) >> 1) & 1);
      unsigned char* pth = smem + L.pt + buf * 4 * NP * 128;
      unsigned char* ptl = pth + 2 * NP * 128;
      const int row = qd * 32 + lane;  // token within the tile
      const bool valid = t * 128 + row < it.chunk_len;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4];
        tmem_ld4(tmem_row(static_cast<uint32_t>(t * NP + gbase + c0)), v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          const float pv = (valid && h < H) ? __expf(v[e] - m_loc[h]) : 0.f;
          zp[c0 + e] += pv;
          __nv_bfloat16 hi, lo;
          split_bf16(pv, hi, lo);
          const uint32_t off = (row >> 6) * NP * 128 + sw128_off(h, row & 63);
          *reinterpret_cast<__nv_bfloat16*>(pth + off) = hi;
          *reinterpret_cast<__nv_bfloat16*>(ptl + off) = lo;
        }
      }
      fence_proxy_async();
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) mbar_arrive(&bars[kPFull0 + buf]);
    }
#pragma unroll
    for (int c0 = 0; c0 < gcols; ++c0) {
      const float z = warp_sum(zp[c0]);
      if (lane == 0) part_s[cw * NP + gbase + c0] = z;
    }
    // tail: local p in place of the logits
    for (int w = tid; w < it.n_tk * H; w += kComputeThreads) {
      const int j = w / H, h = w % H;
      stail[j * NP + h] = __expf(stail[j * NP + h] - m_loc[h]);
    }
    named_bar(kBarCompute, kComputeThreads);
    if (tid < H) {
      const int h = tid, w0 = (h / gcols) * 4;
      float z = 0.f;
      for (int w = 0; w < 4; ++w) z += part_s[(w0 + w) * NP + h];
      for (int j = 0; j < it.n_tk; ++j) z += stail[j * NP + h];
      z_loc[h] = z;
    }
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 3] = global_ns();

    // ---- U readback (TMEM -> U_loc[h][r]); publish (m_loc, z_loc, U_loc) to the cluster
    mbar_wait(&bars[kUFull], 0);
    tc_fence_after();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 4] = global_ns();
    float* uloc = reinterpret_cast<float*>(smem + L.uloc);
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int r = mt * 128 + qd * 32 + lane;
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (it.tiles > 0) tmem_ld4(tmem_row(s_cols + static_cast<uint32_t>(mt * NP + gbase + c0)), v);
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          if (h < H && r < p.s.rank_v) uloc[h * L.uloc_stride + r] = v[e];
        }
      }
    }
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kUReady], static_cast<uint32_t>(tid));
    mbar_wait_cluster(&bars[kUReady], 0);

    // ---- global softmax statistics from the peers' (m, z)
    if (tid < H) {
      const int h = tid;
      float mp[8], zp[8];
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) {
          mp[peer] = ld_dsmem_f32(&m_loc[h], static_cast<uint32_t>(peer));
          zp[peer] = ld_dsmem_f32(&z_loc[h], static_cast<uint32_t>(peer));
        }
      float mg = -INFINITY;
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) mg = fmaxf(mg, mp[peer]);
      float zg = 0.f;
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) {
          const float sc = mp[peer] == -INFINITY ? 0.f : __expf(mp[peer] - mg);
          scale_c[peer * NP + h] = sc;
          zg += zp[peer] * sc;
        }
      const float zi = 1.0f / zg;
      m_g[h] = mg;
      zi_g[h] = zi;
      f_me[h] = (m_loc[h] == -INFINITY ? 0.f : __expf(m_loc[h] - mg)) * zi;
    }
    named_bar(kBarCompute, kComputeThreads);

    // ---- reduce-scatter U over the cluster: heads h = c, c + C, ...; U / z -> workspace
    const int r4 = L.uloc_stride / 4;
    const int my_heads = (H - c + C - 1) / C;
    for (int w = tid; w < my_heads * r4; w += kComputeThreads) {
      const int h = c + (w / r4) * C, r = (w % r4) * 4;
      uint4 u[8];
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) u[peer] = ld_dsmem_v4(&uloc[h * L.uloc_stride + r], static_cast<uint32_t>(peer));
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int peer = 0; peer < 8; ++peer) {
        if (peer >= C) break;
        const float sc = scale_c[peer * NP + h];
        s4.x = fmaf(sc, __uint_as_float(u[peer].x), s4.x);
        s4.y = fmaf(sc, __uint_as_float(u[peer].y), s4.y);
        s4.z = fmaf(sc, __uint_as_float(u[peer].z), s4.z);
        s4.w = fmaf(sc, __uint_as_float(u[peer].w), s4.w);
      }
      const float zi = zi_g[h];
      float* dst = a.ws_u + (static_cast<long>(b) * H + h) * p.s.rank_v + r;
      const float vals[4] = {s4.x * zi, s4.y * zi, s4.z * zi, s4.w * zi};
      for (int e = 0; e < 4; ++e)
        if (r + e < p.s.rank_v) dst[e] = vals[e];
    }
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kDone], static_cast<uint32_t>(tid));

    // ---- head-averaged attention + importance EMA (importance.cpp:33-65), S re-read from TMEM
    float* ha_part = part;  // [4 groups][128] (part_m / part_s are dead)
    const float inv_h = 1.0f / static_cast<float>(H);
    for (int t = 0; t < it.tiles; ++t) {
      const int row = qd * 32 + lane;
      float hsum = 0.f;
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4];
        tmem_ld4(tmem_row(static_cast<uint32_t>(t * NP + gbase + c0)), v);
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          if (h < H) hsum = fmaf(__expf(v[e] - m_loc[h]), f_me[h], hsum);
        }
      }
      ha_part[cg * 128 + row] = hsum;
      named_bar(kBarCompute, kComputeThreads);
      if (tid < 128) {
        const int tk = t * 128 + tid;
        if (tk < it.chunk_len) {
          const float ha = (ha_part[tid] + ha_part[128 + tid] + ha_part[256 + tid] + ha_part[384 + tid]) * inv_h;
          const long gi = it.c_first + tk;
          if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + p.s.tail_cap) + gi] = ha;
          if (a.importance)
            a.importance[static_cast<long>(b) * a.imp_stride + gi] =
                __dadd_rn(__dmul_rn(a.ema_decay, imps[tk]), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
        }
      }
      named_bar(kBarCompute, kComputeThreads);
    }
    tc_fence_before();
    if (tid == 0) mbar_arrive(&bars[kTmemFree]);
    // tail tokens: normalised p -> workspace (for vsum), head average, EMA
    for (int w = tid; w < it.n_tk * H; w += kComputeThreads) {
      const int j = w % it.n_tk, h = w / it.n_tk;
      const float pn = stail[j * NP + h] * f_me[h];
      a.ws_tail[(static_cast<long>(b) * H + h) * p.s.tail_cap + it.t_first + j] = pn;
    }
    for (int j = tid; j < it.n_tk; j += kComputeThreads) {
      float hs = 0.f;
      for (int h = 0; h < H; ++h) hs = fmaf(stail[j * NP + h], f_me[h], hs);
      const float ha = hs * inv_h;
      const long gi = p.s.n_comp + it.t_first + j;
      if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + p.s.tail_cap) + gi] = ha;
      if (a.importance)
        a.importance[static_cast<long>(b) * a.imp_stride + gi] =
            __dadd_rn(__dmul_rn(a.ema_decay, imps[p.chunk + j]), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
    }
    mbar_wait_cluster(&bars[kDone], 0);  // peers may still be reading my U_loc / stats
    if (a.trace && tid == 0) a.trace[blockIdx.x * 16ull + 5] = global_ns();
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    KVP_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
    require(q == cudaDriverEntryPointSuccess && p != nullptr, KVP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes,
               uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tmap_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, KVP_ERR_CUDA, "cuTensorMapEncodeTiled failed");
}

}  // namespace

FusedPlan plan_fused(const FusedShape& s) {
  FusedPlan p{};
  p.s = s;
  p.ok = false;
  auto bad = [&](const char* why) {
    p.why = why;
    return p;
  };
  if (s.H % s.Hkv != 0) return bad("num_kv_heads must divide num_query_heads");
  const int per_kv = s.H / s.Hkv;
  if (per_kv != 1 && per_kv != 2 && per_kv != 4) return bad("fused path needs 1, 2 or 4 query heads per kv head");
  if (s.D != 128 && s.D != 64) return bad("fused path needs head_dim 64 or 128");
  if (s.H > 64) return bad("fused path supports up to 64 query heads");
  if (s.rank_k < 1 || s.rank_v < 1) return bad("fused path needs low-rank K and V");
  if (s.ld_left % 8 != 0 || s.ld_left < std::max(s.rank_k, s.rank_v))
    return bad("left-factor stride must be a multiple of 8 and cover both ranks");
  if (s.cluster < 1 || s.cluster > 8) return bad("cluster size must be 1..8");
  p.np = (s.H + 15) / 16 * 16;
  p.kpk = (s.rank_k + 63) / 64;
  p.vpanels = ((s.rank_v + 63) / 64 + 1) / 2 * 2;
  p.mtiles = p.vpanels / 2;
  const int per = (s.n_comp + s.cluster - 1) / s.cluster;
  p.chunk = (per + 31) / 32 * 32;
  p.max_tiles = (p.chunk + 127) / 128;
  p.tail_max = (s.tail_cap + s.cluster - 1) / s.cluster;
  if (p.tail_max > kTailMax) return bad("too many tail tokens per CTA (raise the cluster size)");
  p.heads_per_cta = (s.H + s.cluster - 1) / s.cluster;
  const int cols = p.max_tiles * p.np + p.mtiles * p.np;
  if (cols > 512) return bad("TMEM budget exceeded (raise the cluster size)");
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.stages = 4;
  if (smem_layout(p).total > 227 * 1024) return bad("shared-memory budget exceeded");
  while (p.stages + 2 <= kMaxStages) {
    FusedPlan q = p;
    q.stages = p.stages + 2;
    if (smem_layout(q).total > 227 * 1024) break;
    p.stages = q.stages;
  }
  if (const char* e = std::getenv("KVP_FUSED_STAGES")) {  // tuning override
    const int want = std::atoi(e);
    if (want >= 2 && want <= kMaxStages && want % 2 == 0 && want < p.stages) p.stages = want;
  }
  p.box32_only = std::getenv("KVP_FUSED_BOX32") != nullptr;
  p.smem_bytes = smem_layout(p).total;
  const size_t vs = (static_cast<size_t>(per_kv) * ((s.rank_v + s.tail_cap + 3) & ~3) + 8 * (256 / s.D) * per_kv * s.D) * 4;
  if (vs > 200 * 1024) return bad("vsum weights exceed shared memory");
  p.ok = true;
  p.why = "";
  return p;
}

size_t fused_workspace_bytes(const FusedShape& s) {
  const size_t np = (s.H + 15) / 16 * 16, kpk = (s.rank_k + 63) / 64;
  const size_t pimg = 2 * kpk * np * 128;
  return static_cast<size_t>(s.batch) * (pimg + sizeof(float) * s.H * (static_cast<size_t>(s.tail_cap) + s.rank_v));
}

void encode_fused_maps(const FusedShape& s, const void* left_k, const void* left_v, CUtensorMap* maps) {
  const uint64_t rows = static_cast<uint64_t>(s.batch) * s.n_comp;
  const uint64_t ld = static_cast<uint64_t>(s.ld_left) * 2;
  encode_2d(&maps[0], left_k, s.rank_k, rows, ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  encode_2d(&maps[1], left_v, s.rank_v, rows, ld, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  encode_2d(&maps[2], left_k, s.rank_k, rows, ld, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  encode_2d(&maps[3], left_v, s.rank_v, rows, ld, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int PER_KV, int D>
void launch_stream_pair(const FusedPlan& p, const FusedArgs& a, cudaStream_t st, bool first) {
  const dim3 grid(static_cast<unsigned>(p.s.Hkv), static_cast<unsigned>(p.s.batch));
  if (first) {
    qdots_kernel<PER_KV, D><<<grid, kStreamThreads, 0, st>>>(p, a);
    KVP_LAUNCHED();
  } else {
    const size_t smem = (static_cast<size_t>(PER_KV) * ((p.s.rank_v + p.s.tail_cap + 3) & ~3) + 8 * (256 / D) * PER_KV * D) * 4;
    static size_t attr = 0;
    if (attr < smem) {
      KVP_CUDA(cudaFuncSetAttribute(vsum_kernel<PER_KV, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      attr = smem;
    }
    vsum_kernel<PER_KV, D><<<grid, kStreamThreads, smem, st>>>(p, a);
    KVP_LAUNCHED();
  }
}

void launch_stream(const FusedPlan& p, const FusedArgs& a, cudaStream_t st, bool first) {
  const int per_kv = p.s.H / p.s.Hkv;
  if (p.s.D == 128) {
    if (per_kv == 1) launch_stream_pair<1, 128>(p, a, st, first);
    else if (per_kv == 2) launch_stream_pair<2, 128>(p, a, st, first);
    else launch_stream_pair<4, 128>(p, a, st, first);
  } else {
    if (per_kv == 1) launch_stream_pair<1, 64>(p, a, st, first);
    else if (per_kv == 2) launch_stream_pair<2, 64>(p, a, st, first);
    else launch_stream_pair<4, 64>(p, a, st, first);
  }
}

using CoreFn = void (*)(const FusedPlan, const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,
                       const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap, const FusedArgs);
CoreFn core_for(int np) {
  switch (np) {
    case 16: return core_kernel<16>;
    case 32: return core_kernel<32>;
    case 48: return core_kernel<48>;
    default: return core_kernel<64>;
  }
}

void launch_fused(const FusedPlan& p, const CUtensorMap* maps, const FusedArgs& a, cudaStream_t st) {
  require(p.ok, KVP_ERR_PARAMETER, p.why);
  launch_stream(p, a, st, true);
  auto kernel = core_for(p.np);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.s.batch * p.s.cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.s.cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KVP_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, maps[0], maps[1], maps[2], maps[3], a));
  KVP_LAUNCHED();
  launch_stream(p, a, st, false);
}

int max_active_clusters(const FusedPlan& p) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.s.batch * p.s.cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.s.cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto kernel = core_for(p.np);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  int n = 0;
  KVP_CUDA(cudaOccupancyMaxActiveClusters(&n, kernel, &cfg));
  return n;
}

}  // namespace kvp

// Debug hooks (not part of the public header).
static unsigned long long* g_trace = nullptr;
extern "C" void kvp_debug_fused_trace(void* dev_buffer) { g_trace = static_cast<unsigned long long*>(dev_buffer); }

namespace {
// Cluster size: 4 CTAs per instance when the plan fits (measured fastest on
// B200 for the C2/C5 shapes), else 8, 2, 1.
int auto_cluster(kvp::FusedShape s) {
  for (int c : {4, 8, 2, 1}) {
    s.cluster = c;
    if (kvp::plan_fused(s).ok) return c;
  }
  return 8;
}
kvp::FusedShape shape_of(const kvp_fused_desc* d) {
  kvp::FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, d->ld_left,
                    d->tail_cap, d->batch, d->cluster};
  if (s.cluster <= 0) s.cluster = auto_cluster(s);
  return s;
}
}  // namespace

extern "C" int kvp_debug_fused_max_clusters(const kvp_fused_desc* d) {
  int n = -1;
  kvp::guarded([&] { n = kvp::max_active_clusters(kvp::plan_fused(shape_of(d))); });
  return n;
}

extern "C" size_t kvp_decode_fused_workspace(const kvp_fused_desc* d) {
  return d ? kvp::fused_workspace_bytes(shape_of(d)) : 0;
}

extern "C" int kvp_decode_fused(const kvp_fused_desc* d, void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(d != nullptr, KVP_ERR_PARAMETER, "decode_fused: null descriptor");
    require(d->heads > 0 && d->kv_heads > 0 && d->head_dim > 0 && d->batch > 0, KVP_ERR_PARAMETER,
            "HeadGeometry: head counts and head_dim must be positive");
    require(d->n_comp > 0, KVP_ERR_PARAMETER, "decode_fused: empty compressed block");
    require(d->n_tail_dev != nullptr || (d->n_tail >= 0 && d->n_tail <= d->tail_cap), KVP_ERR_SHAPE,
            "decode_fused: tail length exceeds capacity");
    require(d->alpha >= 0.0 && d->alpha <= 1.0, KVP_ERR_PARAMETER, "update_importance: alpha must be in [0, 1]");
    const FusedShape s = shape_of(d);
    const FusedPlan p = plan_fused(s);
    require(p.ok, KVP_ERR_PARAMETER, (std::string("decode_fused: ") + p.why).c_str());
    const size_t ws_bytes = fused_workspace_bytes(s);
    cudaStream_t st = as_stream(stream);
    std::unique_ptr<Scratch> own;
    float* ws = static_cast<float*>(d->workspace);
    if (ws == nullptr) {
      own = std::make_unique<Scratch>(ws_bytes, st);
      ws = own->as<float>();
    } else {
      require(d->workspace_bytes >= ws_bytes, KVP_ERR_PARAMETER, "decode_fused: workspace too small");
    }
    CUtensorMap maps[4];
    encode_fused_maps(s, d->left_k, d->left_v, maps);
    FusedArgs a{};
    a.right_k = static_cast<const __nv_bfloat16*>(d->right_k);
    a.right_v = static_cast<const __nv_bfloat16*>(d->right_v);
    a.tail_k = static_cast<const __nv_bfloat16*>(d->tail_k);
    a.tail_v = static_cast<const __nv_bfloat16*>(d->tail_v);
    a.n_tail_dev = d->n_tail_dev;
    a.n_tail = d->n_tail;
    a.q = d->queries;
    a.importance = d->importance;
    a.imp_stride = d->imp_stride;
    const double decay = std::pow(d->alpha, 1.0);  // alpha^T_q, importance.cpp:58
    a.ema_decay = decay;
    a.ema_blend = 1.0 - decay;
    a.head_avg = d->head_avg;
    a.ctx_out = d->context;
    a.ctx_bf16 = d->context_bf16;
    a.ws_pimg = reinterpret_cast<unsigned char*>(ws);
    a.ws_tail = reinterpret_cast<float*>(a.ws_pimg + static_cast<size_t>(s.batch) * 2 * p.kpk * p.np * 128);
    a.ws_u = a.ws_tail + static_cast<size_t>(s.batch) * s.H * s.tail_cap;
    a.trace = g_trace;
    launch_fused(p, maps, a, st);
  });
}
