// Fused decode attention over the compressed KV cache — one thread-block
// cluster per (instance, layer), bf16 storage, tcgen05 tensor cores.
//
// Replaces the reference's decode hot loop (decoder.cpp:555-601: build plan ->
// attend_{materialized,fused} -> head-average -> update_importance), whose
// cost is ~100% store_decompress_row (cache.cpp:63-101).  Nothing of width
// W = H_kv*D is ever rebuilt; every byte of the cache is read once:
//
//   phase P  P[r,h]  = right_k[r, g(h)-slice] . q_h / sqrt(D)      CUDA cores, rows split over the cluster,
//                                                                 slices exchanged through DSMEM
//   phase S  S[t,h]  = left_k[t,:] . P[:,h]                         tcgen05, M=128 tokens, N=heads, K=rank,
//                                                                 accumulators stay resident in TMEM
//            tail    s[t,h] = tail_k[t, g-slice] . q_h / sqrt(D)     CUDA cores
//   stats    cluster-wide max / normaliser per head via DSMEM (no online rescaling)
//   phase U  U^T[r,h] += left_v[t,r] * p[t,h]   (r < rank_v(t))     tcgen05, M=128 ranks, N=heads, K=tokens
//            tail    c[h,:] += p[t,h] * tail_v[t, g-slice]          CUDA cores
//   output   out[h,:] = (sum_cluster U[h,:] . right_v[:, g-slice] + sum_cluster c[h,:]) / z_h
//   EMA      importance[t] <- decay*imp + blend*mean_h p[t,h]/z_h  (importance.cpp:33-65), fp64
//
// bf16 operands: the cached factors are bf16 (the serving format); the
// on-the-fly operands P and p are split into hi+lo bf16 pairs (two MMAs into
// the same fp32 accumulator), so the only rounding vs an fp64 oracle fed the
// same bf16 factors is fp32 accumulation.
//
// Warp roles (320 threads): warp 0 = TMA/bulk-copy producer, warp 1 = MMA
// issuer + TMEM owner, warps 2..9 = compute (CUDA-core phases, TMEM
// epilogues, DSMEM exchanges).  Every global byte the CTA consumes streams
// through one 6-stage, 16 KB/stage mbarrier ring in a fixed item order that
// producer and consumers derive identically.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "decode_fused.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {

using namespace sm100;

constexpr int kStages = 6;  // even: V panel pairs never straddle the ring wrap
constexpr uint32_t kStageBytes = 16384;
constexpr int kThreads = 320;
constexpr int kComputeThreads = 256;
constexpr uint32_t kBarCompute = 1;  // named barrier id for the compute warps
constexpr int kTailMax = 64;

struct Smem {
  uint32_t ring, phi, plo, pt, stail, part, stats, bars, tslot, total;
  uint32_t uloc, ctxloc, ufin, tfin, red;  // late-phase aliases over [phi, stail)
  int uloc_stride;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_layout(const FusedPlan& p) {
  Smem s{};
  const uint32_t np = p.np;
  s.ring = 0;
  s.phi = s.ring + kStages * kStageBytes;
  s.plo = s.phi + p.kpk * np * 128;
  s.pt = align_up(s.plo + p.kpk * np * 128, 1024);  // 2 buffers x {hi, lo} x 2 panels
  s.stail = s.pt + 8 * np * 128;
  s.part = s.stail + kTailMax * np * 4;
  s.stats = s.part + 8 * np * 4 + 2 * 128 * 4;
  s.bars = align_up(s.stats + 4 * np * 4, 8);
  s.tslot = s.bars + 32 * 8;
  s.total = align_up(s.tslot + 16, 1024);
  // aliases, valid once the U MMAs have completed
  s.uloc_stride = static_cast<int>(align_up(p.s.rank_v, 4));
  s.uloc = s.phi;
  s.ctxloc = s.uloc + np * s.uloc_stride * 4;
  s.ufin = s.ctxloc + p.s.H * p.s.D * 4;
  const int per_kv = p.s.H / p.s.Hkv;
  s.tfin = s.ufin + p.heads_per_cta * per_kv * s.uloc_stride * 4;
  s.red = s.tfin + p.heads_per_cta * per_kv * p.s.D * 4;
  return s;
}

enum Bar : int {
  kFull = 0,                      // [kStages]
  kEmpty = kStages,               // [kStages]
  kPopReady = 2 * kStages,        // P operand assembled (compute -> MMA)
  kSFull,                         // S MMAs complete (MMA -> compute)
  kPFull0, kPFull1,               // p tile buffer ready (compute -> MMA)
  kPEmpty0, kPEmpty1,             // p tile buffer consumed (MMA -> compute)
  kUFull,                         // U MMAs complete
  kTmemFree,                      // compute finished reading TMEM
  kSlices,                        // cluster: all P slices published (count C)
  kStats,                         // cluster: all (m, z) published (count C)
  kUReady,                        // cluster: all U / tail contexts published (count C)
  kDone,                          // cluster: all peers finished reading my smem (count C)
  kNumBars
};

struct Items {
  int rk0, n_rk, tk0, n_tk, lk0, lv0, tv0, rv0, total;
  int tiles, chunk_len, c_first, t_first, p_first;
  int n_heads, nrb;
};

__device__ __forceinline__ Items make_items(const FusedPlan& p, int c, int n_tail) {
  Items it{};
  const int C = p.s.cluster;
  it.p_first = c * p.prow_chunk;
  const int p_last = min(p.s.rank_k, (c + 1) * p.prow_chunk);
  it.n_rk = max(0, p_last - it.p_first);
  const int tail_per = (n_tail + C - 1) / C;
  it.t_first = c * tail_per;
  it.n_tk = max(0, min(n_tail, it.t_first + tail_per) - it.t_first);
  it.c_first = c * p.chunk;
  it.chunk_len = max(0, min(p.s.n_comp, it.c_first + p.chunk) - it.c_first);
  it.tiles = (it.chunk_len + 127) / 128;
  it.n_heads = 0;
  for (int g = c; g < p.s.Hkv; g += C) ++it.n_heads;
  it.nrb = (p.s.rank_v + 31) / 32;
  it.rk0 = 0;
  it.tk0 = it.n_rk;
  it.lk0 = it.tk0 + it.n_tk;
  const int after_lk = it.lk0 + it.tiles * p.kpk;
  it.lv0 = after_lk + (after_lk & 1);  // pad to even: V panel pairs sit in adjacent stages
  it.tv0 = it.lv0 + it.tiles * p.vpanels;
  it.rv0 = it.tv0 + it.n_tk;
  it.total = it.rv0 + it.n_heads * it.nrb;
  return it;
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

__global__ void __launch_bounds__(kThreads, 1)
    fused_decode_kernel(const FusedPlan p, const __grid_constant__ CUtensorMap map_lk,
                        const __grid_constant__ CUtensorMap map_lv, const __grid_constant__ CUtensorMap map_rv,
                        const FusedArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const Smem L = smem_layout(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.s.cluster;
  const int c = static_cast<int>(cluster_rank());
  const int b = blockIdx.x / C;
  const int H = p.s.H, Hkv = p.s.Hkv, D = p.s.D, W = Hkv * D, NP = p.np;
  const int per_kv = H / Hkv;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const Items it = make_items(p, c, n_tail);
  const uint32_t s_cols = static_cast<uint32_t>(p.max_tiles * NP);

  // ---- prologue: zero ring + P operand, barriers, TMEM -------------------------
  {
    uint4* z = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = L.pt / 16;  // ring + P hi/lo
    for (uint32_t i = threadIdx.x; i < n16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars[kFull + s], 1);
      mbar_init(&bars[kEmpty + s], 1);
    }
    for (int i = kPopReady; i <= kTmemFree; ++i) mbar_init(&bars[i], 1);
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
    // ===================== producer =====================
    if (lane == 0) {
      prefetch_tmap(&map_lk);
      prefetch_tmap(&map_lv);
      prefetch_tmap(&map_rv);
      const long wb = static_cast<long>(W) * 2;
      for (int i = 0; i < it.total; ++i) {
        const int s = i % kStages;
        mbar_wait(&bars[kEmpty + s], ((i / kStages) & 1) ^ 1);
        unsigned char* dst = smem + L.ring + s * kStageBytes;
        uint64_t* full = &bars[kFull + s];
        if (i < it.tk0) {  // right_k rows
          const int r = it.p_first + (i - it.rk0);
          mbar_expect_tx(full, static_cast<uint32_t>(wb));
          bulk_load(dst, a.right_k + (static_cast<long>(b) * p.s.rank_k + r) * W, static_cast<uint32_t>(wb), full);
        } else if (i < it.lk0) {  // tail_k rows
          const int t = it.t_first + (i - it.tk0);
          mbar_expect_tx(full, static_cast<uint32_t>(wb));
          bulk_load(dst, a.tail_k + (static_cast<long>(b) * p.s.tail_cap + t) * W, static_cast<uint32_t>(wb), full);
        } else if (i < it.lv0 || i < it.tv0) {  // left_k / left_v panels (or the even-pad slot)
          const bool is_v = i >= it.lv0;
          const int rel = is_v ? i - it.lv0 : i - it.lk0;
          const int per_tile = is_v ? p.vpanels : p.kpk;
          if (!is_v && rel >= it.tiles * p.kpk) {  // pad slot
            mbar_arrive(full);
            continue;
          }
          const int tile = rel / per_tile, panel = rel % per_tile;
          const int rank = is_v ? p.s.rank_v : p.s.rank_k;
          if (panel * 64 >= rank) {  // V pad panel: rows >= rank_v of U are never read
            mbar_arrive(full);
            continue;
          }
          const int row0 = tile * 128;
          const int nbox = min(4, (it.chunk_len - row0 + 31) / 32);
          mbar_expect_tx(full, static_cast<uint32_t>(nbox) * 4096u);
          const int grow = b * p.s.n_comp + it.c_first + row0;
          for (int k = 0; k < nbox; ++k)
            tma_load_2d(dst + k * 4096, is_v ? &map_lv : &map_lk, panel * 64, grow + 32 * k, full);
        } else if (i < it.rv0) {  // tail_v rows
          const int t = it.t_first + (i - it.tv0);
          mbar_expect_tx(full, static_cast<uint32_t>(wb));
          bulk_load(dst, a.tail_v + (static_cast<long>(b) * p.s.tail_cap + t) * W, static_cast<uint32_t>(wb), full);
        } else {  // right_v boxes [32 rows x D] for my kv heads
          const int rel = i - it.rv0;
          const int hg = c + (rel / it.nrb) * C, rb = rel % it.nrb;
          mbar_expect_tx(full, static_cast<uint32_t>(D) * 64u);
          tma_load_2d(dst, &map_rv, hg * D, b * p.s.rank_v + rb * 32, full);
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
      for (int t = 0; t < it.tiles; ++t) {
        for (int kp = 0; kp < p.kpk; ++kp) {
          const int i = it.lk0 + t * p.kpk + kp, s = i % kStages;
          mbar_wait(&bars[kFull + s], (i / kStages) & 1);
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
      if (it.lv0 > it.lk0 + it.tiles * p.kpk) {  // release the even-pad slot
        const int i = it.lv0 - 1, s = i % kStages;
        mbar_wait(&bars[kFull + s], (i / kStages) & 1);
        mbar_arrive(&bars[kEmpty + s]);
      }
      mma_commit(&bars[kSFull]);
      for (int t = 0; t < it.tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(&bars[kPFull0 + buf], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t pth = pt + buf * 4 * NP * 128, ptl = pth + 2 * NP * 128;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const int i0 = it.lv0 + t * p.vpanels + 2 * mt;
          const int s0 = i0 % kStages, s1 = (i0 + 1) % kStages;
          mbar_wait(&bars[kFull + s0], (i0 / kStages) & 1);
          mbar_wait(&bars[kFull + s1], ((i0 + 1) / kStages) & 1);
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
    const int cw = warp - 2;                 // 0..7
    const int tid = threadIdx.x - 64;        // 0..255
    const float inv_sqrt_d = rsqrtf(static_cast<float>(D));
    float* q = reinterpret_cast<float*>(smem + L.pt);  // alias: dead before p tiles are written
    float* stail = reinterpret_cast<float*>(smem + L.stail);
    float* part = reinterpret_cast<float*>(smem + L.part);
    float* stats = reinterpret_cast<float*>(smem + L.stats);
    float* m_loc = stats;
    float* z_loc = stats + NP;
    float* m_g = stats + 2 * NP;
    float* z_g = stats + 3 * NP;
    const int dl = D / 32;  // columns per lane within one kv-head slice (D in {64, 128})

    for (int i = tid; i < H * D; i += kComputeThreads) q[i] = a.q[static_cast<long>(b) * H * D + i];
    named_bar(kBarCompute, kComputeThreads);

    // Per-row dot products against q: row = [W] bf16 in a ring stage.
    // Writes out(h) for every query head h (lane 0 of the owning warp).
    auto row_dots = [&](const __nv_bfloat16* row, auto&& emit) {
      for (int g = cw; g < Hkv; g += 8) {
        float v[4];
        const __nv_bfloat16* src = row + g * D + lane * dl;
        if (dl == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(src);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
          const float2 f0 = __bfloat1622float2(h2[0]), f1 = __bfloat1622float2(h2[1]);
          v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
        } else {
          const __nv_bfloat162 raw = *reinterpret_cast<const __nv_bfloat162*>(src);
          const float2 f0 = __bfloat1622float2(raw);
          v[0] = f0.x; v[1] = f0.y; v[2] = 0.f; v[3] = 0.f;
        }
        for (int hh = 0; hh < per_kv; ++hh) {
          const int h = g * per_kv + hh;
          const float* qh = q + h * D + lane * dl;
          float acc = 0.f;
          for (int e = 0; e < dl; ++e) acc = fmaf(v[e], qh[e], acc);
          acc = warp_sum(acc);
          if (lane == 0) emit(h, acc * inv_sqrt_d);
        }
      }
    };
    auto consume = [&](int i) {
      mbar_wait(&bars[kFull + i % kStages], (i / kStages) & 1);
      return reinterpret_cast<const __nv_bfloat16*>(smem + L.ring + (i % kStages) * kStageBytes);
    };
    auto release = [&](int i) {
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) mbar_arrive(&bars[kEmpty + i % kStages]);
    };

    // ---- phase P: my slice of P = right_k q / sqrt(D), bf16 hi/lo, swizzled B operand
    unsigned char* phi = smem + L.phi;
    unsigned char* plo = smem + L.plo;
    for (int j = 0; j < it.n_rk; ++j) {
      const int i = it.rk0 + j, r = it.p_first + j;
      const __nv_bfloat16* row = consume(i);
      row_dots(row, [&](int h, float val) {
        __nv_bfloat16 hi, lo;
        split_bf16(val, hi, lo);
        const uint32_t off = (r >> 6) * NP * 128 + sw128_off(h, r & 63);
        *reinterpret_cast<__nv_bfloat16*>(phi + off) = hi;
        *reinterpret_cast<__nv_bfloat16*>(plo + off) = lo;
      });
      release(i);
    }
    // ---- tail K scores
    for (int j = 0; j < it.n_tk; ++j) {
      const int i = it.tk0 + j;
      const __nv_bfloat16* row = consume(i);
      row_dots(row, [&](int h, float val) { stail[j * NP + h] = val; });
      release(i);
    }
    // ---- publish my P rows; assemble the full P operand from the peers
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kSlices], static_cast<uint32_t>(tid));
    mbar_wait_cluster(&bars[kSlices], 0);
    for (int peer = 0; peer < C; ++peer) {
      if (peer == c) continue;
      const int r0 = peer * p.prow_chunk, r1 = min(p.s.rank_k, r0 + p.prow_chunk);
      const int n_oct = max(0, (r1 - r0 + 7) / 8);
      for (int w = tid; w < n_oct * NP * 2; w += kComputeThreads) {
        const int which = w / (n_oct * NP), rem = w % (n_oct * NP);
        const int oct = r0 / 8 + rem / NP, h = rem % NP;
        const uint32_t off = (oct >> 3) * NP * 128 + sw128_off(h, (oct & 7) * 8);
        unsigned char* base = which ? plo : phi;
        *reinterpret_cast<uint4*>(base + off) = ld_dsmem_v4(base + off, static_cast<uint32_t>(peer));
      }
    }
    fence_proxy_async();
    named_bar(kBarCompute, kComputeThreads);
    if (tid == 0) mbar_arrive(&bars[kPopReady]);

    // ---- softmax statistics over my tokens, then cluster-wide
    const int qd = warp & 3, hf = cw >> 2;  // TMEM lane quadrant, head half
    const int hcols = NP / 2, hbase = hf * hcols;
    mbar_wait(&bars[kSFull], 0);
    tc_fence_after();
    auto tmem_row = [&](uint32_t col) { return tmem + (static_cast<uint32_t>(qd * 32) << 16) + col; };
    for (int pass = 0; pass < 2; ++pass) {
      // pass 0: max, pass 1: sum exp(s - m_loc)
      for (int h0 = 0; h0 < hcols; h0 += 8) {
        float acc[8];
        for (int e = 0; e < 8; ++e) acc[e] = pass == 0 ? -INFINITY : 0.f;
        for (int t = 0; t < it.tiles; ++t) {
          float v[8];
          tmem_ld8(tmem_row(static_cast<uint32_t>(t * NP + hbase + h0)), v);
          const bool valid = t * 128 + qd * 32 + lane < it.chunk_len;
          for (int e = 0; e < 8; ++e) {
            const int h = hbase + h0 + e;
            if (!valid || h >= H) continue;
            acc[e] = pass == 0 ? fmaxf(acc[e], v[e]) : acc[e] + expf(v[e] - m_loc[h]);
          }
        }
        for (int e = 0; e < 8; ++e) {
          const float r = pass == 0 ? warp_max(acc[e]) : warp_sum(acc[e]);
          if (lane == 0) part[(cw) * NP + hbase + h0 + e] = r;  // cw in [4hf, 4hf+3]: one per quadrant
        }
      }
      named_bar(kBarCompute, kComputeThreads);
      if (tid < H) {
        const int h = tid, hb = (h / hcols) * 4;
        float r = pass == 0 ? -INFINITY : 0.f;
        for (int w = 0; w < 4; ++w) r = pass == 0 ? fmaxf(r, part[(hb + w) * NP + h]) : r + part[(hb + w) * NP + h];
        for (int j = 0; j < it.n_tk; ++j)
          r = pass == 0 ? fmaxf(r, stail[j * NP + h]) : r + expf(stail[j * NP + h] - m_loc[h]);
        if (pass == 0) m_loc[h] = r; else z_loc[h] = r;
      }
      named_bar(kBarCompute, kComputeThreads);
    }
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kStats], static_cast<uint32_t>(tid));
    mbar_wait_cluster(&bars[kStats], 0);
    if (tid < H) {
      const int h = tid;
      float mg = -INFINITY;
      for (int peer = 0; peer < C; ++peer) mg = fmaxf(mg, ld_dsmem_f32(&m_loc[h], static_cast<uint32_t>(peer)));
      float zg = 0.f;
      for (int peer = 0; peer < C; ++peer) {
        const float mp = ld_dsmem_f32(&m_loc[h], static_cast<uint32_t>(peer));
        const float zp = ld_dsmem_f32(&z_loc[h], static_cast<uint32_t>(peer));
        if (zp > 0.f) zg += zp * expf(mp - mg);
      }
      m_g[h] = mg;
      z_g[h] = zg;
    }
    named_bar(kBarCompute, kComputeThreads);

    // ---- p tiles (bf16 hi/lo B operand, K-major over tokens) + importance EMA
    float* ha_half = part + 8 * NP;  // [2][128]
    const float inv_h = 1.0f / static_cast<float>(H);
    for (int t = 0; t < it.tiles; ++t) {
      const int buf = t & 1;
      if (t >= 2) mbar_wait(&bars[kPEmpty0 + buf], ((t - 2) >> 1) & 1);
      unsigned char* pth = smem + L.pt + buf * 4 * NP * 128;
      unsigned char* ptl = pth + 2 * NP * 128;
      const int row = qd * 32 + lane;  // token within the tile
      const int tok = t * 128 + row;
      const bool valid = tok < it.chunk_len;
      float hsum = 0.f;
      for (int h0 = 0; h0 < hcols; h0 += 8) {
        float v[8];
        tmem_ld8(tmem_row(static_cast<uint32_t>(t * NP + hbase + h0)), v);
        for (int e = 0; e < 8; ++e) {
          const int h = hbase + h0 + e;
          float pv = 0.f;
          if (valid && h < H) {
            pv = expf(v[e] - m_g[h]);
            hsum += pv / z_g[h];
          }
          __nv_bfloat16 hi, lo;
          split_bf16(pv, hi, lo);
          const uint32_t off = (row >> 6) * NP * 128 + sw128_off(h, row & 63);
          *reinterpret_cast<__nv_bfloat16*>(pth + off) = hi;
          *reinterpret_cast<__nv_bfloat16*>(ptl + off) = lo;
        }
      }
      ha_half[hf * 128 + row] = hsum;
      fence_proxy_async();
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) mbar_arrive(&bars[kPFull0 + buf]);
      if (tid < 128) {
        const int tk = t * 128 + tid;
        if (tk < it.chunk_len) {
          const float ha = (ha_half[tid] + ha_half[128 + tid]) * inv_h;
          const long gi = it.c_first + tk;
          if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + p.s.tail_cap) + gi] = ha;
          if (a.importance) {
            double* imp = a.importance + static_cast<long>(b) * a.imp_stride + gi;
            *imp = __dadd_rn(__dmul_rn(a.ema_decay, *imp), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
          }
        }
      }
      named_bar(kBarCompute, kComputeThreads);
    }
    // tail tokens: p in place of the scores, head average, EMA
    for (int w = tid; w < it.n_tk * H; w += kComputeThreads) {
      const int j = w / H, h = w % H;
      stail[j * NP + h] = expf(stail[j * NP + h] - m_g[h]);
    }
    named_bar(kBarCompute, kComputeThreads);
    for (int j = tid; j < it.n_tk; j += kComputeThreads) {
      float hs = 0.f;
      for (int h = 0; h < H; ++h) hs += stail[j * NP + h] / z_g[h];
      const float ha = hs * inv_h;
      const long gi = p.s.n_comp + it.t_first + j;
      if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + p.s.tail_cap) + gi] = ha;
      if (a.importance) {
        double* imp = a.importance + static_cast<long>(b) * a.imp_stride + gi;
        *imp = __dadd_rn(__dmul_rn(a.ema_decay, *imp), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
      }
    }

    // ---- tail V: c[h, :] += p[t, h] * tail_v[t, g-slice]  (registers until U completes)
    float cacc[8][4];
    for (int x = 0; x < 8; ++x)
      for (int e = 0; e < 4; ++e) cacc[x][e] = 0.f;
    for (int j = 0; j < it.n_tk; ++j) {
      const int i = it.tv0 + j;
      const __nv_bfloat16* row = consume(i);
      int x = 0;
      for (int g = cw; g < Hkv; g += 8) {
        const __nv_bfloat16* src = row + g * D + lane * dl;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (dl == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(src);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
          const float2 f0 = __bfloat1622float2(h2[0]), f1 = __bfloat1622float2(h2[1]);
          v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
        } else {
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(src));
          v[0] = f0.x; v[1] = f0.y;
        }
        for (int hh = 0; hh < per_kv && x < 8; ++hh, ++x) {
          const float pw = stail[j * NP + g * per_kv + hh];
          for (int e = 0; e < 4; ++e) cacc[x][e] = fmaf(pw, v[e], cacc[x][e]);
        }
      }
      release(i);
    }

    // ---- U readback (TMEM -> U_loc[h][r]) and tail-context publish
    mbar_wait(&bars[kUFull], 0);
    tc_fence_after();
    float* uloc = reinterpret_cast<float*>(smem + L.uloc);
    float* ctxloc = reinterpret_cast<float*>(smem + L.ctxloc);
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int r = mt * 128 + qd * 32 + lane;
      for (int h0 = 0; h0 < hcols; h0 += 8) {
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (it.tiles > 0) tmem_ld8(tmem_row(s_cols + static_cast<uint32_t>(mt * NP + hbase + h0)), v);
        for (int e = 0; e < 8; ++e) {
          const int h = hbase + h0 + e;
          if (h < H && r < p.s.rank_v) uloc[h * L.uloc_stride + r] = v[e];
        }
      }
    }
    {
      int x = 0;
      for (int g = cw; g < Hkv; g += 8)
        for (int hh = 0; hh < per_kv && x < 8; ++hh, ++x)
          for (int e = 0; e < dl; ++e) ctxloc[(g * per_kv + hh) * D + lane * dl + e] = cacc[x][e];
    }
    tc_fence_before();
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid == 0) mbar_arrive(&bars[kTmemFree]);
    if (tid < C) mbar_arrive_cluster(&bars[kUReady], static_cast<uint32_t>(tid));
    mbar_wait_cluster(&bars[kUReady], 0);

    // ---- gather U rows / tail contexts of my output heads from the cluster
    float* ufin = reinterpret_cast<float*>(smem + L.ufin);
    float* tfin = reinterpret_cast<float*>(smem + L.tfin);
    float* red = reinterpret_cast<float*>(smem + L.red);
    const int my_q = it.n_heads * per_kv;
    const int r4 = L.uloc_stride / 4;
    for (int w = tid; w < my_q * r4; w += kComputeThreads) {
      const int hl = w / r4, r = (w % r4) * 4;
      const int h = (c + (hl / per_kv) * C) * per_kv + hl % per_kv;
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int peer = 0; peer < C; ++peer) {
        const uint4 u = ld_dsmem_v4(&uloc[h * L.uloc_stride + r], static_cast<uint32_t>(peer));
        s4.x += __uint_as_float(u.x); s4.y += __uint_as_float(u.y);
        s4.z += __uint_as_float(u.z); s4.w += __uint_as_float(u.w);
      }
      *reinterpret_cast<float4*>(&ufin[hl * L.uloc_stride + r]) = s4;
    }
    for (int w = tid; w < my_q * (D / 4); w += kComputeThreads) {
      const int hl = w / (D / 4), d = (w % (D / 4)) * 4;
      const int h = (c + (hl / per_kv) * C) * per_kv + hl % per_kv;
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int peer = 0; peer < C; ++peer) {
        const uint4 u = ld_dsmem_v4(&ctxloc[h * D + d], static_cast<uint32_t>(peer));
        s4.x += __uint_as_float(u.x); s4.y += __uint_as_float(u.y);
        s4.z += __uint_as_float(u.z); s4.w += __uint_as_float(u.w);
      }
      *reinterpret_cast<float4*>(&tfin[hl * D + d]) = s4;
    }
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kDone], static_cast<uint32_t>(tid));

    // ---- output: out[h, :] = (U[h,:] . right_v[:, g-slice] + c[h, :]) / z_h
    // Thread owns 8 columns (16 B) of one row parity; warp cw covers rows 2cw, 2cw+1 (+16k).
    const int col8 = (lane & 15) * 8, rpar = lane >> 4;
    const int rows_per_box = 32;
    for (int hl0 = 0; hl0 < it.n_heads; ++hl0) {
      const int g = c + hl0 * C;
      float oacc[4][8];
      for (int x = 0; x < 4; ++x)
        for (int e = 0; e < 8; ++e) oacc[x][e] = 0.f;
      for (int rb = 0; rb < it.nrb; ++rb) {
        const int i = it.rv0 + hl0 * it.nrb + rb;
        const __nv_bfloat16* box = consume(i);
        if (col8 < D) {
          for (int k = 0; k < rows_per_box / 16; ++k) {
            const int rr = 16 * k + 2 * cw + rpar;
            const int r = rb * 32 + rr;
            if (r < p.s.rank_v) {
              const uint4 raw = *reinterpret_cast<const uint4*>(box + rr * D + col8);
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
              float v[8];
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h2[e]);
                v[2 * e] = f.x;
                v[2 * e + 1] = f.y;
              }
              for (int hh = 0; hh < per_kv && hh < 4; ++hh) {
                const float u = ufin[(hl0 * per_kv + hh) * L.uloc_stride + r];
                for (int e = 0; e < 8; ++e) oacc[hh][e] = fmaf(u, v[e], oacc[hh][e]);
              }
            }
          }
        }
        release(i);
      }
      // reduce the 16 (warp, row-parity) partials per column
      if (col8 < D)
        for (int hh = 0; hh < per_kv && hh < 4; ++hh)
          for (int e = 0; e < 8; ++e) red[((cw * 2 + rpar) * per_kv + hh) * D + col8 + e] = oacc[hh][e];
      named_bar(kBarCompute, kComputeThreads);
      for (int w = tid; w < per_kv * D; w += kComputeThreads) {
        const int hh = w / D, col = w % D;
        const int h = g * per_kv + hh;
        float sacc = tfin[(hl0 * per_kv + hh) * D + col];
        for (int k = 0; k < 16; ++k) sacc += red[(k * per_kv + hh) * D + col];
        const float o = sacc / z_g[h];
        const long oi = static_cast<long>(b) * H * D + static_cast<long>(h) * D + col;
        if (a.ctx_bf16)
          reinterpret_cast<__nv_bfloat16*>(a.ctx_out)[oi] = __float2bfloat16_rn(o);
        else
          reinterpret_cast<float*>(a.ctx_out)[oi] = o;
      }
      named_bar(kBarCompute, kComputeThreads);
    }
    // peers may still be reading my U_loc / contexts
    mbar_wait_cluster(&bars[kDone], 0);
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
  if (s.D != 128 && s.D != 64) return bad("fused path needs head_dim 64 or 128");
  if (s.H > 128) return bad("fused path supports up to 128 query heads");
  if (s.H / s.Hkv > 4) return bad("fused path supports up to 4 query heads per kv head");
  const int W = s.Hkv * s.D;
  if (W * 2 > static_cast<int>(kStageBytes)) return bad("cache width exceeds one ring stage");
  if (s.rank_k < 1 || s.rank_v < 1) return bad("fused path needs low-rank K and V");
  if (s.ld_left % 8 != 0 || s.ld_left < std::max(s.rank_k, s.rank_v)) return bad("left-factor stride must be a multiple of 8");
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
  const int prow = (s.rank_k + s.cluster - 1) / s.cluster;
  p.prow_chunk = (prow + 7) / 8 * 8;
  p.heads_per_cta = (s.Hkv + s.cluster - 1) / s.cluster;
  const int cols = p.max_tiles * p.np + p.mtiles * p.np;
  if (cols > 512) return bad("TMEM budget exceeded (raise the cluster size)");
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  const Smem L = smem_layout(p);
  const uint32_t late = L.red + 16 * (s.H / s.Hkv) * s.D * 4;
  if (late > L.stail) return bad("late-phase buffers do not fit the operand region");
  p.smem_bytes = L.total;
  if (p.smem_bytes > 227 * 1024) return bad("shared-memory budget exceeded");
  p.ok = true;
  p.why = "";
  return p;
}

void encode_fused_maps(const FusedShape& s, const void* left_k, const void* left_v, const void* right_v,
                       CUtensorMap* maps) {
  const uint64_t rows = static_cast<uint64_t>(s.batch) * s.n_comp;
  encode_2d(&maps[0], left_k, s.rank_k, rows, static_cast<uint64_t>(s.ld_left) * 2, 64, 32,
            CU_TENSOR_MAP_SWIZZLE_128B);
  encode_2d(&maps[1], left_v, s.rank_v, rows, static_cast<uint64_t>(s.ld_left) * 2, 64, 32,
            CU_TENSOR_MAP_SWIZZLE_128B);
  const uint64_t W = static_cast<uint64_t>(s.Hkv) * s.D;
  encode_2d(&maps[2], right_v, W, static_cast<uint64_t>(s.batch) * s.rank_v, W * 2, s.D, 32,
            CU_TENSOR_MAP_SWIZZLE_NONE);
}

void launch_fused(const FusedPlan& p, const CUtensorMap* maps, const FusedArgs& a, cudaStream_t st) {
  require(p.ok, KVP_ERR_PARAMETER, p.why);
  static size_t attr_bytes = 0;
  if (attr_bytes < p.smem_bytes) {
    KVP_CUDA(cudaFuncSetAttribute(fused_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(p.smem_bytes)));
    attr_bytes = p.smem_bytes;
  }
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
  KVP_CUDA(cudaLaunchKernelEx(&cfg, fused_decode_kernel, p, maps[0], maps[1], maps[2], a));
  KVP_LAUNCHED();
}

}  // namespace kvp

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
    FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, d->ld_left,
                 d->tail_cap, d->batch, d->cluster > 0 ? d->cluster : 8};
    const FusedPlan p = plan_fused(s);
    require(p.ok, KVP_ERR_PARAMETER, (std::string("decode_fused: ") + p.why).c_str());
    CUtensorMap maps[3];
    encode_fused_maps(s, d->left_k, d->left_v, d->right_v, maps);
    FusedArgs a{};
    a.right_k = static_cast<const __nv_bfloat16*>(d->right_k);
    a.right_v = static_cast<const __nv_bfloat16*>(d->right_v);
    a.tail_k = static_cast<const __nv_bfloat16*>(d->tail_k);
    a.tail_v = static_cast<const __nv_bfloat16*>(d->tail_v);
    a.n_tail_dev = d->n_tail_dev;
    a.n_tail = d->n_tail;
    a.q = d->queries;
    a.rank_v_tok = nullptr;
    a.importance = d->importance;
    a.imp_stride = d->imp_stride;
    const double decay = std::pow(d->alpha, 1.0);  // alpha^T_q, importance.cpp:58
    a.ema_decay = decay;
    a.ema_blend = 1.0 - decay;
    a.head_avg = d->head_avg;
    a.ctx_out = d->context;
    a.ctx_bf16 = d->context_bf16;
    launch_fused(p, maps, a, as_stream(stream));
  });
}
