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

constexpr int kMaxStages = 6;
constexpr uint32_t kStageBytes = 16384;  // one packed 128 x 64 bf16 operand panel
constexpr uint32_t kRing = 32768;        // ring stage: a panel pair, one 32 KB bulk copy (measured on
                                         // B200: a warp-specialised ring's per-SM stream rate grows with
                                         // the copy size, ~40 GB/s at 16 KB vs ~70 GB/s at 32 KB)
constexpr int kThreads = 576;         // warp 0 TMA, warp 1 MMA, warps 2..17 compute
constexpr int kComputeThreads = 512;
constexpr int kComputeWarps = 16;
constexpr uint32_t kBarCompute = 1;  // named barrier id for the compute warps
constexpr int kTailMax = 96;
#ifndef KVP_STREAM_THREADS
#define KVP_STREAM_THREADS 256
#endif
constexpr int kStreamThreads = KVP_STREAM_THREADS;  // qdots / vsum blocks
constexpr int kStreamWarps = kStreamThreads / 32;
// 4 resident blocks per SM (<= 64 registers): 512 (slice, instance) blocks fit one wave of 592 slots
#ifndef KVP_STREAM_MINB
#define KVP_STREAM_MINB 4
#endif
constexpr int kStreamMinBlocks = KVP_STREAM_MINB;
#ifndef QD_UNROLL
#define QD_UNROLL 1
#endif

struct Smem {
  uint32_t ring, phi, plo, pt, pt2, stail, part, stats, imps, vts, bars, tslot, total;
  uint32_t uloc;  // late-phase alias over [phi, ...), valid once the U MMAs completed
  int uloc_stride;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_layout(const FusedPlan& p) {
  Smem s{};
  const uint32_t np = p.np;
  s.ring = 0;
  s.phi = s.ring + p.stages * kRing;
  s.plo = s.phi + p.kpk * np * 128;
  // p tiles: 2 buffers x {hi, lo} x 2 panels (x 2 for the second value tier).  For large
  // ranks (pt_alias) they reuse the P image's bytes: the image is dead once the S MMAs
  // completed, which precedes the first p tile.
  const uint32_t pimg_bytes = 2 * p.kpk * np * 128, pt_bytes = 8 * np * 128 * (p.nb2 > 0 ? 2 : 1);
  s.pt = p.pt_alias ? s.phi : align_up(s.phi + pimg_bytes, 1024);
  s.pt2 = s.pt + 8 * np * 128;  // two-tier values: the second tier's p tiles
  const uint32_t pt_end = (s.pt + pt_bytes) > (s.phi + pimg_bytes) ? s.pt + pt_bytes : s.phi + pimg_bytes;
  s.uloc_stride = static_cast<int>(align_up(p.s.rank_v, 4));
  s.uloc = s.phi;
  const uint32_t uloc_end = s.uloc + np * s.uloc_stride * 4;
  s.stail = align_up(pt_end > uloc_end ? pt_end : uloc_end, 16);
  s.part = s.stail + p.tail_max * np * 4;
  // part: per-warp softmax partials, then (split) every peer's (m, z), then the EMA's head sums
  const uint32_t part_bytes = 2 * kComputeWarps * np * 4 + 4 * 128 * 4;
  const uint32_t peer_bytes = p.split ? static_cast<uint32_t>(p.s.cluster) * 2 * np * 4 : 0;
  s.stats = s.part + (part_bytes > peer_bytes ? part_bytes : peer_bytes);
  s.imps = align_up(s.stats + (5 + 8) * np * 4, 16);
  s.vts = s.imps + (p.chunk + p.tail_max) * 8;  // two-tier values: the chunk's tier flags (prefetched)
  s.bars = align_up(s.vts + (p.nb2 > 0 ? p.chunk : 0), 8);
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
  int n_tk, tiles, tile0, chunk_len, c_first, t_first;
};

__device__ __forceinline__ Items make_items(const FusedPlan& p, int c, int n_tail) {
  Items it{};
  const int C = p.s.cluster;
  const int tail_per = (n_tail + C - 1) / C;
  it.t_first = c * tail_per;
  it.n_tk = max(0, min(n_tail, it.t_first + tail_per) - it.t_first);
  it.tile0 = c * p.max_tiles;
  it.tiles = max(0, min(p.ntiles, it.tile0 + p.max_tiles) - it.tile0);
  it.c_first = it.tile0 * 128;
  it.chunk_len = max(0, min(p.s.n_comp - it.c_first, it.tiles * 128));
  // ring items (MMA operands only): left_k panels, even-pad, left_v panels
  it.lk0 = 0;
  it.lv0 = it.tiles * p.kst;                 // left_k: panel pairs, one ring stage each
  it.total = it.lv0 + it.tiles * p.mtiles;   // left_v: 128-rank panel pairs
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

// Operands that carry an fp32 quantity as a bf16 hi/lo pair (P, p) are stacked
// along N when `st` (NP <= 32): one MMA reads the A panel once and the two halves
// of the accumulator are summed at readback (measured: the tensor core's A-operand
// read from smem, ~64 B/cycle, bounds these skinny MMAs, so two MMAs per K step
// halved the stream rate).  Otherwise two MMAs accumulate into one tile.
// Byte offset of (panel, row, k) in an image of n rows x `panels` 64-wide K panels.
__host__ __device__ __forceinline__ uint32_t bimg_off(bool st, int n, int panels, int panel, int row, int k,
                                                      bool lo) {
  if (st) return static_cast<uint32_t>(panel * 2 * n * 128) + sw128_off(row + (lo ? n : 0), k);
  return static_cast<uint32_t>((lo ? panels * n * 128 : 0) + panel * n * 128) + sw128_off(row, k);
}
template <bool ST>
__device__ __forceinline__ void mma_hilo(uint32_t d, uint64_t adesc, uint32_t img, int n, int panels, int panel,
                                         int kb, uint32_t idesc, uint32_t acc) {
  if (ST) {
    mma_bf16(d, adesc, smem_desc(img + panel * 2 * n * 128 + kb, 16, 1024, kSwizzle128B), idesc, acc);
  } else {
    mma_bf16(d, adesc, smem_desc(img + panel * n * 128 + kb, 16, 1024, kSwizzle128B), idesc, acc);
    mma_bf16(d, adesc, smem_desc(img + panels * n * 128 + panel * n * 128 + kb, 16, 1024, kSwizzle128B), idesc, 1);
  }
}
// G consecutive accumulator columns of one TMEM row quadrant (hi + lo halves summed when
// stacked): every tcgen05.ld is issued before a single wait::ld, one TMEM round trip
// instead of one per 4 columns.
template <bool ST, int G>
__device__ __forceinline__ void tld_row_hilo(uint32_t taddr, int n, float (&v)[G]) {
  static_assert(G % 4 == 0, "column group must be a multiple of 4");
  uint32_t r[G / 4][4], w[ST ? G / 4 : 1][4];
#pragma unroll
  for (int i = 0; i < G / 4; ++i) tmem_ld4_nowait(taddr + static_cast<uint32_t>(4 * i), r[i]);
  if (ST) {
#pragma unroll
    for (int i = 0; i < G / 4; ++i) tmem_ld4_nowait(taddr + static_cast<uint32_t>(n + 4 * i), w[ST ? i : 0]);
  }
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < G / 4; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if constexpr (ST)
        v[4 * i + e] = __uint_as_float(r[i][e]) + __uint_as_float(w[i][e]);
      else
        v[4 * i + e] = __uint_as_float(r[i][e]);
    }
}

// ============================================================================
// 1. qdots: one block per (kv head g, instance b).  Rows = right_k (rank_k)
//    then tail_k (n_tail); each lane owns 8 columns of the g-slice, D/8 lanes
//    span one row segment and reduce with shuffles.
// ============================================================================
template <int PER_KV, int D>
__global__ void __launch_bounds__(kStreamThreads, kStreamMinBlocks) qdots_kernel(const FusedPlan p, const FusedArgs a) {
  // A group of LPH = D/8 lanes covers one row segment (D bf16, one kv-head
  // slice); each lane owns one 16-byte chunk and keeps its 8 query values in
  // registers.  A group walks blocks of 8 consecutive rows: 8 independent
  // 16-byte loads in flight per lane, one butterfly transpose-reduction
  // (8 values over LPH lanes in log2(LPH) rounds), and the 8 results land as
  // one 16-byte chunk of the swizzled P operand image (k = 8 consecutive ranks).
  constexpr int LPH = D / 8, GPW = 32 / LPH;  // lanes per row segment, groups per warp
  const int g = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LPH, gl = lane % LPH;
  const int H = p.s.H, W = p.s.Hkv * D;
  griddep_wait();               // q (and the new k, v) come from the projection GEMM
  griddep_launch_dependents();  // core may start its q-independent prologue and left_k stream
  if (p.split && g == 0 && threadIdx.x == 0) a.ws_count[b] = 0u;  // core's per-instance barrier (after its wait)
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const int rk = p.s.rank_k, rows = rk + n_tail;
  const float scale = rsqrtf(static_cast<float>(D));
  float qv[PER_KV][8];
#pragma unroll
  for (int y = 0; y < PER_KV; ++y)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      qv[y][e] = a.q[static_cast<long>(b) * a.q_stride + (g * PER_KV + y) * D + gl * 8 + e] * scale;
  const __nv_bfloat16* rkb = a.right_k + static_cast<long>(b) * rk * W + g * D + gl * 8;
  const __nv_bfloat16* tkb = a.tail_k + static_cast<long>(b) * p.s.tail_cap * W + g * D + gl * 8;
  if (a.append_kv) {  // the new token's k, v (this block's kv-head slice) -> tail row n_tail - 1
    const float* src = a.q + static_cast<long>(b) * a.q_stride + static_cast<long>(H) * D + g * D;
    const long row = static_cast<long>(b) * p.s.tail_cap + (n_tail - 1);
    __nv_bfloat16* tk = const_cast<__nv_bfloat16*>(a.tail_k) + row * W + g * D;
    __nv_bfloat16* tv = const_cast<__nv_bfloat16*>(a.tail_v) + row * W + g * D;
    for (int i = threadIdx.x; i < D; i += kStreamThreads) {
      tk[i] = __float2bfloat16_rn(src[i]);
      tv[i] = __float2bfloat16_rn(src[W + i]);
    }
    if (g == 0 && threadIdx.x == 0 && a.importance)
      a.importance[static_cast<long>(b) * a.imp_stride + p.s.n_comp + n_tail - 1] = 0.0;
    __threadfence_block();
    __syncthreads();
  }
  const int NP = p.np;
  const bool st = p.stack;
  const uint32_t plane = static_cast<uint32_t>(p.kpk) * NP * 128;  // bytes of one (hi or lo) operand
  unsigned char* pimg = a.ws_pimg + static_cast<size_t>(b) * 2 * plane;
  float* tout = a.ws_tail + static_cast<long>(b) * H * p.s.tail_cap;
  // zero padding of the operand image: ranks >= rank_k of my heads; heads >= H (block g == 0)
  for (int i = threadIdx.x; i < PER_KV * (p.kpk * 64 - rk); i += kStreamThreads) {
    const int h = g * PER_KV + i / (p.kpk * 64 - rk), r = rk + i % (p.kpk * 64 - rk);
    *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, false)) = __float2bfloat16_rn(0.f);
    *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, true)) = __float2bfloat16_rn(0.f);
  }
  if (g == 0)
    for (int i = threadIdx.x; i < (NP - H) * p.kpk * 64; i += kStreamThreads) {
      const int h = H + i / (p.kpk * 64), r = i % (p.kpk * 64);
      *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, false)) = __float2bfloat16_rn(0.f);
      *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, true)) = __float2bfloat16_rn(0.f);
    }
  // The appended row is this kernel's own write: the stream loop stops before it
  // (a non-coherent ld.global.nc of data written by the same kernel is undefined) and
  // its logits come from the fp32 source rounded to bf16, exactly the stored row.
  const int rows_ld = a.append_kv ? rows - 1 : rows;
  const int nblk = (rows_ld + 7) / 8;
  const int gid = warp * GPW + grp, ngroups = (kStreamThreads / 32) * GPW;
  constexpr int UNR = QD_UNROLL;  // 8-row blocks in flight per group
  for (int blk0 = gid; blk0 < nblk; blk0 += UNR * ngroups) {
    uint4 rawb[UNR][8];
#pragma unroll
    for (int ub = 0; ub < UNR; ++ub)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // unconditional load of a clamped row (no select right after the load, so
        // all loads stay in flight); rows >= `rows` are discarded at emit
        const int r = min((blk0 + ub * ngroups) * 8 + u, rows_ld - 1);
        rawb[ub][u] = ldg_stream(r < rk ? rkb + static_cast<long>(r) * W : tkb + static_cast<long>(r - rk) * W);
      }
#pragma unroll
    for (int ub = 0; ub < UNR; ++ub) {
    const int blk = blk0 + ub * ngroups;
    if (blk >= nblk) break;
    const int r0 = blk * 8;
    const uint4* raw = rawb[ub];
#pragma unroll
    for (int y = 0; y < PER_KV; ++y) {
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float v[8];
        unpack8(raw[u], v);
        float t = v[0] * qv[y][0];
#pragma unroll
        for (int e = 1; e < 8; ++e) t = fmaf(v[e], qv[y][e], t);
        acc[u] = t;
      }
      // butterfly transpose-reduction of acc[0..7] across the LPH lanes of the group:
      // after the rounds, lane gl holds the full dot of row r0 + (gl % 8).
      int n = 8;
#pragma unroll
      for (int o = LPH / 2; o >= 1; o >>= 1) {
        if (n > 1) {
          const bool upper = (gl & o) != 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= n / 2) break;
            const float send = upper ? acc[i] : acc[i + n / 2];
            const float keep = upper ? acc[i + n / 2] : acc[i];
            acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
          n /= 2;
        } else {
          acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], o);
        }
      }
      // lane gl now owns row r0 + j where j = bit-reversed (gl / (LPH/8)) pattern of the kept halves
      int j = 0;
      {
        int half = 8, lanebit = LPH / 2;
#pragma unroll
        for (int step = 0; step < 3; ++step) {
          half /= 2;
          if (gl & lanebit) j += half;
          lanebit >>= 1;
        }
      }
      const int r = r0 + j;
      const int h = g * PER_KV + y;
      const bool owner = (gl < 8 * (LPH / 8)) && ((gl % (LPH / 8)) == 0);
      if (owner && r < rows_ld) {
        if (r < rk) {
          __nv_bfloat16 hi, lo;
          split_bf16(acc[0], hi, lo);
          *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, false)) = hi;
          *reinterpret_cast<__nv_bfloat16*>(pimg + bimg_off(st, NP, p.kpk, r >> 6, h, r & 63, true)) = lo;
        } else {
          tout[static_cast<long>(h) * p.s.tail_cap + (r - rk)] = acc[0];
        }
      }
    }
    }
  }
  if (a.append_kv && gid == ngroups - 1) {  // the appended row (tail row n_tail - 1), one lane group
    const float* src = a.q + static_cast<long>(b) * a.q_stride + static_cast<long>(H) * D + g * D + gl * 8;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(__float2bfloat16_rn(src[e]));
#pragma unroll
    for (int y = 0; y < PER_KV; ++y) {
      float t = v[0] * qv[y][0];
#pragma unroll
      for (int e = 1; e < 8; ++e) t = fmaf(v[e], qv[y][e], t);
#pragma unroll
      for (int o = LPH / 2; o >= 1; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (gl == 0) tout[static_cast<long>(g * PER_KV + y) * p.s.tail_cap + (n_tail - 1)] = t;
    }
  }
}

// ============================================================================
// 3. vsum: out[h, :] = sum_r U[h, r] right_v[r, g-slice] + sum_t p_tail[h, t] tail_v[t, g-slice]
// ============================================================================
template <int PER_KV, int D>
__global__ void __launch_bounds__(kStreamThreads, kStreamMinBlocks) vsum_kernel(const FusedPlan p, const FusedArgs a) {
  constexpr int LPH = D / 8, RPI = 32 / LPH, NPART = kStreamWarps * RPI;
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
  const __nv_bfloat16* rvb = a.right_v + static_cast<long>(b) * rv * W + g * D + col8;
  const __nv_bfloat16* tvb = a.tail_v + static_cast<long>(b) * p.s.tail_cap * W + g * D + col8;
  constexpr int U = 8;
  const int stride = kStreamWarps * RPI;
  uint4 raw[U];
  auto issue = [&](int r0) {  // clamped, unconditional loads: all stay in flight
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = min(r0 + u * stride, rows - 1);
      raw[u] = ldg_stream(r < rv ? rvb + static_cast<long>(r) * W : tvb + static_cast<long>(r - rv) * W);
    }
  };
  int r0 = warp * RPI + rsub;
  // The value basis and the tail (appended by qdots, which completed before core
  // triggered this launch) do not depend on core: the first batch is in flight
  // while core finishes.  The weights U / p_tail are core's output.
  issue(r0);
  griddep_wait();
  if (p.split) {  // U = sum of the token chunks' partials (each already scaled by its softmax correction)
    const int C = p.s.cluster;
    for (int i = threadIdx.x; i < PER_KV * rows; i += kStreamThreads) {
      const int y = i / rows, r = i % rows, h = g * PER_KV + y;
      float u = 0.f;
      if (r < rv) {
        // the C partial loads are independent: unrolled so they are all in flight at once (a rolled
        // loop serialises C L2 round trips on vsum's critical path)
        const float* up = a.ws_u + (static_cast<long>(b) * C * H + h) * rv + r;
        const long cs = static_cast<long>(H) * rv;
#pragma unroll 8
        for (int cc = 0; cc < C; ++cc) u += __ldcg(up + cc * cs);
      } else
        u = a.ws_tail[(static_cast<long>(b) * H + h) * p.s.tail_cap + (r - rv)];
      wts[y * wstride + r] = u;
    }
  } else {
    for (int i = threadIdx.x; i < PER_KV * rows; i += kStreamThreads) {
      const int y = i / rows, r = i % rows, h = g * PER_KV + y;
      wts[y * wstride + r] = r < rv ? a.ws_u[(static_cast<long>(b) * H + h) * rv + r]
                                    : a.ws_tail[(static_cast<long>(b) * H + h) * p.s.tail_cap + (r - rv)];
    }
  }
  __syncthreads();
  float acc[PER_KV][8];
#pragma unroll
  for (int y = 0; y < PER_KV; ++y)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[y][e] = 0.f;
  for (; r0 < rows; r0 += U * stride) {
    if (r0 != warp * RPI + rsub) issue(r0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * stride;
      float v[8];
      unpack8(raw[u], v);
#pragma unroll
      for (int y = 0; y < PER_KV; ++y) {
        const float w = r < rows ? wts[y * wstride + r] : 0.f;
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
// SPLIT: the instance's token chunks run as independent CTAs (any count, all SMs) that exchange their
// softmax statistics through global memory behind a per-instance arrival counter, and write U partials
// (scaled by their correction factor) for vsum to sum; otherwise one thread-block cluster per instance
// exchanges through DSMEM and reduce-scatters U.
template <int NPT, bool ST, bool SPLIT>  // ST: hi/lo stacked along N (plan.stack)
__global__ void __launch_bounds__(kThreads, 1)
    core_kernel(const FusedPlan p, const FusedArgs a) {
  constexpr int NPW = ST ? 2 * NPT : NPT;      // TMEM columns of one S / U tile
  extern __shared__ __align__(1024) unsigned char smem[];
  const Smem L = smem_layout(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.s.cluster;
  const int c = SPLIT ? static_cast<int>(blockIdx.x % C) : static_cast<int>(cluster_rank());
  const int b = blockIdx.x / C;
  const int H = p.s.H;
  constexpr int NP = NPT;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const Items it = make_items(p, c, n_tail);
  const uint32_t s_cols = static_cast<uint32_t>(p.max_tiles * NPW);
  const int NS = p.stages;

  // ---- prologue: zero ring + P operand, barriers, TMEM -------------------------
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
  if (!SPLIT) cluster_sync();  // every CTA's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tslot;

  // Programmatic dependent launch: everything above and the first ring of left_k
  // stages is independent of qdots; qdots' outputs (P image, tail logits, the
  // appended tail row's zeroed importance) are read only after griddep_wait.
  // Split mode triggers its dependents only once every CTA of its instance arrived at the
  // instance barrier (so vsum's CTAs can never take the SMs a waiting chunk still needs).
  const bool defer_wait = warp == 0 && lane == 0;
  if (!defer_wait) {
    griddep_wait();
    if (!SPLIT) griddep_launch_dependents();
  }
  if (warp == 0) {
    // ===================== producer: left_k / left_v panels =====================
    if (lane == 0) {
      auto load_p = [&] {  // P operand image (bf16 hi/lo, already swizzled by qdots) -> smem in one bulk copy
        griddep_wait();
        if (!SPLIT) griddep_launch_dependents();
        const uint32_t pbytes = 2u * p.kpk * NP * 128;
        mbar_expect_tx(&bars[kPopReady], pbytes);
        bulk_load(smem + L.phi, reinterpret_cast<const unsigned char*>(a.ws_pimg) + static_cast<size_t>(b) * pbytes,
                  pbytes, &bars[kPopReady]);
      };
      bool p_loaded = false;
      for (int i = 0; i < it.total; ++i) {
        if (i == NS) {  // the ring is full: the MMAs that free it need P
          load_p();
          p_loaded = true;
        }
        const int s = i % NS;
        mbar_wait(&bars[kEmpty + s], ((i / NS) & 1) ^ 1);
        unsigned char* dst = smem + L.ring + s * kRing;
        uint64_t* full = &bars[kFull + s];
        const bool is_v = i >= it.lv0;
        const int rel = is_v ? i - it.lv0 : i - it.lk0;
        const int per_tile = is_v ? p.mtiles : p.kst;
        const int tile = rel / per_tile, pair = rel % per_tile;
        if (a.trace && i == it.lv0) a.trace[blockIdx.x * 32ull + 10] = global_ns();
        if (a.trace && i == it.total - 1) a.trace[blockIdx.x * 32ull + 14] = global_ns();  // last stage issued
        // packed panel-major layout: the panels (2 pair, 2 pair + 1) of a tile are contiguous;
        // a missing odd V panel stays unloaded (U rows >= rank_v are never read)
        const long gtile = static_cast<long>(a.inst0 + b) * p.ntiles + it.tile0 + tile;
        const int panels = is_v ? p.vpanels_st : p.kpk;
        const uint32_t bytes = static_cast<uint32_t>(min(2, panels - 2 * pair)) * kStageBytes;
        const unsigned char* src = (is_v ? a.left_v_packed : a.left_k_packed) +
                                   (gtile * panels + 2 * pair) * static_cast<long>(kStageBytes);
        mbar_expect_tx(full, bytes);
        bulk_load(dst, src, bytes, full);
      }
      if (!p_loaded) load_p();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, NPW, false, false);
      const uint32_t idesc_u = idesc_bf16(128, NPW, true, false);
      const uint32_t ring = smem_addr(smem + L.ring);
      const uint32_t phi = smem_addr(smem + L.phi);
      const uint32_t pt = smem_addr(smem + L.pt);
      const uint32_t pt2 = smem_addr(smem + L.pt2);
      mbar_wait(&bars[kPopReady], 0);
      tc_fence_after();
      if (a.trace) a.trace[blockIdx.x * 32ull + 8] = global_ns();
      for (int t = 0; t < it.tiles; ++t) {
        for (int pp = 0; pp < p.kst; ++pp) {
          const int i = it.lk0 + t * p.kst + pp, s = i % NS;
          mbar_wait(&bars[kFull + s], (i / NS) & 1);
          tc_fence_after();
          for (int q = 0; q < 2 && 2 * pp + q < p.kpk; ++q) {
            const int kp = 2 * pp + q;
            for (int kk = 0; kk < 4; ++kk)
              mma_hilo<ST>(tmem + static_cast<uint32_t>(t * NPW),
                           smem_desc(ring + s * kRing + q * kStageBytes + kk * 32, 16, 1024, kSwizzle128B), phi, NP,
                           p.kpk, kp, kk * 32, idesc_s, (kp | kk) != 0);
          }
          mma_commit(&bars[kEmpty + s]);
        }
      }
      mma_commit(&bars[kSFull]);
      if (a.trace) a.trace[blockIdx.x * 32ull + 9] = global_ns();
      for (int t = 0; t < it.tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(&bars[kPFull0 + buf], (t >> 1) & 1);
        tc_fence_after();
        if (a.trace && t < 3) a.trace[blockIdx.x * 32ull + 11 + t] = global_ns();  // p tile t seen by the MMA
        const uint32_t pth = pt + buf * 4 * NP * 128;
        const uint32_t pth2 = pt2 + buf * 4 * NP * 128;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const int i0 = it.lv0 + t * p.mtiles + mt, s0 = i0 % NS;
          mbar_wait(&bars[kFull + s0], (i0 / NS) & 1);
          tc_fence_after();
          const uint32_t d = tmem + s_cols + static_cast<uint32_t>(mt * NPW);
          for (int ks = 0; ks < 8; ++ks)
            mma_hilo<ST>(d, smem_desc(ring + s0 * kRing + ks * 2048, kStageBytes, 1024, kSwizzle128B), pth, NP, 2,
                         ks >> 2, (ks & 3) * 32, idesc_u, (t | ks) != 0);
          if (mt < p.nb2) {  // second value tier: same A tile, its own p image and accumulator
            const uint32_t d2 = tmem + s_cols + static_cast<uint32_t>((p.mtiles + mt) * NPW);
            for (int ks = 0; ks < 8; ++ks)
              mma_hilo<ST>(d2, smem_desc(ring + s0 * kRing + ks * 2048, kStageBytes, 1024, kSwizzle128B), pth2, NP,
                           2, ks >> 2, (ks & 3) * 32, idesc_u, (t | ks) != 0);
          }
          mma_commit(&bars[kEmpty + s0]);
        }
        mma_commit(&bars[kPEmpty0 + buf]);
      }
      if (a.trace) a.trace[blockIdx.x * 32ull + 7] = global_ns();  // last U MMA issued
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
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 0] = global_ns();

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
    // the chunk's value-tier flags (written at the previous step's end): off the p-tile critical path
    unsigned char* vts = smem + L.vts;
    if (p.nb2 > 0) {
      const unsigned char* vt = a.vtier + static_cast<long>(a.inst0 + b) * p.s.n_comp + it.c_first;
      for (int i = tid; i < it.chunk_len; i += kComputeThreads) vts[i] = vt[i];
    }

    // ---- local softmax: max over TMEM-resident S + my tail logits (no exponentials)
    const int qd = warp & 3;                 // TMEM lane quadrant this warp may access
    const int cg = cw >> 2;                  // column group 0..3
    constexpr int gcols = NP / 4;            // multiple of 4 columns
    const int gbase = cg * gcols;
    auto tmem_row = [&](uint32_t col) { return tmem + (static_cast<uint32_t>(qd * 32) << 16) + col; };
    mbar_wait(&bars[kSFull], 0);
    tc_fence_after();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 1] = global_ns();
    float* part_m = part;                         // [16 warps][NP]
    float* part_s = part + kComputeWarps * NP;    // [16 warps][NP]
    {
      float mx[gcols];
#pragma unroll
      for (int e = 0; e < gcols; ++e) mx[e] = -INFINITY;
      for (int t = 0; t < it.tiles; ++t) {
        float v[gcols];
        tld_row_hilo<ST, gcols>(tmem_row(static_cast<uint32_t>(t * NPW + gbase)), NP, v);
        if (t * 128 + qd * 32 + lane < it.chunk_len)
#pragma unroll
          for (int e = 0; e < gcols; ++e) mx[e] = fmaxf(mx[e], v[e]);
      }
#pragma unroll
      for (int e = 0; e < gcols; ++e) {
        const float m = warp_max(mx[e]);
        if (lane == 0) part_m[cw * NP + gbase + e] = m;
      }
    }
    named_bar(kBarCompute, kComputeThreads);
    if (tid < H) {
      const int h = tid, w0 = (h / gcols) * 4;
      float m = -INFINITY;
      for (int w = 0; w < 4; ++w) m = fmaxf(m, part_m[(w0 + w) * NP + h]);
      for (int j = 0; j < it.n_tk; ++j) m = fmaxf(m, stail[j * NP + h]);
      m_loc[h] = m;
    }
    named_bar(kBarCompute, kComputeThreads);
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 2] = global_ns();

    // ---- p tiles with the local max (bf16 hi/lo B operand, K-major over tokens); z from the same pass
    float zp[gcols];
#pragma unroll
    for (int e = 0; e < gcols; ++e) zp[e] = 0.f;
    for (int t = 0; t < it.tiles; ++t) {
      const int buf = t & 1;
      if (t >= 2) mbar_wait(&bars[kPEmpty0 + buf], ((t - 2) >> 1) & 1);
      unsigned char* pth = smem + L.pt + buf * 4 * NP * 128;
      unsigned char* pth2 = smem + L.pt2 + buf * 4 * NP * 128;
      const int row = qd * 32 + lane;  // token within the tile
      const bool valid = t * 128 + row < it.chunk_len;
      // two-tier values: a second-tier token's p goes to the second image only (U rows < rv2)
      const bool tier2 = p.nb2 > 0 && valid && vts[t * 128 + row] != 0;
      float sv[gcols];
      tld_row_hilo<ST, gcols>(tmem_row(static_cast<uint32_t>(t * NPW + gbase)), NP, sv);
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          const float pv = (valid && h < H) ? __expf(sv[c0 + e] - m_loc[h]) : 0.f;
          zp[c0 + e] += pv;
          __nv_bfloat16 hi, lo, zero = __float2bfloat16_rn(0.f);
          split_bf16(pv, hi, lo);
          *reinterpret_cast<__nv_bfloat16*>(pth + bimg_off(ST, NP, 2, row >> 6, h, row & 63, false)) = tier2 ? zero : hi;
          *reinterpret_cast<__nv_bfloat16*>(pth + bimg_off(ST, NP, 2, row >> 6, h, row & 63, true)) = tier2 ? zero : lo;
          if (p.nb2 > 0) {
            *reinterpret_cast<__nv_bfloat16*>(pth2 + bimg_off(ST, NP, 2, row >> 6, h, row & 63, false)) = tier2 ? hi : zero;
            *reinterpret_cast<__nv_bfloat16*>(pth2 + bimg_off(ST, NP, 2, row >> 6, h, row & 63, true)) = tier2 ? lo : zero;
          }
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
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 3] = global_ns();

    // ---- publish (m_loc, z_loc); global statistics while the U MMAs still run
    if constexpr (SPLIT) {
      float* st_me = a.ws_stats + (static_cast<long>(b) * C + c) * 2 * H;
      if (tid < H) {
        st_me[tid] = m_loc[tid];
        st_me[H + tid] = z_loc[tid];
      }
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) {
        // release: the stats the compute warps wrote before the barrier above are visible to any
        // CTA that acquires the counter (the CUTLASS generic-barrier pattern, no full fence)
        if (a.trace) a.trace[blockIdx.x * 32ull + 16] = global_ns();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&a.ws_count[b]) : "memory");
        if (a.trace) a.trace[blockIdx.x * 32ull + 17] = global_ns();
        unsigned seen;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&a.ws_count[b]) : "memory");
          if (seen < static_cast<unsigned>(C)) __nanosleep(32);
        } while (seen < static_cast<unsigned>(C));
        if (a.trace) a.trace[blockIdx.x * 32ull + 18] = global_ns();
        griddep_launch_dependents();
      }
      named_bar(kBarCompute, kComputeThreads);
      // every peer's (m, z) in one round of independent loads -> shared memory (the part buffer is free)
      float* peer_st = part;
      const float* st0 = a.ws_stats + static_cast<long>(b) * C * 2 * H;
      for (int i = tid; i < C * 2 * H; i += kComputeThreads) peer_st[i] = __ldcg(&st0[i]);
      named_bar(kBarCompute, kComputeThreads);
      if (tid < H) {
        const int h = tid;
        float mg = -INFINITY;
        for (int peer = 0; peer < C; ++peer) mg = fmaxf(mg, peer_st[peer * 2 * H + h]);
        float zg = 0.f;
        for (int peer = 0; peer < C; ++peer) {
          const float mp = peer_st[peer * 2 * H + h];
          if (mp != -INFINITY) zg += peer_st[peer * 2 * H + H + h] * __expf(mp - mg);
        }
        const float zi = 1.0f / zg;
        m_g[h] = mg;
        zi_g[h] = zi;
        f_me[h] = (m_loc[h] == -INFINITY ? 0.f : __expf(m_loc[h] - mg)) * zi;
      }
    } else {
    if (tid == 0) fence_acq_rel_cluster();
    named_bar(kBarCompute, kComputeThreads);
    if (tid < C) mbar_arrive_cluster(&bars[kStats], static_cast<uint32_t>(tid));
    mbar_wait_cluster(&bars[kStats], 0);
    if (tid < H) {
      const int h = tid;
      float mp[8], zq[8];
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) {
          mp[peer] = ld_dsmem_f32(&m_loc[h], static_cast<uint32_t>(peer));
          zq[peer] = ld_dsmem_f32(&z_loc[h], static_cast<uint32_t>(peer));
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
          zg += zq[peer] * sc;
        }
      const float zi = 1.0f / zg;
      m_g[h] = mg;
      zi_g[h] = zi;
      f_me[h] = (m_loc[h] == -INFINITY ? 0.f : __expf(m_loc[h] - mg)) * zi;
    }
    }
    named_bar(kBarCompute, kComputeThreads);
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 6] = global_ns();  // cluster statistics in hand

    // ---- head-averaged attention + importance EMA (importance.cpp:33-65); S re-read
    //      from TMEM concurrently with the U MMAs (disjoint TMEM columns)
    float* ha_part = part;  // [4 groups][kMaxTilesEma][128]
    const float inv_h = 1.0f / static_cast<float>(H);
    for (int t = 0; t < it.tiles; ++t) {
      const int row = qd * 32 + lane;
      float hsum = 0.f;
      {
        float v[gcols];
        tld_row_hilo<ST, gcols>(tmem_row(static_cast<uint32_t>(t * NPW + gbase)), NP, v);
#pragma unroll
        for (int e = 0; e < gcols; ++e) {
          const int h = gbase + e;
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
    // tail tokens: normalised p -> workspace (for vsum), head average, EMA
    for (int w = tid; w < it.n_tk * H; w += kComputeThreads) {
      const int j = w % it.n_tk, h = w / it.n_tk;
      a.ws_tail[(static_cast<long>(b) * H + h) * p.s.tail_cap + it.t_first + j] = stail[j * NP + h] * f_me[h];
    }
    for (int j = cw; j < it.n_tk; j += kComputeWarps) {  // one warp per tail token, lanes over heads
      float hs = 0.f;
      for (int h = lane; h < H; h += 32) hs = fmaf(stail[j * NP + h], f_me[h], hs);
      const float ha = warp_sum(hs) * inv_h;
      if (lane == 0) {
        const long gi = p.s.n_comp + it.t_first + j;
        if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + p.s.tail_cap) + gi] = ha;
        if (a.importance)
          a.importance[static_cast<long>(b) * a.imp_stride + gi] =
              __dadd_rn(__dmul_rn(a.ema_decay, imps[p.chunk + j]), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
      }
    }

    // ---- U readback (TMEM -> U_loc[h][r]); publish U_loc to the cluster
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 15] = global_ns();  // EMA + tail work done
    mbar_wait(&bars[kUFull], 0);
    tc_fence_after();
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 4] = global_ns();
    if constexpr (SPLIT) {
      // this chunk's U, scaled by its softmax correction exp(m_c - m_g) / z_g, as a partial for vsum
      float* up = a.ws_u + (static_cast<long>(b) * C + c) * H * p.s.rank_v;
      for (int mt = 0; mt < p.mtiles; ++mt) {
        const int r = mt * 128 + qd * 32 + lane;
        float v[gcols];
#pragma unroll
        for (int e = 0; e < gcols; ++e) v[e] = 0.f;
        if (it.tiles > 0) tld_row_hilo<ST, gcols>(tmem_row(s_cols + static_cast<uint32_t>(mt * NPW + gbase)), NP, v);
        if (it.tiles > 0 && mt < p.nb2) {
          float v2[gcols];
          tld_row_hilo<ST, gcols>(tmem_row(s_cols + static_cast<uint32_t>((p.mtiles + mt) * NPW + gbase)), NP, v2);
          if (r < p.s.rv2)
#pragma unroll
            for (int e = 0; e < gcols; ++e) v[e] += v2[e];
        }
#pragma unroll
        for (int e = 0; e < gcols; ++e) {
          const int h = gbase + e;
          if (h < H && r < p.s.rank_v) up[static_cast<long>(h) * p.s.rank_v + r] = v[e] * f_me[h];
        }
      }
      tc_fence_before();
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) mbar_arrive(&bars[kTmemFree]);
    } else {
      float* uloc = reinterpret_cast<float*>(smem + L.uloc);
      for (int mt = 0; mt < p.mtiles; ++mt) {
        const int r = mt * 128 + qd * 32 + lane;
        float v[gcols];
#pragma unroll
        for (int e = 0; e < gcols; ++e) v[e] = 0.f;
        if (it.tiles > 0) tld_row_hilo<ST, gcols>(tmem_row(s_cols + static_cast<uint32_t>(mt * NPW + gbase)), NP, v);
        if (it.tiles > 0 && mt < p.nb2) {  // second tier contributes to the value-rank prefix only
          float v2[gcols];
          tld_row_hilo<ST, gcols>(tmem_row(s_cols + static_cast<uint32_t>((p.mtiles + mt) * NPW + gbase)), NP, v2);
          if (r < p.s.rv2)
#pragma unroll
            for (int e = 0; e < gcols; ++e) v[e] += v2[e];
        }
#pragma unroll
        for (int e = 0; e < gcols; ++e) {
          const int h = gbase + e;
          if (h < H && r < p.s.rank_v) uloc[h * L.uloc_stride + r] = v[e];
        }
      }
      tc_fence_before();
      if (tid == 0) fence_acq_rel_cluster();
      named_bar(kBarCompute, kComputeThreads);
      if (tid == 0) mbar_arrive(&bars[kTmemFree]);
      if (tid < C) mbar_arrive_cluster(&bars[kUReady], static_cast<uint32_t>(tid));
      mbar_wait_cluster(&bars[kUReady], 0);

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
      mbar_wait_cluster(&bars[kDone], 0);  // peers may still be reading my U_loc / stats
    }
    if (a.trace && tid == 0) a.trace[blockIdx.x * 32ull + 5] = global_ns();
  }
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
  p.split = s.split == 1;
  if (s.cluster < 1 || (!p.split && s.cluster > 8)) return bad("cluster size must be 1..8");
  p.np = (s.H + 15) / 16 * 16;
  p.kpk = (s.rank_k + 63) / 64;
  p.vpanels = ((s.rank_v + 63) / 64 + 1) / 2 * 2;
  p.mtiles = p.vpanels / 2;
  p.kst = (p.kpk + 1) / 2;
  p.ntiles = (s.n_comp + 127) / 128;
  p.vpanels_st = (s.rank_v + 63) / 64;  // stored V panels (the even-pad panel is never stored)
  p.max_tiles = (p.ntiles + s.cluster - 1) / s.cluster;
  p.chunk = p.max_tiles * 128;
  p.tail_max = (s.tail_cap + s.cluster - 1) / s.cluster;
  if (p.tail_max > kTailMax) return bad("too many tail tokens per CTA (raise the cluster size)");
  p.heads_per_cta = (s.H + s.cluster - 1) / s.cluster;
  // hi/lo stacked along N (one MMA per A panel) when the doubled tiles fit TMEM;
  // otherwise two MMAs per K step into one tile (e.g. rank 1024)
  if (s.rv2 < 0 || s.rv2 >= s.rank_v) return bad("tier-2 value rank must be in [0, rank_v)");
  p.nb2 = s.rv2 > 0 ? (s.rv2 + 127) / 128 : 0;
  p.stack = p.np <= 32;
  int cols = (p.max_tiles + p.mtiles + p.nb2) * (p.stack ? 2 * p.np : p.np);
  if (cols > 512 && p.stack) {
    p.stack = false;
    cols = (p.max_tiles + p.mtiles + p.nb2) * p.np;
  }
  if (cols > 512) return bad("TMEM budget exceeded (raise the cluster size)");
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.stages = 2;
  p.pt_alias = false;
  if (smem_layout(p).total > 227 * 1024 && 8u * p.np * 128 * (p.nb2 > 0 ? 2 : 1) <= 2u * p.kpk * p.np * 128)
    p.pt_alias = true;  // large ranks (e.g. C4 2x, rank 1024): p tiles over the dead P image
  if (smem_layout(p).total > 227 * 1024) return bad("shared-memory budget exceeded");
  while (p.stages + 1 <= kMaxStages) {
    FusedPlan q = p;
    q.stages = p.stages + 1;
    if (smem_layout(q).total > 227 * 1024) break;
    p.stages = q.stages;
  }
  p.smem_bytes = smem_layout(p).total;
  const size_t vs = (static_cast<size_t>(per_kv) * ((s.rank_v + s.tail_cap + 3) & ~3) + kStreamWarps * (256 / s.D) * per_kv * s.D) * 4;
  if (vs > 200 * 1024) return bad("vsum weights exceed shared memory");
  p.ok = true;
  p.why = "";
  return p;
}

namespace {
struct WsLayout {
  size_t pimg, tail, u, stats, count, total;
};
WsLayout ws_layout(const FusedShape& s) {
  const size_t np = (s.H + 15) / 16 * 16, kpk = (s.rank_k + 63) / 64, B = s.batch;
  const size_t parts = s.split == 1 ? static_cast<size_t>(s.cluster) : 1;
  WsLayout w{};
  w.pimg = 0;
  w.tail = w.pimg + B * 2 * kpk * np * 128;
  w.u = w.tail + sizeof(float) * B * s.H * s.tail_cap;
  w.stats = w.u + sizeof(float) * B * parts * s.H * s.rank_v;
  w.count = w.stats + (s.split == 1 ? sizeof(float) * B * parts * 2 * s.H : 0);
  w.total = w.count + (s.split == 1 ? sizeof(unsigned) * B : 0);
  return w;
}
}  // namespace

size_t fused_workspace_bytes(const FusedShape& s) { return ws_layout(s).total; }

void bind_workspace(const FusedPlan& p, FusedArgs& a, void* ws) {
  const WsLayout w = ws_layout(p.s);
  unsigned char* base = static_cast<unsigned char*>(ws);
  a.ws_pimg = base + w.pimg;
  a.ws_tail = reinterpret_cast<float*>(base + w.tail);
  a.ws_u = reinterpret_cast<float*>(base + w.u);
  a.ws_stats = p.split ? reinterpret_cast<float*>(base + w.stats) : nullptr;
  a.ws_count = p.split ? reinterpret_cast<unsigned*>(base + w.count) : nullptr;
}

// Programmatic dependent launch of the three decode kernels (each waits with
// griddepcontrol.wait before reading its predecessor's output).  KVP_PDL=0 turns it off.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KVP_PDL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}
int pdl_attr(cudaLaunchAttribute& at) {
  if (!pdl_enabled()) return 0;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  return 1;
}

template <int PER_KV, int D>
void launch_stream_pair(const FusedPlan& p, const FusedArgs& a, cudaStream_t st, bool first) {
  const dim3 grid(static_cast<unsigned>(p.s.Hkv), static_cast<unsigned>(p.s.batch));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kStreamThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = pdl_attr(attr[0]);
  if (first) {
    KVP_CUDA(cudaLaunchKernelEx(&cfg, qdots_kernel<PER_KV, D>, p, a));
    KVP_LAUNCHED();
  } else {
    const size_t smem = (static_cast<size_t>(PER_KV) * ((p.s.rank_v + p.s.tail_cap + 3) & ~3) + kStreamWarps * (256 / D) * PER_KV * D) * 4;
    static size_t smem_attr = 0;
    if (smem_attr < smem) {
      KVP_CUDA(cudaFuncSetAttribute(vsum_kernel<PER_KV, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      smem_attr = smem;
    }
    cfg.dynamicSmemBytes = smem;
    KVP_CUDA(cudaLaunchKernelEx(&cfg, vsum_kernel<PER_KV, D>, p, a));
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

using CoreFn = void (*)(const FusedPlan, const FusedArgs);
template <bool SPLIT>
CoreFn core_for_mode(int np, bool stack) {
  switch (np) {
    case 16: return stack ? core_kernel<16, true, SPLIT> : core_kernel<16, false, SPLIT>;
    case 32: return stack ? core_kernel<32, true, SPLIT> : core_kernel<32, false, SPLIT>;
    case 48: return core_kernel<48, false, SPLIT>;
    default: return core_kernel<64, false, SPLIT>;
  }
}
CoreFn core_for(const FusedPlan& p) { return p.split ? core_for_mode<true>(p.np, p.stack) : core_for_mode<false>(p.np, p.stack); }

void launch_qdots(const FusedPlan& p, const FusedArgs& a, cudaStream_t st) { launch_stream(p, a, st, true); }
void launch_vsum(const FusedPlan& p, const FusedArgs& a, cudaStream_t st) { launch_stream(p, a, st, false); }

int max_active_clusters(const FusedPlan& p);

void launch_core(const FusedPlan& p, const FusedArgs& a, cudaStream_t st, int priority) {
  auto kernel = core_for(p);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.s.batch * p.s.cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (!p.split) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(p.s.cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  if (priority != 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na++].val.priority = priority;
  }
  na += pdl_attr(attr[na]);
  cfg.attrs = attr;
  cfg.numAttrs = static_cast<unsigned>(na);
  KVP_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, a));
  KVP_LAUNCHED();
}

void launch_fused(const FusedPlan& p, const FusedArgs& a, cudaStream_t st) {
  require(p.ok, KVP_ERR_PARAMETER, p.why);
  launch_qdots(p, a, st);
  launch_core(p, a, st, 0);
  launch_vsum(p, a, st);
}

FusedArgs offset_args(const FusedPlan& full, const FusedArgs& a, int b0) {
  FusedArgs o = a;
  const long W = static_cast<long>(full.s.Hkv) * full.s.D, H = full.s.H;
  o.right_k += b0 * full.s.rank_k * W;
  o.right_v += b0 * full.s.rank_v * W;
  o.tail_k += b0 * full.s.tail_cap * W;
  o.tail_v += b0 * full.s.tail_cap * W;
  o.q += b0 * a.q_stride;
  if (o.importance) o.importance += b0 * a.imp_stride;
  if (o.head_avg) o.head_avg += static_cast<long>(b0) * (full.s.n_comp + full.s.tail_cap);
  const long ctx_elem = H * full.s.D;
  o.ctx_out = static_cast<char*>(a.ctx_out) + b0 * ctx_elem * (a.ctx_bf16 ? 2 : 4);
  o.ws_pimg += static_cast<size_t>(b0) * 2 * full.kpk * full.np * 128;
  o.ws_tail += b0 * H * full.s.tail_cap;
  o.ws_u += b0 * H * full.s.rank_v;
  o.inst0 = a.inst0 + b0;
  return o;
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
  auto kernel = core_for(p);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  int n = 0;
  KVP_CUDA(cudaOccupancyMaxActiveClusters(&n, kernel, &cfg));
  return n;
}

}  // namespace kvp

namespace kvp {
namespace {
// Row-major left factor [n][ld] (bf16) -> packed panel-major, pre-swizzled tiles.
__global__ void pack_left_kernel(const __nv_bfloat16* src, long ld, int n, int rank, int ntiles, int panels,
                                 unsigned char* dst) {
  const long total = static_cast<long>(ntiles) * panels * 128 * 64;  // elements per instance
  const int b = blockIdx.y;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i % 64), row = static_cast<int>((i / 64) % 128);
    const long blk = i / (64 * 128);
    const int panel = static_cast<int>(blk % panels), tile = static_cast<int>(blk / panels);
    const int t = tile * 128 + row, r = panel * 64 + k;
    const __nv_bfloat16 v = (t < n && r < rank) ? src[(static_cast<long>(b) * n + t) * ld + r] : __float2bfloat16_rn(0.f);
    unsigned char* out = dst + (static_cast<long>(b) * ntiles * panels + blk) * static_cast<long>(kStageBytes);
    *reinterpret_cast<__nv_bfloat16*>(out + sm100::sw128_off(row, k)) = v;
  }
}
}  // namespace

size_t packed_left_bytes(int batch, int n, int rank) {
  return static_cast<size_t>(batch) * ((n + 127) / 128) * ((rank + 63) / 64) * kStageBytes;
}

void pack_left(const void* src, long ld, int batch, int n, int rank, void* dst, cudaStream_t st) {
  const int ntiles = (n + 127) / 128, panels = (rank + 63) / 64;
  pack_left_kernel<<<dim3(64, batch), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), ld, n, rank, ntiles, panels,
                                                     static_cast<unsigned char*>(dst));
  KVP_LAUNCHED();
}
}  // namespace kvp

extern "C" size_t kvp_packed_left_bytes(int32_t batch, int32_t n, int32_t rank) {
  return kvp::packed_left_bytes(batch, n, rank);
}

extern "C" int kvp_pack_left(const void* src, int64_t ld, int32_t batch, int32_t n, int32_t rank, void* dst,
                             void* stream) {
  return kvp::guarded([&] {
    kvp::require(src && dst && batch > 0 && n > 0 && rank > 0 && ld >= rank, KVP_ERR_PARAMETER,
                 "pack_left: bad arguments");
    kvp::pack_left(src, ld, batch, n, rank, dst, kvp::as_stream(stream));
  });
}

// Debug hooks (not part of the public header).
static unsigned long long* g_trace = nullptr;
extern "C" void kvp_debug_fused_trace(void* dev_buffer) { g_trace = static_cast<unsigned long long*>(dev_buffer); }

namespace {
// Cluster size (CTAs per instance): minimise waves x tiles-per-CTA, where
// waves = ceil(batch / co-resident clusters of that size).  Measured on B200
// for the C2 shape: 6 (1 wave x 3 tiles) beats 4, 5, 7 and 8.
int auto_cluster(kvp::FusedShape s) {
  static std::map<std::tuple<int, int, int, int, int, int, int, int, int>, int> cache;
  const auto key = std::make_tuple(s.H, s.Hkv, s.D, s.n_comp, s.rank_k, s.rank_v, s.tail_cap, s.batch, s.rv2);
  if (auto it = cache.find(key); it != cache.end()) return it->second;
  int best = 0;
  long best_cost = 1L << 40;
  for (int c = 8; c >= 1; --c) {
    s.cluster = c;
    const kvp::FusedPlan p = kvp::plan_fused(s);
    if (!p.ok) continue;
    int active = 1;
    try {
      active = std::max(1, kvp::max_active_clusters(p));
    } catch (...) {
      active = 148 / c;
    }
    const long waves = (s.batch + active - 1) / active;
    const long cost = waves * p.max_tiles;
    if (cost < best_cost) {
      best_cost = cost;
      best = c;
    }
  }
  cache[key] = best > 0 ? best : 8;
  return cache[key];
}
}  // namespace
int kvp::auto_cluster_size(const kvp::FusedShape& s) { return auto_cluster(s); }

// Work split of the core: token chunks over all SMs when every CTA of the batch can be
// co-resident (the per-instance barrier in global memory needs it), else one cluster per
// instance.  Split: chunks per instance = SMs / batch (capped by the tile count), rounded so
// every chunk holds the same number of 128-token tiles.
kvp::FusedShape kvp::resolve_fused_shape(kvp::FusedShape s) {
  if (s.split == 1 || (s.split < 0 && s.cluster <= 0)) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ntiles = (s.n_comp + 127) / 128;
    int C = s.split == 1 && s.cluster > 0 ? s.cluster : std::min(ntiles, sms / std::max(1, s.batch));
    if (C >= 1) {
      const int per = (ntiles + C - 1) / C;
      C = (ntiles + per - 1) / per;
      kvp::FusedShape t = s;
      t.split = 1;
      t.cluster = C;
      const kvp::FusedPlan p = kvp::plan_fused(t);
      if ((p.ok && static_cast<long>(s.batch) * C <= sms) || s.split == 1) return t;
    }
  }
  s.split = 0;
  if (s.cluster <= 0) s.cluster = auto_cluster(s);
  return s;
}
namespace {
kvp::FusedShape shape_of(const kvp_fused_desc* d) {
  kvp::FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, 0,
                    d->tail_cap, d->batch, d->cluster};
  s.rv2 = d->tier2_value_rank;
  s.split = d->cluster > 0 ? 0 : -1;  // an explicit cluster size keeps the cluster path
  return kvp::resolve_fused_shape(s);
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
    FusedArgs a{};
    a.left_k_packed = static_cast<const unsigned char*>(d->left_k);
    a.left_v_packed = static_cast<const unsigned char*>(d->left_v);
    a.right_k = static_cast<const __nv_bfloat16*>(d->right_k);
    a.right_v = static_cast<const __nv_bfloat16*>(d->right_v);
    a.tail_k = static_cast<const __nv_bfloat16*>(d->tail_k);
    a.tail_v = static_cast<const __nv_bfloat16*>(d->tail_v);
    require(d->tier2_value_rank <= 0 || d->value_tier != nullptr, KVP_ERR_PARAMETER,
            "decode_fused: tier2_value_rank needs the per-token value_tier flags");
    a.vtier = d->tier2_value_rank > 0 ? d->value_tier : nullptr;
    a.n_tail_dev = d->n_tail_dev;
    a.n_tail = d->n_tail;
    a.q = d->queries;
    a.q_stride = static_cast<long>(s.H) * s.D;
    a.append_kv = 0;
    a.inst0 = 0;
    a.importance = d->importance;
    a.imp_stride = d->imp_stride;
    const double decay = std::pow(d->alpha, 1.0);  // alpha^T_q, importance.cpp:58
    a.ema_decay = decay;
    a.ema_blend = 1.0 - decay;
    a.head_avg = d->head_avg;
    a.ctx_out = d->context;
    a.ctx_bf16 = d->context_bf16;
    bind_workspace(p, a, ws);
    a.trace = g_trace;
    launch_fused(p, a, st);
  });
}
