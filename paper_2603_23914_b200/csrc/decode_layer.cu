// Compressed-cache decode attention for one layer in ONE launch (bf16
// storage, T_q = 1) — the serving hot path.  Replaces the reference's
// per-(instance, layer) loop decoder.cpp:555-601 (build_retrieval_plan ->
// attend_{materialized,fused} -> head average -> update_importance), whose
// cost is ~100% row rebuilding in store_decompress_row (cache.cpp:63-101).
// Nothing of width W = H_kv*D is rebuilt and every cache byte is read once.
//
// One thread-block cluster of C CTAs per instance; every byte goes TMA ->
// shared memory -> tcgen05 tensor cores (accumulators in TMEM).  right_k /
// right_v / tail_k / tail_v are stored per kv head in the same packed,
// pre-swizzled 128-row tile layout as the left factors (kvp_pack_left applied
// to the head-major [batch*H_kv][rows][D] matrices), so one 32 KB bulk copy
// lands a tile in the operand layout the MMAs read (K-major for the
// projections, MN-major for the value-basis multiply).  The producer also
// prefetches upcoming tiles into L2, so the ring's depth is not bounded by the
// HBM latency.  The 128-row tiles of
// every phase are split evenly over the cluster.  One ring of 32 KB stages
// carries, in this order:
//   A  my right_k tiles, my tail_k tiles:  [P | s_tail] (128 x NQ) = tile (128 x D) . Q^T
//        Q = the scaled queries of every head my tiles touch (bf16 hi/lo, one N operand);
//        P chunks are pushed into every peer's operand image (DSMEM)
//   B  left_k tiles:  S[t, h] = left_k[t, :].P[h, :]      M=128 tokens, N=heads; S stays in TMEM
//        local (m, z) per head (tiles + my tail rows), exchanged once through DSMEM
//   C  left_v tiles:  U^T[r, h] += left_v[t, r] p[t, h]    M=128 ranks, N=heads
//        importance EMA (importance.cpp:33-65) from the head average, fp64, reference op order
//        U partials gathered for my right_v rows, normalised
//   D  my right_v tiles, my tail_v tiles:  ctx^T (D x 16) += tile^T (D x 128 rows) . [U | p]^T
//        accumulated in TMEM per (kind, kv head), added into the head owner's smem with DSMEM
//        atomics; owners write the context.
// Every address is known at launch, so the producer keeps streaming the next
// phase's bytes while the consumers cross a cluster exchange; CUDA cores only
// handle softmax statistics, operand images and epilogues.
//
// Warp roles (576 threads): warp 0 = TMA producer, warp 1 = MMA issuer + TMEM
// owner, warps 2..17 = compute (epilogues, softmax, EMA, DSMEM exchanges).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "decode_fused.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {

using namespace sm100;

constexpr int kMaxStages = 6;
constexpr uint32_t kStage = 32768;  // ring stage: 32 KB (measured on B200: the per-SM stream rate of a
                                    // warp-specialised ring scales with the copy size — ~40 GB/s at
                                    // 16 KB, ~70 GB/s at 32 KB)
constexpr uint32_t kPanel = 16384;  // one 128 x 64 bf16 SWIZZLE_128B operand panel
constexpr int kThreads = 608;  // + warp 18: L2 prefetcher
constexpr int kCompute = 512;
constexpr int kCWarps = 16;
constexpr uint32_t kBarCompute = 1;
constexpr uint32_t kBarBuild = 2;   // phase-D operand builders (compute warps 0..7)
constexpr int kTile = 128;          // rows of a right / tail tile
constexpr int kND = 16;             // N of the phase-D MMAs (query heads of one kv head, padded)
constexpr int kMaxAB = 8;           // phase-A TMEM result buffers (MMA -> epilogue round trip)
constexpr int kMaxOB = 8;           // phase-D operand buffers (8 KB each, in the U-partial region)

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }
__host__ __device__ inline int cdivi(int a, int b) { return (a + b - 1) / b; }

struct LSmem {
  uint32_t ring, pimg, opimg, plocal, stail, hatp, pout, tstat, part, stats, imps, bars, tslot, total;
  int uv;      // fp32 row stride of the U partial [NP][uv]
  int qslots;  // kv heads one phase-A range can touch
  int nq;      // N of the phase-A MMAs (rows of the query operand)
  int tmax_k, tmax_v, tmax_t;  // tiles per CTA (upper bounds)
};

__host__ __device__ inline LSmem layer_smem(const LayerPlan& p) {
  LSmem s{};
  const uint32_t np = p.np;
  const int per_kv = p.s.H / p.s.Hkv, C = p.s.cluster, D = p.s.D, Hkv = p.s.Hkv;
  s.uv = static_cast<int>(align_up(p.s.rank_v, 4));
  s.tmax_k = cdivi(Hkv * cdivi(p.s.rank_k, kTile), C);
  s.tmax_v = cdivi(Hkv * cdivi(p.s.rank_v, kTile), C);
  s.tmax_t = cdivi(Hkv * cdivi(max(p.s.tail_cap, 1), kTile), C);
  s.qslots = min(Hkv, cdivi(Hkv, C) + 2);
  s.nq = static_cast<int>(align_up(2 * s.qslots * per_kv + 4, 16));
  const int owned = cdivi(Hkv, C);
  s.ring = 0;
  s.pimg = s.ring + p.stages * kStage;
  uint32_t pimg_bytes = 2u * p.kpk * np * 128;                          // P operand (hi, lo)
  pimg_bytes = max(pimg_bytes, 8u * np * 128);                          // p tiles: 2 buffers x {hi, lo} x 2 panels
  pimg_bytes = max(pimg_bytes, np * static_cast<uint32_t>(s.uv) * 4u);  // U partial [NP][uv] (DSMEM-read)
  pimg_bytes = max(pimg_bytes, 4u * 2u * 2u * 2u * kND * 128u);         // >= 4 phase-D operand buffers
  s.opimg = align_up(s.pimg + pimg_bytes, 1024);  // phase A: Q image; phase D: 2 x [U | p] images
  const uint32_t qimg = static_cast<uint32_t>(s.nq) * (D / 64) * 128u * 2u;
  const uint32_t dimg = 2u * 2u * 2u * kND * 128u;  // 2 buffers x {hi, lo} x 2 K panels x 16 rows
  s.plocal = align_up(s.opimg + max(qimg, dimg), 16);  // P of my right_k tiles, later U of my right_v tiles
  s.stail = align_up(s.plocal + max(s.tmax_k, s.tmax_v) * kTile * per_kv * 4u, 16);
  s.hatp = align_up(s.stail + (s.tmax_t * kTile + owned) * per_kv * 4u, 16);  // [cap]
  s.pout = align_up(s.hatp + static_cast<uint32_t>(p.s.tail_cap) * 4u, 16);
  s.tstat = s.pout;  // per tail tile and y: max, then sum
  s.part = s.tstat + s.tmax_t * per_kv * 4u;
  s.stats = s.part + 2u * kCWarps * np * 4u + 4u * 128u * 4u;
  s.imps = align_up(s.stats + (5u + 16u) * np * 4u, 16);
  s.bars = align_up(s.imps + (p.max_tiles * 128u + p.tpc) * 8u, 8);
  s.tslot = s.bars + 64 * 8;
  s.total = align_up(s.tslot + 16, 1024);
  return s;
}

// Per-instance exchange area in global memory (L2-resident): the G CTAs of an
// instance publish P chunks, softmax statistics, U partials, tail head sums and
// context partials here.  [sync | P image | stats [G][2][NP] | U [G][NP][uv] |
// head sums [G][cap] | context [H][D]]
struct GroupWs {
  uint32_t pimg, stats, uloc, hatp, pout, bytes;
};
__host__ __device__ inline GroupWs group_ws(const LayerPlan& p) {
  GroupWs w;
  const uint32_t G = p.s.cluster, np = p.np, uv = align_up(p.s.rank_v, 4);
  w.pimg = 256;
  w.stats = w.pimg + 2u * p.kpk * np * 128;
  w.uloc = align_up(w.stats + G * 2u * np * 4u, 256);
  w.hatp = align_up(w.uloc + G * np * uv * 4u, 256);
  w.pout = align_up(w.hatp + G * static_cast<uint32_t>(p.s.tail_cap) * 4u, 256);
  w.bytes = align_up(w.pout + static_cast<uint32_t>(p.s.H) * p.s.D * 4u, 256);
  return w;
}
// Split-phase barrier of the G CTAs of one instance (sense reversal on a flag
// word; called by one thread per CTA after the CTA's writes are fenced).
__device__ __forceinline__ uint32_t group_arrive(unsigned int* sync, int G) {
  volatile unsigned int* flag = sync + 1;
  const uint32_t gen = *flag;
  __threadfence();
  if (atomicAdd(sync, 1u) == static_cast<unsigned>(G - 1)) {
    sync[0] = 0;
    __threadfence();
    atomicExch(sync + 1, gen + 1);
  }
  return gen;
}
__device__ __forceinline__ void group_wait(unsigned int* sync, uint32_t gen) {
  volatile unsigned int* flag = sync + 1;
  while (*flag == gen) __nanosleep(32);
  __threadfence();
}

enum Bar : int {
  kFull = 0,                  // [stages] data landed
  kFree = kMaxStages,         // [stages] released by the MMAs
  kQReady = 2 * kMaxStages,   // phase-A query operand written
  kAOut0,                     // [kMaxAB] phase-A tile result in TMEM
  kAFree0 = kAOut0 + 8,       // [kMaxAB] phase-A TMEM buffer read (count 4 warps)
  kSFull = kAFree0 + 8,       // S MMAs complete
  kPFull0, kPFull1,           // p tile buffer written
  kPEmpty0, kPEmpty1,         // p tile buffer consumed
  kUFull,                     // U MMAs complete
  kDOpFull0,                  // [kMaxOB] phase-D [U | p] operand written
  kDOpFree0 = kDOpFull0 + 8,  // [kMaxOB] phase-D operand consumed by its MMA
  kDAccBase = kDOpFree0 + 8,
  kDAcc0 = kDAccBase, kDAcc1, // phase-D accumulator complete (segment end)
  kDFree0, kDFree1,           // phase-D accumulator read (count 4 warps)
  kTmemFree,
  kPReady,                    // the group's P image landed in my smem (bulk copy)
  kNumBars
};
static_assert(kNumBars <= 64, "barrier area");

struct Work {
  int tile0, tiles;  // 128-token tiles of the left factors (phases B, C)
  int tk, tv, tt;    // row tiles per kv head: right_k, right_v, tail (in memory)
  int uk0, uk1;      // my right_k tiles [uk0, uk1) of [H_kv x tk]
  int uv0, uv1;      // my right_v tiles
  int ut0, ut1;      // my tail tiles
  int n_mem;         // tail rows per head in memory (the appended row comes from the q buffer)
  int na, lv0, d0, total;
};

__host__ __device__ inline Work make_work(const LayerPlan& p, int c, int n_tail, int append) {
  Work w;
  const int C = p.s.cluster, Hkv = p.s.Hkv;
  const int tb = p.ntiles / C, tr = p.ntiles % C;
  w.tiles = tb + (c < tr ? 1 : 0);
  w.tile0 = c * tb + min(c, tr);
  w.n_mem = max(0, n_tail - (append ? 1 : 0));
  w.tk = cdivi(p.s.rank_k, kTile);
  w.tv = cdivi(p.s.rank_v, kTile);
  w.tt = cdivi(w.n_mem, kTile);
  const long uk = static_cast<long>(Hkv) * w.tk, uv = static_cast<long>(Hkv) * w.tv,
             ut = static_cast<long>(Hkv) * w.tt;
  w.uk0 = static_cast<int>(uk * c / C);
  w.uk1 = static_cast<int>(uk * (c + 1) / C);
  w.uv0 = static_cast<int>(uv * c / C);
  w.uv1 = static_cast<int>(uv * (c + 1) / C);
  w.ut0 = static_cast<int>(ut * c / C);
  w.ut1 = static_cast<int>(ut * (c + 1) / C);
  w.na = (w.uk1 - w.uk0) + (w.ut1 - w.ut0);
  w.lv0 = w.na + w.tiles * p.kst;      // K: panel pairs per stage
  w.d0 = w.lv0 + w.tiles * p.mtiles;   // V: one 128-rank pair per stage
  w.total = w.d0 + (w.uv1 - w.uv0) + (w.ut1 - w.ut0);
  return w;
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
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ void red_add_dsmem(float* local, uint32_t cta, float v) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "red.shared::cluster.add.f32 [ra], %2;\n\t}" ::"r"(smem_addr(local)),
      "r"(cta), "f"(v)
      : "memory");
}
// 8 values -> bf16 hi/lo 16-byte chunks
__device__ __forceinline__ void split8(const float (&v)[8], uint4& h4, uint4& l4) {
  __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) split_bf16(v[e], hi[e], lo[e]);
  h4 = *reinterpret_cast<const uint4*>(hi);
  l4 = *reinterpret_cast<const uint4*>(lo);
}

// Compute-warp waits: one thread polls the mbarrier, the rest park on a named barrier.
__device__ __forceinline__ void cta_wait(uint64_t* bar, uint32_t parity, int tid) {
  if (tid == 0) mbar_wait(bar, parity);
  named_bar(kBarCompute, kCompute);
}
__device__ __forceinline__ void cta_wait_cluster(uint64_t* bar, uint32_t parity, int tid) {
  if (tid == 0) mbar_wait_cluster(bar, parity);
  named_bar(kBarCompute, kCompute);
}
__device__ __forceinline__ void warp_wait(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) mbar_wait(bar, parity);
  __syncwarp();
}

// B operands that carry an fp32 quantity as a bf16 hi/lo pair (P, p, Q, [U | p]) are
// stacked along N when ST (one MMA reads the A tile once; the two halves of the
// accumulator are summed at readback), else issued as two MMAs into one accumulator.
// Image of n rows x `panels` 64-wide K panels, K-major SW128: byte offset of (panel, row, k).
template <bool ST>
__device__ __forceinline__ uint32_t bimg_off(int n, int panels, int panel, int row, int k, bool lo) {
  if (ST) return static_cast<uint32_t>(panel * 2 * n * 128) + sw128_off(row + (lo ? n : 0), k);
  return static_cast<uint32_t>((lo ? panels * n * 128 : 0) + panel * n * 128) + sw128_off(row, k);
}
// D (+)= A . B^T for a hi/lo B image of n rows; `kb` = byte offset of the K step inside a panel row.
template <bool ST>
__device__ __forceinline__ void mma_hilo(uint32_t d, uint64_t adesc, uint64_t bdesc_base, uint32_t img, int n,
                                         int panels, int panel, int kb, uint32_t idesc, uint32_t acc) {
  if (ST) {
    mma_bf16(d, adesc, bdesc_base | (((img + panel * 2 * n * 128 + kb) >> 4) & 0x3FFFu), idesc, acc);
  } else {
    mma_bf16(d, adesc, bdesc_base | (((img + panel * n * 128 + kb) >> 4) & 0x3FFFu), idesc, acc);
    mma_bf16(d, adesc, bdesc_base | (((img + panels * n * 128 + panel * n * 128 + kb) >> 4) & 0x3FFFu), idesc, 1);
  }
}
// 32 lanes x 4 columns of a hi/lo accumulator (n columns per half when ST)
template <bool ST>
__device__ __forceinline__ void tld4_hilo(uint32_t taddr, int n, float (&v)[4]) {
  tmem_ld4(taddr, v);
  if (ST) {
    float w[4];
    tmem_ld4(taddr + static_cast<uint32_t>(n), w);
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] += w[e];
  }
}

template <int NP, int PER_KV, int D, bool ST>
__global__ void __launch_bounds__(kThreads, 1)
    layer_kernel(const LayerPlan p, const FusedArgs a) {
  constexpr int KP = D / 64;  // 64-element panels per row
  constexpr int NPW = ST ? 2 * NP : NP;  // TMEM columns of one S / U tile
  extern __shared__ __align__(1024) unsigned char smem[];
  const LSmem L = layer_smem(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.s.cluster;  // CTAs per instance (one group)
  const int c = blockIdx.x % C;
  const int b = blockIdx.x / C;
  const GroupWs GW = group_ws(p);
  unsigned char* gws = a.group_ws + static_cast<size_t>(b) * GW.bytes;
  unsigned int* gsync = reinterpret_cast<unsigned int*>(gws);
  const int H = p.s.H, Hkv = p.s.Hkv, W = Hkv * D, cap = p.s.tail_cap;
  const int Rk = p.s.rank_k, Rv = p.s.rank_v;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const Work wk = make_work(p, c, n_tail, a.append_kv);
  const int NS = p.stages;
  const int owned = cdivi(Hkv, C);                                   // kv heads g with g % C == c
  const int NQ = L.nq;
  const int gk0 = wk.uk0 / max(wk.tk, 1), gt0 = wk.tt > 0 ? wk.ut0 / wk.tt : 0;
  // TMEM columns: S | U | 4 phase-A buffers | 2 phase-D accumulators
  const uint32_t s_cols = static_cast<uint32_t>(p.max_tiles * NPW);  // U region starts here
  const uint32_t a_col = static_cast<uint32_t>(p.a_col);  // phase-A result buffers (alias the U region)
  const uint32_t d_col = static_cast<uint32_t>(p.d_col);  // phase-D accumulators
  const int NAB = p.nab;
  const int NOB = p.nob;
  const int NQW = ST ? 2 * NQ : NQ;  // TMEM columns of one phase-A result buffer
  constexpr int NDW = ST ? 2 * kND : kND;
  unsigned long long* trace = a.trace ? a.trace + blockIdx.x * 16ull : nullptr;
  // per-item clock64 trace of CTA 0 (debug): [issue, MMA acquire, MMA issued] x item
  unsigned long long* ict = (a.trace && blockIdx.x == 0) ? a.trace + gridDim.x * 16ull : nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[kFull + s], 1);
      mbar_init(&bars[kFree + s], 1);
    }
    for (int i = kQReady; i <= kPReady; ++i) mbar_init(&bars[i], 1);
    for (int k = 0; k < kMaxAB; ++k) mbar_init(&bars[kAFree0 + k], 4);
    mbar_init(&bars[kDFree0], 4);
    mbar_init(&bars[kDFree1], 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, static_cast<uint32_t>(p.tmem_cols));
  if (warp == 0 && lane == 0) *reinterpret_cast<volatile int*>(tslot + 1) = 0;
  if (warp >= 2 && warp < 18) {
    const int tid = threadIdx.x - 64;
    // zero the P operand image rows h >= H and rank chunks no CTA pushes
    const int uph = (Rk + 7) / 8;
    for (int i = tid; i < NP * p.kpk * 8; i += kCompute) {
      const int h = i / (p.kpk * 8), ch = i % (p.kpk * 8);
      if (h < H && ch < uph) continue;
      *reinterpret_cast<uint4*>(smem + L.pimg + bimg_off<ST>(NP, p.kpk, ch >> 3, h, (ch & 7) * 8, false)) =
          make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(smem + L.pimg + bimg_off<ST>(NP, p.kpk, ch >> 3, h, (ch & 7) * 8, true)) =
          make_uint4(0, 0, 0, 0);
    }
    // the group's context accumulator: each CTA zeroes its owned heads (ordered before any
    // add by the P barrier); CTA 0 zeroes the P image chunks nobody pushes
    float* gpout = reinterpret_cast<float*>(gws + GW.pout);
    for (int i = tid; i < owned * PER_KV * D; i += kCompute) {
      const int g = c + (i / (PER_KV * D)) * C;
      if (g < Hkv) gpout[(g * PER_KV + (i / D) % PER_KV) * D + i % D] = 0.f;
    }
    if (c == 0)
      for (int i = tid; i < NP * p.kpk * 8; i += kCompute) {
        const int h = i / (p.kpk * 8), ch = i % (p.kpk * 8);
        if (h < H && ch < (Rk + 7) / 8) continue;
        *reinterpret_cast<uint4*>(gws + GW.pimg + bimg_off<ST>(NP, p.kpk, ch >> 3, h, (ch & 7) * 8, false)) =
            make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(gws + GW.pimg + bimg_off<ST>(NP, p.kpk, ch >> 3, h, (ch & 7) * 8, true)) =
            make_uint4(0, 0, 0, 0);
      }
    // partial tail tiles leave ring rows unwritten: start from zeros (never NaN garbage)
    for (int i = tid; i < NS * static_cast<int>(kStage / 16); i += kCompute)
      reinterpret_cast<uint4*>(smem + L.ring)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

    const int nka = wk.uk1 - wk.uk0, nvk = wk.uv1 - wk.uv0;
    const int tcap = cdivi(cap, kTile);  // tail tiles per kv head in memory
    constexpr uint32_t kTileBytes = KP * kPanel;
    // source of ring item k: (address, bytes per panel, panels); right / left tiles are
    // one contiguous copy, a tail tile copies only its rows in memory, panel by panel
    auto item_src = [&](int k, const unsigned char*& src, uint32_t& bytes, int& parts) {
      parts = 1;
      if (k < wk.na || k >= wk.d0) {
        const bool is_a = k < wk.na;
        const int rel = is_a ? k : k - wk.d0, nr = is_a ? nka : nvk;
        if (rel < nr) {  // right factor tile
          const int u = (is_a ? wk.uk0 : wk.uv0) + rel, per = is_a ? wk.tk : wk.tv;
          src = reinterpret_cast<const unsigned char*>(is_a ? a.right_k : a.right_v) +
                ((static_cast<long>(b) * Hkv + u / per) * per + u % per) * kTileBytes;
          bytes = kTileBytes;
        } else {  // tail tile
          const int u = wk.ut0 + rel - nr, j = u % wk.tt;
          src = reinterpret_cast<const unsigned char*>(is_a ? a.tail_k : a.tail_v) +
                ((static_cast<long>(b) * Hkv + u / wk.tt) * tcap + j) * kTileBytes;
          bytes = static_cast<uint32_t>(min(kTile, wk.n_mem - j * kTile)) * 128u;
          parts = KP;
        }
      } else if (k < wk.lv0) {  // left_k: panels (2pp, 2pp+1) of a tile, contiguous when packed
        const int t = (k - wk.na) / p.kst, pp = (k - wk.na) % p.kst;
        const long gtile = static_cast<long>(a.inst0 + b) * p.ntiles + wk.tile0 + t;
        src = a.left_k_packed + (gtile * p.kpk + 2 * pp) * static_cast<long>(kPanel);
        bytes = static_cast<uint32_t>(min(2, p.kpk - 2 * pp)) * kPanel;
      } else {  // left_v: 128-rank panel pair (a missing odd panel stays unloaded: U rows
                // >= rank_v are never read)
        const int t = (k - wk.lv0) / p.mtiles, mt = (k - wk.lv0) % p.mtiles;
        const long gtile = static_cast<long>(a.inst0 + b) * p.ntiles + wk.tile0 + t;
        src = a.left_v_packed + (gtile * p.vpanels_st + 2 * mt) * static_cast<long>(kPanel);
        bytes = static_cast<uint32_t>(min(2, p.vpanels_st - 2 * mt)) * kPanel;
      }
    };
  volatile int* prog = reinterpret_cast<volatile int*>(tslot + 1);  // items issued by the producer
  if (warp == 0) {
    // ============================ producer ============================
    if (lane == 0) {
      for (int i = 0; i < wk.total; ++i) {
        const int s = i % NS;
        if (i >= NS) mbar_wait(&bars[kFree + s], ((i / NS) - 1) & 1);
        const unsigned char* src;
        uint32_t bytes;
        int parts;
        item_src(i, src, bytes, parts);
        if (ict && i < 512) ict[3 * i] = clock64();
        mbar_expect_tx(&bars[kFull + s], bytes * parts);
        unsigned char* dst = smem + L.ring + s * kStage;
        for (int q = 0; q < parts; ++q) bulk_load(dst + q * kPanel, src + q * kPanel, bytes, &bars[kFull + s]);
        *prog = i + 1;
        if (i == wk.na - 1 && (p.debug & 8)) break;  // timing experiment: phase A only
      }
      if (trace) trace[7] = global_ns();
    }
  } else if (warp == 18) {
    // ======================= L2 prefetcher (LSU path) =======================
    // Keeps the next p.prefetch items (beyond the ring) in L2 with per-line
    // prefetches, so the ring's bulk copies see L2 latency, not HBM latency, and
    // the TMA engine is not spent on prefetching.
    const int pf = NS + p.prefetch;
    for (int k = 0; k < wk.total; ++k) {
      if (k >= pf)
        while (k >= *prog + pf) __nanosleep(64);
      const unsigned char* src;
      uint32_t bytes;
      int parts;
      item_src(k, src, bytes, parts);
      for (int q = 0; q < parts; ++q)
        for (uint32_t off = lane * 128u; off < bytes; off += 32u * 128u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(src + q * kPanel + off));
      if ((p.debug & 8) && k == wk.na - 1) break;
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      const uint32_t ring = smem_addr(smem + L.ring);
      const uint32_t phi = smem_addr(smem + L.pimg);
      const uint32_t pt = smem_addr(smem + L.pimg);  // p tiles reuse the P image once S is done
      const uint32_t opi = smem_addr(smem + L.opimg);
      // descriptors differ only in the start-address field (bits 0-13 = addr >> 4): build the
      // K-major / MN-major bases once
      const uint64_t dk = smem_desc(0, 16, 1024, kSwizzle128B);       // K-major, SW128
      const uint64_t dm = smem_desc(0, kPanel, 1024, kSwizzle128B);   // MN-major pair (LBO = 16 KB)
      auto kdesc = [&](uint32_t addr) { return dk | ((addr >> 4) & 0x3FFFu); };
      auto mdesc = [&](uint32_t addr) { return dm | ((addr >> 4) & 0x3FFFu); };
      auto wait_full = [&](int i) {
        mbar_wait(&bars[kFull + i % NS], (i / NS) & 1);
        if (ict && i < 512) ict[3 * i + 1] = clock64();
        tc_fence_after();
      };
      // ---- phase A: [P | s_tail] tile = row tile (M=128, K=D, K-major) . Q^T (N=NQ)
      {
        const uint32_t idesc_a = idesc_bf16(128, static_cast<uint32_t>(NQW), false, false);
        mbar_wait(&bars[kQReady], 0);
        tc_fence_after();
        for (int i = 0; i < wk.na; ++i) {
          const int ab = i % NAB;
          if (i >= NAB) {
            mbar_wait(&bars[kAFree0 + ab], ((i / NAB) - 1) & 1);
            tc_fence_after();
          }
          wait_full(i);
          const int s = i % NS;
          const uint32_t d = tmem + a_col + static_cast<uint32_t>(ab * NQW);
          for (int q = 0; q < KP; ++q)
            for (int kk = 0; kk < 4; ++kk)
              mma_hilo<ST>(d, kdesc(ring + s * kStage + q * kPanel + kk * 32), dk, opi, NQ, KP, q, kk * 32, idesc_a,
                           (q | kk) != 0);
          mma_commit(&bars[kFree + s]);
          mma_commit(&bars[kAOut0 + ab]);
          if (ict && i < 512) ict[3 * i + 2] = clock64();
        }
      }
      if (p.debug & 8) {
        mbar_wait(&bars[kTmemFree], 0);
      } else {
      // ---- phase B: S = left_k . P
      const uint32_t idesc_s = idesc_bf16(128, NPW, false, false);
      const uint32_t idesc_u = idesc_bf16(128, NPW, true, false);
      mbar_wait(&bars[kPReady], 0);
      tc_fence_after();
      if (trace) trace[8] = global_ns();
      for (int t = 0; t < wk.tiles; ++t) {
        for (int pp = 0; pp < p.kst; ++pp) {
          const int i = wk.na + t * p.kst + pp, s = i % NS;
          wait_full(i);
          for (int q = 0; q < 2 && 2 * pp + q < p.kpk; ++q) {
            const int kp = 2 * pp + q;
            for (int kk = 0; kk < 4; ++kk)
              mma_hilo<ST>(tmem + static_cast<uint32_t>(t * NPW), kdesc(ring + s * kStage + q * kPanel + kk * 32), dk,
                           phi, NP, p.kpk, kp, kk * 32, idesc_s, (kp | kk) != 0);
          }
          mma_commit(&bars[kFree + s]);
        }
      }
      mma_commit(&bars[kSFull]);
      // ---- phase C: U^T += left_v^T . p
      for (int t = 0; t < wk.tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(&bars[kPFull0 + buf], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t pth = pt + buf * 4 * NP * 128;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const int i0 = wk.lv0 + t * p.mtiles + mt, s0 = i0 % NS;
          wait_full(i0);
          const uint32_t d = tmem + s_cols + static_cast<uint32_t>(mt * NPW);
          for (int ks = 0; ks < 8; ++ks)
            mma_hilo<ST>(d, mdesc(ring + s0 * kStage + ks * 2048), dk, pth, NP, 2, ks >> 2, (ks & 3) * 32, idesc_u,
                         (t | ks) != 0);
          mma_commit(&bars[kFree + s0]);
        }
        mma_commit(&bars[kPEmpty0 + buf]);
      }
      mma_commit(&bars[kUFull]);
      // ---- phase D: ctx^T (M=128 dims, N=16) += tile^T (MN-major) . [U | p]^T
      {
        const uint32_t idesc_d = idesc_bf16(128, NDW, true, false);
        const int nvk = wk.uv1 - wk.uv0;
        int seg = -1, prev_key = -1;
        for (int i = wk.d0; i < wk.total; ++i) {
          const int di = i - wk.d0;
          const bool is_tail = di >= nvk;
          const int u = is_tail ? wk.ut0 + (di - nvk) : wk.uv0 + di;
          const int g = is_tail ? u / wk.tt : u / wk.tv;
          const int key = is_tail ? Hkv + g : g;
          const bool first = key != prev_key;
          if (first) {
            ++seg;
            prev_key = key;
            if (seg >= 2) {
              mbar_wait(&bars[kDFree0 + (seg & 1)], ((seg >> 1) - 1) & 1);
              tc_fence_after();
            }
          }
          const int nxt = i + 1 - wk.d0;  // does the next item start a new segment?
          bool last = i + 1 == wk.total;
          if (!last) {
            const bool nt = nxt >= nvk;
            const int un = nt ? wk.ut0 + (nxt - nvk) : wk.uv0 + nxt;
            last = (nt ? Hkv + un / wk.tt : un / wk.tv) != key;
          }
          const int ob = di % NOB;
          mbar_wait(&bars[kDOpFull0 + ob], (di / NOB) & 1);
          if (ict && i < 512) ict[3 * i + 2] = clock64();
          wait_full(i);
          const int s = i % NS;
          const uint32_t d = tmem + d_col + static_cast<uint32_t>((seg & 1) * NDW);
          const uint32_t oh = phi + ob * 2 * 2 * kND * 128;  // operand ring in the U-partial region
          for (int ks = 0; ks < 8; ++ks)
            mma_hilo<ST>(d, mdesc(ring + s * kStage + ks * 2048), dk, oh, kND, 2, ks >> 2, (ks & 3) * 32, idesc_d,
                         (!first || ks != 0) ? 1u : 0u);
          mma_commit(&bars[kFree + s]);
          mma_commit(&bars[kDOpFree0 + ob]);
          if (last) mma_commit(&bars[kDAcc0 + (seg & 1)]);
        }
      }
      mbar_wait(&bars[kTmemFree], 0);
      }
    }
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, static_cast<uint32_t>(p.tmem_cols));
  } else {
    // ============================ compute warps ============================
    const int cw = warp - 2;
    const int tid = threadIdx.x - 64;
    const int qd = warp & 3;  // TMEM lane quadrant this warp may access
    const float scale = rsqrtf(static_cast<float>(D));
    float* plocal = reinterpret_cast<float*>(smem + L.plocal);  // phase A: P of my right_k tiles [row][y]
    float* umine = plocal;                                       // phase D: U of my right_v tiles [row][y]
    float* stail = reinterpret_cast<float*>(smem + L.stail);    // my tail slots [slot][y]: logits -> p
    float* hatp = reinterpret_cast<float*>(smem + L.hatp);      // [cap]: my slots' share of the head average
    float* gpout = reinterpret_cast<float*>(gws + GW.pout);  // the group's context accumulator [H][D]
    float* part = reinterpret_cast<float*>(smem + L.part);
    float* stats = reinterpret_cast<float*>(smem + L.stats);
    double* imps = reinterpret_cast<double*>(smem + L.imps);
    float* m_loc = stats;
    float* z_loc = stats + NP;
    float* m_g = stats + 2 * NP;
    float* f_me = stats + 3 * NP;      // exp(m_loc - m_g) / z_g
    float* zi_g = stats + 4 * NP;      // 1 / z_g
    float* scale_c = stats + 5 * NP;   // [C][NP] exp(m_c - m_g)
    const int tpc = p.tpc, t_lo = c * tpc, t_hi = min(n_tail, t_lo + tpc);  // my tail tokens for the EMA
    const float* qrow = a.q + static_cast<long>(b) * a.q_stride;
    const int ntt = wk.ut1 - wk.ut0;              // my tail tiles
    const int nslot = ntt * kTile + owned;        // my tail slots (tile rows, then appended rows)
    const bool append = a.append_kv && n_tail > 0;
    // slot -> token index (g = its kv head), -1 when the slot holds no token
    auto slot_token = [&](int sl, int& g) -> int {
      if (sl < ntt * kTile) {
        const int u = wk.ut0 + sl / kTile;
        g = u / wk.tt;
        const int t = (u % wk.tt) * kTile + sl % kTile;
        return t < wk.n_mem ? t : -1;
      }
      g = c + (sl - ntt * kTile) * C;
      return (append && g < Hkv) ? n_tail - 1 : -1;
    };
    if (trace && tid == 0) trace[0] = global_ns();

    // query operand of phase A: rows (slot, y) for the kv heads my right_k range (slots
    // 0..qslots-1) and my tail range (slots qslots..) touch; bf16 hi/lo, K-major SW128
    {
      unsigned char* qh = smem + L.opimg;
      for (int w = tid; w < NQ * (D / 8); w += kCompute) {
        const int row = w / (D / 8), ch = w % (D / 8);
        const int sl = row / PER_KV, y = row % PER_KV;
        const int g = sl < L.qslots ? gk0 + sl : gt0 + (sl - L.qslots);
        float v[8];
        const bool ok = sl < 2 * L.qslots && g < Hkv;
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = ok ? qrow[(g * PER_KV + y) * D + ch * 8 + e] * scale : 0.f;
        uint4 h4, l4;
        split8(v, h4, l4);
        *reinterpret_cast<uint4*>(qh + bimg_off<ST>(NQ, KP, ch >> 3, row, (ch & 7) * 8, false)) = h4;
        *reinterpret_cast<uint4*>(qh + bimg_off<ST>(NQ, KP, ch >> 3, row, (ch & 7) * 8, true)) = l4;
      }
      fence_proxy_async();
      named_bar(kBarCompute, kCompute);
      if (tid == 0) mbar_arrive(&bars[kQReady]);
    }
    // prefetch the old importance of my compressed tokens and my EMA tail tokens
    const int c_first = wk.tile0 * 128;
    const int chunk_len = max(0, min(p.s.n_comp - c_first, wk.tiles * 128));
    if (a.importance) {
      const double* ib = a.importance + static_cast<long>(b) * a.imp_stride;
      for (int i = tid; i < chunk_len; i += kCompute) imps[i] = ib[c_first + i];
      for (int t = t_lo + tid; t < t_hi; t += kCompute)
        imps[p.max_tiles * 128 + (t - t_lo)] =
            (a.append_kv && t == n_tail - 1) ? 0.0 : ib[p.s.n_comp + t];  // appended row: importance 0
    }
    for (int t = tid; t < cap; t += kCompute) hatp[t] = 0.f;

    // ---------------- phase A epilogue: tile i -> warp group i % 4 ----------------
    {
      const int grp = cw >> 2;
      const int nk = wk.uk1 - wk.uk0;
      for (int i = grp; i < wk.na; i += 4) {
        const int ab = i % NAB;
        warp_wait(&bars[kAOut0 + ab], (i / NAB) & 1);
        tc_fence_after();
        const bool is_tail = i >= nk;
        const int u = is_tail ? wk.ut0 + (i - nk) : wk.uk0 + i;
        const int g = is_tail ? u / wk.tt : u / wk.tk;
        const int sl = is_tail ? L.qslots + (g - gt0) : g - gk0;
        float v[4];
        tld4_hilo<ST>(tmem + (static_cast<uint32_t>(qd * 32) << 16) + a_col + static_cast<uint32_t>(ab * NQW + sl * PER_KV),
                      NQ, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[kAFree0 + ab]);
        const int row = qd * 32 + lane;
        const int r = (is_tail ? u % wk.tt : u % wk.tk) * kTile + row;
        if (r < (is_tail ? wk.n_mem : Rk)) {
          float* dst = is_tail ? stail + ((u - wk.ut0) * kTile + row) * PER_KV
                               : plocal + ((u - wk.uk0) * kTile + row) * PER_KV;
#pragma unroll
          for (int y = 0; y < PER_KV; ++y) dst[y] = v[y];
        }
      }
    }
    if (p.debug & 8) {
      named_bar(kBarCompute, kCompute);
      if (trace && tid == 0) trace[1] = global_ns();
      if (tid == 0) mbar_arrive(&bars[kTmemFree]);
      return;
    }
    named_bar(kBarCompute, kCompute);
    // push my P rows (16-byte chunks of 8 ranks, bf16 hi/lo) into every peer's operand image
    for (int w = tid; w < (wk.uk1 - wk.uk0) * 16 * PER_KV; w += kCompute) {
      const int ti = w / (16 * PER_KV), m = (w / PER_KV) % 16, y = w % PER_KV;
      const int u = wk.uk0 + ti, g = u / wk.tk, r0 = (u % wk.tk) * kTile + m * 8;
      if (r0 >= Rk) continue;
      const int h = g * PER_KV + y;
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = r0 + e < Rk ? plocal[(ti * kTile + m * 8 + e) * PER_KV + y] : 0.f;
      uint4 h4, l4;
      split8(v, h4, l4);
      *reinterpret_cast<uint4*>(gws + GW.pimg + bimg_off<ST>(NP, p.kpk, r0 >> 6, h, r0 & 63, false)) = h4;
      *reinterpret_cast<uint4*>(gws + GW.pimg + bimg_off<ST>(NP, p.kpk, r0 >> 6, h, r0 & 63, true)) = l4;
    }
    __threadfence();
    named_bar(kBarCompute, kCompute);
    if (tid == 0) {  // group barrier, then one bulk copy of the complete image into my smem
      group_wait(gsync, group_arrive(gsync, C));
      fence_proxy_async_all();  // generic-proxy writes of the peers -> async-proxy (bulk copy) read
      const uint32_t pbytes = 2u * p.kpk * NP * 128;
      mbar_expect_tx(&bars[kPReady], pbytes);
      bulk_load(smem + L.pimg, gws + GW.pimg, pbytes, &bars[kPReady]);
    }
    if (trace && tid == 0) trace[1] = global_ns();
    // appended token of kv heads g = c, c + C, ...: k, v straight from the projection,
    // bf16-rounded as stored; written back to the tail (cache.cpp:147-170)
    if (append) {
      for (int w = cw; w < owned * PER_KV; w += kCWarps) {
        const int k = w / PER_KV, y = w % PER_KV, g = c + k * C;
        if (g >= Hkv) continue;
        const int h = g * PER_KV + y;
        float t = 0.f;
        for (int j = lane; j < D; j += 32) t = fmaf(bf16r(qrow[H * D + g * D + j]), qrow[h * D + j] * scale, t);
        t = warp_sum(t);
        if (lane == 0) stail[(ntt * kTile + k) * PER_KV + y] = t;
        if (y == 0) {  // into the packed tail tile (row t % 128 of tile t / 128, swizzled panels)
          const int t = n_tail - 1, tcap = cdivi(cap, kTile);
          const long tile = (static_cast<long>(b) * Hkv + g) * tcap + t / kTile;
          unsigned char* tk = reinterpret_cast<unsigned char*>(const_cast<__nv_bfloat16*>(a.tail_k)) +
                              tile * (KP * kPanel);
          unsigned char* tv = reinterpret_cast<unsigned char*>(const_cast<__nv_bfloat16*>(a.tail_v)) +
                              tile * (KP * kPanel);
          for (int j = lane; j < D; j += 32) {
            const uint32_t off = (j >> 6) * kPanel + sw128_off(t % kTile, j & 63);
            *reinterpret_cast<__nv_bfloat16*>(tk + off) = __float2bfloat16_rn(qrow[H * D + g * D + j]);
            *reinterpret_cast<__nv_bfloat16*>(tv + off) = __float2bfloat16_rn(qrow[H * D + W + g * D + j]);
          }
        }
      }
    }

    // ---------------- phase B epilogue: local softmax statistics ----------------
    const int cg = cw >> 2;        // column group 0..3
    constexpr int gcols = NP / 4;
    const int gbase = cg * gcols;
    auto tmem_row = [&](uint32_t col) { return tmem + (static_cast<uint32_t>(qd * 32) << 16) + col; };
    cta_wait(&bars[kSFull], 0, tid);
    tc_fence_after();
    if (trace && tid == 0) trace[2] = global_ns();
    float* part_m = part;
    float* part_s = part + kCWarps * NP;
    for (int c0 = 0; c0 < gcols; c0 += 4) {
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int t = 0; t < wk.tiles; ++t) {
        float v[4];
        tld4_hilo<ST>(tmem_row(static_cast<uint32_t>(t * NPW + gbase + c0)), NP, v);
        if (t * 128 + qd * 32 + lane < chunk_len)
          for (int e = 0; e < 4; ++e) mx[e] = fmaxf(mx[e], v[e]);
      }
      for (int e = 0; e < 4; ++e) {
        const float m = warp_max(mx[e]);
        if (lane == 0) part_m[cw * NP + gbase + c0 + e] = m;
      }
    }
    // per tail tile (one warp each): max over its rows in memory
    float* tstat = reinterpret_cast<float*>(smem + L.tstat);
    for (int ti = cw; ti < ntt; ti += kCWarps) {
      const int u = wk.ut0 + ti, t0 = (u % wk.tt) * kTile;
#pragma unroll
      for (int y = 0; y < PER_KV; ++y) {
        float m = -INFINITY;
        for (int row = lane; row < kTile; row += 32)
          if (t0 + row < wk.n_mem) m = fmaxf(m, stail[(ti * kTile + row) * PER_KV + y]);
        m = warp_max(m);
        if (lane == 0) tstat[ti * PER_KV + y] = m;
      }
    }
    named_bar(kBarCompute, kCompute);
    if (tid < H) {
      const int h = tid, g = h / PER_KV, y = h % PER_KV, w0 = (h / gcols) * 4;
      float m = -INFINITY;
      for (int w = 0; w < 4; ++w) m = fmaxf(m, part_m[(w0 + w) * NP + h]);
      const int u0 = max(wk.ut0, g * wk.tt), u1 = min(wk.ut1, (g + 1) * wk.tt);
      for (int u = u0; u < u1; ++u) m = fmaxf(m, tstat[(u - wk.ut0) * PER_KV + y]);
      if (append && g % C == c) m = fmaxf(m, stail[(ntt * kTile + g / C) * PER_KV + y]);
      m_loc[h] = m;
    }
    named_bar(kBarCompute, kCompute);
    if (trace && tid == 0) trace[9] = global_ns();

    // ---------------- p tiles (bf16 hi/lo, K-major over tokens) -> U MMAs ----------------
    float zp[gcols];
#pragma unroll
    for (int e = 0; e < gcols; ++e) zp[e] = 0.f;
    for (int t = 0; t < wk.tiles; ++t) {
      const int buf = t & 1;
      if (t >= 2) cta_wait(&bars[kPEmpty0 + buf], ((t - 2) >> 1) & 1, tid);
      unsigned char* pth = smem + L.pimg + buf * 4 * NP * 128;
      const int row = qd * 32 + lane;
      const bool valid = t * 128 + row < chunk_len;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4];
        tld4_hilo<ST>(tmem_row(static_cast<uint32_t>(t * NPW + gbase + c0)), NP, v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          const float pv = (valid && h < H) ? __expf(v[e] - m_loc[h]) : 0.f;
          zp[c0 + e] += pv;
          __nv_bfloat16 hi, lo;
          split_bf16(pv, hi, lo);
          *reinterpret_cast<__nv_bfloat16*>(pth + bimg_off<ST>(NP, 2, row >> 6, h, row & 63, false)) = hi;
          *reinterpret_cast<__nv_bfloat16*>(pth + bimg_off<ST>(NP, 2, row >> 6, h, row & 63, true)) = lo;
        }
      }
      fence_proxy_async();
      named_bar(kBarCompute, kCompute);
      if (tid == 0) mbar_arrive(&bars[kPFull0 + buf]);
      if (trace && tid == 0 && t == 0) trace[10] = global_ns();
    }
#pragma unroll
    for (int c0 = 0; c0 < gcols; ++c0) {
      const float z = warp_sum(zp[c0]);
      if (lane == 0) part_s[cw * NP + gbase + c0] = z;
    }
    // my tail slots: local p in place of the logits (empty slots -> 0)
    for (int w = tid; w < nslot * PER_KV; w += kCompute) {
      int g;
      const int t = slot_token(w / PER_KV, g);
      stail[w] = t >= 0 ? __expf(stail[w] - m_loc[g * PER_KV + w % PER_KV]) : 0.f;
    }
    named_bar(kBarCompute, kCompute);
    for (int ti = cw; ti < ntt; ti += kCWarps) {  // per tail tile: sum of the local p
#pragma unroll
      for (int y = 0; y < PER_KV; ++y) {
        float z = 0.f;
        for (int row = lane; row < kTile; row += 32) z += stail[(ti * kTile + row) * PER_KV + y];
        z = warp_sum(z);
        if (lane == 0) tstat[ti * PER_KV + y] = z;
      }
    }
    named_bar(kBarCompute, kCompute);
    if (tid < H) {
      const int h = tid, g = h / PER_KV, y = h % PER_KV, w0 = (h / gcols) * 4;
      float z = 0.f;
      for (int w = 0; w < 4; ++w) z += part_s[(w0 + w) * NP + h];
      const int u0 = max(wk.ut0, g * wk.tt), u1 = min(wk.ut1, (g + 1) * wk.tt);
      for (int u = u0; u < u1; ++u) z += tstat[(u - wk.ut0) * PER_KV + y];
      if (append && g % C == c) z += stail[(ntt * kTile + g / C) * PER_KV + y];
      z_loc[h] = z;
    }
    if (trace && tid == 0) trace[3] = global_ns();

    // ---------------- group statistics (while the U MMAs run) ----------------
    named_bar(kBarCompute, kCompute);
    float* gstats = reinterpret_cast<float*>(gws + GW.stats);
    if (tid < NP) {
      gstats[(c * 2) * NP + tid] = m_loc[tid];
      gstats[(c * 2 + 1) * NP + tid] = z_loc[tid];
    }
    __threadfence();
    named_bar(kBarCompute, kCompute);
    if (tid == 0) group_wait(gsync, group_arrive(gsync, C));
    named_bar(kBarCompute, kCompute);
    if (tid < H) {
      const int h = tid;
      float mg = -INFINITY;
      for (int peer = 0; peer < C; ++peer) mg = fmaxf(mg, __ldcg(&gstats[(peer * 2) * NP + h]));
      float zg = 0.f;
      for (int peer = 0; peer < C; ++peer) {
        const float mp = __ldcg(&gstats[(peer * 2) * NP + h]);
        const float sc = mp == -INFINITY ? 0.f : __expf(mp - mg);
        scale_c[peer * NP + h] = sc;
        zg += __ldcg(&gstats[(peer * 2 + 1) * NP + h]) * sc;
      }
      const float zi = 1.0f / zg;
      m_g[h] = mg;
      zi_g[h] = zi;
      f_me[h] = (m_loc[h] == -INFINITY ? 0.f : __expf(m_loc[h] - mg)) * zi;
    }
    named_bar(kBarCompute, kCompute);

    // my tail slots: normalised p, and their share of the head average
    for (int w = tid; w < nslot * PER_KV; w += kCompute) {
      int g;
      const int t = slot_token(w / PER_KV, g);
      if (t < 0) continue;
      const float pv = stail[w] * f_me[g * PER_KV + w % PER_KV];
      stail[w] = pv;
      atomicAdd(&hatp[t], pv);
    }

    // ---------------- U readback, gather U for my right_v tiles ----------------
    cta_wait(&bars[kUFull], 0, tid);
    tc_fence_after();
    if (trace && tid == 0) trace[4] = global_ns();
    float* uloc = reinterpret_cast<float*>(gws + GW.uloc) + static_cast<size_t>(c) * NP * L.uv;  // my U partial
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int r = mt * 128 + qd * 32 + lane;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (wk.tiles > 0) tld4_hilo<ST>(tmem_row(s_cols + static_cast<uint32_t>(mt * NPW + gbase + c0)), NP, v);
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          if (h < H && r < Rv) uloc[h * L.uv + r] = v[e];
        }
      }
    }
    tc_fence_before();
    {  // my tail head sums, then arrive (split phase: the EMA below overlaps the slowest peer)
      float* ghat = reinterpret_cast<float*>(gws + GW.hatp) + static_cast<size_t>(c) * cap;
      for (int t = tid; t < n_tail; t += kCompute) ghat[t] = hatp[t];
    }
    __threadfence();
    named_bar(kBarCompute, kCompute);
    uint32_t ugen = 0;
    if (tid == 0) ugen = group_arrive(gsync, C);
    // head average + importance EMA of my compressed tokens (while the peers publish U)
    float* ha_part = part;  // [4 groups][128]
    const float inv_h = 1.0f / static_cast<float>(H);
    for (int t = 0; t < wk.tiles; ++t) {
      const int row = qd * 32 + lane;
      float hsum = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4];
        tld4_hilo<ST>(tmem_row(static_cast<uint32_t>(t * NPW + gbase + c0)), NP, v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          if (h < H) hsum = fmaf(__expf(v[e] - m_loc[h]), f_me[h], hsum);
        }
      }
      ha_part[cg * 128 + row] = hsum;
      named_bar(kBarCompute, kCompute);
      if (tid < 128) {
        const int tk = t * 128 + tid;
        if (tk < chunk_len) {
          const float ha = (ha_part[tid] + ha_part[128 + tid] + ha_part[256 + tid] + ha_part[384 + tid]) * inv_h;
          const long gi = c_first + tk;
          if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + cap) + gi] = ha;
          if (a.importance)
            a.importance[static_cast<long>(b) * a.imp_stride + gi] =
                __dadd_rn(__dmul_rn(a.ema_decay, imps[tk]), __dmul_rn(a.ema_blend, static_cast<double>(ha)));
        }
      }
      named_bar(kBarCompute, kCompute);
    }
    if (trace && tid == 0) trace[11] = global_ns();
    if (tid == 0) group_wait(gsync, ugen);
    named_bar(kBarCompute, kCompute);
    const float* gul = reinterpret_cast<const float*>(gws + GW.uloc);
    if (trace && tid == 0) trace[12] = global_ns();
    // 4 consecutive ranks of one query head per thread: one 16-byte DSMEM load per peer
    for (int w = tid; w < (wk.uv1 - wk.uv0) * (kTile / 4) * PER_KV; w += kCompute) {
      const int ti = w / ((kTile / 4) * PER_KV), y = w % PER_KV, row = ((w / PER_KV) % (kTile / 4)) * 4;
      const int u = wk.uv0 + ti, g = u / wk.tv, r = (u % wk.tv) * kTile + row, h = g * PER_KV + y;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      if (r < Rv) {  // uv is a multiple of 4: the chunk never leaves the row
        for (int peer = 0; peer < C; ++peer) {
          const float4 uu = __ldcg(reinterpret_cast<const float4*>(gul + (static_cast<size_t>(peer) * NP + h) * L.uv + r));
          const float sc = scale_c[peer * NP + h];
          acc[0] = fmaf(sc, uu.x, acc[0]);
          acc[1] = fmaf(sc, uu.y, acc[1]);
          acc[2] = fmaf(sc, uu.z, acc[2]);
          acc[3] = fmaf(sc, uu.w, acc[3]);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) umine[(ti * kTile + row + e) * PER_KV + y] = r + e < Rv ? acc[e] * zi_g[h] : 0.f;
    }
    if (trace && tid == 0) trace[13] = global_ns();
    // tail tokens t_lo..t_hi: head average over every peer's slots, EMA
    for (int t = t_lo + tid; t < t_hi; t += kCompute) {
      const float* ghat = reinterpret_cast<const float*>(gws + GW.hatp);
      float hs = 0.f;
      for (int peer = 0; peer < C; ++peer) hs += __ldcg(&ghat[static_cast<size_t>(peer) * cap + t]);
      const float ha = hs * inv_h;
      const long gi = p.s.n_comp + t;
      if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + cap) + gi] = ha;
      if (a.importance)
        a.importance[static_cast<long>(b) * a.imp_stride + gi] =
            __dadd_rn(__dmul_rn(a.ema_decay, imps[p.max_tiles * 128 + (t - t_lo)]),
                      __dmul_rn(a.ema_blend, static_cast<double>(ha)));
    }
    named_bar(kBarCompute, kCompute);  // umine final; the U-partial smem region is the operand ring now
    if (trace && tid == 0) trace[5] = global_ns();

    // ---------------- phase D: [U | p] operands (warps 0..7), accumulator epilogues (8..11) ----------------
    {
      const int nvk = wk.uv1 - wk.uv0, nd = wk.total - wk.d0;
      if (cw < 8) {
        const int bt = tid;  // 0..255: (operand row n, 8-row chunk of K)
        const int n = bt >> 4, ch = bt & 15;
        for (int di = 0; di < nd; ++di) {
          const int ob = di % NOB;
          if (di >= NOB) {
            if (bt == 0) mbar_wait(&bars[kDOpFree0 + ob], ((di / NOB) - 1) & 1);
            named_bar(kBarBuild, 256);
          }
          const bool is_tail = di >= nvk;
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = 0.f;
          if (n < PER_KV) {
            if (!is_tail) {
              const int ti = di, u = wk.uv0 + ti;
              const int r0 = (u % wk.tv) * kTile + ch * 8;
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (r0 + e < Rv) v[e] = umine[(ti * kTile + ch * 8 + e) * PER_KV + n];
            } else {
              const int ti = di - nvk;
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = stail[(ti * kTile + ch * 8 + e) * PER_KV + n];
            }
          }
          uint4 h4, l4;
          split8(v, h4, l4);
          unsigned char* oh = smem + L.pimg + ob * 2 * 2 * kND * 128;
          *reinterpret_cast<uint4*>(oh + bimg_off<ST>(kND, 2, ch >> 3, n, (ch & 7) * 8, false)) = h4;
          *reinterpret_cast<uint4*>(oh + bimg_off<ST>(kND, 2, ch >> 3, n, (ch & 7) * 8, true)) = l4;
          fence_proxy_async();
          named_bar(kBarBuild, 256);
          if (bt == 0) mbar_arrive(&bars[kDOpFull0 + ob]);
        }
      } else if (cw < 12) {
        int seg = -1, prev_key = -1;
        for (int di = 0; di < nd; ++di) {
          const bool is_tail = di >= nvk;
          const int u = is_tail ? wk.ut0 + (di - nvk) : wk.uv0 + di;
          const int g = is_tail ? u / wk.tt : u / wk.tv;
          const int key = is_tail ? Hkv + g : g;
          if (key == prev_key) continue;
          ++seg;
          prev_key = key;
          // segment `seg` = (kind, g): wait for its accumulator, add into owner(g)'s context
          warp_wait(&bars[kDAcc0 + (seg & 1)], (seg >> 1) & 1);
          tc_fence_after();
          float v[4];
          tld4_hilo<ST>(tmem + (static_cast<uint32_t>(qd * 32) << 16) + d_col + static_cast<uint32_t>((seg & 1) * NDW), kND, v);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[kDFree0 + (seg & 1)]);
          const int dim = qd * 32 + lane;
          if (dim < D)
#pragma unroll
            for (int y = 0; y < PER_KV; ++y)
              atomicAdd(&gpout[(g * PER_KV + y) * D + dim], v[y]);
        }
      } else if (cw == 12 && append) {
        // appended token: p_new * v_new (bf16-rounded as stored)
        for (int k = 0; k < owned; ++k) {
          const int g = c + k * C;
          if (g >= Hkv) break;
          for (int y = 0; y < PER_KV; ++y) {
            const float pn = stail[(ntt * kTile + k) * PER_KV + y];
            for (int j = lane; j < D; j += 32)
              atomicAdd(&gpout[(g * PER_KV + y) * D + j], pn * bf16r(qrow[H * D + W + g * D + j]));
          }
        }
      }
    }
    named_bar(kBarCompute, kCompute);
    if (tid == 0) mbar_arrive(&bars[kTmemFree]);  // every TMEM read (phase-D epilogues included) done
    __threadfence();
    named_bar(kBarCompute, kCompute);
    if (tid == 0) group_wait(gsync, group_arrive(gsync, C));
    named_bar(kBarCompute, kCompute);
    // owners write the context of kv heads g = c, c + C, ...
    for (int w = tid; w < owned * PER_KV * D; w += kCompute) {
      const int g = c + (w / (PER_KV * D)) * C, y = (w / D) % PER_KV, j = w % D;
      if (g >= Hkv) continue;
      const float v = __ldcg(&gpout[(g * PER_KV + y) * D + j]);
      const long oi = static_cast<long>(b) * H * D + static_cast<long>(g * PER_KV + y) * D + j;
      if (a.ctx_bf16)
        reinterpret_cast<__nv_bfloat16*>(a.ctx_out)[oi] = __float2bfloat16_rn(v);
      else
        reinterpret_cast<float*>(a.ctx_out)[oi] = v;
    }
    if (trace && tid == 0) trace[6] = global_ns();
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using LayerFn = void (*)(const LayerPlan, const FusedArgs);

template <int NP>
LayerFn pick_geom(int per_kv, int D) {
  if (D == 128) {
    if (per_kv == 1) return layer_kernel<NP, 1, 128, (NP <= 32)>;
    if (per_kv == 2) return layer_kernel<NP, 2, 128, (NP <= 32)>;
    return layer_kernel<NP, 4, 128, (NP <= 32)>;
  }
  if (per_kv == 1) return layer_kernel<NP, 1, 64, (NP <= 32)>;
  if (per_kv == 2) return layer_kernel<NP, 2, 64, (NP <= 32)>;
  return layer_kernel<NP, 4, 64, (NP <= 32)>;
}

LayerFn layer_fn(const LayerPlan& p) {
  const int per_kv = p.s.H / p.s.Hkv;
  switch (p.np) {
    case 16: return pick_geom<16>(per_kv, p.s.D);
    case 32: return pick_geom<32>(per_kv, p.s.D);
    case 48: return pick_geom<48>(per_kv, p.s.D);
    default: return pick_geom<64>(per_kv, p.s.D);
  }
}

cudaLaunchConfig_t layer_config(const LayerPlan& p, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.s.batch * p.s.cluster));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.smem_bytes;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeCooperative;  // every group's CTAs co-resident (L2 barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

}  // namespace

LayerPlan plan_layer(const FusedShape& s) {
  LayerPlan p{};
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
  if (s.n_comp < 1) return bad("fused path needs a compressed block");
  if (s.cluster < 1 || s.cluster > 16) return bad("CTAs per instance must be 1..16");
  if (s.tail_cap < 0) return bad("negative tail capacity");
  p.np = (s.H + 15) / 16 * 16;
  p.kpk = (s.rank_k + 63) / 64;
  p.vpanels = ((s.rank_v + 63) / 64 + 1) / 2 * 2;
  p.mtiles = p.vpanels / 2;
  p.vpanels_st = (s.rank_v + 63) / 64;
  p.kst = (p.kpk + 1) / 2;
  p.ntiles = (s.n_comp + 127) / 128;
  p.max_tiles = (p.ntiles + s.cluster - 1) / s.cluster;
  p.max_qh = (s.Hkv + s.cluster - 1) / s.cluster * per_kv;
  p.tpc = (s.tail_cap + s.cluster - 1) / s.cluster;
  p.stages = 2;
  const LSmem l0 = layer_smem(p);
  // TMEM (512 columns, one CTA per SM): S tiles | U tiles; the phase-A result buffers and the
  // phase-D accumulators reuse the U region (phase A ends before the U MMAs, phase D starts
  // after the U readback).  hi/lo operands stacked along N double the widths when NP <= 32.
  const bool st = p.np <= 32;
  const int npw = st ? 2 * p.np : p.np, nqw = st ? 2 * l0.nq : l0.nq, ndw = st ? 2 * kND : kND;
  const int s_cols = p.max_tiles * npw;
  if (s_cols + p.mtiles * npw > 512 || s_cols + 2 * ndw > 512)
    return bad("TMEM budget exceeded (raise the cluster size)");
  p.a_col = s_cols;
  p.d_col = s_cols;
  p.nab = std::min(kMaxAB, (512 - s_cols) / nqw);
  if (p.nab < 2) return bad("TMEM budget exceeded (raise the cluster size)");
  p.tmem_cols = 512;
  p.nob = std::min(kMaxOB, static_cast<int>((l0.opimg - l0.pimg) / (2u * 2u * 2u * kND * 128u)));
  if (p.nob < 2) return bad("phase-D operand ring does not fit");
  if (l0.total > 227 * 1024) return bad("shared-memory budget exceeded (raise the cluster size)");
  while (p.stages + 1 <= kMaxStages) {
    LayerPlan q = p;
    q.stages = p.stages + 1;
    if (layer_smem(q).total > 227 * 1024) break;
    p.stages = q.stages;
  }
  if (const char* e = std::getenv("KVP_LAYER_STAGES")) {  // tuning override
    const int want = std::atoi(e);
    if (want >= 2 && want < p.stages) p.stages = want;
  }
  if (const char* e = std::getenv("KVP_LAYER_DEBUG")) p.debug = std::atoi(e);
  p.prefetch = 4;
  if (const char* e = std::getenv("KVP_LAYER_PREFETCH")) p.prefetch = std::atoi(e);
  p.smem_bytes = layer_smem(p).total;
  p.ok = true;
  p.why = "";
  return p;
}

size_t layer_group_ws_bytes(const LayerPlan& p) { return static_cast<size_t>(p.s.batch) * group_ws(p).bytes; }

void launch_layer(const LayerPlan& p, const FusedArgs& a, cudaStream_t st) {
  require(p.ok, KVP_ERR_PARAMETER, p.why);
  const LayerFn kernel = layer_fn(p);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = layer_config(p, st, attr);
  KVP_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, a));
  KVP_LAUNCHED();
}

int layer_max_active_clusters(const LayerPlan& p) {
  const LayerFn kernel = layer_fn(p);
  KVP_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem_bytes)));
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = layer_config(p, nullptr, attr);
  int n = 0;
  KVP_CUDA(cudaOccupancyMaxActiveClusters(&n, kernel, &cfg));
  return n;
}

// CTAs per instance: as many as fit one co-resident wave (148 SMs, one CTA per
// SM), at most 16, and at least the smallest group the TMEM / smem budget allows.
int auto_layer_cluster(FusedShape s) {
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int g = std::max(1, std::min(16, sms / std::max(1, s.batch)));
  for (; g <= 16; ++g) {
    s.cluster = g;
    if (plan_layer(s).ok) return g;
  }
  return 16;
}

}  // namespace kvp
