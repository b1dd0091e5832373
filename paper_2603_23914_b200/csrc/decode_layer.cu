// Compressed-cache decode attention for one layer in ONE launch (bf16
// storage, T_q = 1) — the serving hot path.  Replaces the reference's
// per-(instance, layer) loop decoder.cpp:555-601 (build_retrieval_plan ->
// attend_{materialized,fused} -> head average -> update_importance), whose
// cost is ~100% row rebuilding in store_decompress_row (cache.cpp:63-101).
// Nothing of width W = H_kv*D is rebuilt and every cache byte is read once.
//
// One thread-block cluster of C CTAs per instance.  right_k / right_v /
// tail_k / tail_v are stored head-major ([batch][H_kv][rows][D]); viewed as
// flat row arrays they are split into C equal contiguous row ranges (right
// factors in units of 8 ranks, so a P chunk never straddles two CTAs), and
// the 128-token tiles of the packed left factors are split evenly.  A single
// TMA ring of 32 KB stages carries, in this order:
//   A  my right_k rows, my tail_k rows                                     (CUDA cores)
//        P[h, r] = right_k[g, r, :].q_h/sqrt(D) -> bf16 hi/lo swizzled chunks pushed to every
//        peer's operand image (DSMEM);  s_tail[h, t] = tail_k[g, t, :].q_h/sqrt(D)
//   B  left_k tiles:  S[t, h] = left_k[t, :].P[h, :]     tcgen05, M=128 tokens, N=heads; S stays in TMEM
//        local (m, z) per head (tiles + my tail rows), exchanged once through DSMEM
//   C  left_v tiles:  U^T[r, h] += left_v[t, r] p[t, h]   tcgen05, M=128 ranks, N=heads
//        importance EMA (importance.cpp:33-65) from the head average, fp64, reference op order
//        U partials gathered for my right_v rows, normalised
//   D  my right_v rows, my tail_v rows: out partials U[h, r] right_v[g, r, :] + p[h, t] tail_v[g, t, :],
//        reduced into the head owner's smem with DSMEM atomics; owners write the context.
// Every address is known at launch, so the producer keeps streaming the next
// phase's bytes while the consumers cross a cluster exchange.  Consumers copy
// a stage into registers and release it before doing arithmetic.
//
// Warp roles (576 threads): warp 0 = TMA producer, warp 1 = MMA issuer +
// TMEM owner, warps 2..17 = compute (phases A and D, softmax, EMA, DSMEM).
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
constexpr uint32_t kStage = 32768;  // ring stage: 32 KB bulk copies (measured on B200: the per-SM
                                    // stream rate of a warp-specialised ring scales with the copy
                                    // size — ~40 GB/s at 16 KB, ~70 GB/s at 32 KB)
constexpr uint32_t kPanel = 16384;  // one packed 128 x 64 bf16 operand panel
constexpr int kThreads = 576;
constexpr int kCompute = 512;
constexpr int kCWarps = 16;
constexpr uint32_t kBarCompute = 1;

template <int D>
constexpr int item_rows() { return 16384 / D; }  // rows of one 32 KB right/tail item
__host__ __device__ inline int item_rows_rt(int D) { return 16384 / D; }

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Upper bounds of the per-CTA ranges (rows of the flat head-major arrays).
__host__ __device__ inline int max_right_rows(int Hkv, int R, int C) {
  const long units = static_cast<long>(Hkv) * ((R + 7) / 8);
  return static_cast<int>((units + C - 1) / C) * 8;
}
__host__ __device__ inline int max_tail_rows(int Hkv, int cap, int C) {
  return static_cast<int>((static_cast<long>(Hkv) * cap + C - 1) / C);
}

struct LSmem {
  uint32_t ring, pimg, umine, stail, hatp, dscr, qs, pout, part, stats, imps, bars, desc, tslot, total;
  int uv;         // fp32 row stride of the U partial [NP][uv]
  int qslots;     // q slots per range (kv heads a range can touch)
};

__host__ __device__ inline LSmem layer_smem(const LayerPlan& p) {
  LSmem s{};
  const uint32_t np = p.np;
  const int per_kv = p.s.H / p.s.Hkv, C = p.s.cluster, D = p.s.D;
  s.uv = static_cast<int>(align_up(p.s.rank_v, 4));
  s.qslots = (p.s.Hkv + C - 1) / C + 2;
  const uint32_t rows_kv = static_cast<uint32_t>(
      max(max_right_rows(p.s.Hkv, p.s.rank_k, C), max_right_rows(p.s.Hkv, p.s.rank_v, C)));
  s.ring = 0;
  s.pimg = s.ring + p.stages * kStage;
  uint32_t pimg_bytes = 2u * p.kpk * np * 128;                          // P operand (hi, lo)
  pimg_bytes = max(pimg_bytes, 8u * np * 128);                          // p tiles: 2 buffers x {hi, lo} x 2 panels
  pimg_bytes = max(pimg_bytes, np * static_cast<uint32_t>(s.uv) * 4u);  // U partial [NP][uv] (DSMEM-read)
  s.umine = align_up(s.pimg + pimg_bytes, 16);                          // P_local, later U_mine [rows][per_kv]
  s.stail = align_up(s.umine + rows_kv * per_kv * 4u, 16);              // s_tail -> p_tail [rows][per_kv]
  s.hatp = align_up(s.stail + (max_tail_rows(p.s.Hkv, p.s.tail_cap, C) + 1u) * per_kv * 4u, 16);  // [cap]
  s.dscr = align_up(s.hatp + static_cast<uint32_t>(p.s.tail_cap) * 4u, 16);  // [16][D]
  s.qs = s.dscr + kCWarps * D * 4u;                                     // [2 ranges][qslots][per_kv][D]
  s.pout = s.qs + 2u * s.qslots * per_kv * D * 4u;                      // owned heads' context [owned][per_kv][D]
  s.part = s.pout + static_cast<uint32_t>((p.s.Hkv + C - 1) / C) * per_kv * D * 4u;
  s.stats = s.part + 2u * kCWarps * np * 4u + 4u * 128u * 4u;
  s.imps = align_up(s.stats + (5u + 8u) * np * 4u, 16);
  s.bars = align_up(s.imps + (p.max_tiles * 128u + p.tpc) * 8u, 8);
  s.desc = align_up(s.bars + 48 * 8, 16);  // [stages] int4 item descriptors (phase A / D)
  s.tslot = s.desc + kMaxStages * 16;
  s.total = align_up(s.tslot + 16, 1024);
  return s;
}

enum Bar : int {
  kFull = 0,                 // [stages] data landed
  kEmpty = kMaxStages,       // [stages] released by the 16 compute warps (phase A / D items)
  kMmaDone = 2 * kMaxStages, // [stages] released by the MMAs (phase B / C items)
  kSFull = 3 * kMaxStages,   // S MMAs complete
  kPFull0, kPFull1,         // p tile buffer written
  kPEmpty0, kPEmpty1,       // p tile buffer consumed
  kUFull,                   // U MMAs complete
  kTmemFree,
  kPReady,                  // cluster: every peer pushed its P chunks (count C)
  kStats,                   // cluster: (m, z) published (count C)
  kUReady,                  // cluster: U partials + tail head sums published (count C)
  kOut,                     // cluster: every peer added its context partials (count C)
  kNumBars
};

// Rows [f, e) of a flat head-major array with `per` rows per head; rows r >= lm
// of a head are not in memory (the appended tail row).  Items are cut at head
// boundaries and at `ir` rows.
struct ItemIter {
  int cur, e, per, lm, ir;
  __host__ __device__ bool next(int& g, int& r0, int& rows) {
    while (cur < e) {
      g = cur / per;
      r0 = cur - g * per;
      const int hend = min(e, (g + 1) * per);
      const int mend = min(hend, g * per + lm);
      if (cur < mend) {
        rows = min(ir, mend - cur);
        cur += rows;
        return true;
      }
      cur = hend;
    }
    return false;
  }
  __host__ __device__ int count() const {
    ItemIter t = *this;
    int g, r0, rows, n = 0;
    while (t.next(g, r0, rows)) ++n;
    return n;
  }
};

struct Work {
  int tile0, tiles;  // 128-token tiles (phases B, C)
  int ka, kb;        // right_k flat rows [ka, kb) over [H_kv][rank_k]
  int va, vb;        // right_v flat rows over [H_kv][rank_v]
  int ta, tb;        // tail flat rows over [H_kv][n_tail] (n_tail includes the appended row)
  int n_mem;         // tail rows per head in memory
  int nak, ndk;      // right-factor items of phases A and D (the tail items follow them)
  int na, lv0, d0;   // first item index of phases B, C, D
  int total;
};

__host__ __device__ inline int unit_row(long u, int R) {
  const int uph = (R + 7) / 8;
  return static_cast<int>(u / uph) * R + min(R, static_cast<int>(u % uph) * 8);
}

__host__ __device__ inline Work make_work(const LayerPlan& p, int c, int n_tail, int append) {
  Work w;
  const int C = p.s.cluster, Hkv = p.s.Hkv;
  const int tb = p.ntiles / C, tr = p.ntiles % C;
  w.tiles = tb + (c < tr ? 1 : 0);
  w.tile0 = c * tb + min(c, tr);
  const long uk = static_cast<long>(Hkv) * ((p.s.rank_k + 7) / 8);
  const long uv = static_cast<long>(Hkv) * ((p.s.rank_v + 7) / 8);
  w.ka = unit_row(uk * c / C, p.s.rank_k);
  w.kb = unit_row(uk * (c + 1) / C, p.s.rank_k);
  w.va = unit_row(uv * c / C, p.s.rank_v);
  w.vb = unit_row(uv * (c + 1) / C, p.s.rank_v);
  const long nt = static_cast<long>(Hkv) * n_tail;
  w.ta = static_cast<int>(nt * c / C);
  w.tb = static_cast<int>(nt * (c + 1) / C);
  w.n_mem = max(0, n_tail - (append ? 1 : 0));
  const int ir = item_rows_rt(p.s.D);
  w.nak = ItemIter{w.ka, w.kb, p.s.rank_k, p.s.rank_k, ir}.count();
  w.ndk = ItemIter{w.va, w.vb, p.s.rank_v, p.s.rank_v, ir}.count();
  const int nat = ItemIter{w.ta, w.tb, max(n_tail, 1), w.n_mem, ir}.count();
  w.na = w.nak + nat;
  w.lv0 = w.na + w.tiles * p.kst;      // K: panel pairs per stage
  w.d0 = w.lv0 + w.tiles * p.mtiles;   // V: one 128-rank pair per stage
  w.total = w.d0 + w.ndk + nat;
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
__device__ __forceinline__ void unpack8(const uint4& raw, float (&v)[8]) {
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h2[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
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

// Compute-warp waits: one thread polls the mbarrier, the rest park on a named barrier.
__device__ __forceinline__ void cta_wait(uint64_t* bar, uint32_t parity, int tid) {
  if (tid == 0) mbar_wait(bar, parity);
  named_bar(kBarCompute, kCompute);
}
__device__ __forceinline__ void cta_wait_cluster(uint64_t* bar, uint32_t parity, int tid) {
  if (tid == 0) mbar_wait_cluster(bar, parity);
  named_bar(kBarCompute, kCompute);
}
// Release a ring stage once every compute thread copied it into registers.
__device__ __forceinline__ void cta_release(uint64_t* bar, int tid) {
  named_bar(kBarCompute, kCompute);
  if (tid == 0) mbar_arrive(bar);
}

template <int NP, int PER_KV, int D>
__global__ void __launch_bounds__(kThreads, 1) layer_kernel(const LayerPlan p, const FusedArgs a) {
  constexpr int IR = item_rows<D>();
  constexpr int TPR = D / 16;                 // phase A: threads per row (16 elements each)
  constexpr int APASS = IR * TPR / kCompute;  // phase A: row passes per item
  constexpr int CPR = D / 8;                  // phase D: 16-byte chunks per row
  constexpr int RG = kCompute / CPR;          // phase D: row groups
  constexpr int DROWS = IR / RG;              // phase D: rows per thread per item
  extern __shared__ __align__(1024) unsigned char smem[];
  const LSmem L = layer_smem(p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L.tslot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.s.cluster;
  const int c = static_cast<int>(cluster_rank());
  const int b = blockIdx.x / C;
  const int H = p.s.H, Hkv = p.s.Hkv, W = Hkv * D, cap = p.s.tail_cap;
  const int Rk = p.s.rank_k, Rv = p.s.rank_v;
  const int n_tail = a.n_tail_dev ? *a.n_tail_dev : a.n_tail;
  const int tper = max(n_tail, 1);  // rows per head of the flat tail array
  const Work wk = make_work(p, c, n_tail, a.append_kv);
  const uint32_t s_cols = static_cast<uint32_t>(p.max_tiles * NP);
  const int NS = p.stages;
  const uint32_t plane = static_cast<uint32_t>(p.kpk) * NP * 128;  // bytes of one (hi or lo) P operand
  const int owned = (Hkv + C - 1) / C;                               // kv heads g with g % C == c
  unsigned long long* trace = a.trace ? a.trace + blockIdx.x * 16ull : nullptr;
  // per-item clock64 trace of CTA 0 (debug): [issue, acquire, release] x item
  unsigned long long* ict = (a.trace && blockIdx.x == 0) ? a.trace + gridDim.x * 16ull : nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[kFull + s], 1);
      mbar_init(&bars[kEmpty + s], kCWarps);
      mbar_init(&bars[kMmaDone + s], 1);
    }
    for (int i = kSFull; i <= kTmemFree; ++i) mbar_init(&bars[i], 1);
    for (int i = kPReady; i <= kOut; ++i) mbar_init(&bars[i], C);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, static_cast<uint32_t>(p.tmem_cols));
  if (warp >= 2) {
    const int tid = threadIdx.x - 64;
    // zero the P operand image rows h >= H and rank chunks past the last pushed unit
    const int uph = (Rk + 7) / 8;
    for (int i = tid; i < NP * p.kpk * 8; i += kCompute) {
      const int h = i / (p.kpk * 8), ch = i % (p.kpk * 8);
      if (h < H && ch < uph) continue;
      const uint32_t off = (ch >> 3) * NP * 128 + sw128_off(h, (ch & 7) * 8);
      *reinterpret_cast<uint4*>(smem + L.pimg + off) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(smem + L.pimg + plane + off) = make_uint4(0, 0, 0, 0);
    }
    float* pout = reinterpret_cast<float*>(smem + L.pout);
    for (int i = tid; i < owned * PER_KV * D; i += kCompute) pout[i] = 0.f;
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's barriers and zeroed buffers exist before any remote access
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ============================ producer ============================
    if (lane == 0) {
      int i = 0;
      // per stage: was the previous occupant consumed by the MMAs (bit set) or the compute
      // warps, and the phase parity of each release barrier
      uint32_t prev_mma = 0, eph = 0, mph = 0;
      int4* desc = reinterpret_cast<int4*>(smem + L.desc);
      auto stage = [&](uint32_t bytes, bool mma_item) -> unsigned char* {
        const int s = i % NS;
        if (i >= NS) {
          if ((prev_mma >> s) & 1) {
            mbar_wait(&bars[kMmaDone + s], (mph >> s) & 1);
            mph ^= 1u << s;
          } else {
            mbar_wait(&bars[kEmpty + s], (eph >> s) & 1);
            eph ^= 1u << s;
          }
        }
        prev_mma = mma_item ? (prev_mma | (1u << s)) : (prev_mma & ~(1u << s));
        return smem + L.ring + s * kStage;
      };
      auto rows_phase = [&](ItemIter itr, const __nv_bfloat16* base, int head_rows) {
        int g, r0, rows;
        while (itr.next(g, r0, rows)) {
          const uint32_t bytes = static_cast<uint32_t>(rows) * D * 2;
          unsigned char* dst = stage(bytes, false);
          desc[i % NS] = make_int4(g, r0, rows, 0);
          mbar_expect_tx(&bars[kFull + i % NS], bytes);
          bulk_load(dst, base + ((static_cast<long>(b) * Hkv + g) * head_rows + r0) * D, bytes,
                    &bars[kFull + i % NS]);
          if (ict && i < 512) ict[3 * i] = clock64();
          ++i;
        }
      };
      rows_phase(ItemIter{wk.ka, wk.kb, Rk, Rk, IR}, a.right_k, Rk);
      rows_phase(ItemIter{wk.ta, wk.tb, tper, wk.n_mem, IR}, a.tail_k, cap);
      if (p.debug & 8) return;
      for (int t = 0; t < wk.tiles; ++t) {  // left_k: panels (2pp, 2pp+1) of a tile, contiguous when packed
        const long gtile = static_cast<long>(a.inst0 + b) * p.ntiles + wk.tile0 + t;
        for (int pp = 0; pp < p.kst; ++pp) {
          const uint32_t bytes = static_cast<uint32_t>(min(2, p.kpk - 2 * pp)) * kPanel;
          unsigned char* dst = stage(bytes, true);
          mbar_expect_tx(&bars[kFull + i % NS], bytes);
          bulk_load(dst, a.left_k_packed + (gtile * p.kpk + 2 * pp) * static_cast<long>(kPanel), bytes,
                    &bars[kFull + i % NS]);
          if (ict && i < 512) ict[3 * i] = clock64();
          ++i;
        }
      }
      for (int t = 0; t < wk.tiles; ++t) {  // left_v: 128-rank panel pairs (a missing odd panel stays
                                            // unloaded: U rows >= rank_v are never read)
        const long gtile = static_cast<long>(a.inst0 + b) * p.ntiles + wk.tile0 + t;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const uint32_t bytes = static_cast<uint32_t>(min(2, p.vpanels_st - 2 * mt)) * kPanel;
          unsigned char* dst = stage(bytes, true);
          mbar_expect_tx(&bars[kFull + i % NS], bytes);
          bulk_load(dst, a.left_v_packed + (gtile * p.vpanels_st + 2 * mt) * static_cast<long>(kPanel), bytes,
                    &bars[kFull + i % NS]);
          if (ict && i < 512) ict[3 * i] = clock64();
          ++i;
        }
      }
      rows_phase(ItemIter{wk.va, wk.vb, Rv, Rv, IR}, a.right_v, Rv);
      rows_phase(ItemIter{wk.ta, wk.tb, tper, wk.n_mem, IR}, a.tail_v, cap);
      if (trace) trace[7] = global_ns();
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, NP, false, false);
      const uint32_t idesc_u = idesc_bf16(128, NP, true, false);
      const uint32_t ring = smem_addr(smem + L.ring);
      const uint32_t phi = smem_addr(smem + L.pimg), plo = phi + plane;
      const uint32_t pt = smem_addr(smem + L.pimg);  // p tiles reuse the P image once S is done
      if (!(p.debug & 8)) {
      mbar_wait_cluster(&bars[kPReady], 0);
      fence_proxy_async_all();
      tc_fence_after();
      if (trace) trace[8] = global_ns();
      for (int t = 0; t < wk.tiles; ++t) {
        for (int pp = 0; pp < p.kst; ++pp) {
          const int i = wk.na + t * p.kst + pp, s = i % NS;
          mbar_wait(&bars[kFull + s], (i / NS) & 1);
          if (ict && i < 512) ict[3 * i + 1] = clock64();
          tc_fence_after();
          for (int q = 0; q < 2 && 2 * pp + q < p.kpk; ++q) {
            const int kp = 2 * pp + q;
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = smem_desc(ring + s * kStage + q * kPanel + kk * 32, 16, 1024, kSwizzle128B);
              const uint64_t bh = smem_desc(phi + kp * NP * 128 + kk * 32, 16, 1024, kSwizzle128B);
              const uint64_t bl = smem_desc(plo + kp * NP * 128 + kk * 32, 16, 1024, kSwizzle128B);
              const uint32_t d = tmem + static_cast<uint32_t>(t * NP);
              mma_bf16(d, ad, bh, idesc_s, (kp | kk) != 0);
              mma_bf16(d, ad, bl, idesc_s, 1);
            }
          }
          mma_commit(&bars[kMmaDone + s]);
        }
      }
      mma_commit(&bars[kSFull]);
      for (int t = 0; t < wk.tiles; ++t) {
        const int buf = t & 1;
        mbar_wait(&bars[kPFull0 + buf], (t >> 1) & 1);
        tc_fence_after();
        const uint32_t pth = pt + buf * 4 * NP * 128, ptl = pth + 2 * NP * 128;
        for (int mt = 0; mt < p.mtiles; ++mt) {
          const int i0 = wk.lv0 + t * p.mtiles + mt, s0 = i0 % NS;
          mbar_wait(&bars[kFull + s0], (i0 / NS) & 1);
          if (ict && i0 < 512) ict[3 * i0 + 1] = clock64();
          tc_fence_after();
          const uint32_t d = tmem + s_cols + static_cast<uint32_t>(mt * NP);
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t ad = smem_desc(ring + s0 * kStage + ks * 2048, kPanel, 1024, kSwizzle128B);
            const uint32_t boff = (ks >> 2) * NP * 128 + (ks & 3) * 32;
            const uint64_t bh = smem_desc(pth + boff, 16, 1024, kSwizzle128B);
            const uint64_t bl = smem_desc(ptl + boff, 16, 1024, kSwizzle128B);
            mma_bf16(d, ad, bh, idesc_u, (t | ks) != 0);
            mma_bf16(d, ad, bl, idesc_u, 1);
          }
          mma_commit(&bars[kMmaDone + s0]);
        }
        mma_commit(&bars[kPEmpty0 + buf]);
      }
      mma_commit(&bars[kUFull]);
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
    const float scale = rsqrtf(static_cast<float>(D));
    float* plocal = reinterpret_cast<float*>(smem + L.umine);  // phase A: P for my right_k rows [row][y]
    float* umine = plocal;                                      // phase D: U for my right_v rows [row][y]
    float* stail = reinterpret_cast<float*>(smem + L.stail);   // my tail rows [row][y]: logits -> p
    float* hatp = reinterpret_cast<float*>(smem + L.hatp);     // [cap]: my rows' share of the head average
    float* dscr = reinterpret_cast<float*>(smem + L.dscr);
    float* qs = reinterpret_cast<float*>(smem + L.qs);
    float* pout = reinterpret_cast<float*>(smem + L.pout);
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
    const int gk0 = wk.ka / Rk, gt0 = wk.ta / tper;  // first kv head of my right_k / tail ranges
    const int ntr = wk.tb - wk.ta;                    // my tail rows (flat)
    if (trace && tid == 0) trace[0] = global_ns();

    // stage the scaled queries of the kv heads my two phase-A ranges touch
    for (int i = tid; i < 2 * L.qslots * PER_KV * D; i += kCompute) {
      const int rng = i / (L.qslots * PER_KV * D), rem = i % (L.qslots * PER_KV * D);
      const int g = (rng == 0 ? gk0 : gt0) + rem / (PER_KV * D), hy = rem % (PER_KV * D);
      qs[i] = g < Hkv ? qrow[g * PER_KV * D + hy] * scale : 0.f;
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
    named_bar(kBarCompute, kCompute);

    // ---------------- phase A: P = right_k . q, tail logits ----------------
    {
      const int arow = tid / TPR, aseg = tid % TPR;
      int i = 0;
      float qv[PER_KV][16];  // this thread's query segment of the current kv head (reloaded per head)
      int q_loaded = -1;
      const int4* desc = reinterpret_cast<const int4*>(smem + L.desc);
      for (; i < wk.na; ++i) {
        {
          const bool is_tail = i >= wk.nak;
          const int s = i % NS;
          // per-warp wait: the 16 compute warps stream through the ring independently
          if (lane == 0) mbar_wait(&bars[kFull + s], (i / NS) & 1);
          __syncwarp();
          const int4 dsc = desc[s];
          const int g = dsc.x, r0 = dsc.y, rows = dsc.z;
          const int qkey = is_tail ? Hkv + g : g;
          if (qkey != q_loaded && !(p.debug & 1)) {  // issue before the wait: latency hidden by it
            const float* qg = qs + ((is_tail ? L.qslots + g - gt0 : g - gk0) * PER_KV) * D;
#pragma unroll
            for (int y = 0; y < PER_KV; ++y) {
              const float4* q0 = reinterpret_cast<const float4*>(qg + y * D + aseg * 8);
              const float4* q1 = reinterpret_cast<const float4*>(qg + y * D + D / 2 + aseg * 8);
              const float4 a0 = q0[0], a1 = q0[1], b0 = q1[0], b1 = q1[1];
              qv[y][0] = a0.x; qv[y][1] = a0.y; qv[y][2] = a0.z; qv[y][3] = a0.w;
              qv[y][4] = a1.x; qv[y][5] = a1.y; qv[y][6] = a1.z; qv[y][7] = a1.w;
              qv[y][8] = b0.x; qv[y][9] = b0.y; qv[y][10] = b0.z; qv[y][11] = b0.w;
              qv[y][12] = b1.x; qv[y][13] = b1.y; qv[y][14] = b1.z; qv[y][15] = b1.w;
            }
            q_loaded = qkey;
          }
          if (ict && tid == 0 && i < 512) ict[3 * i + 1] = clock64();
          uint4 raw[APASS][2];
#pragma unroll
          for (int ps = 0; ps < APASS; ++ps) {
            const unsigned char* src = smem + L.ring + s * kStage + (ps * (kCompute / TPR) + arow) * D * 2;
            raw[ps][0] = *reinterpret_cast<const uint4*>(src + aseg * 16);
            raw[ps][1] = *reinterpret_cast<const uint4*>(src + D + aseg * 16);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[kEmpty + s]);
          if (ict && tid == 0 && i < 512) ict[3 * i + 2] = clock64();
          if (p.debug & 1) continue;
          const int flat0 = g * (is_tail ? tper : Rk) + r0 - (is_tail ? wk.ta : wk.ka);
#pragma unroll
          for (int y = 0; y < PER_KV; ++y) {
#pragma unroll
            for (int ps = 0; ps < APASS; ++ps) {
              const int row = ps * (kCompute / TPR) + arow;
              float v0[8], v1[8];
              unpack8(raw[ps][0], v0);
              unpack8(raw[ps][1], v1);
              float t0 = 0.f, t1 = 0.f;
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                t0 = fmaf(v0[e], qv[y][e], t0);
                t1 = fmaf(v1[e], qv[y][8 + e], t1);
              }
              float t = t0 + t1;
              if (!(p.debug & 16)) {
#pragma unroll
                for (int o = TPR / 2; o >= 1; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
              }
              if (aseg == 0 && row < rows) (is_tail ? stail : plocal)[(flat0 + row) * PER_KV + y] = t;
            }
          }
        }
      };
    }
    if (p.debug & 8) {
      if (trace && tid == 0) trace[1] = global_ns();
      named_bar(kBarCompute, kCompute);
      if (tid == 0) mbar_arrive(&bars[kTmemFree]);
      return;
    }
    // appended token (row n_tail - 1 of every kv head whose flat index is mine): k, v straight
    // from the projection, bf16-rounded as stored; written back to the tail (cache.cpp:147-170)
    if (a.append_kv && n_tail > 0) {
      for (int w = cw; w < Hkv * PER_KV; w += kCWarps) {
        const int g = w / PER_KV, y = w % PER_KV;
        const int f = g * tper + n_tail - 1;
        if (f < wk.ta || f >= wk.tb) continue;
        const int h = g * PER_KV + y;
        float t = 0.f;
        for (int j = lane; j < D; j += 32) t = fmaf(bf16r(qrow[H * D + g * D + j]), qrow[h * D + j] * scale, t);
        t = warp_sum(t);
        if (lane == 0) stail[(f - wk.ta) * PER_KV + y] = t;
        if (y == 0) {
          const long row = (static_cast<long>(b) * Hkv + g) * cap + (n_tail - 1);
          __nv_bfloat16* tk = const_cast<__nv_bfloat16*>(a.tail_k) + row * D;
          __nv_bfloat16* tv = const_cast<__nv_bfloat16*>(a.tail_v) + row * D;
          for (int j = lane; j < D; j += 32) {
            tk[j] = __float2bfloat16_rn(qrow[H * D + g * D + j]);
            tv[j] = __float2bfloat16_rn(qrow[H * D + W + g * D + j]);
          }
        }
      }
    }
    named_bar(kBarCompute, kCompute);
    // push my P units (8 ranks of one kv head, bf16 hi/lo 16-byte chunks) into every peer's image
    {
      const int uph = (Rk + 7) / 8;
      const long uk = static_cast<long>(Hkv) * uph;
      const long u0 = uk * c / C, u1 = uk * (c + 1) / C;
      for (long w = tid; w < (u1 - u0) * PER_KV; w += kCompute) {
        const long u = u0 + w / PER_KV;
        const int y = static_cast<int>(w % PER_KV);
        const int g = static_cast<int>(u / uph), kc = static_cast<int>(u % uph), r0 = kc * 8;
        const int h = g * PER_KV + y;
        const int flat0 = g * Rk + r0 - wk.ka;
        __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float v = r0 + e < Rk ? plocal[(flat0 + e) * PER_KV + y] : 0.f;
          split_bf16(v, hi[e], lo[e]);
        }
        const uint32_t off = (kc >> 3) * NP * 128 + sw128_off(h, (kc & 7) * 8);
        const uint4 h4 = *reinterpret_cast<const uint4*>(hi), l4 = *reinterpret_cast<const uint4*>(lo);
        for (int peer = 0; peer < C; ++peer) {
          st_dsmem_v4(smem + L.pimg + off, static_cast<uint32_t>(peer), h4);
          st_dsmem_v4(smem + L.pimg + plane + off, static_cast<uint32_t>(peer), l4);
        }
      }
    }
    fence_proxy_async_all();
    fence_acq_rel_cluster();
    named_bar(kBarCompute, kCompute);
    if (tid < C) mbar_arrive_cluster(&bars[kPReady], static_cast<uint32_t>(tid));
    if (trace && tid == 0) trace[1] = global_ns();

    // ---------------- phase B epilogue: local softmax statistics ----------------
    const int qd = warp & 3;       // TMEM lane quadrant this warp may access
    const int cg = cw >> 2;        // column group 0..3
    constexpr int gcols = NP / 4;
    const int gbase = cg * gcols;
    auto tmem_row = [&](uint32_t col) { return tmem + (static_cast<uint32_t>(qd * 32) << 16) + col; };
    // heads my tail rows touch: kv heads gt0 .. gt1
    const int gt1 = ntr > 0 ? (wk.tb - 1) / tper : gt0 - 1;
    cta_wait(&bars[kSFull], 0, tid);
    tc_fence_after();
    if (trace && tid == 0) trace[2] = global_ns();
    float* part_m = part;
    float* part_s = part + kCWarps * NP;
    for (int c0 = 0; c0 < gcols; c0 += 4) {
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      for (int t = 0; t < wk.tiles; ++t) {
        float v[4];
        tmem_ld4(tmem_row(static_cast<uint32_t>(t * NP + gbase + c0)), v);
        if (t * 128 + qd * 32 + lane < chunk_len)
          for (int e = 0; e < 4; ++e) mx[e] = fmaxf(mx[e], v[e]);
      }
      for (int e = 0; e < 4; ++e) {
        const float m = warp_max(mx[e]);
        if (lane == 0) part_m[cw * NP + gbase + c0 + e] = m;
      }
    }
    named_bar(kBarCompute, kCompute);
    if (tid < H) {
      const int h = tid, g = h / PER_KV, y = h % PER_KV, w0 = (h / gcols) * 4;
      float m = -INFINITY;
      for (int w = 0; w < 4; ++w) m = fmaxf(m, part_m[(w0 + w) * NP + h]);
      if (g >= gt0 && g <= gt1) {
        const int f0 = max(wk.ta, g * tper), f1 = min(wk.tb, (g + 1) * tper);
        for (int f = f0; f < f1; ++f) m = fmaxf(m, stail[(f - wk.ta) * PER_KV + y]);
      }
      m_loc[h] = m;
    }
    named_bar(kBarCompute, kCompute);

    // ---------------- p tiles (bf16 hi/lo, K-major over tokens) -> U MMAs ----------------
    float zp[gcols];
#pragma unroll
    for (int e = 0; e < gcols; ++e) zp[e] = 0.f;
    for (int t = 0; t < wk.tiles; ++t) {
      const int buf = t & 1;
      if (t >= 2) cta_wait(&bars[kPEmpty0 + buf], ((t - 2) >> 1) & 1, tid);
      unsigned char* pth = smem + L.pimg + buf * 4 * NP * 128;
      unsigned char* ptl = pth + 2 * NP * 128;
      const int row = qd * 32 + lane;
      const bool valid = t * 128 + row < chunk_len;
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
      named_bar(kBarCompute, kCompute);
      if (tid == 0) mbar_arrive(&bars[kPFull0 + buf]);
    }
#pragma unroll
    for (int c0 = 0; c0 < gcols; ++c0) {
      const float z = warp_sum(zp[c0]);
      if (lane == 0) part_s[cw * NP + gbase + c0] = z;
    }
    // my tail rows: local p in place of the logits
    for (int w = tid; w < ntr * PER_KV; w += kCompute) {
      const int f = wk.ta + w / PER_KV, y = w % PER_KV, h = (f / tper) * PER_KV + y;
      stail[w] = __expf(stail[w] - m_loc[h]);
    }
    named_bar(kBarCompute, kCompute);
    if (tid < H) {
      const int h = tid, g = h / PER_KV, y = h % PER_KV, w0 = (h / gcols) * 4;
      float z = 0.f;
      for (int w = 0; w < 4; ++w) z += part_s[(w0 + w) * NP + h];
      if (g >= gt0 && g <= gt1) {
        const int f0 = max(wk.ta, g * tper), f1 = min(wk.tb, (g + 1) * tper);
        for (int f = f0; f < f1; ++f) z += stail[(f - wk.ta) * PER_KV + y];
      }
      z_loc[h] = z;
    }
    if (trace && tid == 0) trace[3] = global_ns();

    // ---------------- cluster statistics (while the U MMAs run) ----------------
    named_bar(kBarCompute, kCompute);
    if (tid < C) mbar_arrive_cluster(&bars[kStats], static_cast<uint32_t>(tid));
    cta_wait_cluster(&bars[kStats], 0, tid);
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
    named_bar(kBarCompute, kCompute);

    // ---------------- head average + importance EMA of my compressed tokens ----------------
    float* ha_part = part;  // [4 groups][128]
    const float inv_h = 1.0f / static_cast<float>(H);
    for (int t = 0; t < wk.tiles; ++t) {
      const int row = qd * 32 + lane;
      float hsum = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4];
        tmem_ld4(tmem_row(static_cast<uint32_t>(t * NP + gbase + c0)), v);
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
    // my tail rows: normalised p, and their share of the head average
    for (int w = tid; w < ntr * PER_KV; w += kCompute) {
      const int f = wk.ta + w / PER_KV, y = w % PER_KV, h = (f / tper) * PER_KV + y;
      const float pv = stail[w] * f_me[h];
      stail[w] = pv;
      atomicAdd(&hatp[f % tper], pv);
    }

    // ---------------- U readback, gather U for my right_v rows ----------------
    cta_wait(&bars[kUFull], 0, tid);
    tc_fence_after();
    if (trace && tid == 0) trace[4] = global_ns();
    float* uloc = reinterpret_cast<float*>(smem + L.pimg);  // [NP][uv], peers read it
    for (int mt = 0; mt < p.mtiles; ++mt) {
      const int r = mt * 128 + qd * 32 + lane;
#pragma unroll
      for (int c0 = 0; c0 < gcols; c0 += 4) {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (wk.tiles > 0) tmem_ld4(tmem_row(s_cols + static_cast<uint32_t>(mt * NP + gbase + c0)), v);
        for (int e = 0; e < 4; ++e) {
          const int h = gbase + c0 + e;
          if (h < H && r < Rv) uloc[h * L.uv + r] = v[e];
        }
      }
    }
    tc_fence_before();
    named_bar(kBarCompute, kCompute);
    if (tid == 0) mbar_arrive(&bars[kTmemFree]);
    if (tid < C) mbar_arrive_cluster(&bars[kUReady], static_cast<uint32_t>(tid));
    cta_wait_cluster(&bars[kUReady], 0, tid);
    for (int w = tid; w < (wk.vb - wk.va) * PER_KV; w += kCompute) {
      const int f = wk.va + w / PER_KV, y = w % PER_KV;
      const int g = f / Rv, r = f - g * Rv, h = g * PER_KV + y;
      float u[8];
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) u[peer] = ld_dsmem_f32(&uloc[h * L.uv + r], static_cast<uint32_t>(peer));
      float acc = 0.f;
#pragma unroll
      for (int peer = 0; peer < 8; ++peer)
        if (peer < C) acc = fmaf(scale_c[peer * NP + h], u[peer], acc);
      umine[w] = acc * zi_g[h];
    }
    // tail tokens t_lo..t_hi: head average over every peer's rows, EMA
    for (int t = t_lo + tid; t < t_hi; t += kCompute) {
      float hs = 0.f;
      for (int peer = 0; peer < C; ++peer) hs += ld_dsmem_f32(&hatp[t], static_cast<uint32_t>(peer));
      const float ha = hs * inv_h;
      const long gi = p.s.n_comp + t;
      if (a.head_avg) a.head_avg[static_cast<long>(b) * (p.s.n_comp + cap) + gi] = ha;
      if (a.importance)
        a.importance[static_cast<long>(b) * a.imp_stride + gi] =
            __dadd_rn(__dmul_rn(a.ema_decay, imps[p.max_tiles * 128 + (t - t_lo)]),
                      __dmul_rn(a.ema_blend, static_cast<double>(ha)));
    }
    named_bar(kBarCompute, kCompute);  // umine visible to every compute warp
    if (trace && tid == 0) trace[5] = global_ns();

    // ---------------- phase D: context partials -> head owners (DSMEM atomics) ----------------
    {
      const int cc = tid % CPR, rg = tid / CPR;
      int i = wk.d0;
      int cur_g = -1;
      float acc[PER_KV][8];
#pragma unroll
      for (int y = 0; y < PER_KV; ++y)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[y][e] = 0.f;
      auto flush = [&](int g) {  // reduce the row groups, add into owner(g)'s context accumulator
#pragma unroll
        for (int y = 0; y < PER_KV; ++y) {
#pragma unroll
          for (int o = CPR; o < 32; o <<= 1)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[y][e] += __shfl_xor_sync(0xffffffffu, acc[y][e], o);
          if (lane < CPR) {
            float* dst = dscr + cw * D + cc * 8;
            *reinterpret_cast<float4*>(dst) = make_float4(acc[y][0], acc[y][1], acc[y][2], acc[y][3]);
            *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[y][4], acc[y][5], acc[y][6], acc[y][7]);
          }
          named_bar(kBarCompute, kCompute);
          if (tid < D) {
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < kCWarps; ++w) sum += dscr[w * D + tid];
            red_add_dsmem(&pout[((g / C) * PER_KV + y) * D + tid], static_cast<uint32_t>(g % C), sum);
          }
          named_bar(kBarCompute, kCompute);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[y][e] = 0.f;
        }
      };
      const int4* desc = reinterpret_cast<const int4*>(smem + L.desc);
      for (; i < wk.total; ++i) {
        {
          const bool is_tail = i >= wk.d0 + wk.ndk;
          const int s = i % NS;
          if (lane == 0) mbar_wait(&bars[kFull + s], (i / NS) & 1);
          __syncwarp();
          const int4 dsc = desc[s];
          const int g = dsc.x, r0 = dsc.y, rows = dsc.z;
          if (ict && tid == 0 && i < 512) ict[3 * i + 1] = clock64();
          uint4 raw[DROWS];
#pragma unroll
          for (int rr = 0; rr < DROWS; ++rr)
            raw[rr] = *reinterpret_cast<const uint4*>(smem + L.ring + s * kStage + (rg + rr * RG) * D * 2 + cc * 16);
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[kEmpty + s]);
          if (ict && tid == 0 && i < 512) ict[3 * i + 2] = clock64();
          if (g != cur_g) {  // every warp sees the same item sequence: flush together
            if (cur_g >= 0) flush(cur_g);
            cur_g = g;
          }
          if (p.debug & 1) continue;
          const float* wsrc = is_tail ? stail : umine;
          const int flat0 = g * (is_tail ? tper : Rv) + r0 - (is_tail ? wk.ta : wk.va);
#pragma unroll
          for (int rr = 0; rr < DROWS; ++rr) {
            const int row = rg + rr * RG;
            if (row < rows) {
              float v[8];
              unpack8(raw[rr], v);
#pragma unroll
              for (int y = 0; y < PER_KV; ++y) {
                const float wgt = wsrc[(flat0 + row) * PER_KV + y];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[y][e] = fmaf(wgt, v[e], acc[y][e]);
              }
            }
          }
        }
      }
      if (cur_g >= 0) flush(cur_g);
      // appended token: p_new * v_new (bf16-rounded as stored)
      if (a.append_kv && n_tail > 0) {
        for (int w = cw; w < Hkv * PER_KV; w += kCWarps) {
          const int g = w / PER_KV, y = w % PER_KV;
          const int f = g * tper + n_tail - 1;
          if (f < wk.ta || f >= wk.tb) continue;
          const float pn = stail[(f - wk.ta) * PER_KV + y];
          for (int j = lane; j < D; j += 32)
            red_add_dsmem(&pout[((g / C) * PER_KV + y) * D + j], static_cast<uint32_t>(g % C),
                          pn * bf16r(qrow[H * D + W + g * D + j]));
        }
      }
    }
    fence_acq_rel_cluster();
    named_bar(kBarCompute, kCompute);
    if (tid < C) mbar_arrive_cluster(&bars[kOut], static_cast<uint32_t>(tid));
    cta_wait_cluster(&bars[kOut], 0, tid);
    // owners write the context of kv heads g = c, c + C, ...
    for (int w = tid; w < owned * PER_KV * D; w += kCompute) {
      const int g = c + (w / (PER_KV * D)) * C, y = (w / D) % PER_KV, j = w % D;
      if (g >= Hkv) continue;
      const long oi = static_cast<long>(b) * H * D + static_cast<long>(g * PER_KV + y) * D + j;
      if (a.ctx_bf16)
        reinterpret_cast<__nv_bfloat16*>(a.ctx_out)[oi] = __float2bfloat16_rn(pout[w]);
      else
        reinterpret_cast<float*>(a.ctx_out)[oi] = pout[w];
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
    if (per_kv == 1) return layer_kernel<NP, 1, 128>;
    if (per_kv == 2) return layer_kernel<NP, 2, 128>;
    return layer_kernel<NP, 4, 128>;
  }
  if (per_kv == 1) return layer_kernel<NP, 1, 64>;
  if (per_kv == 2) return layer_kernel<NP, 2, 64>;
  return layer_kernel<NP, 4, 64>;
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
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.s.cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
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
  if (s.cluster < 1 || s.cluster > 8) return bad("cluster size must be 1..8");
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
  const int cols = p.max_tiles * p.np + p.mtiles * p.np;
  if (cols > 512) return bad("TMEM budget exceeded (raise the cluster size)");
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.stages = 2;
  if (layer_smem(p).total > 227 * 1024) return bad("shared-memory budget exceeded (raise the cluster size)");
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
  p.smem_bytes = layer_smem(p).total;
  p.ok = true;
  p.why = "";
  return p;
}

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

// Cluster size: minimise waves x bytes streamed per CTA (the row-range split
// balances every CTA to within one 8-rank unit / one 128-token tile).
int auto_layer_cluster(FusedShape s) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int, int, int>, int> cache;
  const auto key = std::make_tuple(s.H, s.Hkv, s.D, s.n_comp, s.rank_k, s.rank_v, s.tail_cap, s.batch);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (auto f = cache.find(key); f != cache.end()) return f->second;
  }
  int best = 0;
  double best_cost = 1e300;
  const double tail = 0.5 * s.tail_cap;  // mid-run tail length
  for (int c = 8; c >= 1; --c) {
    s.cluster = c;
    const LayerPlan p = plan_layer(s);
    if (!p.ok) continue;
    int active = 1;
    try {
      active = std::max(1, layer_max_active_clusters(p));
    } catch (...) {
      active = 148 / c;
    }
    const long waves = (s.batch + active - 1) / active;
    const double rows = static_cast<double>(s.Hkv) * (s.rank_k + s.rank_v + 2.0 * tail) / c;
    const double bytes = 2.0 * s.D * rows + 2.0 * p.max_tiles * 128.0 * (s.rank_k + s.rank_v);
    const double cost = waves * bytes;
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = c;
    }
  }
  best = best > 0 ? best : 8;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = best;
  return best;
}

}  // namespace kvp
