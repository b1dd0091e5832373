// The decode step's projections (decoder.cpp:574-576 q/k/v = x W, :590 x' = ctx W_o; `matmul`
// linalg.cpp:167-173) as a hand-written sm_100a weight-streaming GEMM.
//
// y[m, n] = sum_k x[m, k] W[k, n] with m = the batch's tokens (<= 256) and W [K][N] the layer's
// weights: HBM-bound (16 flop per weight byte at batch 16), so the kernel's only job is to stream W
// once at full bandwidth.  It is computed transposed, y^T = W^T x^T, so the weights are the tcgen05
// A operand (M = 128 output features, MN-major) and the tokens are N:
//   * W is stored pre-tiled ("packed"): per (128-feature tile, 64-deep k step) one contiguous 16 KB
//     block holding the MN-major SWIZZLE_128B operand image (two 64-feature halves of 64 k rows x
//     128 B), so one 1-D bulk copy fills a stage and a CTA's weight range is one sequential stream;
//   * x (bf16 [B][K], the previous kernel's output) is the K-major B operand, loaded per stage by a
//     TMA tensor map (rows >= B zero-filled);
//   * stream-K: the tiles x k-steps stages are dealt to one CTA per SM in equal contiguous ranges;
//     a tile split over several CTAs is reduced by its last-arriving CTA in fixed segment order
//     (deterministic), the others leave fp32 partials in a workspace;
//   * programmatic dependent launch: the first ring of weight stages is in flight before
//     griddepcontrol.wait (the weights do not depend on the previous kernel).
// Warp roles (192 threads): warp 0 bulk/TMA producer, warp 1 MMA issuer + TMEM owner, warps 2..5
// epilogue (TMEM lane quadrants = 32 output features each).
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "compact.cuh"
#include "proj_gemm.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {

using namespace sm100;

constexpr int kPThreads = 192;
constexpr uint32_t kWBlock = 16384;  // one packed 128 x 64 weight block
constexpr int kPMaxStages = 12;

__host__ __device__ inline long seg_start(long i, long S, long G) { return i * S / G; }
// the CTA whose stage range holds stage s
__device__ inline int cta_of(long s, long S, int G) {
  int c = static_cast<int>(s * G / S);
  while (c + 1 < G && seg_start(c + 1, S, G) <= s) ++c;
  while (c > 0 && seg_start(c, S, G) > s) --c;
  return c;
}

template <int NB>
__global__ void __launch_bounds__(kPThreads, 1)
    proj_gemm_kernel(const unsigned char* __restrict__ wpk, const __grid_constant__ CUtensorMap map_x, int N, int B,
                     int kst, int stages, void* __restrict__ out, int ldo, int out_bf16, float* __restrict__ ws,
                     unsigned* __restrict__ counters, int maxseg, unsigned long long* __restrict__ trace) {
  extern __shared__ __align__(1024) unsigned char psmem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(psmem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kXBytes = NB * 128;               // one 64-deep x tile (NB token rows x 128 B)
  constexpr uint32_t kStage = 2 * kWBlock + 2 * kXBytes;  // a stage = two k steps (32 KB of weights)
  __shared__ uint64_t full[kPMaxStages], empty[kPMaxStages], tfull[2], tfree[2];
  __shared__ uint32_t tslot;
  __shared__ int last_flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, me = blockIdx.x;
  const long S = static_cast<long>((N + 127) / 128) * kst;
  const long s0 = seg_start(me, S, G), s1 = seg_start(me + 1, S, G);
  auto stamp = [&](int i) {
    if (trace) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[me * 8 + i] = t;
    }
  };
  if (threadIdx.x == 0) {
    stamp(0);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tfree[b], 4);
    }
    fence_mbar_init();
    prefetch_tmap(&map_x);
  }
  constexpr uint32_t kCols = 2 * NB <= 32 ? 32 : 2 * NB <= 64 ? 64 : 2 * NB <= 128 ? 128 : 2 * NB <= 256 ? 256 : 512;
  if (warp == 1) tmem_alloc(&tslot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (lane == 0) {
      stamp(1);
      auto load_x = [&](unsigned char* dst, long q, uint64_t* bar) {
        const int k0 = static_cast<int>((q % kst) * 128);
        tma_load_3d(dst + 2 * kWBlock, &map_x, k0, 0, 0, bar);
        tma_load_3d(dst + 2 * kWBlock + kXBytes, &map_x, k0 + 64, 0, 0, bar);
      };
      // weights of the first ring before the dependency wait; x (the previous kernel's output) after
      const long pre = s1 - s0 < stages ? s1 - s0 : stages;
      for (long j = 0; j < pre; ++j) {
        mbar_expect_tx(&full[j], kStage);
        bulk_load(smem + j * kStage, wpk + (s0 + j) * static_cast<long>(2 * kWBlock), 2 * kWBlock, &full[j]);
      }
      stamp(2);
      griddep_wait();
      stamp(3);
      for (long j = 0; j < pre; ++j) load_x(smem + j * kStage, s0 + j, &full[j]);
      for (long j = pre; j < s1 - s0; ++j) {
        const int st = static_cast<int>(j % stages);
        mbar_wait(&empty[st], static_cast<uint32_t>(((j / stages) - 1) & 1));
        unsigned char* dst = smem + st * kStage;
        mbar_expect_tx(&full[st], kStage);
        bulk_load(dst, wpk + (s0 + j) * static_cast<long>(2 * kWBlock), 2 * kWBlock, &full[st]);
        load_x(dst, s0 + j, &full[st]);
      }
      griddep_launch_dependents();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, NB, true, false);
      const uint32_t base = smem_addr(smem);
      int seg = 0;
      for (long s = s0; s < s1; ++seg) {
        const long t = s / kst, se = s1 < (t + 1) * kst ? s1 : (t + 1) * kst;
        const int buf = seg & 1;
        if (seg >= 2) mbar_wait(&tfree[buf], static_cast<uint32_t>(((seg >> 1) - 1) & 1));
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(buf * NB);
        for (long q = s; q < se; ++q) {
          const long j = q - s0;
          const int st = static_cast<int>(j % stages);
          mbar_wait(&full[st], static_cast<uint32_t>((j / stages) & 1));
          if (j == 0) stamp(4);
          tc_fence_after();
          const uint32_t sa = base + st * kStage, sb = sa + 2 * kWBlock;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16(d, smem_desc(sa + (kk >> 2) * kWBlock + (kk & 3) * 2048, kWBlock / 2, 1024, kSwizzle128B),
                       smem_desc(sb + (kk >> 2) * kXBytes + (kk & 3) * 32, 16, 1024, kSwizzle128B), idesc,
                       (q != s || kk != 0) ? 1u : 0u);
          mma_commit(&empty[st]);
        }
        mma_commit(&tfull[buf]);
        s = se;
      }
      stamp(5);
    }
    __syncwarp();
  } else {
    // epilogue: TMEM lane quadrant qd holds output features n0 + qd*32 + lane, columns = tokens
    const int qd = warp & 3, et = threadIdx.x - 64, row = qd * 32 + lane;
    int seg = 0;
    for (long s = s0; s < s1; ++seg) {
      const long t = s / kst, se = s1 < (t + 1) * kst ? s1 : (t + 1) * kst;
      const int buf = seg & 1;
      mbar_wait(&tfull[buf], static_cast<uint32_t>((seg >> 1) & 1));
      tc_fence_after();
      const int n = static_cast<int>(t) * 128 + row;
      const bool whole = s == t * kst && se == (t + 1) * kst;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(qd * 32) << 16) + static_cast<uint32_t>(buf * NB);
      const int first = cta_of(t * kst, S, G), nseg = cta_of((t + 1) * kst - 1, S, G) - first + 1;
      float* part = ws + (static_cast<long>(t) * maxseg + (me - first)) * NB * 128;
      for (int c0 = 0; c0 < NB && c0 < B; c0 += 8) {
        float v[8];
        tmem_ld8(taddr + static_cast<uint32_t>(c0), v);
        if (whole) {
          if (n < N)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (c0 + e < B) {
                const long oi = static_cast<long>(c0 + e) * ldo + n;
                if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[oi] = __float2bfloat16_rn(v[e]);
                else reinterpret_cast<float*>(out)[oi] = v[e];
              }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) __stcg(&part[(c0 + e) * 128 + row], v[e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfree[buf]);
      if (!whole) {  // split tile: the last-arriving segment reduces all of them in segment order
        __threadfence();
        named_bar(1, 128);
        if (et == 0) {
          const unsigned prev = atomicAdd(&counters[t], 1u);
          last_flag = prev == static_cast<unsigned>(nseg - 1);
          if (last_flag) counters[t] = 0u;  // every segment arrived: ready for the next launch
        }
        named_bar(1, 128);
        if (last_flag) {
          __threadfence();
          const float* p0 = ws + static_cast<long>(t) * maxseg * NB * 128 + row;
          for (int c0 = 0; c0 < NB && c0 < B; c0 += 8) {
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.f;
            for (int j0 = 0; j0 < nseg; j0 += 4) {  // 32 independent loads in flight, summed in segment order
              float v[4][8];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  v[jj][e] = j0 + jj < nseg ? __ldcg(&p0[(static_cast<long>(j0 + jj) * NB + c0 + e) * 128]) : 0.f;
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] += v[jj][e];
            }
            if (n < N)
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (c0 + e < B) {
                  const long oi = static_cast<long>(c0 + e) * ldo + n;
                  if (out_bf16) reinterpret_cast<__nv_bfloat16*>(out)[oi] = __float2bfloat16_rn(acc[e]);
                  else reinterpret_cast<float*>(out)[oi] = acc[e];
                }
          }
        }
      }
      s = se;
    }
    if (et == 0) stamp(6);
  }
  __syncthreads();
  if (threadIdx.x == 0) stamp(7);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// W [K][N] row-major bf16 -> packed blocks [N/128][K/64][16 KB] (MN-major SW128 operand images).
// ksteps = blocks per tile (even: a stage streams two; a zero block pads an odd count).
__global__ void pack_weight_kernel(const __nv_bfloat16* __restrict__ w, int K, int N, int ksteps,
                                   unsigned char* __restrict__ dst) {
  const long total = static_cast<long>((N + 127) / 128) * ksteps * 128 * 64;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int nn = static_cast<int>(i % 128), kk = static_cast<int>((i / 128) % 64);
    const long blk = i / (128 * 64);
    const int ks = static_cast<int>(blk % ksteps), t = static_cast<int>(blk / ksteps);
    const int n = t * 128 + nn, k = ks * 64 + kk;
    const __nv_bfloat16 v = (n < N && k < K) ? w[static_cast<long>(k) * N + n] : __float2bfloat16_rn(0.f);
    *reinterpret_cast<__nv_bfloat16*>(dst + blk * kWBlock + (nn >> 6) * (kWBlock / 2) + sw128_off(kk, nn & 63)) = v;
  }
}

unsigned long long* g_ptrace = nullptr;

template <int NB>
void launch_nb(const ProjGemm& g, const unsigned char* wpk, const CUtensorMap& mx, void* out, int ldo, bool out_bf16,
               cudaStream_t st) {
  constexpr uint32_t stage = 2 * kWBlock + 2 * NB * 128;
  const size_t smem = static_cast<size_t>(g.stages) * stage + 1024;
  static size_t attr = 0;
  if (attr < smem) {
    KVP_CUDA(cudaFuncSetAttribute(proj_gemm_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr = smem;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(g.grid));
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  KVP_CUDA(cudaLaunchKernelEx(&cfg, proj_gemm_kernel<NB>, wpk, mx, g.N, g.B, g.kst, g.stages, out, ldo,
                              out_bf16 ? 1 : 0, g.ws, g.counters, g.maxseg, g_ptrace));
  KVP_LAUNCHED();
}

}  // namespace

void g_ptrace_set(void* p) { g_ptrace = static_cast<unsigned long long*>(p); }

size_t packed_weight_bytes(int K, int N) {
  return static_cast<size_t>((N + 127) / 128) * ((K + 127) / 128) * 2 * kWBlock;
}

void pack_weight(const __nv_bfloat16* w, int K, int N, void* dst, cudaStream_t st) {
  pack_weight_kernel<<<1184, 256, 0, st>>>(w, K, N, (K + 127) / 128 * 2, static_cast<unsigned char*>(dst));
  KVP_LAUNCHED();
}

ProjGemm proj_gemm_plan(int K, int N, int B, int sms) {
  require(B >= 1 && B <= 256, KVP_ERR_PARAMETER, "projection GEMM: batch must be in [1, 256]");
  require(K % 8 == 0, KVP_ERR_PARAMETER, "projection GEMM: K must be a multiple of 8");
  ProjGemm g{};
  g.K = K;
  g.N = N;
  g.B = B;
  g.nb = B <= 16 ? 16 : B <= 32 ? 32 : B <= 48 ? 48 : B <= 64 ? 64 : B <= 128 ? 128 : 256;
  g.kst = (K + 127) / 128;
  const long S = static_cast<long>((N + 127) / 128) * g.kst;
  g.grid = static_cast<int>(std::min<long>(sms, S));
  const long per = S / g.grid;  // every CTA holds >= per stages, so a tile spans <= ceil(kst/per) + 1 CTAs
  g.maxseg = static_cast<int>((g.kst + per - 1) / per + 1);
  const uint32_t stage = 2 * kWBlock + 2 * static_cast<uint32_t>(g.nb) * 128;
  g.stages = std::min<int>(kPMaxStages, static_cast<int>((220u * 1024u) / stage));
  g.ws_bytes = sizeof(float) * static_cast<size_t>((N + 127) / 128) * g.maxseg * g.nb * 128 +
               sizeof(unsigned) * static_cast<size_t>((N + 127) / 128);
  return g;
}

void proj_gemm_bind(ProjGemm& g, void* ws, cudaStream_t st) {
  g.ws = static_cast<float*>(ws);
  const size_t ntiles = static_cast<size_t>((g.N + 127) / 128);
  g.counters = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + g.ws_bytes - sizeof(unsigned) * ntiles);
  KVP_CUDA(cudaMemsetAsync(g.counters, 0, sizeof(unsigned) * ntiles, st));
}

void proj_gemm(const ProjGemm& g, const void* w_packed, const __nv_bfloat16* x, void* out, int ldo, bool out_bf16,
               cudaStream_t st) {
  require(g.ws != nullptr, KVP_ERR_PARAMETER, "projection GEMM: workspace not bound");
  const CUtensorMap mx = encode_bf16_map(x, g.K, g.B, 1, g.nb);
  const auto* wpk = static_cast<const unsigned char*>(w_packed);
  switch (g.nb) {
    case 16: launch_nb<16>(g, wpk, mx, out, ldo, out_bf16, st); break;
    case 32: launch_nb<32>(g, wpk, mx, out, ldo, out_bf16, st); break;
    case 48: launch_nb<48>(g, wpk, mx, out, ldo, out_bf16, st); break;
    case 64: launch_nb<64>(g, wpk, mx, out, ldo, out_bf16, st); break;
    case 128: launch_nb<128>(g, wpk, mx, out, ldo, out_bf16, st); break;
    default: launch_nb<256>(g, wpk, mx, out, ldo, out_bf16, st);
  }
}

}  // namespace kvp

namespace {
int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
}  // namespace

extern "C" size_t kvp_packed_weight_bytes(int32_t K, int32_t N) {
  return K > 0 && N > 0 ? kvp::packed_weight_bytes(K, N) : 0;
}

extern "C" int kvp_pack_weight(const void* w, int32_t K, int32_t N, void* dst, void* stream) {
  return kvp::guarded([&] {
    kvp::require(w && dst && K > 0 && N > 0, KVP_ERR_PARAMETER, "pack_weight: bad arguments");
    kvp::pack_weight(static_cast<const __nv_bfloat16*>(w), K, N, dst, kvp::as_stream(stream));
  });
}

extern "C" size_t kvp_matmul_packed_workspace(int32_t K, int32_t N, int32_t B) {
  size_t n = 0;
  kvp::guarded([&] { n = kvp::proj_gemm_plan(K, N, B, sm_count()).ws_bytes; });
  return n;
}

extern "C" int kvp_matmul_packed(const void* x, int32_t B, int32_t K, const void* w_packed, int32_t N, void* out,
                                 int32_t ldo, int32_t out_bf16, void* workspace, void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(x && w_packed && out && workspace && K > 0 && N > 0, KVP_ERR_PARAMETER, "matmul: bad arguments");
    require(ldo >= N, KVP_ERR_SHAPE, "matmul: output row stride below N");
    ProjGemm g = proj_gemm_plan(K, N, B, sm_count());
    g.ws = static_cast<float*>(workspace);
    g.counters = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + g.ws_bytes -
                                             sizeof(unsigned) * static_cast<size_t>((N + 127) / 128));
    proj_gemm(g, w_packed, static_cast<const __nv_bfloat16*>(x), out, ldo, out_bf16 != 0, as_stream(stream));
  });
}

extern "C" void kvp_debug_proj_trace(void* dev_buffer) { kvp::g_ptrace_set(dev_buffer); }
