// Hand-written weight-streaming projection GEMM (proj_gemm.cu): y = x W for the decode step's
// q/k/v and output projections (decoder.cpp:574-576, 590).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>

namespace kvp {

struct ProjGemm {
  int K, N, B;      // y [B][N] = x [B][K] . W [K][N]
  int nb;           // tokens padded to the MMA's N (16, 32, 48, 64, 128 or 256)
  int kst;          // 128-deep k stages (two packed blocks each)
  int grid;         // CTAs (one per SM, stream-K over tiles x k steps)
  int maxseg;       // CTAs a split tile can span
  int stages;       // shared-memory ring depth
  size_t ws_bytes;  // fp32 partials + one arrival counter per tile
  float* ws;
  unsigned* counters;
};

size_t packed_weight_bytes(int K, int N);
// W [K][N] row-major bf16 -> the packed operand blocks the GEMM streams.
void pack_weight(const __nv_bfloat16* w, int K, int N, void* dst, cudaStream_t st);
void g_ptrace_set(void* p);  // debug: per-CTA phase stamps [grid][8]
ProjGemm proj_gemm_plan(int K, int N, int B, int sms);
// Binds a workspace of plan.ws_bytes (zeroes the tile counters on `st`).
void proj_gemm_bind(ProjGemm& g, void* ws, cudaStream_t st);
// out [B][ldo] (bf16 or fp32) = x [B][K] (bf16, row-major) . W (packed).  Launched with programmatic
// stream serialization: the first weight stages stream before the previous kernel's output is read.
void proj_gemm(const ProjGemm& g, const void* w_packed, const __nv_bfloat16* x, void* out, int ldo, bool out_bf16,
               cudaStream_t st);

}  // namespace kvp
