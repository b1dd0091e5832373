// Compressed-cache decode attention (bf16 storage, T_q = 1), the serving hot
// path: three launches per layer, see decode_fused.cu.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace kvp {

struct FusedShape {
  int H, Hkv, D;      // geometry
  int n_comp;         // compressed (visual) tokens per instance
  int rank_k, rank_v; // stored ranks
  int ld_left;        // row stride of left factors (elements, multiple of 8)
  int tail_cap;       // tail rows allocated per instance
  int batch;
  int cluster;        // CTAs per instance in the low-rank core kernel
};

struct FusedArgs {
  const __nv_bfloat16* right_k;  // [batch][rank_k][W]
  const __nv_bfloat16* right_v;  // [batch][rank_v][W]
  const __nv_bfloat16* tail_k;   // [batch][tail_cap][W]
  const __nv_bfloat16* tail_v;
  const int* n_tail_dev;         // device counter of valid tail rows (nullable)
  int n_tail;                    // used when n_tail_dev == nullptr
  const float* q;                // [batch][H*D], raw (unscaled) queries
  double* importance;            // [batch][imp_stride]: compressed then tail (nullable)
  long imp_stride;
  double ema_decay, ema_blend;   // alpha^1, 1 - alpha^1 (T_q = 1)
  float* head_avg;               // [batch][n_comp + tail_cap] (nullable)
  void* ctx_out;                 // [batch][H*D]
  int ctx_bf16;                  // 1: bf16 output, 0: fp32
  // workspace: P operand image (bf16 hi/lo, swizzled) [batch][2][kpk][NP][64],
  //            s_tail / p_tail fp32 [batch][H][tail_cap], U fp32 [batch][H][rank_v]
  unsigned char* ws_pimg;
  float* ws_tail;
  float* ws_u;
  unsigned long long* trace;     // debug: per-CTA phase timestamps [grid][16] (nullable)
};

struct FusedPlan {
  FusedShape s;
  int np;              // heads padded to 16
  int kpk;             // K panels of rank_k (64 ranks each)
  int vpanels;         // V panels, even
  int mtiles;          // vpanels / 2
  int chunk;           // compressed tokens per CTA (multiple of 32)
  int max_tiles;       // ceil(chunk / 128)
  int tail_max;        // max tail tokens per CTA
  int heads_per_cta;   // query heads per CTA in the U reduce-scatter
  int stages;          // TMA ring stages (even)
  bool box32_only;     // tuning: force 32-row TMA boxes
  size_t smem_bytes;
  int tmem_cols;
  bool ok;
  const char* why;
};

FusedPlan plan_fused(const FusedShape& s);
size_t fused_workspace_bytes(const FusedShape& s);
void encode_fused_maps(const FusedShape& s, const void* left_k, const void* left_v, CUtensorMap* maps /*[4]*/);
void launch_fused(const FusedPlan& p, const CUtensorMap* maps, const FusedArgs& a, cudaStream_t st);

}  // namespace kvp
