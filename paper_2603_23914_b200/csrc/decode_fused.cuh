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
  int ld_left;        // unused (left factors are packed)
  int tail_cap;       // tail rows allocated per instance
  int batch;
  int cluster;        // CTAs per instance in the low-rank core kernel
  int rv2 = 0;        // two-tier values: rank prefix of the second tier (0 = untiered)
  int split = -1;     // core work split: 1 = token chunks over all SMs with a per-instance barrier in global
                      // memory (`cluster` = chunks per instance), 0 = one thread-block cluster per instance
                      // (DSMEM exchange), -1 = choose (split when the whole batch is co-resident)
};

struct FusedArgs {
  // left factors in the packed layout (pack_left): per instance, per 128-token
  // tile, per 64-rank panel one contiguous 16 KB block, rows 128 B, 16 B chunks
  // XOR-swizzled by row % 8 (the tcgen05 SWIZZLE_128B K-major operand layout)
  const unsigned char* left_k_packed;  // [batch][ntiles][kpk][16 KB]
  const unsigned char* left_v_packed;  // [batch][ntiles][vpanels_st][16 KB]
  const __nv_bfloat16* right_k;  // [batch][rank_k][W]
  const __nv_bfloat16* right_v;  // [batch][rank_v][W]
  const __nv_bfloat16* tail_k;   // [batch][tail_cap][W]
  const __nv_bfloat16* tail_v;
  const unsigned char* vtier;    // [batch][n_comp] nonzero: second value tier (rank prefix rv2); nullable
  const int* n_tail_dev;         // device counter of valid tail rows (nullable)
  int n_tail;                    // used when n_tail_dev == nullptr
  const float* q;                // [batch][q_stride] raw (unscaled) queries (first H*D of each row)
  long q_stride;                 // row stride of q (H*D, or H*D + 2W when q points into [q|k|v])
  int append_kv;                 // 1: q rows are [q|k|v]; qdots appends k, v as tail row n_tail-1 and
                                 //    zeroes that token's importance (cache.cpp:147-170)
  int inst0;                     // first instance of this launch inside the tensor-mapped left factors
  double* importance;            // [batch][imp_stride]: compressed then tail (nullable)
  long imp_stride;
  double ema_decay, ema_blend;   // alpha^1, 1 - alpha^1 (T_q = 1)
  float* head_avg;               // [batch][n_comp + tail_cap] (nullable)
  void* ctx_out;                 // [batch][H*D]
  int ctx_bf16;                  // 1: bf16 output, 0: fp32
  // workspace: P operand image (bf16 hi/lo, swizzled) [batch][2][kpk][NP][64],
  //            s_tail / p_tail fp32 [batch][H][tail_cap], U fp32 [batch][H][rank_v]
  //            (split mode: U partials [batch][chunks][H][rank_v], then (m, z) [batch][chunks][2][H] and
  //             one arrival counter per instance)
  unsigned char* ws_pimg;
  float* ws_tail;
  float* ws_u;
  float* ws_stats;
  unsigned* ws_count;
  unsigned long long* trace;     // debug: per-CTA phase timestamps [grid][16] (nullable)
};

struct FusedPlan {
  FusedShape s;
  int np;              // heads padded to 16
  int kpk;             // K panels of rank_k (64 ranks each)
  int vpanels;         // V panels, even
  int mtiles;          // vpanels / 2
  int kst;             // ring stages per tile for left_k (panel pairs)
  int nb2;             // two-tier values: U row tiles that need the second-tier accumulator
  bool pt_alias;       // p tiles reuse the P image's shared memory (large ranks; dead after the S MMAs)
  bool stack;          // P / p hi+lo halves stacked along N (np <= 32 and TMEM allows)
  int ntiles;          // 128-token tiles per instance
  int vpanels_st;      // stored V panels (ceil(rank_v / 64))
  int chunk;           // compressed tokens per CTA (max_tiles * 128)
  int max_tiles;       // tiles per CTA
  int tail_max;        // max tail tokens per CTA
  int heads_per_cta;   // query heads per CTA in the U reduce-scatter
  int stages;          // TMA ring stages (even)
  size_t smem_bytes;
  int tmem_cols;
  bool split;          // token-chunk split over all SMs (global-memory barrier) instead of clusters
  bool ok;
  const char* why;
};

FusedPlan plan_fused(const FusedShape& s);
int auto_cluster_size(const FusedShape& s);  // occupancy-aware CTAs per instance
size_t fused_workspace_bytes(const FusedShape& s);
// Resolves split / cluster choices of `s` (auto when cluster <= 0 or split < 0).
FusedShape resolve_fused_shape(FusedShape s);
// Carves a workspace of fused_workspace_bytes() into the FusedArgs buffers.
void bind_workspace(const FusedPlan& p, FusedArgs& a, void* ws);
size_t packed_left_bytes(int batch, int n, int rank);
void pack_left(const void* src, long ld, int batch, int n, int rank, void* dst, cudaStream_t st);
void launch_fused(const FusedPlan& p, const FusedArgs& a, cudaStream_t st);
// The three launches separately (engine pipelining across instance groups).
void launch_qdots(const FusedPlan& p, const FusedArgs& a, cudaStream_t st);
void launch_core(const FusedPlan& p, const FusedArgs& a, cudaStream_t st, int priority);
void launch_vsum(const FusedPlan& p, const FusedArgs& a, cudaStream_t st);
// Offsets every per-instance pointer of `a` by `b0` instances (workspace included).
FusedArgs offset_args(const FusedPlan& full, const FusedArgs& a, int b0);

}  // namespace kvp
