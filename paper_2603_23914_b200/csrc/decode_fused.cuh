// Compressed-cache decode attention (bf16 storage, T_q = 1), the serving hot
// path: one cluster launch per layer, see decode_layer.cu.
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
  int cluster;        // CTAs per instance (one co-resident group exchanging through L2)
};

struct FusedArgs {
  // left factors in the packed layout (pack_left): per instance, per 128-token
  // tile, per 64-rank panel one contiguous 16 KB block, rows 128 B, 16 B chunks
  // XOR-swizzled by row % 8 (the tcgen05 SWIZZLE_128B K-major operand layout)
  const unsigned char* left_k_packed;  // [batch][ntiles][kpk][16 KB]
  const unsigned char* left_v_packed;  // [batch][ntiles][vpanels_st][16 KB]
  // right factors and tails: packed row tiles per kv head (pack_left layout of the head-major
  // [batch*Hkv][rows][D] matrix): [batch*Hkv][ceil(rows/128)][D/64][16 KB]
  const __nv_bfloat16* right_k;  // rows = rank_k
  const __nv_bfloat16* right_v;  // rows = rank_v
  const __nv_bfloat16* tail_k;   // rows = tail_cap
  const __nv_bfloat16* tail_v;
  const int* n_tail_dev;         // device counter of valid tail rows (nullable)
  int n_tail;                    // used when n_tail_dev == nullptr
  const float* q;                // [batch][q_stride] raw (unscaled) queries (first H*D of each row)
  long q_stride;                 // row stride of q (H*D, or H*D + 2W when q points into [q|k|v])
  int append_kv;                 // 1: q rows are [q|k|v]; k, v are appended as tail row n_tail-1 with
                                 //    importance 0 (cache.cpp:147-170)
  int inst0;                     // first instance of this launch inside the packed left factors
  double* importance;            // [batch][imp_stride]: compressed then tail (nullable)
  long imp_stride;
  double ema_decay, ema_blend;   // alpha^1, 1 - alpha^1 (T_q = 1)
  float* head_avg;               // [batch][n_comp + tail_cap] (nullable)
  void* ctx_out;                 // [batch][H*D]
  int ctx_bf16;                  // 1: bf16 output, 0: fp32
  unsigned char* group_ws;       // [batch][layer_group_ws_bytes / batch] exchange area; its barrier
                                 // words (first 8 bytes per instance) zeroed once at allocation
  unsigned long long* trace;     // debug: per-CTA phase timestamps [grid][16] (nullable)
};

size_t packed_left_bytes(int batch, int n, int rank);
void pack_left(const void* src, long ld, int batch, int n, int rank, void* dst, cudaStream_t st);
// [batch][rows][Hkv*D] <-> [batch][Hkv][rows][D] (bf16)
void pack_heads(const void* src, void* dst, int batch, int rows, int Hkv, int D, bool to_heads, cudaStream_t st);

// ---- one-launch layer kernel (decode_layer.cu) -----------------------------
struct LayerPlan {
  FusedShape s;
  int np;          // heads padded to 16 (MMA N)
  int kpk;         // K panels of rank_k
  int vpanels;     // V panels, even
  int mtiles;      // vpanels / 2 (U MMA M tiles of 128 ranks)
  int vpanels_st;  // stored V panels
  int kst;         // ring stages per tile for left_k (panel pairs)
  int ntiles;      // 128-token tiles per instance
  int max_tiles;   // tiles of the busiest CTA
  int max_qh;      // query heads of the busiest CTA
  int tpc;         // tail tokens per CTA in the tail EMA
  int stages;      // TMA ring stages (even)
  int tmem_cols;
  int nab;         // phase-A TMEM result buffers
  int nob;         // phase-D operand buffers
  int a_col, d_col;  // TMEM column of the phase-A buffers / phase-D accumulators
  int debug;       // timing experiments only (KVP_LAYER_DEBUG): 8 = phase A only
  int prefetch;    // L2 prefetch distance beyond the ring, in items
  size_t smem_bytes;
  bool ok;
  const char* why;
};
LayerPlan plan_layer(const FusedShape& s);
int auto_layer_cluster(FusedShape s);
int layer_max_active_clusters(const LayerPlan& p);
size_t layer_group_ws_bytes(const LayerPlan& p);
void launch_layer(const LayerPlan& p, const FusedArgs& a, cudaStream_t st);

}  // namespace kvp
