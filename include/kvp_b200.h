/*
 * kvp_b200.h — C-ABI of the B200-native AttentionPack KV-cache path.
 *
 * This is the drop-in boundary.  Every entry point takes plain pointers,
 * sizes and POD descriptors (no C++ or torch types), returns an int status,
 * never throws, and leaves a thread-local message behind on failure:
 *
 *   0 KVP_OK            1 KVP_ERR_PARAMETER   (kvpack::parameter_error)
 *   2 KVP_ERR_SHAPE     (kvpack::shape_error) 3 KVP_ERR_DATA (kvpack::data_error)
 *   4 KVP_ERR_IO        (kvpack::io_error)    5 KVP_ERR_CUDA (device failure)
 *
 * The codes map 1:1 onto the reference's exception hierarchy
 * (/root/reference/proj/include/kvpack/errors.hpp:11-36); the C++ facade
 * and the Python layer turn them back into the same exception types
 * (bindings/module.cpp:117-127: io -> OSError, parameter/shape/data -> ValueError).
 *
 * Streams are caller-owned (`stream` is a cudaStream_t passed as void*;
 * NULL = legacy default stream).  Device pointers are marked [dev], host
 * pointers [host].  A kvp_ctx is single-writer, like a reference LayerCache
 * (SPEC.md:151).
 *
 * Which reference interface each entry point replaces is cited beside it.
 */
#ifndef KVP_B200_H
#define KVP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVP_ABI_VERSION 1

enum kvp_status {
  KVP_OK = 0,
  KVP_ERR_PARAMETER = 1,
  KVP_ERR_SHAPE = 2,
  KVP_ERR_DATA = 3,
  KVP_ERR_IO = 4,
  KVP_ERR_CUDA = 5
};

/* Storage precision of cache payloads (the reference instantiates float and
 * double, cache.cpp:241-242; bf16 is the B200 serving format). */
enum kvp_dtype { KVP_F32 = 0, KVP_F64 = 1, KVP_BF16 = 2 };

/* Store forms (cache.hpp:35-60 BlockStore): dense rows or low-rank factors. */
enum kvp_form { KVP_DENSE = 0, KVP_LOWRANK = 1 };

int kvp_abi_version(void);
const char* kvp_last_error_message(void);
/* Number of CUDA kernel launches issued by this library so far (process-wide). */
uint64_t kvp_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Retrieval-plan attention (generic path, any dtype, any plan).             */
/* ------------------------------------------------------------------------ */

/* One stored matrix.  KVP_DENSE: a = rows (n x width, row stride lda).
 * KVP_LOWRANK: a = left (n x rank, stride lda), b = right (rank x width,
 * stride ldb).  [dev] pointers in `dtype`. */
typedef struct {
  int32_t form;
  int32_t rank;
  const void* a;
  const void* b;
  int64_t lda;
  int64_t ldb;
} kvp_store;

/* One RetrievalPlan entry (decoder.hpp:84-98): which K/V stores the row
 * comes from, the row inside them, the tier rank prefixes (0 = full stored
 * rank / dense), the global position (causal visibility), and the column of
 * the importance table it maps to (decoder.cpp:596-600; -1 = none). */
typedef struct {
  int32_t k_store;
  int32_t v_store;
  uint32_t row;
  uint32_t rank_k;
  uint32_t rank_v;
  int32_t table_index;
  uint64_t position;
} kvp_plan_entry;

typedef struct {
  int32_t heads;      /* H   (HeadGeometry, cache.hpp:21-31) */
  int32_t kv_heads;   /* H_kv */
  int32_t head_dim;   /* D */
  int32_t dtype;      /* kvp_dtype of every store */
  int32_t n_stores;
  int32_t n_entries;
  int32_t tq;         /* query rows */
  int32_t table_size; /* importance-table width for head_avg_table (0 = skip) */
  const kvp_store* stores;          /* [host] n_stores */
  const kvp_plan_entry* entries;    /* [host] n_entries, plan order */
  const double* queries;            /* [dev] tq x H*D */
  const uint64_t* query_positions;  /* [dev] tq */
  double* context;                  /* [dev] out tq x H*D (pre-W_o) */
  double* head_avg;                 /* [dev] out tq x n_entries, plan order (nullable) */
  double* head_avg_table;           /* [dev] out tq x table_size, table order (nullable) */
} kvp_attend_desc;

/* attend_materialized / attend_fused (decoder.hpp:127-135, decoder.cpp:190-344)
 * evaluated in the low-rank space: P = right_k·q, S = left_k·P, softmax,
 * U = p·left_v, out = U·right_v — never rebuilding K~/V~.  fp64 accumulation
 * (the reference accumulates in double for both T=float and T=double). */
int kvp_attend_plan(const kvp_attend_desc* desc, void* stream);

/* ------------------------------------------------------------------------ */
/* Importance (importance.cpp:33-117).                                       */
/* ------------------------------------------------------------------------ */

/* EMA update of `n_tables` tables of `n` scores each (importance.cpp:33-65):
 * s <- decay*s + blend*mean_t attn[t, :], decay = alpha^tq (computed on the
 * host with std::pow like the reference), bit-exact (no FMA contraction).
 * Rows must be distributions within 1e-4 (else KVP_ERR_DATA after the sync
 * when `check` != 0; *bad_rows receives the count when non-NULL). */
int kvp_update_importance(int32_t n_tables, int32_t n, double* scores /*[dev] n_tables x n*/,
                          int32_t tq, const double* attn /*[dev] n_tables x tq x n*/,
                          double alpha, int32_t check, void* stream);

/* Tier assignment (importance.cpp:67-117 assign_groups + decoder.cpp:105-139
 * resolve_tiering): per table, stable order by (score desc, index asc) of the
 * n compressed tokens; group f gets floor(ratio_f*n+0.5) tokens (last takes
 * the rest).  Outputs the group id per token and the per-token rank prefixes
 * rank_k[f], rank_v[f].  Bit-exact vs the reference for identical scores. */
int kvp_assign_tiers(int32_t n_tables, int32_t n, const double* scores /*[dev] stride score_stride*/,
                     int64_t score_stride, int32_t n_groups, const double* ratios /*[host]*/,
                     const int32_t* key_ranks /*[host]*/, const int32_t* value_ranks /*[host]*/,
                     uint8_t* tier_out /*[dev] n_tables x n (nullable)*/,
                     uint16_t* rank_k_out /*[dev] n_tables x n (nullable)*/,
                     uint16_t* rank_v_out /*[dev] n_tables x n (nullable)*/, void* stream);

/* Host-buffer convenience forms used by the kvpack-compatible Python surface
 * (bindings/module.cpp:186-225 ema_update / assign_groups). */
int kvp_update_importance_host(int32_t n, double* scores, int32_t tq, const double* attn, double alpha);
int kvp_assign_groups_host(int32_t n, const double* scores, int32_t n_groups, const double* ratios,
                           const int32_t* ranks, uint32_t* tier_out);

/* ------------------------------------------------------------------------ */
/* Truncated SVD (linalg.hpp:29-30 truncated_svd, linalg.cpp:68-105).         */
/* ------------------------------------------------------------------------ */

/* Rank-R factorisation of `batch` row-major fp32 matrices a[b] (T x W):
 * left[b] (T x R, singular values folded in), right[b] (R x W, orthonormal
 * rows), sv[b] (R singular values, descending; nullable).  method 1 =
 * randomized (Halko: k = min(R + oversampling, min(T, W)), q power
 * iterations, Philox sketch stream 0x72737664), range-finder products on the
 * tcgen05 GEMM in bf16; method 0 = exact up to fp32 rounding (full sketch,
 * fp32 products).  Errors as check_svd_input (linalg.cpp:15-24). */
int kvp_truncated_svd(const float* a, int32_t batch, int32_t T, int32_t W, int32_t rank, int32_t method,
                      uint64_t seed, int32_t oversampling, int32_t power_iterations, float* left, float* right,
                      float* sv, void* stream);

/* quantize_roundtrip (bindings/module.cpp:223-230): quantize_4bit + dequantize
 * (quantize.cpp:10-54) of a row-major f64 matrix, groups of group_size rows per column;
 * a, out [dev].  Bit-identical to the reference. */
int kvp_quantize_roundtrip(const double* a, int64_t rows, int64_t cols, int64_t group_size, double* out,
                           void* stream);

/* gaussian_matrix (linalg.hpp:55-58): rows x cols N(0,1) draws of the Philox
 * stream (seed, stream_id) (rng.hpp:15-98), row-major, dtype f32 or f64 [dev]. */
int kvp_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint64_t stream_id, int32_t dtype, void* out,
                        void* stream);

/* ------------------------------------------------------------------------ */
/* Fused serving kernel: bf16 compressed cache, T_q = 1, batched instances.  */
/* ------------------------------------------------------------------------ */

/* Left factors live in the packed layout kvp_pack_left produces: per
 * instance, per 128-token tile, per 64-rank panel one contiguous 16 KB block
 * (128 rows of 128 B, 16 B chunks XOR-swizzled by row % 8 — the tcgen05
 * SWIZZLE_128B K-major operand layout), zero padded.  One bulk copy per block
 * feeds the tensor cores. */
size_t kvp_packed_left_bytes(int32_t batch, int32_t n, int32_t rank);
/* Row-major [batch][n][ld] bf16 left factor -> packed layout. */
int kvp_pack_left(const void* src, int64_t ld, int32_t batch, int32_t n, int32_t rank, void* dst, void* stream);

/* Projection GEMM of the decode step (decoder.cpp:574-576 q/k/v = h W_q|W_k|W_v, :590 x = ctx W_o;
 * `matmul` linalg.cpp:167-173) in the serving format: bf16 weights in a packed layout (per
 * 128-column tile, per 64-row step one contiguous 16 KB block — the tcgen05 MN-major SWIZZLE_128B
 * operand image), bf16 tokens, fp32 accumulation.  out[B][ldo] = x[B][K] . W[K][N], B <= 256. */
size_t kvp_packed_weight_bytes(int32_t K, int32_t N);
/* Row-major [K][N] bf16 weight -> packed layout. */
int kvp_pack_weight(const void* w, int32_t K, int32_t N, void* dst, void* stream);
size_t kvp_matmul_packed_workspace(int32_t K, int32_t N, int32_t B);
/* x: [dev] bf16 [B][K]; w_packed: [dev] (kvp_pack_weight); out: [dev] bf16 or fp32 [B][ldo];
 * workspace: [dev] kvp_matmul_packed_workspace bytes, zeroed before its first use. */
int kvp_matmul_packed(const void* x, int32_t B, int32_t K, const void* w_packed, int32_t N, void* out, int32_t ldo,
                      int32_t out_bf16, void* workspace, void* stream);

/* One layer of a batch of caches in the serving layout: every instance holds
 * one factored block of n_comp tokens (left_k/left_v packed, see above;
 * right_k: [batch][rank_k][W], right_v: [batch][rank_v][W]) and a dense tail
 * (tail_k/tail_v: [batch][tail_cap][W], n_tail rows valid — read from
 * n_tail_dev when non-NULL so the call can live in a CUDA graph).  This is
 * the plan build_retrieval_plan produces for the reference's default
 * configuration (visual block factored, textual tail dense; decoder.cpp:141-188)
 * with untiered decompression, or two-tier value decompression (key fractions 1;
 * tier2_value_rank / value_tier).  Outputs the pre-W_o context (decoder.cpp:587-590)
 * and, when `importance` is set, applies the Eq. 1 EMA in place for T_q = 1
 * (importance.cpp:33-65) over [compressed..., tail...] columns. */
typedef struct {
  int32_t heads, kv_heads, head_dim, batch;
  int32_t n_comp, rank_k, rank_v;
  int32_t tier2_value_rank;     /* attention-aware decompression (decoder.cpp:105-188): tokens flagged in
                                   value_tier use only this prefix of the value rank; 0 = untiered */
  int32_t tail_cap, n_tail;
  const int32_t* n_tail_dev;    /* [dev] nullable */
  int32_t cluster;              /* CTAs per instance, 0 = auto */
  int32_t context_bf16;         /* 1: context is bf16, 0: fp32 */
  const void* left_k;           /* [dev] packed (kvp_pack_left) */
  const void* right_k;
  const void* left_v;
  const void* right_v;
  const void* tail_k;
  const void* tail_v;
  const float* queries;         /* [dev] batch x H*D (unscaled) */
  double* importance;           /* [dev] batch x imp_stride, nullable */
  int64_t imp_stride;
  double alpha;
  float* head_avg;              /* [dev] batch x (n_comp + tail_cap), nullable */
  void* context;                /* [dev] batch x H*D */
  void* workspace;              /* [dev] nullable: kvp_decode_fused_workspace() bytes */
  size_t workspace_bytes;
  const uint8_t* value_tier;    /* [dev] batch x n_comp, nonzero = second tier (the group assign_groups puts
                                   after the first ratio, importance.cpp:67-117); read when tier2_value_rank > 0 */
} kvp_fused_desc;

/* Bytes of device workspace kvp_decode_fused needs for `desc` (P, tail
 * weights and U between its three launches); pass it to make the call
 * allocation-free (and CUDA-graph capturable). */
size_t kvp_decode_fused_workspace(const kvp_fused_desc* desc);

/* decode_step's attention + importance for a whole batch (decoder.cpp:583-601):
 * qdots (project q into the key basis + tail logits), the cluster/tcgen05
 * low-rank core, and vsum (value basis multiply + tail values) — 3 launches.  KVP_ERR_PARAMETER when the shape is outside the
 * fused kernel's envelope (then use kvp_attend_plan). */
int kvp_decode_fused(const kvp_fused_desc* desc, void* stream);

/* ------------------------------------------------------------------------ */
/* Device LayerCache batch: the caller-owned cache of decode_step / compress_now */
/* (cache.hpp:120-146 LayerCache, decoder.hpp:166-191).                        */
/* ------------------------------------------------------------------------ */

/* `batch` LayerCaches of one layer, held on the device and stepped together:
 * every instance has the same segment structure (token counts, positions,
 * block layout — what the reference harness builds for a batch of requests,
 * harness.cpp:239-360); payloads, importance scores and stored ranks are per
 * instance.  Storage dtype f32 / f64 (the reference's two instantiations,
 * cache.cpp:241-242) or bf16 (the serving format).  A kvp_cache is
 * single-writer. */
typedef struct kvp_cache kvp_cache;

typedef struct {
  int32_t heads, kv_heads, head_dim; /* HeadGeometry (cache.hpp:21-31) */
  int32_t dtype;                     /* storage: KVP_F32, KVP_F64 or KVP_BF16 */
  int32_t batch;                     /* instances */
  int32_t layer_index;               /* LayerCache.layer_index (rank schemes) */
} kvp_cache_config;

/* DecodeConfig (decoder.hpp:53-75) with TierSpec, MatrixRanks, SvdOptions and
 * RankScheme (compressor.hpp:14-30).  Arrays are [host]. */
typedef struct {
  int64_t compression_period;        /* tail rows that trigger re-factorisation; <= 0 = never (nullopt) */
  int32_t rank_key_visual, rank_value_visual, rank_key_textual, rank_value_textual; /* 0 = dense */
  int32_t rank_scheme;               /* -1 none, 0 fixed, 1 linear_schedule, 2 variance_target */
  int32_t scheme_fixed_rank;
  int32_t scheme_first_layer_rank, scheme_last_layer_rank, scheme_num_layers;
  double scheme_variance_target;
  int32_t scheme_max_rank;
  int32_t n_tiers;                   /* TierSpec groups, 0 = full-rank decompression */
  const double* tier_ratios;
  const double* tier_key_fractions;
  const double* tier_value_fractions;
  double alpha;                      /* importance EMA factor */
  int32_t svd_method;                /* 0 exact, 1 randomized (linalg.hpp:12-19) */
  uint64_t svd_seed;
  int32_t svd_oversampling, svd_power_iterations;
  int32_t recompress;                /* 0 joint, 1 separate_epochs (RecompressMode) */
  int32_t bytes_per_scalar;          /* accounting width of the reports */
} kvp_decode_config;

/* StepReport (decoder.hpp:145-160), one per instance. */
typedef struct {
  uint64_t step, bytes_before, bytes_after, importance_bytes;
  uint64_t decompress_flops, decompress_flops_full;
  double flops_reduction;
  int32_t compression_event;
  int32_t n_warnings;                /* rank-clamp warnings (decoder.cpp:440-449) */
} kvp_step_report;

/* AttentionWeights (decoder.hpp:18-26): [dev] row-major, storage dtype;
 * w_q, w_o: HD x HD, w_k, w_v: HD x W. */
typedef struct {
  const void *w_q, *w_k, *w_v, *w_o;
} kvp_weights;

/* CacheBytes (cache.hpp:158-168) of one instance. */
typedef struct {
  uint64_t visual_scalars, textual_scalars, visual_bytes, textual_bytes, cache_bytes, importance_bytes;
} kvp_cache_bytes;

int kvp_cache_create(const kvp_cache_config* config, kvp_cache** cache);
int kvp_cache_destroy(kvp_cache* cache);
/* append_tokens (cache.cpp:147-170) to every instance: k, v [host] f64,
 * batch x n x W; fresh global positions, importance 0. */
int kvp_cache_append(kvp_cache* cache, int32_t modality, int32_t n, const double* k, const double* v);
/* Upload of a host LayerCache image: the segment's current tail becomes one
 * block (appended after existing blocks) holding the given factors instead of
 * an SVD — left: batch x n x rank, right: batch x rank x W, [host] f64; rank 0
 * keeps that kind dense (the tail rows).  */
int kvp_cache_factor_tail(kvp_cache* cache, int32_t modality, int32_t rank_k, const double* k_left,
                          const double* k_right, int32_t rank_v, const double* v_left, const double* v_right);
/* Importance table (importance.hpp:16-31): scores [host] batch x table_size. */
int kvp_cache_set_importance(kvp_cache* cache, const double* scores);
int kvp_cache_get_importance(kvp_cache* cache, uint64_t* positions /*table_size, nullable*/,
                             double* scores /*batch x table_size, nullable*/);
/* Shape: table size, next_position, steps_taken; per segment blocks and tail length. */
int kvp_cache_shape(kvp_cache* cache, int32_t* table_size, uint64_t* next_position, uint64_t* steps_taken,
                    int32_t* n_blocks /*[2]*/, int32_t* tail_len /*[2]*/);
/* next_position / steps_taken of every instance (LayerCache fields, cache.hpp:137-146), e.g. from a
 * KVPK snapshot (snapshot.cpp:275-276); next_position may not move below an assigned position. */
int kvp_cache_set_counters(kvp_cache* cache, uint64_t next_position, uint64_t steps_taken);
/* One block store of one instance: tokens and stored rank (0 = dense). */
int kvp_cache_block_info(kvp_cache* cache, int32_t instance, int32_t modality, int32_t block, int32_t kind,
                         int32_t* tokens, int32_t* rank);
/* Download: low-rank -> left (tokens x rank) and right (rank x W); dense -> rows
 * (tokens x W) into `left`.  [host] f64; positions: tokens (nullable). */
int kvp_cache_block_get(kvp_cache* cache, int32_t instance, int32_t modality, int32_t block, int32_t kind,
                        double* left, double* right, uint64_t* positions);
int kvp_cache_tail_get(kvp_cache* cache, int32_t instance, int32_t modality, double* k, double* v,
                       uint64_t* positions);
/* memory_bytes (cache.cpp:209-219) of one instance. */
int kvp_cache_memory_bytes(kvp_cache* cache, int32_t instance, int32_t bytes_per_scalar, kvp_cache_bytes* out);

/* segment_full_matrix (decoder.cpp:406-424): dense [blocks at full stored rank;
 * tail] of one segment and kind for every instance, [dev] f64 batch x T x W. */
int kvp_segment_full_matrix(kvp_cache* cache, int32_t modality, int32_t kind, double* out, void* stream);

/* compress_now (decoder.cpp:619-628): re-factorise every compressible segment
 * with a non-empty tail (recompress_segment, decoder.cpp:455-497: joint or
 * separate epochs, rank clamp, dense kinds) on the device.  reports [host]
 * batch entries (nullable); compression_event / n_warnings are set. */
int kvp_compress_now(kvp_cache* cache, const kvp_decode_config* cfg, kvp_step_report* reports, void* stream);

/* decode_step (decoder.cpp:555-617) for every instance: project h (T_q rows),
 * append the new K/V to `modality`'s tail, tier the compressed tokens by
 * importance, attend over the plan in the low-rank space, W_o, EMA update,
 * re-factorise segments whose tail reached the period.  h, out: [dev]
 * batch x tq x HD, f64 for f64 caches, else f32.  Serving-shaped bf16 caches
 * (one factored visual block, dense textual tail, T_q = 1, <= 2 value tiers)
 * run the fused tcgen05 kernel; every other cache the generic plan kernels.
 * Errors as the reference: non-finite h -> KVP_ERR_DATA before any change. */
int kvp_decode_step(kvp_cache* cache, const void* h, int32_t tq, int32_t modality, const kvp_weights* weights,
                    const kvp_decode_config* cfg, void* out, kvp_step_report* reports, void* stream);

/* ------------------------------------------------------------------------ */
/* Device decode engine: the batched serving loop of the synthetic harness   */
/* (harness.cpp:239-360 run_instance, decoder.cpp:555-617 decode_step).      */
/* ------------------------------------------------------------------------ */

/* One modality's synthetic cache profile (harness.hpp:20-25 ModalityProfile). */
typedef struct {
  int32_t true_rank;
  int32_t shared_subspace;
  double spectrum_decay;
  double noise_floor;
} kvp_profile;

/* WorkloadSpec + DecodeConfig subset of the serving layout (harness.hpp:27-38,
 * decoder.hpp:53-75): visual segment factored at rank_k / rank_v right after
 * prefill (compress_now), textual segment dense, decode tokens join the
 * textual tail, importance EMA with `alpha`, untiered or two-tier value decompression. */
typedef struct {
  int32_t heads, kv_heads, head_dim;
  int32_t layers, batch;
  int32_t visual_tokens, textual_tokens, decode_steps;
  int32_t rank_k, rank_v;
  double alpha;
  uint64_t seed;                /* WorkloadSpec.seed (Philox streams, harness.cpp:29-32) */
  kvp_profile visual, textual;
  int32_t svd_method;           /* 0 exact, 1 randomized (linalg.hpp:12-19) */
  uint64_t svd_seed;
  int32_t svd_oversampling, svd_power_iterations;
  int32_t factor_init;          /* 0: compaction of the generated K/V; 1: placeholder factors */
  int32_t cluster;              /* CTAs per instance in the decode core, 0 = auto */
  /* two-tier attention-aware decompression of the visual block (TierSpec, decoder.hpp:31-52): each step the
     first tier_ratio of the tokens by importance (assign_groups) keep the full value rank, the rest use
     resolved_tier_rank(tier_value_fraction, rank_v); key fractions 1.  tier_ratio 0 or fraction 1 = untiered */
  double tier_ratio;
  double tier_value_fraction;
  /* global index of this engine's first instance: instance b draws the Philox
     streams of instance instance_offset + b (harness.cpp:29-32), so a batch
     sharded over ranks reproduces the single-process workload */
  int32_t instance_offset;
} kvp_engine_config;

typedef struct {
  int32_t cluster, rank_k, rank_v, ld_left, tail_cap, steps_taken;
  double compaction_ms;
  uint64_t launches_per_step;          /* kernels of this library per decode step */
  uint64_t weight_bytes_per_step;      /* projection weights read per step */
  uint64_t factor_bytes_per_step;      /* left + right factors read per step */
  uint64_t tail_row_bytes;             /* bytes per tail token (K + V, all layers/instances) */
  uint64_t importance_bytes_per_token; /* fp64 read + write per token, all layers/instances */
} kvp_engine_info;

/* Device pointers of one layer's state (for tests / inspection). */
typedef struct {
  const void *left_k, *left_v, *right_k, *right_v, *tail_k, *tail_v;
  const double* importance;
  const void *w_qkv, *w_o;
  int32_t n_tail;
} kvp_engine_layer_view;

typedef struct kvp_engine kvp_engine;

int kvp_engine_create(const kvp_engine_config* config, kvp_engine** engine);
int kvp_engine_destroy(kvp_engine* engine);
/* Generate the workload on the device (weights, prefill K/V) and compact it. */
int kvp_engine_prefill(kvp_engine* engine);
/* One decode step for every instance: x, y are [dev] batch x H*D fp32. */
int kvp_engine_step(kvp_engine* engine, const float* x, float* y, void* stream);
/* Same with [host] buffers (pinned for best results): H2D, step, D2H, sync. */
int kvp_engine_step_host(kvp_engine* engine, const float* x, float* y);
int kvp_engine_reset_steps(kvp_engine* engine);
int kvp_engine_get_info(kvp_engine* engine, kvp_engine_info* info);
int kvp_engine_layer_state(kvp_engine* engine, int32_t layer, kvp_engine_layer_view* view);
/* Times the attention launches alone (all layers, current tail length) and
 * reports ms per layer and the algorithmic bytes per layer. */
int kvp_engine_time_attention(kvp_engine* engine, int32_t iters, double* ms_per_layer, double* bytes_per_layer);

#ifdef __cplusplus
}
#endif
#endif /* KVP_B200_H */
