// Serving-layout plumbing for the one-launch layer kernel (decode_layer.cu):
// left factors packed into tcgen05 operand tiles, right factors and tails
// stored head-major, and the kvp_decode_fused C-ABI entry (decode_step's
// attention + importance for a batch, decoder.cpp:583-601).
#include <cuda_bf16.h>

#include <cmath>
#include <memory>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "decode_fused.cuh"
#include "sm100.cuh"

namespace kvp {
namespace {
constexpr uint32_t kStageBytes = 16384;
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

// [batch][rows][H_kv*D] (row-major, the reference's Matrix layout) <-> head-major
// [batch][H_kv][rows][D]: each kv head's slice becomes one contiguous run.
__global__ void heads_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int Hkv, int D, int to_heads) {
  const long per = static_cast<long>(rows) * Hkv * D;
  const int b = blockIdx.y;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < per;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long r = i / (static_cast<long>(Hkv) * D);
    const int col = static_cast<int>(i % (static_cast<long>(Hkv) * D)), g = col / D, j = col % D;
    const long hm = (static_cast<long>(g) * rows + r) * D + j;
    if (to_heads) dst[b * per + hm] = src[b * per + i];
    else dst[b * per + i] = src[b * per + hm];
  }
}
}  // namespace

void pack_heads(const void* src, void* dst, int batch, int rows, int Hkv, int D, bool to_heads, cudaStream_t st) {
  heads_kernel<<<dim3(128, batch), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src),
                                                 static_cast<__nv_bfloat16*>(dst), rows, Hkv, D, to_heads ? 1 : 0);
  KVP_LAUNCHED();
}

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

extern "C" int kvp_pack_heads(const void* src, void* dst, int32_t batch, int32_t rows, int32_t kv_heads,
                              int32_t head_dim, int32_t to_heads, void* stream) {
  return kvp::guarded([&] {
    kvp::require(src && dst && src != dst && batch > 0 && rows >= 0 && kv_heads > 0 && head_dim > 0,
                 KVP_ERR_PARAMETER, "pack_heads: bad arguments");
    if (rows > 0) kvp::pack_heads(src, dst, batch, rows, kv_heads, head_dim, to_heads != 0, kvp::as_stream(stream));
  });
}

// Debug hooks (not part of the public header).
static unsigned long long* g_trace = nullptr;
extern "C" void kvp_debug_fused_trace(void* dev_buffer) { g_trace = static_cast<unsigned long long*>(dev_buffer); }

extern "C" int kvp_debug_fused_max_clusters(const kvp_fused_desc* d) {
  int n = -1;
  kvp::guarded([&] {
    kvp::FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, 0, d->tail_cap, d->batch,
                      d->cluster > 0 ? d->cluster : kvp::auto_layer_cluster(kvp::FusedShape{
                                                        d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k,
                                                        d->rank_v, 0, d->tail_cap, d->batch, 0})};
    n = kvp::layer_max_active_clusters(kvp::plan_layer(s));
  });
  return n;
}

extern "C" int kvp_debug_fused_cluster(const kvp_fused_desc* d) {
  int n = -1;
  kvp::guarded([&] {
    n = d->cluster > 0 ? d->cluster
                       : kvp::auto_layer_cluster(kvp::FusedShape{d->heads, d->kv_heads, d->head_dim, d->n_comp,
                                                                 d->rank_k, d->rank_v, 0, d->tail_cap, d->batch, 0});
  });
  return n;
}

// Exchange area of the CTA groups (P image, statistics, U partials, context).
extern "C" size_t kvp_decode_fused_workspace(const kvp_fused_desc* d) {
  size_t n = 0;
  kvp::guarded([&] {
    kvp::FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, 0, d->tail_cap, d->batch,
                      d->cluster};
    if (s.cluster <= 0) s.cluster = kvp::auto_layer_cluster(s);
    const kvp::LayerPlan lp = kvp::plan_layer(s);
    if (lp.ok) n = kvp::layer_group_ws_bytes(lp);
  });
  return n;
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
    require(d->left_k && d->left_v && d->right_k && d->right_v && d->queries && d->context, KVP_ERR_PARAMETER,
            "decode_fused: null buffer");
    require(d->tail_cap == 0 || (d->tail_k && d->tail_v), KVP_ERR_PARAMETER, "decode_fused: null tail buffer");
    FusedShape s{d->heads, d->kv_heads, d->head_dim, d->n_comp, d->rank_k, d->rank_v, 0, d->tail_cap, d->batch,
                 d->cluster};
    if (s.cluster <= 0) s.cluster = auto_layer_cluster(s);
    const LayerPlan lp = plan_layer(s);
    require(lp.ok, KVP_ERR_PARAMETER, (std::string("decode_fused: ") + lp.why).c_str());
    FusedArgs a{};
    a.left_k_packed = static_cast<const unsigned char*>(d->left_k);
    a.left_v_packed = static_cast<const unsigned char*>(d->left_v);
    a.right_k = static_cast<const __nv_bfloat16*>(d->right_k);
    a.right_v = static_cast<const __nv_bfloat16*>(d->right_v);
    a.tail_k = static_cast<const __nv_bfloat16*>(d->tail_k);
    a.tail_v = static_cast<const __nv_bfloat16*>(d->tail_v);
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
    a.trace = g_trace;
    const size_t ws_bytes = layer_group_ws_bytes(lp);
    std::unique_ptr<Scratch> own;
    if (d->workspace == nullptr) {  // stream-ordered scratch, barrier words zeroed
      own = std::make_unique<Scratch>(ws_bytes, as_stream(stream));
      KVP_CUDA(cudaMemsetAsync(own->p, 0, ws_bytes, as_stream(stream)));
      a.group_ws = own->as<unsigned char>();
    } else {
      require(d->workspace_bytes >= ws_bytes, KVP_ERR_PARAMETER, "decode_fused: workspace too small");
      a.group_ws = static_cast<unsigned char*>(d->workspace);
    }
    launch_layer(lp, a, as_stream(stream));
  });
}
