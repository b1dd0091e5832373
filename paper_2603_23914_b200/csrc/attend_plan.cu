// Generic retrieval-plan attention on the GPU, evaluated in the low-rank
// space.  Replaces attend_materialized / attend_fused
// (/root/reference/proj/src/decoder.cpp:190-344) for any plan the reference
// can build: any mix of low-rank / dense stores, tier rank prefixes per
// entry, T_q >= 1 with causal visibility by global position, GQA.
//
// The reference rebuilds every row (store_decompress_row, cache.cpp:63-101:
// W*rank MACs per row) and then attends.  Here nothing of width W is rebuilt:
//
//   P_s[(i,h), r]  = sum_c right_k_s[r, g*D+c] * q[i, h*D+c]          (per K store)
//   logit[(i,h),j] = sum_{r<rk_j} left_k[row_j, r] * P_s[(i,h), r] / sqrt(D)
//   m, z           = max / sum exp over visible j
//   U_s[(i,h), r] += exp(logit-m) * left_v[row_j, r]   (r < rv_j)      (per V store)
//   ctx[(i,h), c]  = (sum_s sum_r U_s[(i,h), r] right_v_s[r, g*D+c] + dense part) / z
//
// Arithmetic is fp64 like the reference's double accumulators, so float and
// double caches agree with the oracle to ~1e-12 relative.  This path is the
// parity workhorse and the general-plan fallback *on the GPU*; the batched
// bf16 serving path is the fused cluster kernel in decode_fused.cu.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "attend_plan.cuh"

namespace kvp {
namespace {

struct DevPlan {
  int H, Hkv, D, per_kv, tq, n, n_stores, table_size;
  const kvp_store* stores;          // [batch][n_stores]
  const kvp_plan_entry* entries;    // [batch][n]
  const double* q;                  // [batch][tq][H*D]
  const uint64_t* qpos;             // [tq] (shared by the batch)
  const long* p_off;  // per store offset of its P block (doubles), -1 if none
  const long* u_off;  // per store offset of its U block (doubles), -1 if none
  long p_total, u_total;            // doubles of P / U per instance
  double* P;
  double* U;
  double* logits;  // [batch] (tq*H) x n
  double* m;       // [batch] tq*H
  double* z;       // [batch] tq*H
  double* ctx_dense;  // [batch] (tq*H) x D
};

// The instance of this block (gridDim.z = batch): every per-instance array is
// offset here, so the kernels below read like the single-instance form.
__device__ __forceinline__ DevPlan at_instance(DevPlan p) {
  const long bi = blockIdx.z;
  const long THq = (long)p.tq * p.H;
  p.stores += bi * p.n_stores;
  p.entries += bi * p.n;
  p.q += bi * THq * p.D;
  p.P += bi * p.p_total;
  p.U += bi * p.u_total;
  p.logits += bi * THq * p.n;
  p.m += bi * THq;
  p.z += bi * THq;
  p.ctx_dense += bi * THq * p.D;
  return p;
}

template <typename T>
__device__ __forceinline__ double ld(const void* base, long idx) {
  return to_d(static_cast<const T*>(base)[idx]);
}

// P_s = right_k_s[:, g-slice] q_h for every low-rank key store.
template <typename T>
__global__ void project_queries(DevPlan p) {
  p = at_instance(p);
  const int s = blockIdx.x, ih = blockIdx.y;
  const kvp_store st = p.stores[s];
  if (p.p_off[s] < 0) return;
  const int i = ih / p.H, h = ih % p.H, g = h / p.per_kv;
  const double* q = p.q + (long)i * p.H * p.D + (long)h * p.D;
  double* out = p.P + p.p_off[s] + (long)ih * st.rank;
  for (int r = threadIdx.x; r < st.rank; r += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < p.D; ++c) acc += ld<T>(st.b, (long)r * st.ldb + (long)g * p.D + c) * q[c];
    out[r] = acc;
  }
}

template <typename T>
__global__ void score_entries(DevPlan p, double inv_sqrt_d) {
  p = at_instance(p);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int ih = blockIdx.y;
  if (j >= p.n) return;
  const int i = ih / p.H, h = ih % p.H, g = h / p.per_kv;
  const kvp_plan_entry e = p.entries[j];
  double logit = -INFINITY;
  if (e.position <= p.qpos[i]) {
    const kvp_store st = p.stores[e.k_store];
    double dot = 0.0;
    if (st.form == KVP_LOWRANK) {
      const int r_use = (e.rank_k == 0 || (int)e.rank_k > st.rank) ? st.rank : (int)e.rank_k;
      const double* P = p.P + p.p_off[e.k_store] + (long)ih * st.rank;
      for (int r = 0; r < r_use; ++r) dot += ld<T>(st.a, (long)e.row * st.lda + r) * P[r];
    } else {
      const double* q = p.q + (long)i * p.H * p.D + (long)h * p.D;
      for (int c = 0; c < p.D; ++c) dot += ld<T>(st.a, (long)e.row * st.lda + (long)g * p.D + c) * q[c];
    }
    logit = dot * inv_sqrt_d;
  }
  p.logits[(long)ih * p.n + j] = logit;
}

__global__ void softmax_stats(DevPlan p) {
  p = at_instance(p);
  const int ih = blockIdx.x;
  const double* l = p.logits + (long)ih * p.n;
  __shared__ double red[256];
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < p.n; j += blockDim.x) mx = fmax(mx, l[j]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  double zs = 0.0;
  for (int j = threadIdx.x; j < p.n; j += blockDim.x)
    if (l[j] != -INFINITY) zs += exp(l[j] - mx);
  red[threadIdx.x] = zs;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    p.m[ih] = mx;
    p.z[ih] = red[0];
  }
}

// head_avg(i, j) += exp(l - m_h) / z_h * (1/H), heads in ascending order
// (decoder.cpp:247-250).
__global__ void head_average(DevPlan p, double* head_avg, double* head_avg_table, long table_stride,
                             double inv_heads) {
  p = at_instance(p);
  if (head_avg) head_avg += (long)blockIdx.z * p.tq * p.n;
  if (head_avg_table) head_avg_table += (long)blockIdx.z * p.tq * table_stride;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= p.n) return;
  double acc = 0.0;
  for (int h = 0; h < p.H; ++h) {
    const int ih = i * p.H + h;
    const double l = p.logits[(long)ih * p.n + j];
    if (l != -INFINITY) acc += exp(l - p.m[ih]) / p.z[ih] * inv_heads;
  }
  if (head_avg) head_avg[(long)i * p.n + j] = acc;
  const int t = p.entries[j].table_index;
  if (head_avg_table && t >= 0) head_avg_table[(long)i * table_stride + t] = acc;
}

// U_s and the dense-value context, one block per (query, head); entries in
// plan order so every accumulator has a single owner (no atomics).
template <typename T>
__global__ void accumulate_values(DevPlan p) {
  p = at_instance(p);
  const int ih = blockIdx.x;
  const int h = ih % p.H, g = h / p.per_kv;
  const double mx = p.m[ih];
  double* cd = p.ctx_dense + (long)ih * p.D;
  for (int c = threadIdx.x; c < p.D; c += blockDim.x) cd[c] = 0.0;
  for (int s = 0; s < p.n_stores; ++s) {
    if (p.u_off[s] < 0) continue;
    double* u = p.U + p.u_off[s] + (long)ih * p.stores[s].rank;
    for (int r = threadIdx.x; r < p.stores[s].rank; r += blockDim.x) u[r] = 0.0;
  }
  __syncthreads();
  for (int j = 0; j < p.n; ++j) {
    const double l = p.logits[(long)ih * p.n + j];
    if (l == -INFINITY) continue;
    const double w = exp(l - mx);
    const kvp_plan_entry e = p.entries[j];
    const kvp_store st = p.stores[e.v_store];
    if (st.form == KVP_LOWRANK) {
      const int r_use = (e.rank_v == 0 || (int)e.rank_v > st.rank) ? st.rank : (int)e.rank_v;
      double* u = p.U + p.u_off[e.v_store] + (long)ih * st.rank;
      for (int r = threadIdx.x; r < r_use; r += blockDim.x) u[r] += w * ld<T>(st.a, (long)e.row * st.lda + r);
    } else {
      for (int c = threadIdx.x; c < p.D; c += blockDim.x)
        cd[c] += w * ld<T>(st.a, (long)e.row * st.lda + (long)g * p.D + c);
    }
  }
}

template <typename T>
__global__ void emit_context(DevPlan p, double* context) {
  p = at_instance(p);
  context += (long)blockIdx.z * p.tq * p.H * p.D;
  const int ih = blockIdx.x;
  const int i = ih / p.H, h = ih % p.H, g = h / p.per_kv;
  const double inv_z = 1.0 / p.z[ih];
  for (int c = threadIdx.x; c < p.D; c += blockDim.x) {
    double acc = p.ctx_dense[(long)ih * p.D + c];
    for (int s = 0; s < p.n_stores; ++s) {
      if (p.u_off[s] < 0) continue;
      const kvp_store st = p.stores[s];
      const double* u = p.U + p.u_off[s] + (long)ih * st.rank;
      for (int r = 0; r < st.rank; ++r) acc += u[r] * ld<T>(st.b, (long)r * st.ldb + (long)g * p.D + c);
    }
    context[(long)i * p.H * p.D + (long)h * p.D + c] = acc * inv_z;
  }
}

// Batched plan attention.  `stores` [host] batch x n_stores (every instance
// has the same store structure, ranks may differ), `entries` [dev or host]
// batch x n, queries [dev] batch x tq x H*D (fp64), context [dev] batch x tq x H*D.
template <typename T>
void run_plan_batched(const PlanBatch& d, cudaStream_t s) {
  DevPlan p{};
  p.H = d.heads;
  p.Hkv = d.kv_heads;
  p.D = d.head_dim;
  p.per_kv = d.heads / d.kv_heads;
  p.tq = d.tq;
  p.n = d.n_entries;
  p.n_stores = d.n_stores;
  p.table_size = d.table_size;
  const long THq = (long)d.tq * d.heads;
  const int B = d.batch;

  // Which stores are referenced as low-rank keys / values (every store of the
  // structure when the plan lives on the device); offsets sized by the batch's
  // largest rank per store.
  std::vector<long> p_off(d.n_stores, -1), u_off(d.n_stores, -1);
  std::vector<char> k_used(d.n_stores, d.entries_on_device ? 1 : 0), v_used(d.n_stores, d.entries_on_device ? 1 : 0);
  if (!d.entries_on_device) {
    for (long j = 0; j < (long)B * d.n_entries; ++j) {
      const kvp_plan_entry& e = d.entries[j];
      require(e.k_store >= 0 && e.k_store < d.n_stores && e.v_store >= 0 && e.v_store < d.n_stores,
              KVP_ERR_PARAMETER, "attend: plan entry references an unknown store");
      k_used[e.k_store] = 1;
      v_used[e.v_store] = 1;
    }
  }
  long p_total = 0, u_total = 0;
  for (int st_i = 0; st_i < d.n_stores; ++st_i) {
    int rmax = 0;
    for (int b = 0; b < B; ++b) {
      const kvp_store& st = d.stores[(long)b * d.n_stores + st_i];
      require(st.form == KVP_DENSE || st.form == KVP_LOWRANK, KVP_ERR_PARAMETER, "attend: bad store form");
      require(st.a != nullptr, KVP_ERR_PARAMETER, "attend: store without payload");
      if (st.form == KVP_LOWRANK) {
        require(st.rank >= 1 && st.b != nullptr, KVP_ERR_PARAMETER,
                "attend: low-rank store needs rank and right factor");
        rmax = rmax > st.rank ? rmax : st.rank;
      }
    }
    if (rmax > 0) {
      if (k_used[st_i]) { p_off[st_i] = p_total; p_total += THq * rmax; }
      if (v_used[st_i]) { u_off[st_i] = u_total; u_total += THq * rmax; }
    }
  }
  p.p_total = p_total;
  p.u_total = u_total;
  const size_t n_bytes = sizeof(kvp_store) * B * d.n_stores +
                         (d.entries_on_device ? 0 : sizeof(kvp_plan_entry) * B * d.n_entries) +
                         2 * sizeof(long) * d.n_stores;
  const size_t f_bytes =
      sizeof(double) * B * (p_total + u_total + THq * (long)d.n_entries + 2 * THq + THq * d.head_dim);
  Scratch scratch(n_bytes + f_bytes + 64, s);
  char* base = scratch.as<char>();
  // Descriptors are tiny: copied from pageable host memory on the stream.
  auto* dstores = reinterpret_cast<kvp_store*>(base);
  auto* dentries = reinterpret_cast<kvp_plan_entry*>(dstores + (long)B * d.n_stores);
  auto* dpoff = reinterpret_cast<long*>(dentries + (d.entries_on_device ? 0 : (long)B * d.n_entries));
  auto* duoff = dpoff + d.n_stores;
  auto* fbase = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(duoff + d.n_stores) + 15) & ~uintptr_t(15));
  KVP_CUDA(cudaMemcpyAsync(dstores, d.stores, sizeof(kvp_store) * B * d.n_stores, cudaMemcpyHostToDevice, s));
  if (!d.entries_on_device)
    KVP_CUDA(cudaMemcpyAsync(dentries, d.entries, sizeof(kvp_plan_entry) * B * d.n_entries, cudaMemcpyHostToDevice,
                             s));
  KVP_CUDA(cudaMemcpyAsync(dpoff, p_off.data(), sizeof(long) * d.n_stores, cudaMemcpyHostToDevice, s));
  KVP_CUDA(cudaMemcpyAsync(duoff, u_off.data(), sizeof(long) * d.n_stores, cudaMemcpyHostToDevice, s));
  p.stores = dstores;
  p.entries = d.entries_on_device ? d.entries : dentries;
  p.p_off = dpoff;
  p.u_off = duoff;
  p.q = d.queries;
  p.qpos = d.query_positions;
  p.P = fbase;
  p.U = p.P + (long)B * p_total;
  p.logits = p.U + (long)B * u_total;
  p.m = p.logits + (long)B * THq * d.n_entries;
  p.z = p.m + (long)B * THq;
  p.ctx_dense = p.z + (long)B * THq;

  const double inv_sqrt_d = 1.0 / std::sqrt(static_cast<double>(d.head_dim));
  if (p_total > 0) {
    project_queries<T><<<dim3(d.n_stores, THq, B), 128, 0, s>>>(p);
    KVP_LAUNCHED();
  }
  score_entries<T><<<dim3(cdiv(d.n_entries, 128), THq, B), 128, 0, s>>>(p, inv_sqrt_d);
  KVP_LAUNCHED();
  softmax_stats<<<dim3(THq, 1, B), 256, 0, s>>>(p);
  KVP_LAUNCHED();
  if (d.head_avg || d.head_avg_table) {
    head_average<<<dim3(cdiv(d.n_entries, 128), d.tq, B), 128, 0, s>>>(
        p, d.head_avg, d.head_avg_table, d.table_stride, 1.0 / static_cast<double>(d.heads));
    KVP_LAUNCHED();
  }
  accumulate_values<T><<<dim3(THq, 1, B), 128, 0, s>>>(p);
  KVP_LAUNCHED();
  emit_context<T><<<dim3(THq, 1, B), 128, 0, s>>>(p, d.context);
  KVP_LAUNCHED();
}

}  // namespace

void run_plan(const PlanBatch& d, cudaStream_t s) {
  switch (d.dtype) {
    case KVP_F32: run_plan_batched<float>(d, s); break;
    case KVP_F64: run_plan_batched<double>(d, s); break;
    case KVP_BF16: run_plan_batched<__nv_bfloat16>(d, s); break;
    default: fail(KVP_ERR_PARAMETER, "attend: unknown dtype");
  }
}
}  // namespace kvp

extern "C" int kvp_attend_plan(const kvp_attend_desc* d, void* stream) {
  return kvp::guarded([&] {
    using namespace kvp;
    require(d != nullptr, KVP_ERR_PARAMETER, "attend: null descriptor");
    require(d->heads > 0 && d->kv_heads > 0 && d->head_dim > 0, KVP_ERR_PARAMETER,
            "HeadGeometry: head counts and head_dim must be positive");
    require(d->heads % d->kv_heads == 0, KVP_ERR_PARAMETER, "HeadGeometry: num_kv_heads must divide num_query_heads");
    require(d->n_entries > 0, KVP_ERR_PARAMETER, "attend: empty retrieval plan");
    require(d->tq > 0, KVP_ERR_SHAPE, "attend: one position per query row required");
    require(d->queries && d->query_positions && d->context, KVP_ERR_PARAMETER, "attend: null buffer");
    PlanBatch pb{};
    pb.heads = d->heads;
    pb.kv_heads = d->kv_heads;
    pb.head_dim = d->head_dim;
    pb.dtype = d->dtype;
    pb.batch = 1;
    pb.n_stores = d->n_stores;
    pb.n_entries = d->n_entries;
    pb.tq = d->tq;
    pb.table_size = d->table_size;
    pb.table_stride = d->table_size;
    pb.stores = d->stores;
    pb.entries = d->entries;
    pb.entries_on_device = false;
    pb.queries = d->queries;
    pb.query_positions = d->query_positions;
    pb.context = d->context;
    pb.head_avg = d->head_avg;
    pb.head_avg_table = d->head_avg_table;
    run_plan(pb, as_stream(stream));
  });
}
