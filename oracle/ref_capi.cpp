// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Plain-C entry points over the reference's own implementation (compiled from
// /root/reference/proj/src by oracle/Makefile) so that the Python tests,
// the golden-fixture generator and bench.py's cpu_baseline leg can drive the
// reference through ctypes.  Values cross as float64 and are cast to the
// engine precision T (float or double) exactly like the reference's pybind11
// module does (bindings/module.cpp:29-47).  Status codes mirror the product
// C-ABI (include/kvp_b200.h): 0 ok, 1 parameter, 2 shape, 3 data, 4 io, 5 other.
#include <cstdint>
#include <cstring>
#include <string>
#include <variant>
#include <vector>

#include "kvpack/cache.hpp"
#include "kvpack/config.hpp"
#include "kvpack/decoder.hpp"
#include "kvpack/harness.hpp"
#include "kvpack/importance.hpp"
#include "kvpack/linalg.hpp"
#include "kvpack/quantize.hpp"
#include "kvpack/snapshot.hpp"

using namespace kvpack;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const shape_error& e) {
        g_err = e.what();
        return 2;
    } catch (const parameter_error& e) {
        g_err = e.what();
        return 1;
    } catch (const data_error& e) {
        g_err = e.what();
        return 3;
    } catch (const io_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

template <typename T>
Matrix<T> mat_in(std::size_t r, std::size_t c, const double* p) {
    Matrix<T> m(r, c);
    for (std::size_t i = 0; i < r * c; ++i) m.data[i] = static_cast<T>(p[i]);
    return m;
}

template <typename T>
void mat_out(const Matrix<T>& m, double* p) {
    for (std::size_t i = 0; i < m.data.size(); ++i) p[i] = static_cast<double>(m.data[i]);
}

DecodeConfig decode_cfg(const char* ini) {
    return parse_config_text(ini ? std::string(ini) : std::string()).decode;
}

template <typename C>
struct scalar_of;
template <typename T>
struct scalar_of<LayerCache<T>> {
    using type = T;
};

using AnyCache = std::variant<LayerCache<double>, LayerCache<float>>;

template <typename F>
void with_cache(void* h, F&& f) {
    std::visit([&](auto& c) { f(c); }, *static_cast<AnyCache*>(h));
}

Modality mod(int m) { return m == 0 ? Modality::visual : Modality::textual; }
MatrixKind kind_of(int k) { return k == 0 ? MatrixKind::key : MatrixKind::value; }

template <typename T>
AttentionWeights<T> weights_in(std::size_t hd, std::size_t cw, const double* wq, const double* wk,
                               const double* wv, const double* wo) {
    AttentionWeights<T> w;
    w.w_q = mat_in<T>(hd, hd, wq);
    w.w_k = mat_in<T>(hd, cw, wk);
    w.w_v = mat_in<T>(hd, cw, wv);
    w.w_o = mat_in<T>(hd, hd, wo);
    return w;
}

} // namespace

extern "C" {

// Plan entry as returned to the tests; `segment` 0 visual / 1 textual,
// `block` = block index inside the segment or -1 for tail rows.
struct kvref_plan_entry {
    std::int32_t segment;
    std::int32_t block;
    std::uint32_t row;
    std::uint32_t rank_k;
    std::uint32_t rank_v;
    std::uint32_t pad;
    std::uint64_t position;
};

struct kvref_step_report {
    std::uint64_t step, bytes_before, bytes_after, importance_bytes;
    std::uint64_t decompress_flops, decompress_flops_full;
    double flops_reduction;
    std::int32_t compression_event;
    std::int32_t n_warnings;
};

const char* kvref_last_error() { return g_err.c_str(); }

void* kvref_cache_new(int dtype, std::size_t heads, std::size_t kv_heads, std::size_t head_dim,
                      std::size_t layer) {
    const HeadGeometry g{heads, kv_heads, head_dim};
    if (dtype == 1) return new AnyCache(std::in_place_type<LayerCache<float>>, g, layer);
    return new AnyCache(std::in_place_type<LayerCache<double>>, g, layer);
}

void kvref_cache_free(void* h) { delete static_cast<AnyCache*>(h); }

// KVPK snapshots through the reference's own save_cache / load_cache (snapshot.cpp:251-371).
int kvref_save_cache(void* h, const char* path, std::size_t width) {
    return guarded([&] { with_cache(h, [&](auto& c) { save_cache(c, std::string(path), width); }); });
}

int kvref_load_cache(int dtype, const char* path, void** out) {
    return guarded([&] {
        if (dtype == 1)
            *out = new AnyCache(std::in_place_type<LayerCache<float>>, load_cache<float>(std::string(path)));
        else
            *out = new AnyCache(std::in_place_type<LayerCache<double>>, load_cache<double>(std::string(path)));
    });
}

int kvref_append(void* h, int modality, std::size_t n, const double* k, const double* v) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            using T = typename scalar_of<std::decay_t<decltype(c)>>::type;
            const std::size_t w = c.geometry.cache_width();
            append_tokens(c, mod(modality), mat_in<T>(n, w, k), mat_in<T>(n, w, v));
        });
    });
}

int kvref_compress_now(void* h, const char* ini) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            StepReport rep;
            compress_now(c, decode_cfg(ini), rep);
        });
    });
}

int kvref_decode_step(void* h, const char* ini, std::size_t tq, const double* x, const double* wq,
                      const double* wk, const double* wv, const double* wo, double* out,
                      kvref_step_report* report) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            using T = typename scalar_of<std::decay_t<decltype(c)>>::type;
            const std::size_t hd = c.geometry.model_width(), cw = c.geometry.cache_width();
            const AttentionWeights<T> w = weights_in<T>(hd, cw, wq, wk, wv, wo);
            StepReport rep;
            const Matrix<T> y = decode_step(mat_in<T>(tq, hd, x), c, w, decode_cfg(ini), rep);
            mat_out(y, out);
            if (report) {
                report->step = rep.step;
                report->bytes_before = rep.bytes_before;
                report->bytes_after = rep.bytes_after;
                report->importance_bytes = rep.importance_bytes;
                report->decompress_flops = rep.decompress_flops;
                report->decompress_flops_full = rep.decompress_flops_full;
                report->flops_reduction = rep.flops_reduction;
                report->compression_event = rep.compression_event ? 1 : 0;
                report->n_warnings = static_cast<std::int32_t>(rep.warnings.size());
            }
        });
    });
}

// Test hook: turn the segment's tail into its single joint block with the
// given factors instead of an SVD (what recompress_segment, decoder.cpp:455-497,
// stores after compress_segment), so the reference can be driven on the exact
// factors a GPU path holds.  rank 0 keeps that kind dense (the tail rows).
// k_left: tokens x rank_k, k_right: rank_k x width (likewise v).
int kvref_factor_tail(void* h, int modality, std::size_t rank_k, const double* k_left,
                      const double* k_right, std::size_t rank_v, const double* v_left,
                      const double* v_right) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            using T = typename scalar_of<std::decay_t<decltype(c)>>::type;
            auto& seg = c.segment(mod(modality));
            if (!seg.blocks.empty()) throw parameter_error("kvref_factor_tail: segment already has blocks");
            const std::size_t n = seg.tail_len(), w = c.geometry.cache_width();
            if (n == 0) throw parameter_error("kvref_factor_tail: empty tail");
            CompressedBlock<T> block;
            block.positions = seg.tail_positions;
            auto store = [&](std::size_t rank, const double* l, const double* r,
                             const Matrix<T>& rows) -> BlockStore<T> {
                if (rank == 0) return DenseStore<T>{rows};
                return LowRankStore<T>{FactorPair<T>{mat_in<T>(n, rank, l), mat_in<T>(rank, w, r)}};
            };
            block.keys = store(rank_k, k_left, k_right, seg.tail_k);
            block.values = store(rank_v, v_left, v_right, seg.tail_v);
            seg.blocks.push_back(std::move(block));
            seg.tail_k = Matrix<T>(0, w);
            seg.tail_v = Matrix<T>(0, w);
            seg.tail_positions.clear();
        });
    });
}

// Plan size for the cache under `ini` (so the caller can size buffers).
int kvref_plan_size(void* h, const char* ini, std::size_t* n) {
    return guarded([&] {
        with_cache(h, [&](auto& c) { *n = build_retrieval_plan(c, decode_cfg(ini)).size(); });
    });
}

// build_retrieval_plan + attend_{materialized,fused}.  context: tq x HD,
// head_avg: tq x n (plan order), entries: n.
int kvref_attend(void* h, const char* ini, std::size_t tq, const double* queries,
                 const std::uint64_t* qpos, int fused, std::size_t tile, double* context,
                 double* head_avg, kvref_plan_entry* entries) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            using T = typename scalar_of<std::decay_t<decltype(c)>>::type;
            const DecodeConfig cfg = decode_cfg(ini);
            const RetrievalPlan<T> plan = build_retrieval_plan(c, cfg);
            const std::vector<std::uint64_t> qp(qpos, qpos + tq);
            const Matrix<T> q = mat_in<T>(tq, c.geometry.model_width(), queries);
            const AttentionResult<T> r = fused ? attend_fused(plan, q, qp, c.geometry, tile)
                                               : attend_materialized(plan, q, qp, c.geometry);
            mat_out(r.context, context);
            mat_out(r.head_avg, head_avg);
            for (std::size_t j = 0; j < plan.size(); ++j) {
                const auto& e = plan.entries[j];
                kvref_plan_entry& o = entries[j];
                o.row = e.row;
                o.rank_k = e.rank_k;
                o.rank_v = e.rank_v;
                o.position = e.position;
                o.pad = 0;
                o.block = -1;
                if (e.keys) {
                    o.segment = -1;
                    for (int s = 0; s < 2; ++s) {
                        const auto& seg = c.segment(mod(s));
                        for (std::size_t b = 0; b < seg.blocks.size(); ++b)
                            if (&seg.blocks[b].keys == e.keys) {
                                o.segment = s;
                                o.block = static_cast<std::int32_t>(b);
                            }
                    }
                } else {
                    o.segment = e.tail_k == &c.visual.tail_k ? 0 : 1;
                }
            }
        });
    });
}

// ---- state accessors -------------------------------------------------------

int kvref_importance_size(void* h, std::size_t* n) {
    return guarded([&] { with_cache(h, [&](auto& c) { *n = c.importance.size(); }); });
}

int kvref_importance_get(void* h, std::uint64_t* positions, double* scores) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            for (std::size_t i = 0; i < c.importance.size(); ++i) {
                positions[i] = c.importance.positions[i];
                scores[i] = c.importance.scores[i];
            }
        });
    });
}

int kvref_importance_set(void* h, const double* scores) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            for (std::size_t i = 0; i < c.importance.size(); ++i) c.importance.scores[i] = scores[i];
        });
    });
}

// Segment shape: number of blocks, tail length, next_position.
int kvref_segment_info(void* h, int modality, std::size_t* n_blocks, std::size_t* tail_len,
                       std::uint64_t* next_position) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            const auto& seg = c.segment(mod(modality));
            *n_blocks = seg.blocks.size();
            *tail_len = seg.tail_len();
            *next_position = c.next_position;
        });
    });
}

// Block store shape: tokens, rank (0 = dense), width.
int kvref_block_info(void* h, int modality, std::size_t block, int kind, std::size_t* tokens,
                     std::size_t* rank, std::size_t* width) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            const auto& b = c.segment(mod(modality)).blocks.at(block);
            const auto& s = kind_of(kind) == MatrixKind::key ? b.keys : b.values;
            *tokens = store_token_count(s);
            *rank = store_rank(s);
            *width = store_width(s);
        });
    });
}

// Copy one block store: low-rank -> left (tokens x rank) + right (rank x width);
// dense -> rows into `left` (tokens x width).  positions: tokens.
int kvref_block_get(void* h, int modality, std::size_t block, int kind, double* left,
                    double* right, std::uint64_t* positions) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            using T = typename scalar_of<std::decay_t<decltype(c)>>::type;
            const auto& b = c.segment(mod(modality)).blocks.at(block);
            const auto& s = kind_of(kind) == MatrixKind::key ? b.keys : b.values;
            if (const auto* lr = std::get_if<LowRankStore<T>>(&s)) {
                mat_out(lr->factors.left, left);
                mat_out(lr->factors.right, right);
            } else if (const auto* d = std::get_if<DenseStore<T>>(&s)) {
                mat_out(d->rows, left);
            } else {
                throw parameter_error("kvref_block_get: quantized stores not exported");
            }
            if (positions)
                for (std::size_t i = 0; i < b.positions.size(); ++i) positions[i] = b.positions[i];
        });
    });
}

int kvref_tail_get(void* h, int modality, double* k, double* v, std::uint64_t* positions) {
    return guarded([&] {
        with_cache(h, [&](auto& c) {
            const auto& seg = c.segment(mod(modality));
            if (k) mat_out(seg.tail_k, k);
            if (v) mat_out(seg.tail_v, v);
            if (positions)
                for (std::size_t i = 0; i < seg.tail_len(); ++i)
                    positions[i] = seg.tail_positions[i];
        });
    });
}

// ---- free functions --------------------------------------------------------

int kvref_truncated_svd(int dtype, std::size_t rows, std::size_t cols, const double* a,
                        std::size_t rank, int randomized, std::uint64_t seed,
                        std::size_t oversampling, std::size_t power_iterations, double* left,
                        double* right) {
    return guarded([&] {
        SvdOptions o;
        o.method = randomized ? SvdMethod::randomized : SvdMethod::exact;
        o.seed = seed;
        o.oversampling = oversampling;
        o.power_iterations = power_iterations;
        if (dtype == 1) {
            const FactorPair<float> f = truncated_svd(mat_in<float>(rows, cols, a), rank, o);
            mat_out(f.left, left);
            mat_out(f.right, right);
        } else {
            const FactorPair<double> f = truncated_svd(mat_in<double>(rows, cols, a), rank, o);
            mat_out(f.left, left);
            mat_out(f.right, right);
        }
    });
}

int kvref_singular_values(std::size_t rows, std::size_t cols, const double* a, double* out) {
    return guarded([&] {
        const std::vector<double> s = singular_values(mat_in<double>(rows, cols, a));
        std::memcpy(out, s.data(), s.size() * sizeof(double));
    });
}

// tier_of[i] = group index of compressed token i (masks are the ascending
// index lists of each group, importance.cpp:67-117).
int kvref_assign_groups(std::size_t n, const double* scores, const std::uint64_t* positions,
                        std::size_t groups, const double* ratios, const std::size_t* ranks,
                        std::uint32_t* tier_of) {
    return guarded([&] {
        ImportanceTable t;
        for (std::size_t i = 0; i < n; ++i) t.append_token(positions[i]);
        t.scores.assign(scores, scores + n);
        const std::vector<std::uint64_t> pos(positions, positions + n);
        const GroupAssignment g = assign_groups(t, pos, std::vector<double>(ratios, ratios + groups),
                                                std::vector<std::size_t>(ranks, ranks + groups));
        for (std::size_t f = 0; f < g.masks.size(); ++f)
            for (std::uint32_t i : g.masks[f]) tier_of[i] = static_cast<std::uint32_t>(f);
    });
}

int kvref_update_importance(std::size_t n, double* scores, std::size_t tq, const double* attn,
                            double alpha) {
    return guarded([&] {
        ImportanceTable t;
        t.alpha = alpha;
        for (std::size_t i = 0; i < n; ++i) t.append_token(i);
        t.scores.assign(scores, scores + n);
        update_importance(t, mat_in<double>(tq, n, attn), tq);
        std::memcpy(scores, t.scores.data(), n * sizeof(double));
    });
}

int kvref_flops_partial_decompress(std::size_t tokens, std::size_t width, std::size_t groups,
                                   const double* ratios, const std::size_t* ranks,
                                   std::uint64_t* flops, double* reduction) {
    return guarded([&] {
        const DecompressCost c = flops_partial_decompress(
            tokens, width, std::vector<double>(ratios, ratios + groups),
            std::vector<std::size_t>(ranks, ranks + groups));
        *flops = c.flops;
        *reduction = c.reduction;
    });
}

// quantize_roundtrip (module.cpp:223-230): dequantize(quantize_4bit(a, group_size)), double.
int kvref_quantize_roundtrip(std::size_t rows, std::size_t cols, const double* a, std::size_t group_size,
                             double* out) {
    return guarded([&] { mat_out(dequantize(quantize_4bit(mat_in<double>(rows, cols, a), group_size)), out); });
}

int kvref_compression_ratio(std::size_t tokens, std::size_t width, std::size_t rank, double* out) {
    return guarded([&] { *out = compression_ratio(tokens, width, rank); });
}

int kvref_gaussian_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed,
                          std::uint64_t stream, double* out) {
    return guarded([&] { mat_out(gaussian_matrix<double>(rows, cols, seed, stream), out); });
}

int kvref_latent_factor_matrix(std::size_t tokens, std::size_t heads, std::size_t kv_heads,
                               std::size_t head_dim, std::size_t true_rank, double decay,
                               std::size_t shared, double noise, std::uint64_t seed,
                               std::uint64_t stream, double* out) {
    return guarded([&] {
        const HeadGeometry g{heads, kv_heads, head_dim};
        const ModalityProfile p{true_rank, decay, shared, noise};
        mat_out(latent_factor_matrix<double>(tokens, g, p, seed, stream), out);
    });
}

// Dense fp64 reference attention (decoder.cpp:346-404) of x (tq rows) against
// the full history (n rows, already containing the new tokens' rows).
int kvref_reference_attention(std::size_t heads, std::size_t kv_heads, std::size_t head_dim,
                              std::size_t tq, const double* x, std::size_t n, const double* k,
                              const double* v, const double* wq, const double* wk,
                              const double* wv, const double* wo, double* out) {
    return guarded([&] {
        const HeadGeometry g{heads, kv_heads, head_dim};
        const std::size_t hd = g.model_width(), cw = g.cache_width();
        const AttentionWeights<double> w = weights_in<double>(hd, cw, wq, wk, wv, wo);
        mat_out(reference_attention(mat_in<double>(tq, hd, x), mat_in<double>(n, cw, k),
                                    mat_in<double>(n, cw, v), w, g),
                out);
    });
}

// Full synthetic experiment (config INI text) -> rendered json-lines report.
// *report is malloc'ed; free with kvref_free.
int kvref_run_simulation(const char* ini, int threads, char** report) {
    return guarded([&] {
        ExperimentConfig cfg = parse_config_text(ini);
        if (threads > 0) cfg.run.threads = static_cast<std::size_t>(threads);
        const RunReport r = cfg.precision == Precision::f64
                                ? run_experiment<double>(cfg.workload, cfg.decode, cfg.run)
                                : run_experiment<float>(cfg.workload, cfg.decode, cfg.run);
        const std::string text = render_report(r, ReportFormat::json_lines);
        *report = static_cast<char*>(std::malloc(text.size() + 1));
        std::memcpy(*report, text.c_str(), text.size() + 1);
    });
}

void kvref_free(void* p) { std::free(p); }

} // extern "C"
