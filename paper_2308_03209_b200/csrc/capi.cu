// capi.cu — the extern "C" boundary of libsagecut_cuda.so (include/sagecut_cuda.h).
//
// Every entry point converts C++ exceptions into sc_status codes with the
// reference's message text in sc_last_error(), the same taxonomy the
// reference's CLI maps to exit codes (proj/tools/main.cpp:822-834).
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sagecut_cuda.h"
#include "internal.hpp"
#include "graph_io.hpp"
#include "io.hpp"
#include "trainer.hpp"

namespace {

thread_local std::string g_err;

template <class F>
sc_status guard(F&& f) {
    try {
        f();
        return SC_OK;
    } catch (const sc::CudaError& e) {
        g_err = e.what();
        return SC_ECUDA;
    } catch (const sc::NcclError& e) {
        g_err = e.what();
        return SC_ENCCL;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SC_EINVAL;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return SC_EINTERNAL;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return SC_ERUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SC_EINTERNAL;
    }
}

#define REQUIRE_ARG(cond, msg) \
    if (!(cond)) throw std::invalid_argument(msg)

void set_device(sc_ctx* ctx) { SC_CUDA(cudaSetDevice(ctx->device)); }

}  // namespace

using namespace sc;

extern "C" {

const char* sc_last_error(void) { return g_err.c_str(); }
const char* sc_version(void) { return "sagecut_cuda 0.1 (sm_100a)"; }

// ---- context ----
sc_status sc_ctx_create(int device, sc_ctx** out) {
    return guard([&] {
        REQUIRE_ARG(out, "sc_ctx_create: null out");
        int count = 0;
        SC_CUDA(cudaGetDeviceCount(&count));
        REQUIRE_ARG(device >= 0 && device < count, "sc_ctx_create: no such CUDA device");
        SC_CUDA(cudaSetDevice(device));
        auto ctx = std::make_unique<sc_ctx>();
        ctx->device = device;
        SC_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        *out = ctx.release();
    });
}
sc_status sc_ctx_destroy(sc_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        set_device(ctx);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->t0) {
            cudaEventDestroy(ctx->t0);
            cudaEventDestroy(ctx->t1);
        }
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}
sc_status sc_ctx_sync(sc_ctx* ctx) {
    return guard([&] { SC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}
int64_t sc_ctx_launch_count(sc_ctx*) { return sc::g_launches; }
sc_status sc_ctx_timer_start(sc_ctx* ctx) {
    return guard([&] {
        set_device(ctx);
        if (!ctx->t0) {
            SC_CUDA(cudaEventCreate(&ctx->t0));
            SC_CUDA(cudaEventCreate(&ctx->t1));
        }
        SC_CUDA(cudaEventRecord(ctx->t0, ctx->stream));
    });
}
sc_status sc_ctx_timer_stop(sc_ctx* ctx, double* ms) {
    return guard([&] {
        REQUIRE_ARG(ctx && ctx->t0, "sc_ctx_timer_stop: timer not started");
        set_device(ctx);
        SC_CUDA(cudaEventRecord(ctx->t1, ctx->stream));
        SC_CUDA(cudaEventSynchronize(ctx->t1));
        float f = 0.f;
        SC_CUDA(cudaEventElapsedTime(&f, ctx->t0, ctx->t1));
        *ms = f;
    });
}

// ---- graph ----
sc_status sc_build_graph_dev(sc_ctx* ctx, int32_t n, const int32_t* raw_dev, int64_t m_raw, sc_graph** out,
                             int64_t* self_loops, int64_t* dups) {
    return guard([&] {
        REQUIRE_ARG(ctx && out, "sc_build_graph: null argument");
        REQUIRE_ARG(m_raw >= 0, "build_graph: negative edge count");
        REQUIRE_ARG(m_raw < (int64_t(1) << 31), "build_graph: more than 2^31 edges");
        set_device(ctx);
        *out = build_graph_device(ctx, n, raw_dev, m_raw, self_loops, dups).release();
    });
}
sc_status sc_build_graph(sc_ctx* ctx, int32_t n, const int32_t* raw_uv, int64_t m_raw, sc_graph** out,
                         int64_t* self_loops, int64_t* dups) {
    return guard([&] {
        REQUIRE_ARG(ctx && out && (raw_uv || m_raw == 0), "sc_build_graph: null argument");
        REQUIRE_ARG(m_raw >= 0, "build_graph: negative edge count");
        set_device(ctx);
        DevBuf<int32_t> raw(std::max<int64_t>(2 * m_raw, 2));
        h2d(raw.get(), raw_uv, 2 * m_raw, ctx->stream);
        *out = build_graph_device(ctx, n, raw.get(), m_raw, self_loops, dups).release();
    });
}
sc_status sc_graph_set_data(sc_graph* g, const float* features, int32_t dim, const int32_t* labels, int32_t classes,
                            const uint8_t* train, const uint8_t* val, const uint8_t* test) {
    return guard([&] {
        REQUIRE_ARG(g && labels && train && val && test, "sc_graph_set_data: null argument");
        REQUIRE_ARG(dim >= 1, "sc_graph_set_data: feature dim must be positive");
        REQUIRE_ARG(classes >= 1, "sc_graph_set_data: num_classes must be positive");
        set_device(g->ctx);
        cudaStream_t s = g->ctx->stream;
        const int64_t n = g->n;
        int64_t train_count = 0;
        for (int64_t v = 0; v < n; ++v) {
            // softmax_ce_loss validates every row's class id (nn.hpp:328-329)
            if (labels[v] < 0 || labels[v] >= classes) throw std::invalid_argument("loss: class id out of range");
            train_count += train[v] ? 1 : 0;
        }
        g->dim = dim;
        g->num_classes = classes;
        g->features.alloc(std::max<int64_t>(n * dim, 1));
        g->labels.alloc(std::max<int64_t>(n, 1));
        g->train.alloc(std::max<int64_t>(n, 1));
        g->val.alloc(std::max<int64_t>(n, 1));
        g->test.alloc(std::max<int64_t>(n, 1));
        if (features) h2d(g->features.get(), features, n * dim, s);
        else SC_CUDA(cudaMemsetAsync(g->features.get(), 0, g->features.bytes(), s));
        h2d(g->labels.get(), labels, n, s);
        h2d(g->train.get(), train, n, s);
        h2d(g->val.get(), val, n, s);
        h2d(g->test.get(), test, n, s);
        g->train_count = train_count;
        g->multilabel = false;  // class ids replace any multi-label matrix (load_labels, graph_io.cpp:230-241)
        g->targets.release();
        g->feat_amax.alloc(1);
        ++g->feat_version;
        SC_CUDA(cudaMemsetAsync(g->feat_amax.get(), 0, sizeof(float), s));
        absmax(n * dim, g->features.get(), g->feat_amax.get(), s);
        SC_CUDA(cudaStreamSynchronize(s));
    });
}
sc_status sc_graph_set_multilabels(sc_graph* g, const float* targets, int32_t classes) {
    return guard([&] {
        REQUIRE_ARG(g && targets, "sc_graph_set_multilabels: null argument");
        REQUIRE_ARG(classes >= 1, "sc_graph_set_multilabels: num_classes must be positive");
        REQUIRE_ARG(g->dim > 0, "sc_graph_set_multilabels: call sc_graph_set_data first");
        set_device(g->ctx);
        const int64_t k = int64_t(g->n) * classes;
        std::vector<uint8_t> y(static_cast<size_t>(std::max<int64_t>(k, 1)));
        for (int64_t i = 0; i < k; ++i) {  // bce_loss's target check (nn.hpp:366-367)
            if (targets[i] != 0.f && targets[i] != 1.f) throw std::invalid_argument("loss: bce targets must be 0 or 1");
            y[size_t(i)] = targets[i] != 0.f ? 1 : 0;
        }
        g->targets.alloc(std::max<int64_t>(k, 1));
        h2d(g->targets.get(), y.data(), k, g->ctx->stream);
        g->num_classes = classes;
        g->multilabel = true;
        SC_CUDA(cudaStreamSynchronize(g->ctx->stream));
    });
}
sc_status sc_graph_set_features(sc_graph* g, const float* features, int is_device) {
    return guard([&] {
        REQUIRE_ARG(g && features && g->dim > 0, "sc_graph_set_features: graph has no feature buffer");
        REQUIRE_ARG(!g->staged, "sc_graph_set_features: features are staged for the next step");
        set_device(g->ctx);
        SC_CUDA(cudaMemcpyAsync(g->features.get(), features, sizeof(float) * size_t(g->n) * g->dim,
                                is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, g->ctx->stream));
        ++g->feat_version;
        SC_CUDA(cudaMemsetAsync(g->feat_amax.get(), 0, sizeof(float), g->ctx->stream));
        absmax(int64_t(g->n) * g->dim, g->features.get(), g->feat_amax.get(), g->ctx->stream);
    });
}
sc_status sc_graph_set_feature_rows(sc_graph* g, int64_t row0, int64_t rows, const float* src, int is_device) {
    return guard([&] {
        REQUIRE_ARG(g && g->dim > 0, "sc_graph_set_feature_rows: graph has no feature buffer");
        REQUIRE_ARG(row0 >= 0 && rows >= 0 && row0 + rows <= g->n, "sc_graph_set_feature_rows: rows out of range");
        REQUIRE_ARG(src || rows == 0, "sc_graph_set_feature_rows: null source");
        REQUIRE_ARG(!g->staged, "sc_graph_set_feature_rows: features are staged for the next step");
        if (rows == 0) return;
        set_device(g->ctx);
        float* dst = g->features.get() + row0 * g->dim;
        const int64_t k = rows * g->dim;
        SC_CUDA(cudaMemcpyAsync(dst, src, sizeof(float) * size_t(k),
                                is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, g->ctx->stream));
        ++g->feat_version;
        absmax(k, dst, g->feat_amax.get(), g->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(g->ctx->stream));  // the caller may reuse src
    });
}
sc_status sc_graph_set_part_ownership(sc_graph* g, int32_t rank, int32_t world) {
    return guard([&] {
        REQUIRE_ARG(g, "sc_graph_set_part_ownership: null graph");
        REQUIRE_ARG(world >= 1 && rank >= 0 && rank < world, "bad rank/world");
        g->own_rank = rank;
        g->own_world = world;
    });
}
sc_status sc_vcut_part_held(sc_vcut* vc, int32_t part, int32_t* held) {
    return guard([&] {
        REQUIRE_ARG(vc && held && part >= 0 && part < vc->p, "sc_vcut_part_held: bad part index");
        *held = vc->parts[part].held ? 1 : 0;
    });
}
sc_status sc_graph_info(sc_graph* g, int32_t* n, int64_t* m, int32_t* dim, int32_t* classes) {
    return guard([&] {
        REQUIRE_ARG(g, "sc_graph_info: null graph");
        if (n) *n = g->n;
        if (m) *m = g->m;
        if (dim) *dim = g->dim;
        if (classes) *classes = g->num_classes;
    });
}
sc_status sc_graph_copy_edges(sc_graph* g, int32_t* uv) {
    return guard([&] {
        set_device(g->ctx);
        std::vector<int32_t> u(g->m), v(g->m);
        d2h(u.data(), g->eu.get(), g->m, g->ctx->stream);
        d2h(v.data(), g->ev.get(), g->m, g->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(g->ctx->stream));
        for (int64_t e = 0; e < g->m; ++e) {
            uv[2 * e] = u[e];
            uv[2 * e + 1] = v[e];
        }
    });
}
sc_status sc_graph_copy_csr(sc_graph* g, int64_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* degrees) {
    return guard([&] {
        set_device(g->ctx);
        cudaStream_t s = g->ctx->stream;
        if (offsets) d2h(offsets, g->offsets.get(), size_t(g->n) + 1, s);
        if (nbrs) d2h(nbrs, g->nbrs.get(), 2 * g->m, s);
        if (eids) d2h(eids, g->eids.get(), 2 * g->m, s);
        if (degrees) d2h(degrees, g->degrees.get(), g->n, s);
        SC_CUDA(cudaStreamSynchronize(s));
    });
}
sc_graph::~sc_graph() {
    if (copy_stream) {
        cudaStreamSynchronize(copy_stream);
        cudaStreamDestroy(copy_stream);
    }
    if (staged_ev) cudaEventDestroy(staged_ev);
    if (released_ev) cudaEventDestroy(released_ev);
}
sc_status sc_graph_destroy(sc_graph* g) {
    return guard([&] {
        if (!g) return;
        set_device(g->ctx);
        delete g;
    });
}

// ---- dataset files (graph_io.cpp:41-296) ----
sc_status sc_load_graph(sc_ctx* ctx, const char* path, int32_t num_nodes, int32_t strict, sc_graph** out,
                        int64_t* self_loops, int64_t* dups) {
    return guard([&] {
        REQUIRE_ARG(ctx && path && out, "sc_load_graph: null argument");
        const std::string p(path);
        const EdgeList el = read_edge_list(p, num_nodes);
        set_device(ctx);
        const int64_t m = static_cast<int64_t>(el.uv.size() / 2);
        DevBuf<int32_t> raw(std::max<int64_t>(2 * m, 2));
        h2d(raw.get(), el.uv.data(), 2 * m, ctx->stream);
        auto g = build_graph_device(ctx, el.num_nodes, raw.get(), m, self_loops, dups);
        if (strict && g->n > 0) {  // ValidationReport::isolated_nodes must be empty (graph_io.cpp:73-76)
            std::vector<int32_t> deg(static_cast<size_t>(g->n));
            d2h(deg.data(), g->degrees.get(), g->n, ctx->stream);
            SC_CUDA(cudaStreamSynchronize(ctx->stream));
            int64_t isolated = 0;
            for (int32_t d : deg) isolated += d == 0;
            if (isolated)
                throw std::runtime_error(p + ": " + std::to_string(isolated) +
                                         " node id(s) absent from the edge list (strict mode)");
        }
        *out = g.release();
    });
}
sc_status sc_read_edge_list(const char* path, int32_t num_nodes, int32_t* uv, int64_t cap, int64_t* m,
                            int32_t* n) {
    return guard([&] {
        REQUIRE_ARG(path && m && n, "sc_read_edge_list: null argument");
        const EdgeList el = read_edge_list(path, num_nodes);
        *m = static_cast<int64_t>(el.uv.size() / 2);
        *n = el.num_nodes;
        if (!uv) return;
        REQUIRE_ARG(cap >= *m, "sc_read_edge_list: output buffer too small");
        std::copy(el.uv.begin(), el.uv.end(), uv);
    });
}
sc_status sc_load_features(const char* path, int32_t expected_nodes, float* out, int64_t cap, int64_t* rows,
                           int64_t* cols) {
    return guard([&] {
        REQUIRE_ARG(path && rows && cols, "sc_load_features: null argument");
        const HostFeatures f = read_features(path, expected_nodes);
        *rows = f.rows;
        *cols = f.cols;
        if (!out) return;
        REQUIRE_ARG(cap >= f.rows * f.cols, "sc_load_features: output buffer too small");
        std::copy(f.values.begin(), f.values.end(), out);
    });
}
sc_status sc_load_labels(const char* path, int32_t num_nodes, int32_t* labels, float* targets, int64_t cap,
                         int32_t* num_classes, int32_t* is_multilabel) {
    return guard([&] {
        REQUIRE_ARG(path && num_classes && is_multilabel, "sc_load_labels: null argument");
        const HostLabels L = read_labels(path, num_nodes);
        *num_classes = L.num_classes;
        *is_multilabel = L.multilabel ? 1 : 0;
        if (L.multilabel && targets) {
            REQUIRE_ARG(cap >= int64_t(L.targets.size()), "sc_load_labels: output buffer too small");
            std::copy(L.targets.begin(), L.targets.end(), targets);
        }
        if (!L.multilabel && labels) std::copy(L.labels.begin(), L.labels.end(), labels);
    });
}
sc_status sc_load_masks(const char* path, int32_t num_nodes, uint8_t* train, uint8_t* val, uint8_t* test) {
    return guard([&] {
        REQUIRE_ARG(path && train && val && test, "sc_load_masks: null argument");
        std::vector<uint8_t> tr, va, te;
        read_masks(path, num_nodes, tr, va, te);
        std::copy(tr.begin(), tr.end(), train);
        std::copy(va.begin(), va.end(), val);
        std::copy(te.begin(), te.end(), test);
    });
}
sc_status sc_save_edge_list(sc_graph* g, const char* path) {
    return guard([&] {
        REQUIRE_ARG(g && path, "sc_save_edge_list: null argument");
        set_device(g->ctx);
        std::vector<int32_t> u(g->m), v(g->m);
        d2h(u.data(), g->eu.get(), g->m, g->ctx->stream);
        d2h(v.data(), g->ev.get(), g->m, g->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(g->ctx->stream));
        write_edge_list(path, u.data(), v.data(), g->m);
    });
}
sc_status sc_save_features(const char* path, const float* features, int64_t rows, int64_t cols, int32_t binary) {
    return guard([&] {
        REQUIRE_ARG(path && (features || rows * cols == 0), "sc_save_features: null argument");
        if (binary) write_features_binary(path, features, rows, cols);
        else write_features_csv(path, features, rows, cols);
    });
}
sc_status sc_save_labels(const char* path, int32_t num_nodes, const int32_t* labels, const float* targets,
                         int32_t num_classes) {
    return guard([&] {
        REQUIRE_ARG(path && (labels || targets), "sc_save_labels: null argument");
        write_labels(path, num_nodes, labels, targets, num_classes);
    });
}
sc_status sc_save_masks(const char* path, int32_t num_nodes, const uint8_t* train, const uint8_t* val,
                        const uint8_t* test) {
    return guard([&] {
        REQUIRE_ARG(path && train && val && test, "sc_save_masks: null argument");
        write_masks(path, num_nodes, train, val, test);
    });
}

// ---- vertex cut ----
sc_status sc_partition_random(sc_graph* g, int32_t p, uint64_t seed, sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && out, "sc_partition_random: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        REQUIRE_ARG(g->m > 0, "partition_random: graph has no edges");
        set_device(g->ctx);
        DevBuf<int32_t> a(g->m);
        assign_random(g, p, seed, a.get());
        *out = build_vertex_cut_device(g, p, std::move(a)).release();
    });
}
sc_status sc_partition_dbh(sc_graph* g, int32_t p, uint64_t seed, sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && out, "sc_partition_dbh: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        DevBuf<int32_t> a(std::max<int64_t>(g->m, 1));
        assign_dbh(g, p, seed, a.get());
        *out = build_vertex_cut_device(g, p, std::move(a)).release();
    });
}
sc_status sc_build_vertex_cut(sc_graph* g, int32_t p, const int32_t* assign, sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && out && (assign || g->m == 0), "sc_build_vertex_cut: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        DevBuf<int32_t> a(std::max<int64_t>(g->m, 1));
        h2d(a.get(), assign, g->m, g->ctx->stream);
        *out = build_vertex_cut_device(g, p, std::move(a)).release();
    });
}
sc_status sc_partition_ne(sc_graph* g, int32_t p, uint64_t seed, double balance_slack, sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && out, "sc_partition_ne: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        REQUIRE_ARG(balance_slack >= 1.0, "partition_ne: balance_slack must be >= 1");
        (void)seed;  // growth order is fully fixed by the tie-break rules (partition.cpp:123)
        set_device(g->ctx);
        std::vector<std::string> warnings;
        const std::vector<int32_t> a = ne_assign_host(g, p, balance_slack, warnings);
        DevBuf<int32_t> d(std::max<int64_t>(g->m, 1));
        h2d(d.get(), a.data(), g->m, g->ctx->stream);
        auto vc = build_vertex_cut_device(g, p, std::move(d));
        vc->warnings = std::move(warnings);
        *out = vc.release();
    });
}
sc_status sc_partition_edge_cut_greedy(sc_graph* g, int32_t p, uint64_t seed, int32_t* node_assignment) {
    return guard([&] {
        REQUIRE_ARG(g && (node_assignment || g->n == 0), "sc_partition_edge_cut_greedy: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        const std::vector<int32_t> a = edge_cut_greedy_host(g, p, seed);
        std::copy(a.begin(), a.end(), node_assignment);
    });
}
sc_status sc_edge_cut_from_assignment(sc_graph* g, int32_t p, const int32_t* node_assignment, int64_t* kept_counts,
                                      int64_t* num_cut, int64_t* halo_counts, int32_t* kept_edges, int32_t* cut_edges,
                                      int32_t* halo_nodes) {
    return guard([&] {
        REQUIRE_ARG(g && num_cut && (node_assignment || g->n == 0), "sc_edge_cut_from_assignment: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        edge_cut_stats_device(g, p, node_assignment, kept_counts, num_cut, halo_counts, kept_edges, cut_edges,
                              halo_nodes);
    });
}
sc_status sc_edge_cut_to_vertex_cut(sc_graph* g, int32_t p, const int32_t* node_assignment, uint64_t seed,
                                    sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && out && (node_assignment || g->n == 0), "sc_edge_cut_to_vertex_cut: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        DevBuf<int32_t> a(std::max<int64_t>(g->m, 1));
        ec2vc_assign_device(g, p, node_assignment, seed, a.get());
        *out = build_vertex_cut_device(g, p, std::move(a)).release();
    });
}
sc_status sc_vcut_warnings(sc_vcut* vc, char* buf, int64_t cap, int64_t* needed) {
    return guard([&] {
        std::string j;
        for (const auto& w : vc->warnings) j += (j.empty() ? "" : "\n") + w;
        if (needed) *needed = static_cast<int64_t>(j.size()) + 1;
        if (buf && cap > 0) {
            const size_t k = std::min<size_t>(j.size(), size_t(cap - 1));
            std::memcpy(buf, j.data(), k);
            buf[k] = 0;
        }
    });
}
sc_status sc_vcut_num_parts(sc_vcut* vc, int32_t* p) {
    return guard([&] { *p = vc->p; });
}
sc_status sc_vcut_assignment(sc_vcut* vc, int32_t* out) {
    return guard([&] {
        set_device(vc->g->ctx);
        d2h(out, vc->assign.get(), vc->g->m, vc->g->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(vc->g->ctx->stream));
    });
}
sc_status sc_vcut_part_sizes(sc_vcut* vc, int32_t part, int64_t* n_local, int64_t* n_edges) {
    return guard([&] {
        REQUIRE_ARG(vc && part >= 0 && part < vc->p, "sc_vcut_part_sizes: bad part index");
        if (n_local) *n_local = vc->parts[part].n_local;
        if (n_edges) *n_edges = vc->parts[part].m_local;
    });
}
sc_status sc_vcut_part_copy(sc_vcut* vc, int32_t part, int32_t* nodes, int32_t* edges_uv, int32_t* gids,
                            int32_t* local_deg, int64_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* g2l) {
    return guard([&] {
        REQUIRE_ARG(vc && part >= 0 && part < vc->p, "sc_vcut_part_copy: bad part index");
        set_device(vc->g->ctx);
        cudaStream_t s = vc->g->ctx->stream;
        const PartDev& pd = vc->held(part);
        if (nodes) d2h(nodes, pd.nodes.get(), pd.n_local, s);
        if (gids) d2h(gids, pd.edge_gids.get(), pd.m_local, s);
        if (local_deg) d2h(local_deg, pd.local_deg.get(), pd.n_local, s);
        if (offsets) d2h(offsets, pd.offsets.get(), pd.n_local + 1, s);
        if (nbrs) d2h(nbrs, pd.nbrs.get(), 2 * pd.m_local, s);
        if (eids) d2h(eids, pd.eids.get(), 2 * pd.m_local, s);
        if (g2l) {
            DevBuf<int32_t> tmp(std::max<int64_t>(vc->g->n, 1));
            part_g2l_device(vc, part, tmp.get());
            d2h(g2l, tmp.get(), vc->g->n, s);
            SC_CUDA(cudaStreamSynchronize(s));
        }
        std::vector<int32_t> u, v;
        if (edges_uv) {
            u.resize(pd.m_local);
            v.resize(pd.m_local);
            d2h(u.data(), pd.lu.get(), pd.m_local, s);
            d2h(v.data(), pd.lv.get(), pd.m_local, s);
        }
        SC_CUDA(cudaStreamSynchronize(s));
        for (int64_t e = 0; edges_uv && e < pd.m_local; ++e) {
            edges_uv[2 * e] = u[e];
            edges_uv[2 * e + 1] = v[e];
        }
    });
}
sc_status sc_replication_stats(sc_vcut* vc, int32_t* per_node_rf, double* rf, double* edge_balance,
                               double* node_balance, int64_t* duplicated) {
    // partition.cpp:310-342
    return guard([&] {
        REQUIRE_ARG(vc, "replication_stats: null partition");
        set_device(vc->g->ctx);
        const sc_graph* g = vc->g;
        if (per_node_rf) {
            d2h(per_node_rf, vc->per_node_rf.get(), g->n, g->ctx->stream);
            SC_CUDA(cudaStreamSynchronize(g->ctx->stream));
        }
        int64_t total = 0, maxn = 0, maxe = 0;
        for (const auto& pd : vc->parts) {
            total += pd.n_local;
            maxn = std::max(maxn, pd.n_local);
            maxe = std::max(maxe, pd.m_local);
        }
        const double n = static_cast<double>(g->n), p = static_cast<double>(vc->p);
        if (rf) *rf = static_cast<double>(total) / n;
        if (duplicated) *duplicated = total - g->n;
        if (edge_balance) *edge_balance = g->m == 0 ? 0.0 : static_cast<double>(maxe) / (static_cast<double>(g->m) / p);
        if (node_balance) *node_balance = total == 0 ? 0.0 : static_cast<double>(maxn) / (static_cast<double>(total) / p);
    });
}
sc_status sc_vcut_destroy(sc_vcut* vc) {
    return guard([&] {
        if (!vc) return;
        set_device(vc->g->ctx);
        delete vc;
    });
}

// ---- reweighting ----
sc_status sc_compute_weights(sc_vcut* vc, int32_t scheme, double* out) {
    return guard([&] {
        REQUIRE_ARG(vc && out, "compute_weights: null argument");
        REQUIRE_ARG(scheme >= 0 && scheme <= 2, "compute_weights: bad scheme");
        set_device(vc->g->ctx);
        int64_t off = 0;
        for (int32_t i = 0; i < vc->p; ++i) {
            const int64_t nl = vc->parts[i].n_local;
            DevBuf<double> w(std::max<int64_t>(nl, 1));
            compute_weights_device(vc, scheme, i, w.get());
            d2h(out + off, w.get(), nl, vc->g->ctx->stream);
            SC_CUDA(cudaStreamSynchronize(vc->g->ctx->stream));
            off += nl;
        }
    });
}

// ---- files (partition_io.cpp, checkpoint.cpp, trainer.cpp:126-140) ----
namespace {
const char* const kSchemeNames[] = {"dar", "vanilla_inv", "none"};
std::vector<std::vector<int32_t>> part_nodes_host(sc_vcut* vc) {
    std::vector<std::vector<int32_t>> nodes(vc->p);
    for (int32_t i = 0; i < vc->p; ++i) {
        const PartDev& pd = vc->held(i);
        nodes[i].resize(pd.n_local);
        d2h(nodes[i].data(), pd.nodes.get(), pd.n_local, vc->g->ctx->stream);
    }
    SC_CUDA(cudaStreamSynchronize(vc->g->ctx->stream));
    return nodes;
}
}  // namespace

sc_status sc_save_partition(sc_vcut* vc, const char* path, int32_t weight_scheme) {
    return guard([&] {
        REQUIRE_ARG(vc && path, "sc_save_partition: null argument");
        REQUIRE_ARG(weight_scheme >= -1 && weight_scheme <= 2, "sc_save_partition: bad weight scheme");
        set_device(vc->g->ctx);
        cudaStream_t s = vc->g->ctx->stream;
        std::vector<int32_t> assign(vc->g->m);
        d2h(assign.data(), vc->assign.get(), vc->g->m, s);
        const auto nodes = part_nodes_host(vc);
        std::vector<std::vector<double>> w;
        if (weight_scheme >= 0) {
            for (int32_t i = 0; i < vc->p; ++i) {
                const int64_t nl = vc->parts[i].n_local;
                DevBuf<double> wd(std::max<int64_t>(nl, 1));
                compute_weights_device(vc, weight_scheme, i, wd.get());
                w.emplace_back(nl);
                d2h(w.back().data(), wd.get(), nl, s);
                SC_CUDA(cudaStreamSynchronize(s));
            }
        }
        write_partition_json(path, vc->p, assign, nodes, weight_scheme >= 0 ? &w : nullptr,
                             weight_scheme >= 0 ? kSchemeNames[weight_scheme] : nullptr);
    });
}
sc_status sc_load_partition(sc_graph* g, const char* path, sc_vcut** out) {
    return guard([&] {
        REQUIRE_ARG(g && path && out, "sc_load_partition: null argument");
        set_device(g->ctx);
        const std::string p(path);
        int32_t np = 0;
        std::vector<int32_t> assign;
        std::vector<std::vector<int32_t>> stored;
        read_partition_json(p, np, assign, stored);
        if (int64_t(assign.size()) != g->m)  // partition_io.cpp:40-43
            throw std::runtime_error(p + ": partition was built for " + std::to_string(assign.size()) +
                                     " edges, graph has " + std::to_string(g->m));
        REQUIRE_ARG(np >= 1, "num_parts must be >= 1");
        for (int32_t a : assign)
            REQUIRE_ARG(a >= 0 && a < np, "edge assignment references an invalid part");
        DevBuf<int32_t> d(std::max<int64_t>(g->m, 1));
        h2d(d.get(), assign.data(), g->m, g->ctx->stream);
        auto vc = build_vertex_cut_device(g, np, std::move(d));
        if (stored.size() != size_t(vc->p)) throw std::runtime_error(p + ": part count mismatch");
        if (part_nodes_host(vc.get()) != stored)
            throw std::runtime_error(p + ": stored node sets do not match this graph");
        *out = vc.release();
    });
}
sc_status sc_save_edge_cut(sc_graph* g, int32_t p, const int32_t* node_assignment, const char* path) {
    return guard([&] {
        REQUIRE_ARG(g && path && (node_assignment || g->n == 0), "sc_save_edge_cut: null argument");
        REQUIRE_ARG(p >= 1, "num_parts must be >= 1");
        set_device(g->ctx);
        std::vector<int64_t> kept(p), halo(p);
        int64_t ncut = 0;
        edge_cut_stats_device(g, p, node_assignment, kept.data(), &ncut, halo.data(), nullptr, nullptr, nullptr);
        int64_t nh = 0;
        for (int64_t h : halo) nh += h;
        std::vector<int32_t> cut(ncut), hn(nh);
        edge_cut_stats_device(g, p, node_assignment, kept.data(), &ncut, halo.data(), nullptr, cut.data(), hn.data());
        std::vector<std::vector<int32_t>> sets(p);
        int64_t o = 0;
        for (int32_t i = 0; i < p; ++i) {
            sets[i].assign(hn.begin() + o, hn.begin() + o + halo[i]);
            o += halo[i];
        }
        write_edge_cut_json(path, p, std::vector<int32_t>(node_assignment, node_assignment + g->n), cut, sets);
    });
}
namespace {
std::vector<std::pair<int64_t, int64_t>> model_shapes(sc_trainer* t) {  // for_each_matrix order
    std::vector<std::pair<int64_t, int64_t>> sh;
    for (const auto& lo : t->lay) {
        sh.emplace_back(lo.H, lo.in);
        sh.emplace_back(lo.H, lo.H + lo.in);
    }
    sh.emplace_back(t->C, t->E);
    return sh;
}
}  // namespace
sc_status sc_trainer_save_checkpoint(sc_trainer* t, const char* path) {
    return guard([&] {
        REQUIRE_ARG(t && path, "sc_trainer_save_checkpoint: null argument");
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);
        std::vector<float> theta(t->P);
        d2h(theta.data(), t->theta.get(), t->P, t->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
        std::vector<HostMatrix> mats;
        int64_t k = 0;
        for (const auto& [r, c] : model_shapes(t)) {  // TrainResult::model is SageModel<double>
            HostMatrix m;
            m.rows = uint64_t(r);
            m.cols = uint64_t(c);
            m.v.assign(theta.begin() + k, theta.begin() + k + r * c);
            k += r * c;
            mats.push_back(std::move(m));
        }
        write_checkpoint(path, mats);
    });
}
sc_status sc_trainer_load_checkpoint(sc_trainer* t, const char* path) {
    return guard([&] {
        REQUIRE_ARG(t && path, "sc_trainer_load_checkpoint: null argument");
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);
        const auto mats = read_checkpoint(path);
        const auto sh = model_shapes(t);
        REQUIRE_ARG(mats.size() == sh.size(), "load_checkpoint: layer count does not match the model");
        std::vector<float> theta;
        for (size_t i = 0; i < sh.size(); ++i) {
            REQUIRE_ARG(mats[i].rows == uint64_t(sh[i].first) && mats[i].cols == uint64_t(sh[i].second),
                        "load_checkpoint: matrix shape does not match the model");
            for (double v : mats[i].v) theta.push_back(static_cast<float>(v));
        }
        h2d(t->theta.get(), theta.data(), t->P, t->ctx->stream);
        // CFCK holds the model only (checkpoint.cpp:44-57): training resumes from
        // fresh Adam state, as a reference run started from these weights would.
        if (t->m1.size()) SC_CUDA(cudaMemsetAsync(t->m1.get(), 0, t->m1.bytes(), t->ctx->stream));
        if (t->m2.size()) SC_CUDA(cudaMemsetAsync(t->m2.get(), 0, t->m2.bytes(), t->ctx->stream));
        t->adam_step = 0;
        t->tc.invalidate();
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_save_checkpoint_params(const float* theta, int32_t in_dim, const int32_t* hidden, int32_t layers,
                                    int32_t num_classes, const char* path) {
    return guard([&] {
        REQUIRE_ARG(theta && path && (hidden || layers == 0), "sc_save_checkpoint_params: null argument");
        REQUIRE_ARG(layers >= 0 && in_dim >= 0 && num_classes >= 0, "sc_save_checkpoint_params: bad dims");
        for (int32_t l = 0; l < layers; ++l)
            REQUIRE_ARG(hidden[l] >= 1, "hidden dims must be positive");
        std::vector<HostMatrix> mats;
        int64_t k = 0, in = in_dim;
        auto add = [&](int64_t r, int64_t c) {
            HostMatrix m;
            m.rows = uint64_t(r);
            m.cols = uint64_t(c);
            m.v.assign(theta + k, theta + k + r * c);
            k += r * c;
            mats.push_back(std::move(m));
        };
        for (int32_t l = 0; l < layers; ++l) {
            add(hidden[l], in);
            add(hidden[l], hidden[l] + in);
            in = hidden[l];
        }
        add(num_classes, in);
        write_checkpoint(path, mats);
    });
}
sc_status sc_load_checkpoint_params(const char* path, float* theta, int64_t cap, int64_t* count) {
    return guard([&] {
        REQUIRE_ARG(path && count, "sc_load_checkpoint_params: null argument");
        const auto mats = read_checkpoint(path);
        int64_t n = 0;
        for (const auto& m : mats) n += int64_t(m.v.size());
        *count = n;
        if (!theta) return;
        REQUIRE_ARG(cap >= n, "sc_load_checkpoint_params: output buffer too small");
        int64_t k = 0;
        for (const auto& m : mats)
            for (double v : m.v) theta[k++] = static_cast<float>(v);
    });
}
sc_status sc_write_metrics_jsonl(const char* path, int32_t n, const sc_epoch_metrics* rows) {
    return guard([&] {
        REQUIRE_ARG(path && (rows || n == 0), "sc_write_metrics_jsonl: null argument");
        std::vector<EpochRow> v(n);
        for (int32_t i = 0; i < n; ++i)
            v[i] = EpochRow{rows[i].epoch, rows[i].train_loss, rows[i].train_metric, rows[i].val_metric,
                            rows[i].test_metric, rows[i].grad_norm, rows[i].comm_floats};
        write_metrics_jsonl(path, v);
    });
}

// ---- DropEdge ----
sc_status sc_precompute_masks(sc_ctx* ctx, int64_t m, int32_t k, double ratio, uint64_t seed, uint8_t* out) {
    return guard([&] {
        REQUIRE_ARG(ctx && (out || m == 0), "precompute_masks: null argument");
        set_device(ctx);
        DevBuf<uint8_t> d(std::max<int64_t>(m * std::max(k, 1), 1));
        precompute_masks_device(ctx, m, k, ratio, seed, d.get());
        d2h(out, d.get(), m * k, ctx->stream);
        SC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
int32_t sc_select_mask(uint64_t seed, uint64_t part, uint64_t epoch, int32_t k) {
    if (k < 1) return -1;
    HostRng rng(substream(seed, "dropedge.select", part, epoch));
    return static_cast<int32_t>(rng.next_below(static_cast<uint64_t>(k)));
}
uint64_t sc_substream(uint64_t seed, const char* tag, int32_t nidx, uint64_t a, uint64_t b) {
    return nidx == 0 ? substream(seed, tag) : (nidx == 1 ? substream(seed, tag, a) : substream(seed, tag, a, b));
}

// ---- model ----
int64_t sc_param_count(int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t classes) {
    int64_t total = 0, in = in_dim;
    for (int32_t l = 0; l < layers; ++l) {
        total += int64_t(hidden[l]) * in + int64_t(hidden[l]) * (hidden[l] + in);
        in = hidden[l];
    }
    return total + int64_t(classes) * in;
}
sc_status sc_init_params(sc_ctx* ctx, int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t classes,
                         uint64_t seed, float* out) {
    return guard([&] {
        REQUIRE_ARG(ctx && out && (hidden || layers == 0), "make_sage_model: null argument");
        set_device(ctx);
        const int64_t P = sc_param_count(in_dim, hidden, layers, classes);
        DevBuf<float> d(std::max<int64_t>(P, 1));
        init_params_device(ctx, in_dim, hidden, layers, classes, seed, d.get());
        d2h(out, d.get(), P, ctx->stream);
        SC_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- trainer ----
sc_status sc_trainer_create(sc_ctx* ctx, sc_graph* g, sc_vcut* vc, const sc_train_config* cfg, int32_t rank,
                            int32_t world, sc_trainer** out) {
    return guard([&] {
        REQUIRE_ARG(ctx && g && vc && cfg && out, "sc_trainer_create: null argument");
        REQUIRE_ARG(cfg->layers >= 0 && (cfg->hidden || cfg->layers == 0), "layers must be >= 0");
        set_device(ctx);
        auto t = std::make_unique<sc_trainer>();
        t->ctx = ctx;
        t->g = g;
        t->vc = vc;
        t->rank = rank;
        t->world = world;
        t->L = cfg->layers;
        t->hidden.assign(cfg->hidden, cfg->hidden + cfg->layers);
        t->lr = cfg->learning_rate;
        t->loss = cfg->loss;
        t->reweight = cfg->reweight;
        t->use_dropedge = cfg->use_dropedge;
        t->K = cfg->dropedge_k;
        t->ratio = cfg->drop_ratio;
        t->seed = cfg->seed;
        t->deterministic = cfg->deterministic;
        t->gemm_mode = cfg->gemm;
        REQUIRE_ARG(t->loss == 0 || t->loss == 1, "unknown loss");
        REQUIRE_ARG(t->reweight >= 0 && t->reweight <= 2, "unknown reweight scheme");
        trainer_init(t.get());
        *out = t.release();
    });
}
sc_status sc_nccl_unique_id(uint8_t out[128]) {
    return guard([&] { nccl_unique_id(out); });
}
sc_status sc_trainer_init_comm(sc_trainer* t, const uint8_t id[128]) {
    return guard([&] {
        REQUIRE_ARG(t && id, "sc_trainer_init_comm: null argument");
        trainer_init_comm(t, id);  // world == 1: a single-rank communicator (exercises the exchange path)
    });
}
sc_status sc_trainer_emulate_rank(sc_trainer* t) {
    return guard([&] {
        REQUIRE_ARG(t, "sc_trainer_emulate_rank: null trainer");
        t->emulate = true;
    });
}
sc_status sc_trainer_set_exchange(sc_trainer* t, sc_exchange_fn fn, void* user) {
    return guard([&] {
        REQUIRE_ARG(t, "sc_trainer_set_exchange: null trainer");
        t->xfn = fn;
        t->xuser = user;
    });
}
sc_status sc_trainer_step(sc_trainer* t, int32_t epoch, double* loss, double* gnorm) {
    return guard([&] {
        set_device(t->ctx);
        trainer_step_async(t, epoch);
        trainer_finish(t, loss, gnorm);
    });
}
sc_status sc_trainer_stage_features(sc_trainer* t, const float* features, int32_t is_device) {
    return guard([&] {
        REQUIRE_ARG(t && features, "sc_trainer_stage_features: null argument");
        set_device(t->ctx);
        trainer_stage_features(t, features, is_device != 0);
    });
}
sc_status sc_trainer_step_async(sc_trainer* t, int32_t epoch) {
    return guard([&] {
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);  // settle the previous step's host bookkeeping
        trainer_step_async(t, epoch);
    });
}
sc_status sc_trainer_last(sc_trainer* t, double* loss, double* gnorm) {
    return guard([&] {
        set_device(t->ctx);
        trainer_finish(t, loss, gnorm);
    });
}
sc_status sc_trainer_param_count(sc_trainer* t, int64_t* n) {
    return guard([&] { *n = t->P; });
}
sc_status sc_trainer_get_params(sc_trainer* t, float* out) {
    return guard([&] {
        set_device(t->ctx);
        d2h(out, t->theta.get(), t->P, t->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_set_params(sc_trainer* t, const float* in) {
    return guard([&] {
        REQUIRE_ARG(t && in, "sc_trainer_set_params: null argument");
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);  // the pending step read the old parameters
        h2d(t->theta.get(), in, t->P, t->ctx->stream);
        t->tc.invalidate();
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_get_grads(sc_trainer* t, float* out) {
    return guard([&] {
        set_device(t->ctx);
        d2h(out, t->gathered.get(), t->P, t->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_get_part_grads(sc_trainer* t, int32_t part, float* out) {
    return guard([&] {
        REQUIRE_ARG(part >= 0 && part < t->p, "bad part index");
        set_device(t->ctx);
        for (int b = 0; b < t->nb(); ++b)  // bucket-major slots -> one flat parameter-ordered vector
            d2h(out + t->b_off[b], t->slot_ptr(b, part), t->b_len(b), t->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_get_part_logits(sc_trainer* t, int32_t part, float* out) {
    return guard([&] {
        REQUIRE_ARG(part >= 0 && part < t->p, "bad part index");
        REQUIRE_ARG(part % t->world == t->rank, "partition is not trained on this rank");
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);
        if (t->shared_logits && part != t->last_part)
            throw std::invalid_argument("logits of partition " + std::to_string(part) +
                                        " were not kept (shared logits buffer: only the last trained partition's)");
        const float* src = t->shared_logits ? t->logits_shared.get() : t->ps[part].logits.get();
        if (t->ps[part].n > 0)
            SC_CUDA(cudaMemcpy2DAsync(out, sizeof(float) * t->C, src, sizeof(float) * t->Cp,
                                      sizeof(float) * t->C, t->ps[part].n, cudaMemcpyDeviceToHost, t->ctx->stream));
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_get_part_loss(sc_trainer* t, int32_t part, double* loss) {
    return guard([&] {
        REQUIRE_ARG(part >= 0 && part < t->p, "bad part index");
        set_device(t->ctx);
        d2h(loss, t->part_loss.get() + part, 1, t->ctx->stream);
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}
sc_status sc_trainer_get_part_mask(sc_trainer* t, int32_t part, int32_t* idx) {
    return guard([&] {
        REQUIRE_ARG(part >= 0 && part < t->p, "bad part index");
        *idx = t->ps[part].chosen;
    });
}
sc_status sc_trainer_evaluate(sc_trainer* t, double* tr, double* va, double* te) {
    return guard([&] {
        set_device(t->ctx);
        trainer_evaluate(t, tr, va, te);
    });
}
sc_status sc_trainer_evaluate_mask(sc_trainer* t, const uint8_t* mask, double* metric) {
    return guard([&] {
        REQUIRE_ARG(t && mask && metric, "sc_trainer_evaluate_mask: null argument");
        set_device(t->ctx);
        const int64_t n = t->g->n;
        int64_t masked = 0;
        for (int64_t v = 0; v < n; ++v) masked += mask[v] ? 1 : 0;
        if (masked == 0) throw std::invalid_argument("evaluate: empty mask");  // trainer.cpp:106-108
        DevBuf<uint8_t> d(std::max<int64_t>(n, 1));
        h2d(d.get(), mask, n, t->ctx->stream);
        *metric = trainer_evaluate_mask(t, d.get());
    });
}
sc_status sc_evaluate(sc_ctx* ctx, sc_graph* g, const float* theta, const int32_t* hidden, int32_t layers,
                      const uint8_t* mask, double* metric) {
    return guard([&] {
        REQUIRE_ARG(ctx && g && theta && mask && metric && (hidden || layers == 0), "sc_evaluate: null argument");
        REQUIRE_ARG(layers >= 0, "layers must be >= 0");
        set_device(ctx);
        if (g->dim == 0 || g->num_classes == 0) throw std::invalid_argument("evaluate: graph lacks features or labels");
        auto t = std::make_unique<sc_trainer>();
        t->ctx = ctx;
        t->g = g;
        t->L = layers;
        t->hidden.assign(hidden, hidden + layers);
        trainer_init_eval_only(t.get());
        h2d(t->theta.get(), theta, t->P, ctx->stream);
        const int64_t n = g->n;
        int64_t masked = 0;
        for (int64_t v = 0; v < n; ++v) masked += mask[v] ? 1 : 0;
        if (masked == 0) throw std::invalid_argument("evaluate: empty mask");
        DevBuf<uint8_t> d(std::max<int64_t>(n, 1));
        h2d(d.get(), mask, n, ctx->stream);
        *metric = trainer_evaluate_mask(t.get(), d.get());
    });
}
sc_status sc_trainer_comm_audit(sc_trainer* t, uint64_t* gradient_floats, uint64_t* embedding_floats) {
    return guard([&] {
        REQUIRE_ARG(t, "sc_trainer_comm_audit: null trainer");
        trainer_finish(t, nullptr, nullptr);
        if (gradient_floats) *gradient_floats = t->audit_floats;
        if (embedding_floats) *embedding_floats = 0;  // no node embedding ever leaves a partition
    });
}
sc_status sc_trainer_fallback_count(sc_trainer* t, int64_t* count) {
    return guard([&] {
        REQUIRE_ARG(t && count, "sc_trainer_fallback_count: null argument");
        *count = t->tc.simt_fallbacks;
    });
}
sc_status sc_trainer_memory_mode(sc_trainer* t, int32_t* flags, int64_t* arena_bytes) {
    return guard([&] {
        REQUIRE_ARG(t, "sc_trainer_memory_mode: null argument");
        if (flags) *flags = (t->compact ? 1 : 0) | (t->shared_x0 ? 2 : 0) | (t->shared_logits ? 4 : 0);
        if (arena_bytes) *arena_bytes = static_cast<int64_t>(t->arena.bytes());
    });
}
sc_status sc_comm_volume(int32_t mode, int32_t num_parts, uint64_t param_count, uint64_t num_layers,
                         uint64_t hidden_dim, uint64_t total_halo, uint64_t* floats_per_iteration,
                         uint64_t* gradient_floats, uint64_t* embedding_floats) {
    return guard([&] {  // trainer.cpp:38-49
        REQUIRE_ARG(mode == 0 || mode == 1, "comm_volume: unknown mode");
        if (num_parts < 1) throw std::invalid_argument("comm_volume: num_parts must be >= 1");
        const uint64_t grad = static_cast<uint64_t>(num_parts) * param_count;
        const uint64_t emb = mode == 1 ? 2ULL * num_layers * total_halo * hidden_dim : 0ULL;
        if (gradient_floats) *gradient_floats = grad;
        if (embedding_floats) *embedding_floats = emb;
        if (floats_per_iteration) *floats_per_iteration = grad + emb;
    });
}
sc_status sc_expected_rf_random(int32_t num_parts, int64_t degree, double* out) {
    return guard([&] {  // partition.cpp:344-349
        REQUIRE_ARG(out, "sc_expected_rf_random: null out");
        if (num_parts < 1) throw std::invalid_argument("expected_rf_random: num_parts must be >= 1");
        if (degree < 0) throw std::invalid_argument("expected_rf_random: degree must be >= 0");
        const double p = static_cast<double>(num_parts);
        *out = p * (1.0 - std::pow(1.0 - 1.0 / p, static_cast<double>(degree)));
    });
}
sc_status sc_imbalance_lower_bound(int32_t num_parts, int64_t max_degree, int64_t min_degree, double* out) {
    return guard([&] {  // partition.cpp:351-362
        REQUIRE_ARG(out, "sc_imbalance_lower_bound: null out");
        if (num_parts < 1) throw std::invalid_argument("num_parts must be >= 1");
        if (min_degree < 1) throw std::invalid_argument("imbalance_lower_bound: min_degree must be >= 1");
        if (max_degree < min_degree) throw std::invalid_argument("imbalance_lower_bound: max_degree < min_degree");
        if (num_parts == 1) {
            *out = 1.0;
            return;
        }
        const double p = static_cast<double>(num_parts);
        *out = (1.0 - std::pow(1.0 - 1.0 / p, static_cast<double>(max_degree))) /
               (1.0 - std::pow(1.0 - 1.0 / p, static_cast<double>(min_degree)));
    });
}
sc_status sc_trainer_profile(sc_trainer* t, int32_t enable) {
    return guard([&] { t->prof.enabled = enable != 0; });
}
sc_status sc_trainer_kernel_times(sc_trainer* t, const char** names, double* ms, double* bytes, int32_t cap,
                                  int32_t* count) {
    return guard([&] {
        int32_t k = 0;
        for (const auto& kv : t->prof.totals) {
            if (k < cap) {
                if (names) names[k] = kv.first.c_str();
                if (ms) ms[k] = kv.second.ms;
                if (bytes) bytes[k] = kv.second.bytes;
            }
            ++k;
        }
        *count = k;
    });
}
sc_status sc_trainer_kernel_flops(sc_trainer* t, double* flops, int32_t cap, int32_t* count) {
    return guard([&] {
        int32_t k = 0;
        for (const auto& kv : t->prof.totals) {  // same order as sc_trainer_kernel_times
            if (k < cap && flops) flops[k] = kv.second.flops;
            ++k;
        }
        *count = k;
    });
}
sc_status sc_debug_gemm(sc_ctx* ctx, int32_t mode, int64_t M, int32_t N, int32_t K1, const float* A1,
                        int64_t a1_rows, int64_t lda1, const int32_t* rows1, const float* B1, int64_t ldb1,
                        int32_t b1_nn, int32_t K2, const float* A2, int64_t lda2, const float* B2, int64_t ldb2,
                        int32_t b2_nn, int32_t epi, const float* scale, float* C) {
    return guard([&] {
        REQUIRE_ARG(ctx && A1 && B1 && C && M >= 0 && N >= 1 && K1 >= 1, "sc_debug_gemm: bad arguments");
        set_device(ctx);
        cudaStream_t s = ctx->stream;
        auto up = [&](const void* h, size_t bytes) {
            DevBuf<unsigned char> d(std::max<size_t>(bytes, 16));
            if (bytes) SC_CUDA(cudaMemcpyAsync(d.get(), h, bytes, cudaMemcpyHostToDevice, s));
            return d;
        };
        auto dA1 = up(A1, sizeof(float) * a1_rows * lda1);
        auto dB1 = up(B1, sizeof(float) * (b1_nn ? int64_t(K1) * ldb1 : int64_t(N) * ldb1));
        DevBuf<unsigned char> dR1, dA2, dB2, dS;
        if (rows1) dR1 = up(rows1, sizeof(int32_t) * M);
        if (K2 > 0) {
            dA2 = up(A2, sizeof(float) * M * lda2);
            dB2 = up(B2, sizeof(float) * (b2_nn ? int64_t(K2) * ldb2 : int64_t(N) * ldb2));
        }
        if (epi == kEpiRowScale) dS = up(scale, sizeof(float) * M);
        const int64_t ldc = (N + 3) / 4 * 4;  // 16-byte output rows, as the trainer's buffers are
        DevBuf<float> dC(std::max<int64_t>(M * ldc, 1));
        const MatA a1{reinterpret_cast<const float*>(dA1.get()), lda1,
                      rows1 ? reinterpret_cast<const int32_t*>(dR1.get()) : nullptr, K1};
        const MatB b1{reinterpret_cast<const float*>(dB1.get()), ldb1, b1_nn != 0};
        const MatA a2{reinterpret_cast<const float*>(dA2.get()), lda2, nullptr, K2};
        const MatB b2{reinterpret_cast<const float*>(dB2.get()), ldb2, b2_nn != 0};
        const float* sc = epi == kEpiRowScale ? reinterpret_cast<const float*>(dS.get()) : nullptr;
        if (mode == 0 && tc_supported(a1, K2 > 0 ? &a2 : nullptr, N)) {
            DevBuf<float> am(2);
            SC_CUDA(cudaMemsetAsync(am.get(), 0, 2 * sizeof(float), s));
            absmax(a1_rows * lda1, a1.ptr, am.get(), s);
            if (K2 > 0) absmax(M * lda2, a2.ptr, am.get() + 1, s);
            BImage i1, i2;
            prep_bimage(i1, b1, N, K1, s);
            if (K2 > 0) prep_bimage(i2, b2, N, K2, s);
            gemm_f16x3(a1, am.get(), i1, K2 > 0 ? &a2 : nullptr, am.get() + 1, K2 > 0 ? &i2 : nullptr, dC.get(), ldc,
                       M, N, epi, sc, nullptr, s);
            SC_CUDA(cudaStreamSynchronize(s));
        } else {
            gemm_nt(a1, b1, K2 > 0 ? &a2 : nullptr, K2 > 0 ? &b2 : nullptr, dC.get(), ldc, M, N, epi, sc, s);
        }
        if (M > 0)
            SC_CUDA(cudaMemcpy2DAsync(C, sizeof(float) * N, dC.get(), sizeof(float) * ldc, sizeof(float) * N, M,
                                      cudaMemcpyDeviceToHost, s));
        SC_CUDA(cudaStreamSynchronize(s));
    });
}

sc_status sc_debug_gemm_tn(sc_ctx* ctx, int32_t mode, int64_t M, const float* A, int32_t N1, const float* B1,
                           int32_t N2a, const float* B2, int64_t b2_rows, int32_t N2b, const int32_t* rows2, float* C) {
    return guard([&] {
        REQUIRE_ARG(ctx && A && B1 && C && M >= 0 && N1 >= 1 && N2a >= 1, "sc_debug_gemm_tn: bad arguments");
        set_device(ctx);
        cudaStream_t s = ctx->stream;
        const int32_t N2 = N2a + (B2 ? N2b : 0);
        const int32_t lda = (N1 + 3) / 4 * 4;  // 16-byte rows, as the trainer's buffers are
        DevBuf<float> dA(std::max<int64_t>(M * lda, 1)), dB1(std::max<int64_t>(M * N2a, 1));
        DevBuf<float> dB2(std::max<int64_t>(B2 ? b2_rows * N2b : 1, 1)), dC(int64_t(N1) * N2);
        DevBuf<int32_t> dR(std::max<int64_t>(rows2 ? M : 1, 1));
        if (M > 0)
            SC_CUDA(cudaMemcpy2DAsync(dA.get(), sizeof(float) * lda, A, sizeof(float) * N1, sizeof(float) * N1, M,
                                      cudaMemcpyHostToDevice, s));
        h2d(dB1.get(), B1, M * N2a, s);
        if (B2) h2d(dB2.get(), B2, b2_rows * N2b, s);
        if (rows2) h2d(dR.get(), rows2, M, s);
        const MatT a{dA.get(), lda, nullptr, N1}, b1{dB1.get(), N2a, nullptr, N2a};
        const MatT b2{dB2.get(), N2b, rows2 ? dR.get() : nullptr, N2b};
        const int64_t wsf = std::max<int64_t>(gemm_tn_workspace_floats(N1, N2), int64_t(256) * N1 * N2);
        DevBuf<float> ws(wsf);
        if (mode == 0 && tn_supported(a, b1, B2 ? &b2 : nullptr)) {
            DevBuf<float> am(3);
            SC_CUDA(cudaMemsetAsync(am.get(), 0, 3 * sizeof(float), s));
            absmax(M * lda, dA.get(), am.get(), s);
            absmax(M * N2a, dB1.get(), am.get() + 1, s);
            if (B2) absmax(b2_rows * N2b, dB2.get(), am.get() + 2, s);
            gemm_tn_f16x3(a, am.get(), b1, am.get() + 1, B2 ? &b2 : nullptr, am.get() + 2, M, dC.get(), N2, ws.get(),
                          wsf, s);
        } else {
            gemm_tn(a, b1, B2 ? &b2 : nullptr, M, dC.get(), N2, ws.get(), wsf, s);
        }
        d2h(C, dC.get(), int64_t(N1) * N2, s);
        SC_CUDA(cudaStreamSynchronize(s));
    });
}

sc_status sc_debug_gemm_tn_dual(sc_ctx* ctx, int64_t M, const float* A1, int32_t N1a, const float* A2, int32_t N1b,
                               const float* B1, int32_t N2a, const float* B2, int32_t N2b, float* C1, float* C2) {
    return guard([&] {
        REQUIRE_ARG(ctx && A1 && A2 && B1 && B2 && C1 && C2 && M >= 0, "sc_debug_gemm_tn_dual: bad arguments");
        set_device(ctx);
        cudaStream_t s = ctx->stream;
        auto up = [&](const float* h, int64_t rows, int32_t cols) {
            DevBuf<float> d(std::max<int64_t>(rows * cols, 1));
            h2d(d.get(), h, rows * cols, s);
            return d;
        };
        auto dA1 = up(A1, M, N1a), dA2 = up(A2, M, N1b), dB1 = up(B1, M, N2a), dB2 = up(B2, M, N2b);
        const MatT a1{dA1.get(), N1a, nullptr, N1a}, a2{dA2.get(), N1b, nullptr, N1b};
        const MatT b1{dB1.get(), N2a, nullptr, N2a}, b2{dB2.get(), N2b, nullptr, N2b};
        REQUIRE_ARG(tn_dual_supported(a1, a2, b1, b2), "sc_debug_gemm_tn_dual: shapes not supported by the dual launch");
        DevBuf<float> am(4), dC1(int64_t(N1a) * (N2a + N2b)), dC2(int64_t(N1b) * N2b);
        SC_CUDA(cudaMemsetAsync(am.get(), 0, 4 * sizeof(float), s));
        absmax(M * N1a, a1.ptr, am.get(), s);
        absmax(M * N1b, a2.ptr, am.get() + 1, s);
        absmax(M * N2a, b1.ptr, am.get() + 2, s);
        absmax(M * N2b, b2.ptr, am.get() + 3, s);
        const int64_t wsf = gemm_tn_workspace_floats(N1a + N1b, N2a + N2b);
        DevBuf<float> ws(wsf);
        gemm_tn_f16x3_dual(a1, am.get(), a2, am.get() + 1, b1, am.get() + 2, b2, am.get() + 3, M, dC1.get(), N2a + N2b,
                           dC2.get(), N2b, ws.get(), wsf, s);
        d2h(C1, dC1.get(), int64_t(N1a) * (N2a + N2b), s);
        d2h(C2, dC2.get(), int64_t(N1b) * N2b, s);
        SC_CUDA(cudaStreamSynchronize(s));
    });
}
sc_status sc_debug_spmm(sc_ctx* ctx, int32_t bwd, int64_t n, int32_t H, const int64_t* offsets,
                        const int32_t* nbrs, const int32_t* eids, int64_t num_edges, const uint8_t* edge_mask,
                        const float* src, const float* msg, float* out) {
    return guard([&] {
        REQUIRE_ARG(ctx && offsets && src && out && n >= 0 && H >= 1, "sc_debug_spmm: bad arguments");
        REQUIRE_ARG(bwd >= 0 && bwd <= 3, "sc_debug_spmm: mode must be 0 .. 3");
        REQUIRE_ARG((bwd != 1 && bwd != 3) || msg, "sc_debug_spmm: modes 1 and 3 need msg (ReLU decisions / addend)");
        set_device(ctx);
        cudaStream_t s = ctx->stream;
        const int64_t nnz = offsets[n] - offsets[0];
        REQUIRE_ARG(offsets[0] == 0 && nnz >= 0 && (nnz == 0 || (nbrs && eids)), "sc_debug_spmm: bad CSR");
        DevBuf<int64_t> d_off(n + 1);
        DevBuf<int32_t> d_nb(std::max<int64_t>(nnz, 1)), d_ei(std::max<int64_t>(nnz, 1));
        DevBuf<float> d_src(std::max<int64_t>(n * H, 1)), d_out(std::max<int64_t>(n * H, 1)), d_inv(std::max<int64_t>(n, 1));
        const bool has_msg = bwd == 1 || bwd == 3;
        DevBuf<float> d_msg(has_msg ? std::max<int64_t>(n * H, 1) : 1);
        h2d(d_off.get(), offsets, n + 1, s);
        h2d(d_nb.get(), nbrs, nnz, s);
        h2d(d_ei.get(), eids, nnz, s);
        h2d(d_src.get(), src, n * H, s);
        if (has_msg) h2d(d_msg.get(), msg, n * H, s);
        DevBuf<uint32_t> bits;
        if (edge_mask) {  // the trainer's CSR-slot bitmap of a per-local-edge DropEdge mask
            DevBuf<uint8_t> d_mask(std::max<int64_t>(num_edges, 1));
            h2d(d_mask.get(), edge_mask, num_edges, s);
            bits.alloc(std::max<int64_t>((nnz + 31) / 32, 1));
            mask_to_bits(nnz, d_ei.get(), d_mask.get(), bits.get(), s);
            SC_CUDA(cudaStreamSynchronize(s));
        }
        HeavyRows hv;
        build_heavy_rows(ctx, n, d_off.get(), hv);
        DevBuf<float> partial(std::max<int64_t>(int64_t(hv.nseg) * H, 1));
        if (bwd != 1) inv_degree(n, d_off.get(), bits.get(), d_inv.get(), s);
        if (bwd == 0) {
            spmm_fwd(n, H, d_off.get(), d_nb.get(), bits.get(), d_inv.get(), d_src.get(), d_out.get(), s, &hv,
                     partial.get());
        } else if (bwd == 2) {  // the projected top layer's backward: sum_kept inv[nbr] src[nbr]
            spmm_sum_scaled(n, H, d_off.get(), d_nb.get(), bits.get(), d_inv.get(), d_src.get(), d_out.get(), s,
                            nullptr, &hv, partial.get());
        } else if (bwd == 3) {  // its forward: msg (the addend) + inv * sum_kept src[nbr]
            SC_CUDA(cudaMemcpyAsync(d_out.get(), d_msg.get(), sizeof(float) * n * H, cudaMemcpyDeviceToDevice, s));
            spmm_fwd_add(n, H, d_off.get(), d_nb.get(), bits.get(), d_inv.get(), d_src.get(), d_out.get(), s, &hv,
                         partial.get());
        } else {
            spmm_bwd(n, H, d_off.get(), d_nb.get(), bits.get(), d_src.get(), d_msg.get(), d_out.get(), s, nullptr, &hv,
                     partial.get());
        }
        d2h(out, d_out.get(), n * H, s);
        SC_CUDA(cudaStreamSynchronize(s));
    });
}
sc_status sc_trainer_debug_buffer(sc_trainer* t, const char* name, int32_t layer, void* dst_dev, int64_t bytes) {
    return guard([&] {
        REQUIRE_ARG(t && name && dst_dev, "sc_trainer_debug_buffer: null argument");
        set_device(t->ctx);
        trainer_finish(t, nullptr, nullptr);
        const std::string nm(name);
        const void* b = nullptr;
        size_t width = 0;  // bytes per row
        const int32_t H = layer >= 0 && layer < t->L ? t->lay[layer].H : 0;
        if (nm == "X" && layer >= 1 && layer <= t->L) {
            b = t->X[layer];
            width = 4 * size_t(t->lay[layer - 1].H);
        } else if (nm == "MSG" && layer >= 0 && layer < t->L) {
            REQUIRE_ARG(!t->compact, "sc_trainer_debug_buffer: compact activations keep only the ReLU bits (POS)");
            b = t->MSG[layer];
            width = 4 * size_t(H);
        } else if (nm == "POS" && layer >= 0 && layer < t->L) {
            REQUIRE_ARG(t->compact, "sc_trainer_debug_buffer: POS exists with compact activations only");
            b = t->POS[layer];
            width = 4 * size_t((H + 31) / 32);
        } else if (nm == "MEAN" && layer >= 0 && layer < t->L) {
            b = t->MEAN[layer];
            width = 4 * size_t(H);
        } else if (nm == "inv") {
            b = t->inv;
            width = 4;
        } else if (nm == "G") {
            b = t->G;
            width = 4 * size_t(t->Cp);
        }
        REQUIRE_ARG(b, "sc_trainer_debug_buffer: unknown buffer");
        REQUIRE_ARG(bytes >= 0 && size_t(bytes) <= width * size_t(t->rows_cap),
                    "sc_trainer_debug_buffer: more bytes than the buffer holds");
        SC_CUDA(cudaMemcpyAsync(dst_dev, b, size_t(bytes), cudaMemcpyDeviceToDevice, t->ctx->stream));
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
    });
}

sc_status sc_trainer_destroy(sc_trainer* t) {
    return guard([&] {
        if (!t) return;
        set_device(t->ctx);
        cudaStreamSynchronize(t->ctx->stream);
        delete t;
    });
}

}  // extern "C"
