// sagecut_b200.hpp — C++ drop-in facade over libsagecut_cuda.so.
//
// Mirrors the reference's C++ API for the CoFree-GNN training path
// (namespace sagecut in /root/reference/proj/include/sagecut/*.hpp) on top of
// the C ABI in sagecut_cuda.h, so a caller such as the reference CLI
// (proj/tools/main.cpp: run_partition :299-318, run_train :430-446) switches
// by changing the namespace and include. Graph / partition state stays on the
// device; the by-value structs below are host copies made on request.
//
// Differences from the reference, by design:
//   * Graph holds a device handle (features fp32 row-major, no Eigen);
//   * precision is always f32 (the reference's Precision::f32 path); TrainConfig::precision
//     defaults to f32 here and f64 is rejected with std::invalid_argument;
//   * train_cofree's per-epoch evaluation is optional (TrainConfig::evaluate).
// Errors: the reference's exception types and message texts are rethrown
// (std::invalid_argument, std::runtime_error, std::logic_error).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sagecut_cuda.h"

namespace sagecut_b200 {

using NodeId = std::int32_t;  // graph.hpp:12
using EdgeId = std::int32_t;  // graph.hpp:13

struct Edge {  // graph.hpp:15-19
    NodeId u = 0;
    NodeId v = 0;
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(sc_status st) {
    if (st == SC_OK) return;
    const std::string msg = sc_last_error();
    switch (st) {
        case SC_EINVAL: throw std::invalid_argument(msg);
        case SC_ERUNTIME: throw std::runtime_error(msg);
        case SC_EINTERNAL: throw std::logic_error(msg);
        default: throw CudaError(msg);
    }
}

class Context {
public:
    explicit Context(int device = 0) { check(sc_ctx_create(device, &h_)); }
    ~Context() { sc_ctx_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    sc_ctx* get() const { return h_; }

private:
    sc_ctx* h_ = nullptr;
};

struct ValidationReport {  // graph.hpp:43-48
    std::int64_t dropped_self_loops = 0;
    std::int64_t merged_duplicate_edges = 0;
};

// sagecut::Graph (graph.hpp:53-80) with its storage on the device.
class Graph {
public:
    Graph() = default;
    Graph(Context& ctx, sc_graph* h) : ctx_(&ctx), h_(h, &sc_graph_destroy) { refresh(); }
    sc_graph* get() const { return h_.get(); }
    Context& context() const { return *ctx_; }
    NodeId num_nodes = 0;
    int num_classes = 0;
    int feature_dim = 0;
    std::size_t num_edges() const { return static_cast<std::size_t>(m_); }
    std::vector<Edge> edges() const {
        std::vector<Edge> e(num_edges());
        check(sc_graph_copy_edges(get(), reinterpret_cast<std::int32_t*>(e.data())));
        return e;
    }
    std::vector<NodeId> degrees() const {
        std::vector<NodeId> d(static_cast<std::size_t>(num_nodes));
        check(sc_graph_copy_csr(get(), nullptr, nullptr, nullptr, d.data()));
        return d;
    }
    // features: num_nodes x dim row-major; labels: class ids; masks: 0/1 per node
    void set_data(const std::vector<float>& features, int dim, const std::vector<NodeId>& labels, int classes,
                  const std::vector<std::uint8_t>& train, const std::vector<std::uint8_t>& val,
                  const std::vector<std::uint8_t>& test) {
        check(sc_graph_set_data(get(), features.data(), dim, labels.data(), classes, train.data(), val.data(),
                                test.data()));
        refresh();
    }

    // Graph::multilabels (graph.hpp:64): num_nodes x C row-major 0/1; replaces the class ids
    // (bce training, micro-F1 evaluation). Call after set_data.
    void set_multilabels(const std::vector<float>& targets, int classes) {
        check(sc_graph_set_multilabels(get(), targets.data(), classes));
        refresh();
        multilabel_ = true;
    }
    bool is_multilabel() const { return multilabel_; }  // graph.hpp:74

private:
    bool multilabel_ = false;
    void refresh() {
        std::int32_t d = 0, c = 0;
        check(sc_graph_info(get(), &num_nodes, &m_, &d, &c));
        feature_dim = d;
        num_classes = c;
    }
    Context* ctx_ = nullptr;
    std::shared_ptr<sc_graph> h_;
    std::int64_t m_ = 0;
};

// build_graph (graph.cpp:8-64), on the device.
inline std::pair<Graph, ValidationReport> build_graph(Context& ctx, NodeId num_nodes, const std::vector<Edge>& raw) {
    sc_graph* h = nullptr;
    ValidationReport rep;
    check(sc_build_graph(ctx.get(), num_nodes, reinterpret_cast<const std::int32_t*>(raw.data()),
                         static_cast<std::int64_t>(raw.size()), &h, &rep.dropped_self_loops,
                         &rep.merged_duplicate_edges));
    return {Graph(ctx, h), rep};
}

// ---- dataset files (graph_io.hpp / graph_io.cpp:41-296) ----------------------------
struct LoadOptions {  // graph_io.hpp:12-19
    std::int32_t num_nodes = -1;  // -1: 1 + max id seen
    bool strict = false;
};
// load_graph (graph_io.cpp:41-80): text edge list -> build_graph on the device.
inline std::pair<Graph, ValidationReport> load_graph(Context& ctx, const std::string& path,
                                                     const LoadOptions& options = {}) {
    sc_graph* h = nullptr;
    ValidationReport rep;
    check(sc_load_graph(ctx.get(), path.c_str(), options.num_nodes, options.strict ? 1 : 0, &h,
                        &rep.dropped_self_loops, &rep.merged_duplicate_edges));
    return {Graph(ctx, h), rep};
}
struct FeatureMatrix {  // Eigen::MatrixXd of load_features, as fp32 row-major
    std::int64_t rows = 0, cols = 0;
    std::vector<float> values;
};
inline FeatureMatrix load_features(const std::string& path, NodeId expected_nodes) {  // graph_io.cpp:82-160
    FeatureMatrix m;
    check(sc_load_features(path.c_str(), expected_nodes, nullptr, 0, &m.rows, &m.cols));
    m.values.resize(static_cast<std::size_t>(m.rows * m.cols));
    check(sc_load_features(path.c_str(), expected_nodes, m.values.data(), static_cast<std::int64_t>(m.values.size()),
                           &m.rows, &m.cols));
    return m;
}
struct LabelData {  // Graph::labels / multilabels / num_classes after load_labels
    std::vector<NodeId> labels;        // multi-class
    std::vector<float> multilabels;    // n x num_classes 0/1
    int num_classes = 0;
    bool is_multilabel() const { return !multilabels.empty(); }
};
inline LabelData load_labels(const std::string& path, NodeId num_nodes) {  // graph_io.cpp:188-242
    LabelData d;
    std::int32_t nc = 0, ml = 0;
    check(sc_load_labels(path.c_str(), num_nodes, nullptr, nullptr, 0, &nc, &ml));
    d.num_classes = nc;
    if (ml) {
        d.multilabels.resize(static_cast<std::size_t>(num_nodes) * static_cast<std::size_t>(nc));
        check(sc_load_labels(path.c_str(), num_nodes, nullptr, d.multilabels.data(),
                             static_cast<std::int64_t>(d.multilabels.size()), &nc, &ml));
    } else {
        d.labels.resize(static_cast<std::size_t>(num_nodes));
        check(sc_load_labels(path.c_str(), num_nodes, d.labels.data(), nullptr, 0, &nc, &ml));
    }
    return d;
}
struct SplitMasks {
    std::vector<std::uint8_t> train, val, test;
};
inline SplitMasks load_masks(const std::string& path, NodeId num_nodes) {  // graph_io.cpp:256-283
    SplitMasks m;
    m.train.resize(static_cast<std::size_t>(num_nodes));
    m.val.resize(m.train.size());
    m.test.resize(m.train.size());
    check(sc_load_masks(path.c_str(), num_nodes, m.train.data(), m.val.data(), m.test.data()));
    return m;
}
// main.cpp:137 load_dataset: graph + features + labels (+ multi-label) + masks on the device
inline std::pair<Graph, ValidationReport> load_dataset(Context& ctx, const std::string& edges,
                                                       const std::string& features, const std::string& labels,
                                                       const std::string& masks, const LoadOptions& options = {}) {
    auto gr = load_graph(ctx, edges, options);
    Graph& g = gr.first;
    const FeatureMatrix f = load_features(features, g.num_nodes);
    const LabelData l = load_labels(labels, g.num_nodes);
    const SplitMasks m = load_masks(masks, g.num_nodes);
    const std::vector<NodeId> ids = l.is_multilabel() ? std::vector<NodeId>(static_cast<std::size_t>(g.num_nodes), 0)
                                                      : l.labels;
    g.set_data(f.values, static_cast<int>(f.cols), ids, l.num_classes, m.train, m.val, m.test);
    if (l.is_multilabel()) g.set_multilabels(l.multilabels, l.num_classes);
    return gr;
}
inline void save_edge_list(const Graph& g, const std::string& path) {  // graph_io.cpp:75-80
    check(sc_save_edge_list(g.get(), path.c_str()));
}
inline void save_features_csv(const FeatureMatrix& m, const std::string& path) {  // graph_io.cpp:162-172
    check(sc_save_features(path.c_str(), m.values.data(), m.rows, m.cols, 0));
}
inline void save_features_binary(const FeatureMatrix& m, const std::string& path) {  // graph_io.cpp:174-186
    check(sc_save_features(path.c_str(), m.values.data(), m.rows, m.cols, 1));
}
inline void save_labels(const LabelData& l, NodeId num_nodes, const std::string& path) {  // graph_io.cpp:244-254
    check(sc_save_labels(path.c_str(), num_nodes, l.is_multilabel() ? nullptr : l.labels.data(),
                         l.is_multilabel() ? l.multilabels.data() : nullptr, l.num_classes));
}
inline void save_masks(const SplitMasks& m, const std::string& path) {  // graph_io.cpp:285-296
    check(sc_save_masks(path.c_str(), static_cast<std::int32_t>(m.train.size()), m.train.data(), m.val.data(),
                        m.test.data()));
}

struct PartSubgraph {  // partition.hpp:14-31 (host copy)
    std::vector<NodeId> nodes;
    std::vector<NodeId> global_to_local;
    std::vector<Edge> edges;
    std::vector<EdgeId> edge_global_ids;
    std::vector<NodeId> local_degrees;
    std::vector<std::int64_t> adj_offsets;  // int64: >2^31 CSR entries fit
    std::vector<NodeId> adj_neighbors;
    std::vector<EdgeId> adj_edge_ids;
    NodeId num_local_nodes() const { return static_cast<NodeId>(nodes.size()); }
};

// sagecut::VertexCutPartition (partition.hpp:35-40), device resident.
class VertexCutPartition {
public:
    VertexCutPartition() = default;
    VertexCutPartition(const Graph& g, sc_vcut* h) : g_(&g), h_(h, &sc_vcut_destroy) {
        check(sc_vcut_num_parts(h, &num_parts));
    }
    sc_vcut* get() const { return h_.get(); }
    int num_parts = 0;
    std::vector<int> edge_assignment() const {
        std::vector<int> a(g_->num_edges());
        check(sc_vcut_assignment(get(), a.data()));
        return a;
    }
    PartSubgraph part(int i) const {
        std::int64_t nl = 0, ne = 0;
        check(sc_vcut_part_sizes(get(), i, &nl, &ne));
        PartSubgraph s;
        s.nodes.resize(nl);
        s.global_to_local.resize(static_cast<std::size_t>(g_->num_nodes));
        s.edges.resize(ne);
        s.edge_global_ids.resize(ne);
        s.local_degrees.resize(nl);
        s.adj_offsets.resize(nl + 1);
        s.adj_neighbors.resize(2 * ne);
        s.adj_edge_ids.resize(2 * ne);
        check(sc_vcut_part_copy(get(), i, s.nodes.data(), reinterpret_cast<std::int32_t*>(s.edges.data()),
                                s.edge_global_ids.data(), s.local_degrees.data(), s.adj_offsets.data(),
                                s.adj_neighbors.data(), s.adj_edge_ids.data(), s.global_to_local.data()));
        return s;
    }
    std::vector<std::string> warnings() const {  // partition.hpp:36
        std::int64_t need = 0;
        check(sc_vcut_warnings(get(), nullptr, 0, &need));
        std::string buf(static_cast<std::size_t>(need), '\0');
        check(sc_vcut_warnings(get(), buf.data(), need, &need));
        buf.resize(std::strlen(buf.c_str()));
        std::vector<std::string> out;
        std::size_t a = 0;
        while (!buf.empty() && a <= buf.size()) {
            const std::size_t b = std::min(buf.find('\n', a), buf.size());
            out.push_back(buf.substr(a, b - a));
            a = b + 1;
        }
        return out;
    }

private:
    const Graph* g_ = nullptr;
    std::shared_ptr<sc_vcut> h_;
};

// partition.hpp:41-52 (host copy)
struct EdgeCutPartition {
    int num_parts = 0;
    std::vector<int> node_assignment;
    std::vector<std::vector<EdgeId>> kept_edges;
    std::vector<EdgeId> cut_edges;
    std::vector<std::vector<NodeId>> halo_sets;
    std::size_t total_halo() const {
        std::size_t h = 0;
        for (const auto& s : halo_sets) h += s.size();
        return h;
    }
};

// partition.cpp:92-114, 22-90
inline VertexCutPartition partition_random(const Graph& g, int num_parts, std::uint64_t seed) {
    sc_vcut* h = nullptr;
    check(sc_partition_random(g.get(), num_parts, seed, &h));
    return VertexCutPartition(g, h);
}
inline VertexCutPartition partition_dbh(const Graph& g, int num_parts, std::uint64_t seed) {
    sc_vcut* h = nullptr;
    check(sc_partition_dbh(g.get(), num_parts, seed, &h));
    return VertexCutPartition(g, h);
}
// partition.cpp:116-201 (same assignment and warnings; O(E log E))
inline VertexCutPartition partition_ne(const Graph& g, int num_parts, std::uint64_t seed, double balance_slack = 1.1) {
    sc_vcut* h = nullptr;
    check(sc_partition_ne(g.get(), num_parts, seed, balance_slack, &h));
    return VertexCutPartition(g, h);
}
// partition.cpp:203-231
inline EdgeCutPartition edge_cut_from_assignment(const Graph& g, int num_parts, std::vector<int> node_assignment) {
    if (node_assignment.size() != static_cast<std::size_t>(g.num_nodes))
        throw std::invalid_argument("node assignment length does not match node count");
    const std::size_t p = static_cast<std::size_t>(std::max(num_parts, 1));
    std::vector<std::int64_t> kept(p), halo(p);
    std::int64_t ncut = 0;
    check(sc_edge_cut_from_assignment(g.get(), num_parts, node_assignment.data(), kept.data(), &ncut, halo.data(),
                                      nullptr, nullptr, nullptr));
    std::int64_t nh = 0;
    for (auto x : halo) nh += x;
    std::vector<std::int32_t> kept_ids(g.num_edges() - static_cast<std::size_t>(ncut)), halo_nodes(nh);
    EdgeCutPartition ec;
    ec.num_parts = num_parts;
    ec.cut_edges.resize(static_cast<std::size_t>(ncut));
    check(sc_edge_cut_from_assignment(g.get(), num_parts, node_assignment.data(), kept.data(), &ncut, halo.data(),
                                      kept_ids.data(), ec.cut_edges.data(), halo_nodes.data()));
    std::size_t ka = 0, ha = 0;
    for (int i = 0; i < num_parts; ++i) {
        ec.kept_edges.emplace_back(kept_ids.begin() + ka, kept_ids.begin() + ka + kept[i]);
        ec.halo_sets.emplace_back(halo_nodes.begin() + ha, halo_nodes.begin() + ha + halo[i]);
        ka += kept[i];
        ha += halo[i];
    }
    ec.node_assignment = std::move(node_assignment);
    return ec;
}
// partition.cpp:233-278
inline EdgeCutPartition partition_edge_cut_greedy(const Graph& g, int num_parts, std::uint64_t seed) {
    std::vector<int> na(static_cast<std::size_t>(g.num_nodes));
    check(sc_partition_edge_cut_greedy(g.get(), num_parts, seed, na.data()));
    return edge_cut_from_assignment(g, num_parts, std::move(na));
}
// partition.cpp:280-308
inline VertexCutPartition edge_cut_to_vertex_cut(const Graph& g, const EdgeCutPartition& ec, std::uint64_t seed) {
    if (ec.node_assignment.size() != static_cast<std::size_t>(g.num_nodes))
        throw std::invalid_argument("edge cut does not match graph");
    sc_vcut* h = nullptr;
    check(sc_edge_cut_to_vertex_cut(g.get(), ec.num_parts, ec.node_assignment.data(), seed, &h));
    return VertexCutPartition(g, h);
}
inline VertexCutPartition build_vertex_cut(const Graph& g, int num_parts, const std::vector<int>& edge_assignment) {
    if (edge_assignment.size() != g.num_edges())
        throw std::invalid_argument("edge assignment length does not match edge count");
    sc_vcut* h = nullptr;
    check(sc_build_vertex_cut(g.get(), num_parts, edge_assignment.data(), &h));
    return VertexCutPartition(g, h);
}

struct ReplicationStats {  // partition.hpp:50-56
    double rf = 0.0;
    std::vector<int> per_node_rf;
    double edge_balance = 0.0;
    double node_balance = 0.0;
    std::int64_t duplicated_nodes = 0;
};
inline ReplicationStats replication_stats(const VertexCutPartition& part, const Graph& g) {  // partition.cpp:310
    ReplicationStats s;
    s.per_node_rf.resize(static_cast<std::size_t>(g.num_nodes));
    check(sc_replication_stats(part.get(), s.per_node_rf.data(), &s.rf, &s.edge_balance, &s.node_balance,
                               &s.duplicated_nodes));
    return s;
}

enum class ReweightScheme { dar, vanilla_inv, none };  // reweight.hpp:10
struct NodeWeights {                                    // reweight.hpp:15-19
    ReweightScheme scheme = ReweightScheme::none;
    std::vector<std::vector<double>> per_part;
};
inline NodeWeights compute_weights(ReweightScheme scheme, const Graph& g, const VertexCutPartition& part) {
    (void)g;
    std::vector<std::int64_t> sizes(static_cast<std::size_t>(part.num_parts));
    std::int64_t total = 0;
    for (int i = 0; i < part.num_parts; ++i) {
        check(sc_vcut_part_sizes(part.get(), i, &sizes[i], nullptr));
        total += sizes[i];
    }
    std::vector<double> flat(static_cast<std::size_t>(total));
    check(sc_compute_weights(part.get(), static_cast<int>(scheme), flat.data()));
    NodeWeights w;
    w.scheme = scheme;
    std::int64_t off = 0;
    for (auto sz : sizes) {
        w.per_part.emplace_back(flat.begin() + off, flat.begin() + off + sz);
        off += sz;
    }
    return w;
}

struct DropEdgeMaskSet {  // dropedge.hpp:13-18
    int num_masks = 0;
    double ratio = 0.0;
    std::uint64_t seed = 0;
    std::vector<std::vector<std::uint8_t>> masks;
};
inline DropEdgeMaskSet precompute_masks(Context& ctx, std::size_t num_edges, int num_masks, double ratio,
                                        std::uint64_t seed) {  // dropedge.cpp:9
    std::vector<std::uint8_t> flat(num_edges * static_cast<std::size_t>(num_masks > 0 ? num_masks : 0) + 1);
    check(sc_precompute_masks(ctx.get(), static_cast<std::int64_t>(num_edges), num_masks, ratio, seed, flat.data()));
    DropEdgeMaskSet s{num_masks, ratio, seed, {}};
    for (int k = 0; k < num_masks; ++k)
        s.masks.emplace_back(flat.begin() + k * num_edges, flat.begin() + (k + 1) * num_edges);
    return s;
}
// select_mask for partition i at an epoch (trainer.hpp:261-266).
inline int select_mask(std::uint64_t seed, std::uint64_t part, std::uint64_t epoch, int num_masks) {
    if (num_masks < 1) throw std::invalid_argument("select_mask: need at least one mask");
    return sc_select_mask(seed, part, epoch, num_masks);
}

enum class LossKind { softmax_ce, bce };  // nn.hpp:296

enum class Precision { f64, f32 };  // trainer.hpp:18

struct TrainConfig {  // trainer.hpp:20-33
    int layers = 2;
    std::vector<int> hidden = {32};
    int epochs = 100;
    double learning_rate = 0.01;
    LossKind loss = LossKind::softmax_ce;
    ReweightScheme reweight = ReweightScheme::dar;
    bool use_dropedge = false;
    int dropedge_k = 10;
    double drop_ratio = 0.5;
    std::uint64_t seed = 0;
    // The device path computes in f32 (the reference's Precision::f32 arithmetic: f32 features,
    // model and Adam; f64 loss, weights and grad-norm). The reference defaults to f64, which
    // this library rejects rather than silently narrowing (train_cofree throws).
    Precision precision = Precision::f32;
    int workers = 1;            // accepted for source compatibility: results never depend on it
    bool evaluate = true;       // per-epoch full-graph metrics (trainer.hpp:306)
    bool deterministic = true;  // ascending-partition gradient sum
};

inline std::vector<int> resolved_hidden_dims(const TrainConfig& c) {  // trainer.cpp:12-19
    if (c.layers == 0) return {};
    if (c.hidden.size() == 1) return std::vector<int>(static_cast<std::size_t>(c.layers), c.hidden.front());
    if (c.hidden.size() != static_cast<std::size_t>(c.layers))
        throw std::invalid_argument("hidden dims must match layer count (or be a single value)");
    return c.hidden;
}

struct EpochMetrics {  // trainer.hpp:38-46
    int epoch = 0;
    double train_loss = 0.0, train_metric = 0.0, val_metric = 0.0, test_metric = 0.0, grad_norm = 0.0;
    std::uint64_t comm_floats = 0;
};
enum class CommMode { cofree, halo_sync_model };  // trainer.hpp:48
struct CommReport {                               // trainer.hpp:50-55
    CommMode mode = CommMode::cofree;
    std::uint64_t floats_per_iteration = 0;
    std::uint64_t gradient_floats = 0;
    std::uint64_t embedding_floats = 0;
};
// trainer.cpp:38-49
inline CommReport comm_volume(CommMode mode, int num_parts, std::size_t param_count, std::size_t num_layers,
                              std::size_t hidden_dim, std::size_t total_halo) {
    CommReport r;
    r.mode = mode;
    check(sc_comm_volume(mode == CommMode::cofree ? 0 : 1, num_parts, param_count, num_layers, hidden_dim,
                         total_halo, &r.floats_per_iteration, &r.gradient_floats, &r.embedding_floats));
    return r;
}
struct CommAudit {  // trainer.hpp:61-67
    std::vector<std::uint64_t> gradient_floats_per_epoch;
    std::uint64_t embedding_floats = 0;
};
// partition.cpp:344-362
inline double expected_rf_random(int num_parts, std::int64_t degree) {
    double x = 0;
    check(sc_expected_rf_random(num_parts, degree, &x));
    return x;
}
inline double imbalance_lower_bound(int num_parts, std::int64_t max_degree, std::int64_t min_degree) {
    double x = 0;
    check(sc_imbalance_lower_bound(num_parts, max_degree, min_degree, &x));
    return x;
}

struct TrainResult {  // trainer.hpp:71-75 (model as the flat for_each_matrix vector)
    std::vector<float> model;
    std::vector<EpochMetrics> metrics;
    CommAudit audit;
    int in_dim = 0, num_classes = 0;  // model dims, for save_checkpoint
    std::vector<int> hidden;
};

// checkpoint.cpp:44-57 (the model as SageModel<double>, "CFCK" format)
inline void save_checkpoint(const TrainResult& r, const std::string& path) {
    check(sc_save_checkpoint_params(r.model.data(), r.in_dim, r.hidden.data(), static_cast<std::int32_t>(r.hidden.size()),
                                    r.num_classes, path.c_str()));
}
// checkpoint.cpp:59-84: the flat parameters, cast to f32
inline std::vector<float> load_checkpoint(const std::string& path) {
    std::int64_t n = 0;
    check(sc_load_checkpoint_params(path.c_str(), nullptr, 0, &n));
    std::vector<float> theta(static_cast<std::size_t>(n));
    check(sc_load_checkpoint_params(path.c_str(), theta.data(), n, &n));
    return theta;
}
// trainer.cpp:126-140
inline void write_metrics_jsonl(const std::vector<EpochMetrics>& metrics, const std::string& path) {
    std::vector<sc_epoch_metrics> rows;
    for (const auto& m : metrics)
        rows.push_back(sc_epoch_metrics{m.epoch, m.train_loss, m.train_metric, m.val_metric, m.test_metric,
                                        m.grad_norm, m.comm_floats});
    check(sc_write_metrics_jsonl(path.c_str(), static_cast<std::int32_t>(rows.size()), rows.data()));
}
// partition_io.cpp:12-29 / :31-56 / :58-68
inline void save_partition(const VertexCutPartition& part, const std::string& path,
                           const ReweightScheme* weights = nullptr) {
    check(sc_save_partition(part.get(), path.c_str(), weights ? static_cast<std::int32_t>(*weights) : -1));
}
inline VertexCutPartition load_partition(const std::string& path, const Graph& g) {
    sc_vcut* h = nullptr;
    check(sc_load_partition(g.get(), path.c_str(), &h));
    return VertexCutPartition(g, h);
}
inline void save_edge_cut(const Graph& g, const EdgeCutPartition& ec, const std::string& path) {
    check(sc_save_edge_cut(g.get(), ec.num_parts, ec.node_assignment.data(), path.c_str()));
}

// train_cofree (trainer.cpp:119 / trainer.hpp:202-313) on one GPU; for a
// multi-GPU run create one sc_trainer per rank through the C ABI.
inline TrainResult train_cofree(const Graph& g, const VertexCutPartition& part, const TrainConfig& c) {
    if (c.epochs < 0) throw std::invalid_argument("epochs must be >= 0");
    if (c.precision != Precision::f32)
        throw std::invalid_argument("sagecut_b200 trains in Precision::f32 only (set TrainConfig::precision)");
    if (c.workers < 1) throw std::invalid_argument("workers must be >= 1");  // trainer.cpp:25
    const std::vector<int> hidden = resolved_hidden_dims(c);
    sc_train_config cfg{};
    cfg.layers = static_cast<std::int32_t>(hidden.size());
    cfg.hidden = hidden.data();
    cfg.learning_rate = c.learning_rate;
    cfg.loss = c.loss == LossKind::softmax_ce ? 0 : 1;
    cfg.reweight = static_cast<std::int32_t>(c.reweight);
    cfg.use_dropedge = c.use_dropedge ? 1 : 0;
    cfg.dropedge_k = c.dropedge_k;
    cfg.drop_ratio = c.drop_ratio;
    cfg.seed = c.seed;
    cfg.deterministic = c.deterministic ? 1 : 0;
    cfg.gemm = 0;
    sc_trainer* t = nullptr;
    check(sc_trainer_create(g.context().get(), g.get(), part.get(), &cfg, 0, 1, &t));
    std::unique_ptr<sc_trainer, sc_status (*)(sc_trainer*)> guard(t, &sc_trainer_destroy);
    std::int64_t P = 0;
    check(sc_trainer_param_count(t, &P));
    TrainResult res;
    for (int e = 0; e < c.epochs; ++e) {
        EpochMetrics m;
        m.epoch = e;
        check(sc_trainer_step(t, e, &m.train_loss, &m.grad_norm));
        std::uint64_t grad_floats = 0, emb_floats = 0;
        check(sc_trainer_comm_audit(t, &grad_floats, &emb_floats));
        res.audit.gradient_floats_per_epoch.push_back(grad_floats);
        res.audit.embedding_floats += emb_floats;
        if (c.evaluate) check(sc_trainer_evaluate(t, &m.train_metric, &m.val_metric, &m.test_metric));
        m.comm_floats = static_cast<std::uint64_t>(part.num_parts) * static_cast<std::uint64_t>(P);
        res.metrics.push_back(m);
    }
    res.in_dim = g.feature_dim;
    res.num_classes = g.num_classes;
    res.hidden = hidden;
    res.model.resize(static_cast<std::size_t>(P));
    check(sc_trainer_get_params(t, res.model.data()));
    return res;
}

// evaluate (trainer.cpp:101-112): full-graph metric of a trained model over one split mask
// (accuracy, or micro-F1 on multi-label graphs), forward-only on the device.
inline double evaluate(const TrainResult& model, const Graph& g, const std::vector<std::uint8_t>& mask) {
    if (mask.size() != static_cast<std::size_t>(g.num_nodes))
        throw std::invalid_argument("evaluate: mask length != node count");
    double x = 0.0;
    check(sc_evaluate(g.context().get(), g.get(), model.model.data(), model.hidden.data(),
                      static_cast<std::int32_t>(model.hidden.size()), mask.data(), &x));
    return x;
}

// train_full_graph (trainer.hpp:164-200): the p = 1 vertex cut (every edge in part 0, local ids =
// global ids) trained with unit loss weights and no DropEdge — the reference's degeneracy
// (test_trainer.cpp:69-79) — on the same device trainer.
inline TrainResult train_full_graph(const Graph& g, const TrainConfig& c) {
    const VertexCutPartition part = build_vertex_cut(g, 1, std::vector<int>(g.num_edges(), 0));
    TrainConfig fc = c;
    fc.reweight = ReweightScheme::none;
    fc.use_dropedge = false;
    TrainResult r = train_cofree(g, part, fc);
    for (auto& m : r.metrics) m.comm_floats = 0;
    r.audit = CommAudit{};  // nothing crosses workers in full-graph training
    return r;
}

}  // namespace sagecut_b200
