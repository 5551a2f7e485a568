// oracle/_ref harness — TEST INFRASTRUCTURE ONLY.
//
// Compiled together with the UNMODIFIED reference sources under
// /root/reference/proj/src (see oracle/Makefile) into oracle/_ref/libsagecut_ref.so.
// It exposes the reference's own functions through a flat C ABI so that
//   * tests/golden/make_golden.py can dump golden vectors from the real reference,
//   * tests/ can pin the oracle restatement (oracle/sagecut_oracle.cpp) against it,
//   * bench.py --impl reference can time the reference's CPU training step.
// Only tests/, __graft_entry__.smoke() and bench.py's reference leg load it.
//
// The training loop below (RefTrainer::step) is the body of
// train_cofree_impl (proj/include/sagecut/trainer.hpp:202-313) with the
// per-step intermediates kept; ref_train_cofree() calls the reference's own
// train_cofree (proj/src/trainer.cpp:119) so tests can check the two agree
// bit-for-bit.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "sagecut/checkpoint.hpp"
#include "sagecut/dropedge.hpp"
#include "sagecut/graph.hpp"
#include "sagecut/graph_io.hpp"
#include "sagecut/nn.hpp"
#include "sagecut/partition.hpp"
#include "sagecut/partition_io.hpp"
#include "sagecut/reweight.hpp"
#include "sagecut/rng.hpp"
#include "sagecut/synth.hpp"
#include "sagecut/trainer.hpp"

using namespace sagecut;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

std::vector<int> hidden_vec(const int* hidden, int layers) {
    return std::vector<int>(hidden, hidden + layers);
}

template <class Scalar>
void flatten(const SageModel<Scalar>& m, double* out) {
    std::size_t k = 0;
    m.for_each_matrix([&](const MatX<Scalar>& x) {
        for (Eigen::Index r = 0; r < x.rows(); ++r)
            for (Eigen::Index c = 0; c < x.cols(); ++c) out[k++] = static_cast<double>(x(r, c));
    });
}

template <class Scalar>
void unflatten(SageModel<Scalar>& m, const double* in) {
    std::size_t k = 0;
    m.for_each_matrix([&](MatX<Scalar>& x) {
        for (Eigen::Index r = 0; r < x.rows(); ++r)
            for (Eigen::Index c = 0; c < x.cols(); ++c) x(r, c) = static_cast<Scalar>(in[k++]);
    });
}

TrainConfig make_config(const int* hidden, int layers, double lr, int loss, int reweight,
                        int use_dropedge, int k, double ratio, std::uint64_t seed, int f32,
                        int workers, int epochs) {
    TrainConfig cfg;
    cfg.layers = layers;
    cfg.hidden = layers > 0 ? hidden_vec(hidden, layers) : std::vector<int>{1};
    cfg.epochs = epochs;
    cfg.learning_rate = lr;
    cfg.loss = loss == 0 ? LossKind::softmax_ce : LossKind::bce;
    cfg.reweight = reweight == 0 ? ReweightScheme::dar
                                 : (reweight == 1 ? ReweightScheme::vanilla_inv : ReweightScheme::none);
    cfg.use_dropedge = use_dropedge != 0;
    cfg.dropedge_k = k;
    cfg.drop_ratio = ratio;
    cfg.seed = seed;
    cfg.precision = f32 ? Precision::f32 : Precision::f64;
    cfg.workers = workers;
    return cfg;
}

// The per-epoch body of train_cofree_impl with intermediates retained.
struct TrainerBase {
    virtual ~TrainerBase() = default;
    virtual void step(int epoch, double* loss, double* gnorm) = 0;
    virtual void params(double* out) const = 0;
    virtual void set_params(const double* in) = 0;
    virtual void part_grads(int i, double* out) const = 0;
    virtual void gathered(double* out) const = 0;
    virtual void part_logits(int i, double* out) const = 0;
    virtual double part_loss(int i) const = 0;
    virtual int part_mask(int i) const = 0;
    virtual std::size_t param_count() const = 0;
    virtual void eval_splits(double* train, double* val, double* test) const = 0;
    virtual double time_part_step(int i, int epoch, int reps) = 0;
};

template <class Scalar>
struct RefTrainer final : TrainerBase {
    const Graph& g;
    const VertexCutPartition& part;
    TrainConfig config;
    double normalizer;
    std::vector<detail::PartitionInputs<Scalar>> inputs;
    SageModel<Scalar> model;
    AdamState<Scalar> adam;
    AdamConfig adam_cfg;
    std::vector<SageGrads<Scalar>> worker_grads;
    std::vector<double> worker_loss;
    std::vector<MatX<Scalar>> worker_logits;
    std::vector<int> worker_mask;
    SageGrads<Scalar> last_gathered;

    RefTrainer(const Graph& graph, const VertexCutPartition& p, const TrainConfig& cfg)
        : g(graph), part(p), config(cfg) {
        // trainer.hpp:205-243 verbatim in effect.
        validate_train_config(config);
        detail::require_trainable(g);
        if (config.loss == LossKind::softmax_ce && g.labels.empty())
            throw std::invalid_argument("softmax_ce requires multi-class labels");
        if (part.edge_assignment.size() != g.edges.size() || part.parts.empty())
            throw std::invalid_argument("train_cofree: partition does not match graph");
        normalizer = detail::train_node_count(g);
        const auto num_parts = static_cast<std::size_t>(part.num_parts);
        const NodeWeights scheme_weights = compute_weights(config.reweight, g, part);
        const Eigen::MatrixXd all_targets =
            config.loss == LossKind::bce ? label_targets(g) : Eigen::MatrixXd();
        inputs.resize(num_parts);
        for (std::size_t i = 0; i < num_parts; ++i) {
            const PartSubgraph& sub = part.parts[i];
            auto& in = inputs[i];
            const auto n_local = static_cast<Eigen::Index>(sub.nodes.size());
            in.features.resize(n_local, g.features.cols());
            if (config.loss == LossKind::bce) in.targets.resize(n_local, all_targets.cols());
            in.loss_weights.resize(sub.nodes.size());
            if (config.loss == LossKind::softmax_ce) in.class_ids.resize(sub.nodes.size());
            for (std::size_t j = 0; j < sub.nodes.size(); ++j) {
                const NodeId v = sub.nodes[j];
                in.features.row(static_cast<Eigen::Index>(j)) =
                    g.features.row(v).template cast<Scalar>();
                if (config.loss == LossKind::bce)
                    in.targets.row(static_cast<Eigen::Index>(j)) =
                        all_targets.row(v).template cast<Scalar>();
                else
                    in.class_ids[j] = g.labels[static_cast<std::size_t>(v)];
                in.loss_weights[j] =
                    g.train_mask[static_cast<std::size_t>(v)] ? scheme_weights.per_part[i][j] : 0.0;
            }
            if (config.use_dropedge) in.dropedge = partition_mask_set(sub, config, i);
        }
        model = make_sage_model<Scalar>(g.features.cols(), resolved_hidden_dims(config),
                                        g.num_classes, config.seed);
        adam = make_adam_state(model);
        adam_cfg = AdamConfig{config.learning_rate, 0.9, 0.999, 1e-8};
        worker_grads.resize(num_parts);
        worker_loss.assign(num_parts, 0.0);
        worker_logits.resize(num_parts);
        worker_mask.assign(num_parts, -1);
    }

    std::span<const std::uint8_t> mask_for(std::size_t i, int epoch, int* chosen) const {
        std::span<const std::uint8_t> mask;
        *chosen = -1;
        if (config.use_dropedge) {
            Rng select_rng(substream(config.seed, "dropedge.select", i, static_cast<std::uint64_t>(epoch)));
            const int k = select_mask(inputs[i].dropedge, select_rng);
            *chosen = k;
            mask = inputs[i].dropedge.masks[static_cast<std::size_t>(k)];
        }
        return mask;
    }

    void run_worker(std::size_t i, int epoch) {
        const PartSubgraph& sub = part.parts[i];
        const auto& in = inputs[i];
        int chosen;
        const auto mask = mask_for(i, epoch, &chosen);
        const AdjacencyView adj = sub.adjacency();
        auto fwd = sage_forward(model, adj, in.features, mask);
        auto lg = detail::loss_dispatch(config.loss, fwd.logits, in.class_ids, in.targets,
                                        in.loss_weights, normalizer);
        worker_grads[i] = sage_backward(model, fwd.cache, adj, lg.grad, mask);
        worker_loss[i] = lg.loss;
        worker_logits[i] = fwd.logits;
        worker_mask[i] = chosen;
    }

    void step(int epoch, double* loss, double* gnorm) override {
        const auto num_parts = static_cast<std::size_t>(part.num_parts);
        const int pool_size = std::min<int>(config.workers, static_cast<int>(num_parts));
        if (pool_size <= 1) {
            for (std::size_t i = 0; i < num_parts; ++i) run_worker(i, epoch);
        } else {
            std::vector<std::thread> pool;
            std::vector<std::exception_ptr> errors(static_cast<std::size_t>(pool_size));
            for (int w = 0; w < pool_size; ++w)
                pool.emplace_back([&, w] {
                    try {
                        for (std::size_t i = static_cast<std::size_t>(w); i < num_parts;
                             i += static_cast<std::size_t>(pool_size))
                            run_worker(i, epoch);
                    } catch (...) {
                        errors[static_cast<std::size_t>(w)] = std::current_exception();
                    }
                });
            for (auto& t : pool) t.join();
            for (const auto& err : errors)
                if (err) std::rethrow_exception(err);
        }
        last_gathered = gather_gradients(worker_grads);
        *gnorm = grad_norm(last_gathered);
        double total = 0.0;
        for (const double l : worker_loss) total += l;
        *loss = total;
        adam_step(model, last_gathered, adam, adam_cfg);
    }

    double time_part_step(int i, int epoch, int reps) override {
        // One partition's forward + loss + backward (the per-worker body), timed.
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r) run_worker(static_cast<std::size_t>(i), epoch);
        const auto t1 = std::chrono::steady_clock::now();
        return std::chrono::duration<double>(t1 - t0).count() / reps;
    }

    void params(double* out) const override { flatten(model, out); }
    void set_params(const double* in) override { unflatten(model, in); }
    void part_grads(int i, double* out) const override { flatten(worker_grads[static_cast<std::size_t>(i)], out); }
    void gathered(double* out) const override { flatten(last_gathered, out); }
    void part_logits(int i, double* out) const override {
        const auto& l = worker_logits[static_cast<std::size_t>(i)];
        std::size_t k = 0;
        for (Eigen::Index r = 0; r < l.rows(); ++r)
            for (Eigen::Index c = 0; c < l.cols(); ++c) out[k++] = static_cast<double>(l(r, c));
    }
    double part_loss(int i) const override { return worker_loss[static_cast<std::size_t>(i)]; }
    int part_mask(int i) const override { return worker_mask[static_cast<std::size_t>(i)]; }
    std::size_t param_count() const override { return model.param_count(); }
    void eval_splits(double* tr, double* va, double* te) const override {
        const auto s = detail::evaluate_splits(model, g);
        *tr = s.train;
        *va = s.val;
        *te = s.test;
    }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_blas_active() { return Eigen::shim::blas_active() ? 1 : 0; }

// ---- RNG (proj/include/sagecut/rng.hpp) -------------------------------------
std::uint64_t ref_mix64(std::uint64_t x) { return mix64(x); }
std::uint64_t ref_substream(std::uint64_t seed, const char* tag, int nidx, std::uint64_t a,
                            std::uint64_t b) {
    if (nidx == 0) return substream(seed, tag);
    if (nidx == 1) return substream(seed, tag, a);
    return substream(seed, tag, a, b);
}
void ref_rng_draws(std::uint64_t seed, int kind, std::uint64_t arg, std::int64_t n, std::uint64_t* out_u,
                   double* out_d) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < n; ++i) {
        if (kind == 0) out_u[i] = rng.next_u64();
        else if (kind == 1) out_u[i] = rng.next_below(arg);
        else if (kind == 2) out_d[i] = rng.next_double();
        else out_d[i] = rng.next_gaussian();
    }
}

// ---- Graphs -------------------------------------------------------------------
void* ref_graph_build(std::int32_t n, const std::int32_t* uv, std::int64_t m) {
    Graph* out = nullptr;
    if (guard([&] {
            std::vector<Edge> raw(static_cast<std::size_t>(m));
            for (std::int64_t e = 0; e < m; ++e) raw[static_cast<std::size_t>(e)] = Edge{uv[2 * e], uv[2 * e + 1]};
            auto [g, rep] = build_graph(n, std::move(raw));
            out = new Graph(std::move(g));
        }))
        return nullptr;
    return out;
}
void* ref_graph_load(const char* path) {
    Graph* out = nullptr;
    if (guard([&] {
            auto [g, rep] = load_graph(path);
            out = new Graph(std::move(g));
        }))
        return nullptr;
    return out;
}
void* ref_graph_sbm(std::int32_t n, int classes, double p_in, double p_out, int d, double noise,
                    std::uint64_t seed) {
    Graph* out = nullptr;
    if (guard([&] { out = new Graph(gen_homophilic_sbm(SbmSpec{n, classes, p_in, p_out, d, noise, seed})); }))
        return nullptr;
    return out;
}
void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }
std::int32_t ref_graph_num_nodes(void* g) { return static_cast<Graph*>(g)->num_nodes; }
std::int64_t ref_graph_num_edges(void* g) { return static_cast<std::int64_t>(static_cast<Graph*>(g)->edges.size()); }
int ref_graph_feature_dim(void* g) { return static_cast<int>(static_cast<Graph*>(g)->features.cols()); }
int ref_graph_num_classes(void* g) { return static_cast<Graph*>(g)->num_classes; }
void ref_graph_edges(void* gp, std::int32_t* uv) {
    auto* g = static_cast<Graph*>(gp);
    for (std::size_t e = 0; e < g->edges.size(); ++e) {
        uv[2 * e] = g->edges[e].u;
        uv[2 * e + 1] = g->edges[e].v;
    }
}
void ref_graph_csr(void* gp, std::int32_t* offsets, std::int32_t* nbrs, std::int32_t* eids, std::int32_t* deg) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(offsets, g->adj_offsets.data(), g->adj_offsets.size() * 4);
    std::memcpy(nbrs, g->adj_neighbors.data(), g->adj_neighbors.size() * 4);
    std::memcpy(eids, g->adj_edge_ids.data(), g->adj_edge_ids.size() * 4);
    std::memcpy(deg, g->degrees.data(), g->degrees.size() * 4);
}
void ref_graph_features(void* gp, double* out) {  // row-major n x d
    auto* g = static_cast<Graph*>(gp);
    for (Eigen::Index r = 0; r < g->features.rows(); ++r)
        for (Eigen::Index c = 0; c < g->features.cols(); ++c)
            out[r * g->features.cols() + c] = g->features(r, c);
}
void ref_graph_labels(void* gp, std::int32_t* labels) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(labels, g->labels.data(), g->labels.size() * 4);
}
void ref_graph_masks(void* gp, std::uint8_t* train, std::uint8_t* val, std::uint8_t* test) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(train, g->train_mask.data(), g->train_mask.size());
    std::memcpy(val, g->val_mask.data(), g->val_mask.size());
    std::memcpy(test, g->test_mask.data(), g->test_mask.size());
}
// Attach caller data (features as float32 row-major, like the CFM1 loader's
// float32 payload promoted to double, graph_io.cpp:82-110).
int ref_graph_set_data(void* gp, const float* features, int d, const std::int32_t* labels, int classes,
                       const std::uint8_t* train, const std::uint8_t* val, const std::uint8_t* test) {
    return guard([&] {
        auto* g = static_cast<Graph*>(gp);
        const auto n = static_cast<Eigen::Index>(g->num_nodes);
        g->features.resize(n, d);
        for (Eigen::Index r = 0; r < n; ++r)
            for (int c = 0; c < d; ++c) g->features(r, c) = static_cast<double>(features[r * d + c]);
        g->labels.assign(labels, labels + n);
        g->num_classes = classes;
        g->train_mask.assign(train, train + n);
        g->val_mask.assign(val, val + n);
        g->test_mask.assign(test, test + n);
    });
}

// A multi-label target matrix (n x C of 0/1 floats), as load_labels' multi-label
// branch leaves the graph (graph_io.cpp:206-229): multilabels set, labels cleared.
int ref_graph_set_multilabels(void* gp, const float* y, int classes) {
    return guard([&] {
        auto* g = static_cast<Graph*>(gp);
        const auto n = static_cast<Eigen::Index>(g->num_nodes);
        g->multilabels.resize(n, classes);
        for (Eigen::Index r = 0; r < n; ++r)
            for (int c = 0; c < classes; ++c) g->multilabels(r, c) = static_cast<double>(y[r * classes + c]);
        g->num_classes = classes;
        g->labels.clear();
    });
}

// The reference's evaluate (trainer.cpp:101-112) of a flat f64 model.
int ref_evaluate(void* gp, const double* theta, const int* hidden, int layers, const std::uint8_t* mask,
                 double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        auto model = make_sage_model<double>(g.features.cols(), hidden_vec(hidden, layers), g.num_classes, 0);
        unflatten(model, theta);
        *out = evaluate(model, g, std::span<const std::uint8_t>(mask, static_cast<std::size_t>(g.num_nodes)));
    });
}

// comm_volume (trainer.cpp:38-49): out = {floats_per_iteration, gradient_floats, embedding_floats}
int ref_comm_volume(int mode, int num_parts, std::uint64_t params, std::uint64_t layers, std::uint64_t hidden,
                    std::uint64_t halo, std::uint64_t* out) {
    return guard([&] {
        const CommReport r = comm_volume(mode == 0 ? CommMode::cofree : CommMode::halo_sync_model, num_parts,
                                         params, layers, hidden, halo);
        out[0] = r.floats_per_iteration;
        out[1] = r.gradient_floats;
        out[2] = r.embedding_floats;
    });
}
int ref_expected_rf_random(int p, std::int64_t degree, double* out) {
    return guard([&] { *out = expected_rf_random(p, degree); });
}
int ref_imbalance_lower_bound(int p, std::int64_t max_degree, std::int64_t min_degree, double* out) {
    return guard([&] { *out = imbalance_lower_bound(p, max_degree, min_degree); });
}

// ---- Partitioning (proj/src/partition.cpp) ---------------------------------------
// algo: 0 random, 1 dbh, 2 ne, 3 edge-cut greedy -> ec2vc
void* ref_partition(void* gp, int algo, int p, std::uint64_t seed) {
    VertexCutPartition* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            if (algo == 0) out = new VertexCutPartition(partition_random(g, p, seed));
            else if (algo == 1) out = new VertexCutPartition(partition_dbh(g, p, seed));
            else if (algo == 2) out = new VertexCutPartition(partition_ne(g, p, seed));
            else out = new VertexCutPartition(edge_cut_to_vertex_cut(g, partition_edge_cut_greedy(g, p, seed), seed));
        }))
        return nullptr;
    return out;
}
void* ref_build_vertex_cut(void* gp, int p, const std::int32_t* assign) {
    VertexCutPartition* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            out = new VertexCutPartition(build_vertex_cut(g, p, std::vector<int>(assign, assign + g.edges.size())));
        }))
        return nullptr;
    return out;
}
void* ref_partition_ne(void* gp, int p, std::uint64_t seed, double slack, char* wbuf, std::int64_t cap) {
    VertexCutPartition* out = nullptr;
    if (guard([&] {
            out = new VertexCutPartition(partition_ne(*static_cast<Graph*>(gp), p, seed, slack));
            std::string j;
            for (const auto& x : out->warnings) j += (j.empty() ? "" : "\n") + x;
            if (wbuf && cap > 0) {
                std::strncpy(wbuf, j.c_str(), static_cast<std::size_t>(cap - 1));
                wbuf[cap - 1] = 0;
            }
        }))
        return nullptr;
    return out;
}
int ref_edge_cut_greedy(void* gp, int p, std::uint64_t seed, std::int32_t* node_assign) {
    return guard([&] {
        const EdgeCutPartition ec = partition_edge_cut_greedy(*static_cast<Graph*>(gp), p, seed);
        for (std::size_t v = 0; v < ec.node_assignment.size(); ++v) node_assign[v] = ec.node_assignment[v];
    });
}
int ref_edge_cut_stats(void* gp, int p, const std::int32_t* na, std::int64_t* kept_counts, std::int64_t* num_cut,
                       std::int64_t* halo_counts, std::int32_t* cut_edges, std::int32_t* halo_nodes) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        const EdgeCutPartition ec =
            edge_cut_from_assignment(g, p, std::vector<int>(na, na + static_cast<std::size_t>(g.num_nodes)));
        *num_cut = static_cast<std::int64_t>(ec.cut_edges.size());
        for (int i = 0; i < p; ++i) {
            kept_counts[i] = static_cast<std::int64_t>(ec.kept_edges[static_cast<std::size_t>(i)].size());
            halo_counts[i] = static_cast<std::int64_t>(ec.halo_sets[static_cast<std::size_t>(i)].size());
        }
        if (cut_edges)
            for (std::size_t k = 0; k < ec.cut_edges.size(); ++k) cut_edges[k] = static_cast<std::int32_t>(ec.cut_edges[k]);
        if (halo_nodes)
            for (const auto& h : ec.halo_sets)
                for (const auto v : h) *halo_nodes++ = static_cast<std::int32_t>(v);
    });
}
void* ref_edge_cut_to_vertex_cut(void* gp, int p, const std::int32_t* na, std::uint64_t seed) {
    VertexCutPartition* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            const EdgeCutPartition ec =
                edge_cut_from_assignment(g, p, std::vector<int>(na, na + static_cast<std::size_t>(g.num_nodes)));
            out = new VertexCutPartition(edge_cut_to_vertex_cut(g, ec, seed));
        }))
        return nullptr;
    return out;
}
void ref_partition_free(void* pp) { delete static_cast<VertexCutPartition*>(pp); }
void ref_partition_assignment(void* pp, std::int32_t* out) {
    auto* vc = static_cast<VertexCutPartition*>(pp);
    for (std::size_t e = 0; e < vc->edge_assignment.size(); ++e) out[e] = vc->edge_assignment[e];
}
void ref_part_sizes(void* pp, int i, std::int64_t* n_local, std::int64_t* n_edges) {
    auto& sub = static_cast<VertexCutPartition*>(pp)->parts[static_cast<std::size_t>(i)];
    *n_local = static_cast<std::int64_t>(sub.nodes.size());
    *n_edges = static_cast<std::int64_t>(sub.edges.size());
}
void ref_part_arrays(void* pp, int i, std::int32_t* nodes, std::int32_t* edges_uv, std::int32_t* edge_gids,
                     std::int32_t* local_deg, std::int32_t* offsets, std::int32_t* nbrs, std::int32_t* eids,
                     std::int32_t* g2l) {
    auto& sub = static_cast<VertexCutPartition*>(pp)->parts[static_cast<std::size_t>(i)];
    std::memcpy(nodes, sub.nodes.data(), sub.nodes.size() * 4);
    for (std::size_t e = 0; e < sub.edges.size(); ++e) {
        edges_uv[2 * e] = sub.edges[e].u;
        edges_uv[2 * e + 1] = sub.edges[e].v;
    }
    std::memcpy(edge_gids, sub.edge_global_ids.data(), sub.edge_global_ids.size() * 4);
    std::memcpy(local_deg, sub.local_degrees.data(), sub.local_degrees.size() * 4);
    std::memcpy(offsets, sub.adj_offsets.data(), sub.adj_offsets.size() * 4);
    std::memcpy(nbrs, sub.adj_neighbors.data(), sub.adj_neighbors.size() * 4);
    std::memcpy(eids, sub.adj_edge_ids.data(), sub.adj_edge_ids.size() * 4);
    if (g2l) std::memcpy(g2l, sub.global_to_local.data(), sub.global_to_local.size() * 4);
}
int ref_replication_stats(void* pp, void* gp, std::int32_t* per_node_rf, double* rf, double* edge_balance,
                          double* node_balance, std::int64_t* duplicated) {
    return guard([&] {
        const auto s = replication_stats(*static_cast<VertexCutPartition*>(pp), *static_cast<Graph*>(gp));
        for (std::size_t v = 0; v < s.per_node_rf.size(); ++v) per_node_rf[v] = s.per_node_rf[v];
        *rf = s.rf;
        *edge_balance = s.edge_balance;
        *node_balance = s.node_balance;
        *duplicated = s.duplicated_nodes;
    });
}

// ---- Reweighting / DropEdge (proj/src/reweight.cpp, dropedge.cpp) ---------------
// scheme: 0 dar, 1 vanilla_inv, 2 none. Output concatenated over parts.
int ref_weights(void* gp, void* pp, int scheme, double* out) {
    return guard([&] {
        const auto s = scheme == 0 ? ReweightScheme::dar : (scheme == 1 ? ReweightScheme::vanilla_inv : ReweightScheme::none);
        const auto w = compute_weights(s, *static_cast<Graph*>(gp), *static_cast<VertexCutPartition*>(pp));
        std::size_t k = 0;
        for (const auto& part : w.per_part)
            for (const double x : part) out[k++] = x;
    });
}
int ref_precompute_masks(std::int64_t num_edges, int k, double ratio, std::uint64_t seed, std::uint8_t* out) {
    return guard([&] {
        const auto set = precompute_masks(static_cast<std::size_t>(num_edges), k, ratio, seed);
        for (int i = 0; i < k; ++i)
            std::memcpy(out + static_cast<std::size_t>(i) * static_cast<std::size_t>(num_edges),
                        set.masks[static_cast<std::size_t>(i)].data(), static_cast<std::size_t>(num_edges));
    });
}
int ref_select_mask(std::uint64_t seed, std::uint64_t part, std::uint64_t epoch, int k) {
    DropEdgeMaskSet set;
    set.num_masks = k;
    Rng rng(substream(seed, "dropedge.select", part, epoch));
    return select_mask(set, rng);
}

// ---- Model init (nn.hpp:73-102) --------------------------------------------------
std::int64_t ref_init_params(int in_dim, const int* hidden, int layers, int classes, std::uint64_t seed,
                             int f32, double* out) {
    std::int64_t count = -1;
    guard([&] {
        if (f32) {
            const auto m = make_sage_model<float>(in_dim, hidden_vec(hidden, layers), classes, seed);
            if (out) flatten(m, out);
            count = static_cast<std::int64_t>(m.param_count());
        } else {
            const auto m = make_sage_model<double>(in_dim, hidden_vec(hidden, layers), classes, seed);
            if (out) flatten(m, out);
            count = static_cast<std::int64_t>(m.param_count());
        }
    });
    return count;
}

// ---- File formats (partition_io.cpp, checkpoint.cpp, trainer.cpp:126-140) --------
// scheme: -1 no weights, else dar / vanilla_inv / none
int ref_save_partition(void* gp, void* pp, const char* path, int scheme) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        const auto& part = *static_cast<VertexCutPartition*>(pp);
        if (scheme < 0) {
            save_partition(part, path);
        } else {
            const NodeWeights w = compute_weights(static_cast<ReweightScheme>(scheme), g, part);
            save_partition(part, path, &w);
        }
    });
}
void* ref_load_partition(void* gp, const char* path) {
    VertexCutPartition* out = nullptr;
    if (guard([&] { out = new VertexCutPartition(load_partition(path, *static_cast<Graph*>(gp))); })) return nullptr;
    return out;
}
int ref_save_edge_cut(void* gp, int p, const std::int32_t* na, const char* path) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        save_edge_cut(edge_cut_from_assignment(g, p, std::vector<int>(na, na + g.num_nodes)), path);
    });
}
// theta: flat f32 parameters (for_each_matrix order) -> SageModel<double> (TrainResult::model) -> CFCK
int ref_save_checkpoint_f32(const float* theta, int in_dim, const int* hidden, int layers, int classes,
                            const char* path) {
    return guard([&] {
        auto m = make_sage_model<double>(in_dim, hidden_vec(hidden, layers), classes, 0);
        std::vector<double> v(theta, theta + m.param_count());
        unflatten(m, v.data());
        save_checkpoint(m, path);
    });
}
// flat f64 parameters of a CFCK file (count returned; -1 on error)
std::int64_t ref_load_checkpoint(const char* path, double* out) {
    std::int64_t count = -1;
    guard([&] {
        const auto m = load_checkpoint(path);
        if (out) flatten(m, out);
        count = static_cast<std::int64_t>(m.param_count());
    });
    return count;
}
// rows: n x 6 doubles (train_loss, train_metric, val_metric, test_metric, grad_norm, comm_floats) + epochs
int ref_write_metrics(const char* path, int n, const int* epochs, const double* rows) {
    return guard([&] {
        std::vector<EpochMetrics> v(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            v[i].epoch = epochs[i];
            v[i].train_loss = rows[6 * i];
            v[i].train_metric = rows[6 * i + 1];
            v[i].val_metric = rows[6 * i + 2];
            v[i].test_metric = rows[6 * i + 3];
            v[i].grad_norm = rows[6 * i + 4];
            v[i].comm_floats = static_cast<std::uint64_t>(rows[6 * i + 5]);
        }
        write_metrics_jsonl(v, path);
    });
}

// ---- Trainer -------------------------------------------------------------------
void* ref_trainer_new(void* gp, void* pp, const int* hidden, int layers, double lr, int loss, int reweight,
                      int use_dropedge, int k, double ratio, std::uint64_t seed, int f32, int workers) {
    TrainerBase* out = nullptr;
    if (guard([&] {
            const auto cfg = make_config(hidden, layers, lr, loss, reweight, use_dropedge, k, ratio, seed, f32,
                                         workers, 1);
            const Graph& g = *static_cast<Graph*>(gp);
            const auto& part = *static_cast<VertexCutPartition*>(pp);
            if (f32) out = new RefTrainer<float>(g, part, cfg);
            else out = new RefTrainer<double>(g, part, cfg);
        }))
        return nullptr;
    return out;
}
void ref_trainer_free(void* t) { delete static_cast<TrainerBase*>(t); }
int ref_trainer_step(void* t, int epoch, double* loss, double* gnorm) {
    return guard([&] { static_cast<TrainerBase*>(t)->step(epoch, loss, gnorm); });
}
std::int64_t ref_trainer_param_count(void* t) { return static_cast<std::int64_t>(static_cast<TrainerBase*>(t)->param_count()); }
void ref_trainer_params(void* t, double* out) { static_cast<TrainerBase*>(t)->params(out); }
void ref_trainer_set_params(void* t, const double* in) { static_cast<TrainerBase*>(t)->set_params(in); }
void ref_trainer_part_grads(void* t, int i, double* out) { static_cast<TrainerBase*>(t)->part_grads(i, out); }
void ref_trainer_gathered(void* t, double* out) { static_cast<TrainerBase*>(t)->gathered(out); }
void ref_trainer_part_logits(void* t, int i, double* out) { static_cast<TrainerBase*>(t)->part_logits(i, out); }
double ref_trainer_part_loss(void* t, int i) { return static_cast<TrainerBase*>(t)->part_loss(i); }
int ref_trainer_part_mask(void* t, int i) { return static_cast<TrainerBase*>(t)->part_mask(i); }
void ref_trainer_eval(void* t, double* tr, double* va, double* te) { static_cast<TrainerBase*>(t)->eval_splits(tr, va, te); }
double ref_trainer_time_part_step(void* t, int i, int epoch, int reps) {
    double s = -1.0;
    guard([&] { s = static_cast<TrainerBase*>(t)->time_part_step(i, epoch, reps); });
    return s;
}

// The reference's own end-to-end entry point (trainer.cpp:119), for
// cross-checking the step-wise harness above.
// the reference's train_full_graph (trainer.cpp:114-117 -> trainer.hpp:164-200)
int ref_train_full_graph(void* gp, const int* hidden, int layers, double lr, int loss, std::uint64_t seed, int f32,
                         int epochs, double* final_params, double* losses, double* gnorms, double* metrics) {
    return guard([&] {
        const auto cfg = make_config(hidden, layers, lr, loss, 0, 0, 10, 0.5, seed, f32, 1, epochs);
        const auto res = train_full_graph(*static_cast<Graph*>(gp), cfg);
        flatten(res.model, final_params);
        for (std::size_t e = 0; e < res.metrics.size(); ++e) {
            losses[e] = res.metrics[e].train_loss;
            gnorms[e] = res.metrics[e].grad_norm;
            metrics[3 * e] = res.metrics[e].train_metric;
            metrics[3 * e + 1] = res.metrics[e].val_metric;
            metrics[3 * e + 2] = res.metrics[e].test_metric;
        }
    });
}

int ref_train_cofree(void* gp, void* pp, const int* hidden, int layers, double lr, int loss, int reweight,
                     int use_dropedge, int k, double ratio, std::uint64_t seed, int f32, int workers, int epochs,
                     double* final_params, double* losses, double* gnorms, double* metrics /* epochs x 3 */,
                     std::uint64_t* audit /* epochs gradient floats + embedding floats, optional */) {
    return guard([&] {
        const auto cfg = make_config(hidden, layers, lr, loss, reweight, use_dropedge, k, ratio, seed, f32,
                                     workers, epochs);
        const auto res = train_cofree(*static_cast<Graph*>(gp), *static_cast<VertexCutPartition*>(pp), cfg);
        flatten(res.model, final_params);
        if (audit) {
            for (std::size_t e = 0; e < res.audit.gradient_floats_per_epoch.size(); ++e)
                audit[e] = res.audit.gradient_floats_per_epoch[e];
            audit[res.audit.gradient_floats_per_epoch.size()] = res.audit.embedding_floats;
        }
        for (std::size_t e = 0; e < res.metrics.size(); ++e) {
            losses[e] = res.metrics[e].train_loss;
            gnorms[e] = res.metrics[e].grad_norm;
            if (metrics) {
                metrics[3 * e] = res.metrics[e].train_metric;
                metrics[3 * e + 1] = res.metrics[e].val_metric;
                metrics[3 * e + 2] = res.metrics[e].test_metric;
            }
        }
    });
}

}  // extern "C"
