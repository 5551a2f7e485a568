// C++ facade smoke/parity driver (include/sagecut_b200.hpp over libsagecut_cuda.so).
// Reads a graph + data + config from argv[1] (text), runs the reference-shaped
// API (build_graph, partition_random, replication_stats, compute_weights,
// precompute_masks, train_cofree) and prints results for tests/test_gpu_facade.py.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <stdexcept>

#include "sagecut_b200.hpp"

namespace sb = sagecut_b200;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: facade_main input.txt\n");
        return 2;
    }
    try {
        std::ifstream in(argv[1]);
        int n, d, C, p, epochs;
        long long m;
        unsigned long long seed;
        in >> n >> m >> d >> C >> p >> seed >> epochs;
        std::vector<sb::Edge> raw(static_cast<std::size_t>(m));
        for (auto& e : raw) in >> e.u >> e.v;
        std::vector<float> feats(static_cast<std::size_t>(n) * d);
        for (auto& x : feats) in >> x;
        std::vector<int> labels(n), tr8(n), va8(n), te8(n);
        for (auto& x : labels) in >> x;
        std::vector<std::uint8_t> tr(n), va(n), te(n);
        for (int i = 0; i < n; ++i) { in >> tr8[i]; tr[i] = static_cast<std::uint8_t>(tr8[i]); }
        for (int i = 0; i < n; ++i) { in >> va8[i]; va[i] = static_cast<std::uint8_t>(va8[i]); }
        for (int i = 0; i < n; ++i) { in >> te8[i]; te[i] = static_cast<std::uint8_t>(te8[i]); }

        sb::Context ctx(0);
        auto [g, rep] = sb::build_graph(ctx, n, raw);
        g.set_data(feats, d, labels, C, tr, va, te);
        auto part = sb::partition_random(g, p, 3);
        const auto stats = sb::replication_stats(part, g);
        const auto w = sb::compute_weights(sb::ReweightScheme::dar, g, part);
        const auto masks = sb::precompute_masks(ctx, part.part(0).edges.size(), 3, 0.5, 17);

        std::printf("edges %zu\nrf %.17g\ndup %lld\n", g.num_edges(), stats.rf, (long long)stats.duplicated_nodes);
        std::printf("assign");
        for (int a : part.edge_assignment()) std::printf(" %d", a);
        std::printf("\nw0");
        for (double x : w.per_part[0]) std::printf(" %.17g", x);
        std::printf("\nmask0");
        for (auto b : masks.masks[0]) std::printf(" %d", int(b));
        std::printf("\n");

        // greedy partitioners (partition.cpp:116-308) through the facade
        const auto ne = sb::partition_ne(g, p, 0, 1.0);
        std::printf("ne");
        for (int a : ne.edge_assignment()) std::printf(" %d", a);
        std::printf("\nne_warnings %zu\n", ne.warnings().size());
        const auto ec = sb::partition_edge_cut_greedy(g, p, 5);
        std::printf("ec_nodes");
        for (int a : ec.node_assignment) std::printf(" %d", a);
        std::printf("\nec_cut %zu\nec_halo %zu\nec2vc", ec.cut_edges.size(), ec.total_halo());
        for (int a : sb::edge_cut_to_vertex_cut(g, ec, 5).edge_assignment()) std::printf(" %d", a);
        std::printf("\n");

        sb::TrainConfig cfg;
        cfg.layers = 2;
        cfg.hidden = {16};
        cfg.epochs = epochs;
        cfg.learning_rate = 0.01;
        cfg.use_dropedge = true;
        cfg.seed = seed;
        const auto res = sb::train_cofree(g, part, cfg);
        // file formats through the facade (partition_io.cpp, checkpoint.cpp, trainer.cpp:126-140)
        if (argc > 2) {
            const std::string dir = argv[2];
            const sb::ReweightScheme dar = sb::ReweightScheme::dar;
            sb::save_partition(part, dir + "/part.json", &dar);
            const auto back = sb::load_partition(dir + "/part.json", g);
            std::printf("reload_same %d\n", back.edge_assignment() == part.edge_assignment() ? 1 : 0);
            sb::save_checkpoint(res, dir + "/model.ckpt");
            std::printf("ckpt_same %d\n", sb::load_checkpoint(dir + "/model.ckpt") == res.model ? 1 : 0);
            sb::write_metrics_jsonl(res.metrics, dir + "/metrics.jsonl");
        }
        // evaluate / CommAudit / analytic helpers (trainer.cpp:38-49, 101-112; partition.cpp:344-362)
        std::printf("eval_test %.17g\n", sb::evaluate(res, g, te));
        std::printf("audit");
        for (auto f : res.audit.gradient_floats_per_epoch) std::printf(" %llu", (unsigned long long)f);
        std::printf(" %llu\n", (unsigned long long)res.audit.embedding_floats);
        const auto cv = sb::comm_volume(sb::CommMode::halo_sync_model, p, res.model.size(), 2, 16, 100);
        std::printf("comm %llu %llu %llu\n", (unsigned long long)cv.floats_per_iteration,
                    (unsigned long long)cv.gradient_floats, (unsigned long long)cv.embedding_floats);
        std::printf("erf %.17g\nilb %.17g\n", sb::expected_rf_random(p, 13), sb::imbalance_lower_bound(p, 9, 2));
        std::printf("loss");
        for (const auto& e : res.metrics) std::printf(" %.17g", e.train_loss);
        std::printf("\nparams");
        for (float x : res.model) std::printf(" %.9g", x);
        std::printf("\n");
        // the reference's error taxonomy survives the boundary
        try {
            sb::partition_random(g, 0, 1);
            std::printf("error none\n");
        } catch (const std::invalid_argument& e) {
            std::printf("error invalid_argument %s\n", e.what());
        }
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "facade_main: %s\n", e.what());
        return 1;
    }
}
