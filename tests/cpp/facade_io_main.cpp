// C++ facade driver over the reference's dataset files: load_dataset (graph_io.cpp:41-296 via
// include/sagecut_b200.hpp) -> partition_random -> train_cofree -> evaluate, printing what
// tests/test_gpu_facade.py compares with the oracle.
//   facade_io_main EDGES FEATURES LABELS MASKS P EPOCHS LOSS(softmax_ce|bce)
#include <cstdio>
#include <string>

#include "sagecut_b200.hpp"

namespace sb = sagecut_b200;

int main(int argc, char** argv) {
    if (argc < 8) return 2;
    try {
        sb::Context ctx(0);
        auto [g, rep] = sb::load_dataset(ctx, argv[1], argv[2], argv[3], argv[4]);
        const int p = std::stoi(argv[5]), epochs = std::stoi(argv[6]);
        std::printf("graph %d %zu %lld %lld %d %d %d\n", g.num_nodes, g.num_edges(), (long long)rep.dropped_self_loops,
                    (long long)rep.merged_duplicate_edges, g.feature_dim, g.num_classes, g.is_multilabel() ? 1 : 0);
        const auto part = sb::partition_random(g, p, 3);
        sb::TrainConfig cfg;
        cfg.layers = 2;
        cfg.hidden = {16};
        cfg.epochs = epochs;
        cfg.use_dropedge = true;
        cfg.seed = 1;
        cfg.loss = std::string(argv[7]) == "bce" ? sb::LossKind::bce : sb::LossKind::softmax_ce;
        const auto res = sb::train_cofree(g, part, cfg);
        std::printf("loss");
        for (const auto& m : res.metrics) std::printf(" %.17g", m.train_loss);
        std::printf("\nmetrics");
        for (const auto& m : res.metrics) std::printf(" %.17g %.17g %.17g", m.train_metric, m.val_metric, m.test_metric);
        std::printf("\nparams");
        for (float x : res.model) std::printf(" %.9g", x);
        std::printf("\n");
        return 0;
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
}
