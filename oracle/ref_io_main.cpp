// oracle/_ref/ref_io_main — TEST INFRASTRUCTURE ONLY.
//
// The reference's own dataset loaders / writers (proj/src/graph_io.cpp, compiled unmodified
// into oracle/_ref) behind a tiny command line, so tests/test_graph_io_cpu.py can compare the
// product's readers (paper_2308_03209_b200/csrc/graph_io.cpp) with them in a separate process
// (the reference's iostream parsers are kept out of processes that have numpy loaded).
//
//   ref_io_main graph PATH NUM_NODES(-1) STRICT        -> "ok n m self_loops dups" + edge lines
//   ref_io_main features PATH N [OUT_CSV OUT_BIN]      -> "ok rows cols" + %.9g values (+ re-saved)
//   ref_io_main labels PATH N [OUT]                    -> "ok multilabel classes" + values
//   ref_io_main masks PATH N [OUT]                     -> "ok" + three 0/1 lines
//   ref_io_main save-edges PATH OUT                    -> load_graph then save_edge_list
// Errors: "error <type> <what>" and exit code 0 (the message is the result).
#include <cstdio>
#include <stdexcept>
#include <string>

#include "sagecut/graph.hpp"
#include "sagecut/graph_io.hpp"

using namespace sagecut;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string cmd = argv[1], path = argv[2];
    try {
        if (cmd == "graph") {
            LoadOptions opt;
            const long n = argc > 3 ? std::stol(argv[3]) : -1;
            if (n >= 0) opt.num_nodes = static_cast<NodeId>(n);
            opt.strict = argc > 4 && std::string(argv[4]) == "1";
            auto [g, rep] = load_graph(path, opt);
            std::printf("ok %d %zu %lld %lld\n", g.num_nodes, g.edges.size(),
                        static_cast<long long>(rep.dropped_self_loops), static_cast<long long>(rep.merged_duplicate_edges));
            for (const Edge& e : g.edges) std::printf("%d %d\n", e.u, e.v);
        } else if (cmd == "save-edges") {
            auto [g, rep] = load_graph(path);
            save_edge_list(g, argv[3]);
            std::printf("ok\n");
        } else if (cmd == "features") {
            const auto m = load_features(path, static_cast<NodeId>(std::stol(argv[3])));
            std::printf("ok %ld %ld\n", static_cast<long>(m.rows()), static_cast<long>(m.cols()));
            for (Eigen::Index r = 0; r < m.rows(); ++r)
                for (Eigen::Index c = 0; c < m.cols(); ++c) std::printf("%.9g\n", static_cast<double>(static_cast<float>(m(r, c))));
            if (argc > 5) {
                save_features_csv(m, argv[4]);
                save_features_binary(m, argv[5]);
            }
        } else if (cmd == "labels" || cmd == "masks") {
            Graph g;
            g.num_nodes = static_cast<NodeId>(std::stol(argv[3]));
            if (cmd == "labels") {
                load_labels(path, g);
                std::printf("ok %d %d\n", g.is_multilabel() ? 1 : 0, g.num_classes);
                if (g.is_multilabel()) {
                    for (Eigen::Index r = 0; r < g.multilabels.rows(); ++r)
                        for (Eigen::Index c = 0; c < g.multilabels.cols(); ++c)
                            std::printf("%d\n", g.multilabels(r, c) != 0.0 ? 1 : 0);
                } else {
                    for (NodeId y : g.labels) std::printf("%d\n", y);
                }
                if (argc > 4) save_labels(g, argv[4]);
            } else {
                load_masks(path, g);
                std::printf("ok\n");
                for (const auto* m : {&g.train_mask, &g.val_mask, &g.test_mask}) {
                    for (auto x : *m) std::printf("%d", int(x));
                    std::printf("\n");
                }
                if (argc > 4) save_masks(g, argv[4]);
            }
        } else {
            return 2;
        }
    } catch (const std::invalid_argument& e) {
        std::printf("error invalid_argument %s\n", e.what());
    } catch (const std::runtime_error& e) {
        std::printf("error runtime_error %s\n", e.what());
    }
    return 0;
}
