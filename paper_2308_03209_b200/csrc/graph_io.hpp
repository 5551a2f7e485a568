// graph_io.hpp — host readers / writers of the reference's dataset files (graph_io.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sc {

struct EdgeList {          // load_graph's parse (graph_io.cpp:41-80), before build_graph
    int32_t num_nodes = 0;
    std::vector<int32_t> uv;  // raw (u, v) pairs in file order
};
struct HostFeatures {      // load_features (graph_io.cpp:82-160), as float32
    int64_t rows = 0, cols = 0;
    std::vector<float> values;  // row-major
};
struct HostLabels {        // load_labels (graph_io.cpp:188-242)
    bool multilabel = false;
    int32_t num_classes = 0;
    std::vector<int32_t> labels;  // multi-class
    std::vector<float> targets;   // multi-label, n x num_classes
};

// num_nodes < 0: 1 + the largest id seen (LoadOptions::num_nodes unset)
EdgeList read_edge_list(const std::string& path, int32_t num_nodes);
HostFeatures read_features(const std::string& path, int32_t expected_nodes);
HostLabels read_labels(const std::string& path, int32_t num_nodes);
void read_masks(const std::string& path, int32_t num_nodes, std::vector<uint8_t>& train, std::vector<uint8_t>& val,
                std::vector<uint8_t>& test);

void write_edge_list(const std::string& path, const int32_t* u, const int32_t* v, int64_t m);
void write_features_csv(const std::string& path, const float* x, int64_t rows, int64_t cols);
void write_features_binary(const std::string& path, const float* x, int64_t rows, int64_t cols);
void write_labels(const std::string& path, int32_t n, const int32_t* labels, const float* targets, int32_t classes);
void write_masks(const std::string& path, int32_t n, const uint8_t* train, const uint8_t* val, const uint8_t* test);

}  // namespace sc
