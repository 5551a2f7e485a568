// io.hpp — host-side writers/readers of the reference's file formats (io.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sc {

struct HostMatrix {  // one SageModel matrix, row-major f64
    uint64_t rows = 0, cols = 0;
    std::vector<double> v;
};

struct EpochRow {  // EpochMetrics (trainer.hpp:38-46)
    int epoch = 0;
    double train_loss = 0, train_metric = 0, val_metric = 0, test_metric = 0, grad_norm = 0;
    uint64_t comm_floats = 0;
};

void write_partition_json(const std::string& path, int32_t num_parts, const std::vector<int32_t>& assignment,
                          const std::vector<std::vector<int32_t>>& nodes,
                          const std::vector<std::vector<double>>* weights, const char* scheme);
void read_partition_json(const std::string& path, int32_t& num_parts, std::vector<int32_t>& assignment,
                         std::vector<std::vector<int32_t>>& nodes);
void write_edge_cut_json(const std::string& path, int32_t num_parts, const std::vector<int32_t>& node_assignment,
                         const std::vector<int32_t>& cut_edges, const std::vector<std::vector<int32_t>>& halo_sets);
void write_checkpoint(const std::string& path, const std::vector<HostMatrix>& mats);
std::vector<HostMatrix> read_checkpoint(const std::string& path);
void write_metrics_jsonl(const std::string& path, const std::vector<EpochRow>& rows);

}  // namespace sc
