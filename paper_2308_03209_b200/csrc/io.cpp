// io.cpp — the reference's file formats, byte-compatible:
//   * partition JSON  (proj/src/partition_io.cpp:12-29 save, :31-56 load, :58-68 edge cut)
//   * CFCK checkpoint (proj/src/checkpoint.cpp:44-84): "CFCK", u64 layer count, then per layer
//     message and update, then the head; each as u64 rows, u64 cols, row-major f64, little-endian
//   * metrics JSONL   (proj/src/trainer.cpp:126-140)
// Host-only C++ (no CUDA): capi.cu moves the device data and calls these. JSON goes through
// nlohmann::json, the library the reference writes with, so dump() output matches byte for byte.
#include "io.hpp"

#include <cstring>
#include <fstream>
#include <json.hpp>
#include <stdexcept>

namespace sc {

using nlohmann::json;

void write_partition_json(const std::string& path, int32_t num_parts, const std::vector<int32_t>& assignment,
                          const std::vector<std::vector<int32_t>>& nodes,
                          const std::vector<std::vector<double>>* weights, const char* scheme) {
    json doc;
    doc["num_parts"] = num_parts;
    doc["edge_assignment"] = assignment;
    json parts = json::array();
    for (size_t i = 0; i < nodes.size(); ++i) {
        json entry{{"nodes", nodes[i]}};
        if (weights) entry["weights"] = (*weights)[i];
        parts.push_back(std::move(entry));
    }
    doc["parts"] = std::move(parts);
    if (weights) doc["weight_scheme"] = scheme;
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    out << doc.dump(2) << '\n';
}

void read_partition_json(const std::string& path, int32_t& num_parts, std::vector<int32_t>& assignment,
                         std::vector<std::vector<int32_t>>& nodes) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open partition file: " + path);
    json doc;
    in >> doc;
    num_parts = doc.at("num_parts").get<int>();
    assignment = doc.at("edge_assignment").get<std::vector<int32_t>>();
    nodes.clear();
    for (const auto& p : doc.at("parts")) nodes.push_back(p.at("nodes").get<std::vector<int32_t>>());
}

void write_edge_cut_json(const std::string& path, int32_t num_parts, const std::vector<int32_t>& node_assignment,
                         const std::vector<int32_t>& cut_edges, const std::vector<std::vector<int32_t>>& halo_sets) {
    json doc;
    doc["num_parts"] = num_parts;
    doc["node_assignment"] = node_assignment;
    doc["cut_edges"] = cut_edges;
    doc["halo_sets"] = halo_sets;
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    out << doc.dump(2) << '\n';
}

namespace {
void write_u64(std::ostream& out, uint64_t v) {
    unsigned char b[8];
    for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
    out.write(reinterpret_cast<const char*>(b), 8);
}
uint64_t read_u64(std::istream& in) {
    unsigned char b[8];
    in.read(reinterpret_cast<char*>(b), 8);
    if (!in) throw std::runtime_error("checkpoint: truncated header");
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
}
}  // namespace

void write_checkpoint(const std::string& path, const std::vector<HostMatrix>& mats) {
    if (mats.empty() || mats.size() % 2 != 1) throw std::logic_error("write_checkpoint: expects 2L + 1 matrices");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    out.write("CFCK", 4);
    write_u64(out, (mats.size() - 1) / 2);
    for (const HostMatrix& m : mats) {
        write_u64(out, m.rows);
        write_u64(out, m.cols);
        out.write(reinterpret_cast<const char*>(m.v.data()), static_cast<std::streamsize>(m.v.size() * sizeof(double)));
    }
    if (!out) throw std::runtime_error("write failed: " + path);
}

std::vector<HostMatrix> read_checkpoint(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open checkpoint: " + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "CFCK", 4) != 0)
        throw std::runtime_error(path + ": not a checkpoint file (bad magic)");
    in.seekg(0, std::ios::end);
    const uint64_t file_bytes = static_cast<uint64_t>(in.tellg());
    in.seekg(4, std::ios::beg);
    const uint64_t layers = read_u64(in);
    // Every matrix costs at least its 16-byte header, so a corrupt count or shape is rejected
    // before anything is allocated from it.
    if (layers > file_bytes / 32) throw std::runtime_error("checkpoint: truncated header");
    std::vector<HostMatrix> mats;
    for (uint64_t k = 0; k < 2 * layers + 1; ++k) {
        HostMatrix m;
        m.rows = read_u64(in);
        m.cols = read_u64(in);
        const uint64_t left = file_bytes - static_cast<uint64_t>(in.tellg());
        if (m.cols != 0 && m.rows > left / sizeof(double) / m.cols)
            throw std::runtime_error("checkpoint: truncated matrix data");
        m.v.resize(static_cast<size_t>(m.rows * m.cols));
        in.read(reinterpret_cast<char*>(m.v.data()), static_cast<std::streamsize>(m.v.size() * sizeof(double)));
        if (!in) throw std::runtime_error("checkpoint: truncated matrix data");
        mats.push_back(std::move(m));
    }
    return mats;
}

void write_metrics_jsonl(const std::string& path, const std::vector<EpochRow>& rows) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    for (const EpochRow& m : rows) {
        json row;
        row["epoch"] = m.epoch;
        row["train_loss"] = m.train_loss;
        row["train_metric"] = m.train_metric;
        row["val_metric"] = m.val_metric;
        row["test_metric"] = m.test_metric;
        row["grad_norm"] = m.grad_norm;
        row["comm_floats"] = m.comm_floats;
        out << row.dump() << '\n';
    }
}

}  // namespace sc
