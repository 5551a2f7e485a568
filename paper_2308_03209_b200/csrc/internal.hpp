// internal.hpp — device-side state behind the opaque handles of sagecut_cuda.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace sc {

// RAII device allocation.
template <class T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void alloc(size_t n) {
        release();
        if (n) SC_CUDA(cudaMalloc(&p_, n * sizeof(T)));
        n_ = n;
    }
    // Grow-only reallocation (contents not preserved).
    void ensure(size_t n) {
        if (n > n_) alloc(n);
    }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

template <class T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n) SC_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (n) SC_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

}  // namespace sc

struct sc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    sc::DevBuf<unsigned char> cub_tmp;  // CUB temp storage (grow-only)
    sc::DevBuf<unsigned char> scratch;  // misc scratch (grow-only)
    int64_t launches = 0;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    void* temp(size_t bytes) {
        cub_tmp.ensure(bytes < 256 ? 256 : bytes);
        return cub_tmp.get();
    }
};

// Canonical undirected graph + symmetric CSR (graph.hpp:53-80).
struct sc_graph {
    sc_ctx* ctx = nullptr;
    int32_t n = 0;
    int64_t m = 0;
    sc::DevBuf<int32_t> eu, ev;        // canonical edges, SoA, u < v, sorted
    sc::DevBuf<int32_t> degrees;       // n
    sc::DevBuf<int64_t> offsets;       // n + 1
    sc::DevBuf<int32_t> nbrs, eids;    // 2m
    // Graph data (features/labels/masks)
    int32_t dim = 0, num_classes = 0;
    sc::DevBuf<float> features;        // n x dim
    sc::DevBuf<float> feat_amax;       // max |features| (tensor-core operand scale)
    uint64_t feat_version = 0;         // bumped whenever the features change
    sc::DevBuf<int32_t> labels;        // n (multi-class ids)
    sc::DevBuf<uint8_t> targets;       // n x num_classes 0/1 (multi-label graphs, graph.hpp:64)
    bool multilabel = false;           // Graph::is_multilabel (graph.hpp:74)
    sc::DevBuf<uint8_t> train, val, test;  // n
    int64_t train_count = 0;
    // Partition ownership (sc_graph_set_part_ownership): vertex cuts built on this
    // graph materialise only parts i with i % own_world == own_rank (the ones this
    // rank trains); the others keep their sizes only. own_world 1 = every part.
    int32_t own_rank = 0, own_world = 1;
    bool owns(int32_t part) const { return own_world <= 1 || part % own_world == own_rank; }
    // Staged next features (sc_trainer_stage_features): H2D on copy_stream into
    // features_next while the current step runs; committed (buffers swapped)
    // at the start of the next step. released: recorded on the compute stream
    // at each commit, after the last use of the buffer that becomes _next.
    sc::DevBuf<float> features_next;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t staged_ev = nullptr, released_ev = nullptr;
    bool staged = false, released_recorded = false;
    ~sc_graph();
};

// One PartSubgraph (partition.hpp:14-31), device resident.
struct PartDev {
    int64_t n_local = 0, m_local = 0;
    bool held = true;                       // arrays materialised on this rank (sc_graph_set_part_ownership)
    sc::DevBuf<int32_t> nodes;              // global ids ascending
    sc::DevBuf<int32_t> lu, lv;             // local endpoints, local-edge order
    sc::DevBuf<int32_t> edge_gids;          // global edge id per local edge
    sc::DevBuf<int32_t> local_deg;          // n_local
    sc::DevBuf<int64_t> offsets;            // n_local + 1
    sc::DevBuf<int32_t> nbrs, eids;         // 2 m_local (eids index local edges)
};

struct sc_vcut {
    sc_graph* g = nullptr;
    int32_t p = 0;
    sc::DevBuf<int32_t> assign;        // m
    int32_t own_rank = 0, own_world = 1;  // the graph's ownership when this cut was built
    const PartDev& held(int32_t i) const {
        if (!parts[i].held)
            throw std::invalid_argument("partition " + std::to_string(i) + " is not held on this rank");
        return parts[i];
    }
    sc::DevBuf<int32_t> per_node_rf;   // n
    std::vector<PartDev> parts;
    std::vector<std::string> warnings; // VertexCutPartition::warnings (partition_ne overshoot reports)
};

namespace sc {
// graph.cu
void build_csr(sc_ctx* ctx, int64_t n, int64_t m, const int32_t* u, const int32_t* v, int64_t* offsets,
               int32_t* nbrs, int32_t* eids, int32_t* degrees_out /* may be null */);
std::unique_ptr<sc_graph> build_graph_device(sc_ctx* ctx, int32_t n, const int32_t* raw_uv_dev, int64_t m_raw,
                                             int64_t* self_loops, int64_t* dups);
std::unique_ptr<sc_vcut> build_vertex_cut_device(sc_graph* g, int32_t p, DevBuf<int32_t>&& assign);
void assign_random(sc_graph* g, int32_t p, uint64_t seed, int32_t* assign);
void assign_dbh(sc_graph* g, int32_t p, uint64_t seed, int32_t* assign);
void compute_weights_device(sc_vcut* vc, int scheme, int32_t part, double* out_dev);
void part_g2l_device(const sc_vcut* vc, int32_t part, int32_t* out_dev);  // global_to_local (n, -1 absent)
// partition_seq.cu (partition.cpp:116-308)
std::vector<int32_t> ne_assign_host(sc_graph* g, int32_t p, double slack, std::vector<std::string>& warnings);
std::vector<int32_t> edge_cut_greedy_host(sc_graph* g, int32_t p, uint64_t seed);
void ec2vc_assign_device(sc_graph* g, int32_t p, const int32_t* node_assign_host, uint64_t seed, int32_t* assign_dev);
void edge_cut_stats_device(sc_graph* g, int32_t p, const int32_t* node_assign_host, int64_t* kept_counts,
                           int64_t* num_cut, int64_t* halo_counts, int32_t* kept_edges_host, int32_t* cut_edges_host,
                           int32_t* halo_nodes_host);
// dropedge.cu
void precompute_masks_device(sc_ctx* ctx, int64_t m, int32_t k, double ratio, uint64_t seed, uint8_t* out_dev);
// init
void init_params_device(sc_ctx* ctx, int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t classes,
                        uint64_t seed, float* out_dev);
}  // namespace sc
