// partition_seq.cu — the reference's greedy partitioners, output-exact
// (proj/src/partition.cpp:116-308):
//
//  * partition_ne (:116-201). The reference rescans its whole boundary for the
//    (unassigned-degree, id)-minimum on every pick, O(picks x |boundary|)
//    (~6 h at 62M edges). Scores only ever decrease and the boundary is reset
//    per part, so a binary min-heap of (score << 32 | id) keys with lazy
//    deletion (an entry is live iff the node is still in the boundary and its
//    score is current) yields the same pick sequence in O(E log E). Greedy
//    expansion is inherently sequential, so it runs on the host over the
//    device graph's CSR (one D2H); the vertex cut is then built on the device.
//  * partition_edge_cut_greedy (:233-278). BFS region growing; a restart takes
//    the r-th unassigned node in ascending id order (r = next_below(#free)),
//    found with a Fenwick order-statistic tree instead of the reference's O(n)
//    rebuild of the free list.
//  * edge_cut_from_assignment (:203-231) and edge_cut_to_vertex_cut (:280-308)
//    on the device: a cut edge not touching the anchor consumes the next
//    next_bool() draw of Rng(substream(seed, "partition.ec2vc")) in ascending
//    edge order, so its draw index is an exclusive scan of that predicate and
//    every edge resolves independently (counter-based stream, rng.hpp:20-30).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

#include "internal.hpp"

namespace sc {

namespace {
constexpr int kBlock = 256;

struct HostCsr {
    std::vector<int64_t> off;
    std::vector<int32_t> nbrs, eids, deg;
};

HostCsr copy_csr(sc_graph* g) {
    HostCsr h;
    cudaStream_t s = g->ctx->stream;
    h.off.resize(size_t(g->n) + 1);
    h.nbrs.resize(size_t(2 * g->m));
    h.eids.resize(size_t(2 * g->m));
    h.deg.resize(size_t(g->n));
    d2h(h.off.data(), g->offsets.get(), h.off.size(), s);
    if (g->m) {
        d2h(h.nbrs.data(), g->nbrs.get(), h.nbrs.size(), s);
        d2h(h.eids.data(), g->eids.get(), h.eids.size(), s);
    }
    if (g->n) d2h(h.deg.data(), g->degrees.get(), h.deg.size(), s);
    SC_CUDA(cudaStreamSynchronize(s));
    return h;
}

// Fenwick tree over "node v is unassigned" with k-th-one search.
struct Fenwick {
    std::vector<int32_t> t;
    int32_t n = 0, top = 1;
    explicit Fenwick(int32_t n_) : t(size_t(n_) + 1, 0), n(n_) {
        for (int32_t i = 1; i <= n; ++i) {  // all ones, O(n) build
            t[i] += 1;
            const int32_t j = i + (i & -i);
            if (j <= n) t[j] += t[i];
        }
        while (top * 2 <= n) top *= 2;
    }
    void clear(int32_t v) {
        for (int32_t i = v + 1; i <= n; i += i & -i) --t[i];
    }
    int32_t kth(int64_t k) const {  // 0-based rank among the set -> node id
        int32_t pos = 0;
        for (int32_t step = top; step > 0; step >>= 1)
            if (pos + step <= n && t[pos + step] <= k) {
                pos += step;
                k -= t[pos];
            }
        return pos;
    }
};

__global__ void ec_flags_kernel(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                const int32_t* __restrict__ na, int32_t* first_cut) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
        if (na[eu[e]] != na[ev[e]]) atomicMin(first_cut, static_cast<int32_t>(e));
}

// draw[e] = 1 for a cut edge away from the anchor (it consumes one next_bool draw)
__global__ void ec_draw_flags_kernel(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                     const int32_t* __restrict__ na, const int32_t* first_cut,
                                     int32_t* __restrict__ draw) {
    const int32_t f = *first_cut;
    const int32_t anchor = f < m ? eu[f] : -1;  // canonical u < v: min endpoint of the first cut edge
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        const int32_t u = eu[e], v = ev[e];
        draw[e] = (na[u] != na[v] && u != anchor && v != anchor) ? 1 : 0;
    }
}

__global__ void ec_assign_kernel(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                 const int32_t* __restrict__ na, const int32_t* first_cut,
                                 const int64_t* __restrict__ draw_idx, uint64_t stream, int32_t* __restrict__ assign) {
    const int32_t f = *first_cut;
    const int32_t anchor = f < m ? eu[f] : -1;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        const int32_t u = eu[e], v = ev[e];
        const int32_t pu = na[u], pv = na[v];
        int32_t a;
        if (pu == pv) a = pu;                               // kept edge stays in its part
        else if (u == anchor || v == anchor) a = na[anchor];  // the anchor's cut edges stay home
        else a = (draw_u64(stream, static_cast<uint64_t>(draw_idx[e])) & 1u) ? pu : pv;  // next_bool
        assign[e] = a;
    }
}

__global__ void halo_keys_kernel(int64_t m, const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                 const int32_t* __restrict__ na, const int64_t* __restrict__ cut_pos,
                                 uint64_t* __restrict__ keys, int32_t* __restrict__ cut_edges,
                                 uint64_t* __restrict__ kept_keys, unsigned long long* kept_counts) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        const int32_t u = eu[e], v = ev[e];
        const int32_t pu = na[u], pv = na[v];
        if (pu == pv) {
            atomicAdd(kept_counts + pu, 1ull);
            kept_keys[e - cut_pos[e]] = (uint64_t(uint32_t(pu)) << 32) | uint32_t(e);  // kept_edges[pu] gets e
        } else {
            const int64_t k = cut_pos[e];
            cut_edges[k] = static_cast<int32_t>(e);
            keys[2 * k] = (uint64_t(uint32_t(pv)) << 32) | uint32_t(u);  // halo_sets[pv] gets u
            keys[2 * k + 1] = (uint64_t(uint32_t(pu)) << 32) | uint32_t(v);
        }
    }
}

__global__ void low_word_kernel(int64_t k, const uint64_t* __restrict__ keys, int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < k; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = static_cast<int32_t>(keys[i] & 0xffffffffu);
}

__global__ void halo_count_kernel(int64_t k, const uint64_t* __restrict__ keys, unsigned long long* halo_counts,
                                  int32_t* __restrict__ nodes) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < k; i += int64_t(gridDim.x) * blockDim.x) {
        atomicAdd(halo_counts + (keys[i] >> 32), 1ull);
        if (nodes) nodes[i] = static_cast<int32_t>(keys[i] & 0xffffffffu);
    }
}

struct IsCut {
    const int32_t *eu, *ev, *na;
    int64_t m;
    __device__ int64_t operator()(int64_t e) const { return e < m && na[eu[e]] != na[ev[e]] ? 1 : 0; }
};

void validate_node_assignment(sc_graph* g, int32_t p, const int32_t* na_host) {
    for (int32_t v = 0; v < g->n; ++v)
        if (na_host[v] < 0 || na_host[v] >= p) throw std::invalid_argument("node assignment references an invalid part");
}
}  // namespace

std::vector<int32_t> ne_assign_host(sc_graph* g, int32_t p, double slack, std::vector<std::string>& warnings) {
    const HostCsr h = copy_csr(g);
    const int64_t m = g->m;
    const int32_t n = g->n;
    const int64_t target = (m + p - 1) / p;
    std::vector<int32_t> assign(size_t(m), p - 1);
    std::vector<uint8_t> done(size_t(m), 0), in_b(size_t(n), 0);
    std::vector<int32_t> deg(h.deg);
    std::priority_queue<uint64_t, std::vector<uint64_t>, std::greater<uint64_t>> heap;
    auto key = [](int32_t score, int32_t v) { return (uint64_t(uint32_t(score)) << 32) | uint32_t(v); };
    int64_t left = m;
    int32_t lowest = 0;
    for (int part = 0; part + 1 < p && left > 0; ++part) {
        heap = decltype(heap)();
        std::fill(in_b.begin(), in_b.end(), 0);
        int64_t filled = 0;
        while (filled < target && left > 0) {
            int32_t pick = -1;
            while (!heap.empty()) {  // (score, id)-minimum live boundary entry (:143-157)
                const uint64_t k = heap.top();
                const int32_t v = int32_t(k & 0xffffffffu), sc = int32_t(k >> 32);
                if (!in_b[v] || deg[v] != sc) {  // stale: left the boundary, or score decreased since
                    heap.pop();
                    continue;
                }
                heap.pop();  // live entries always have score > 0: exhausted nodes only leave stale ones
                pick = v;
                break;
            }
            if (pick < 0) {  // :159-165
                while (lowest < n && deg[lowest] == 0) ++lowest;
                if (lowest >= n) break;
                pick = lowest;
            } else {
                in_b[pick] = 0;
            }
            for (int64_t k = h.off[pick]; k < h.off[pick + 1]; ++k) {  // :170-186
                const int32_t e = h.eids[k];
                if (done[e]) continue;
                done[e] = 1;
                assign[e] = part;
                ++filled;
                --left;
                const int32_t o = h.nbrs[k];
                --deg[pick];
                --deg[o];
                if (deg[o] > 0) {
                    if (!in_b[o]) in_b[o] = 1;
                    heap.push(key(deg[o], o));  // new member, or a boundary node whose score dropped
                }
            }
        }
        const auto limit = static_cast<size_t>(slack * static_cast<double>(target));  // :188-193
        if (static_cast<size_t>(filled) > limit)
            warnings.push_back("part " + std::to_string(part) + " overshoot: " + std::to_string(filled) +
                               " edges > slack limit " + std::to_string(limit));
    }
    return assign;
}

std::vector<int32_t> edge_cut_greedy_host(sc_graph* g, int32_t p, uint64_t seed) {
    const HostCsr h = copy_csr(g);
    const int32_t n = g->n;
    HostRng rng(substream(seed, "partition.edge_cut"));
    std::vector<int32_t> a(size_t(n), -1);
    Fenwick freeset(n);
    const int64_t base = n / p, rem = n % p;
    int64_t assigned = 0;
    std::vector<int32_t> q;
    for (int part = 0; part < p && assigned < n; ++part) {
        const int64_t target = base + (part < rem ? 1 : 0);
        int64_t size = 0;
        q.clear();  // the frontier is per part (:246)
        size_t head = 0;
        auto take = [&](int32_t v) {
            a[v] = part;
            freeset.clear(v);
            ++size;
            ++assigned;
            q.push_back(v);
        };
        while (size < target && assigned < n) {
            if (head == q.size()) {  // seeded restart on an unvisited node (:248-258)
                const int64_t r = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n - assigned)));
                take(freeset.kth(r));
                continue;
            }
            const int32_t v = q[head++];
            for (int64_t k = h.off[v]; k < h.off[v + 1]; ++k) {
                if (size >= target) break;
                const int32_t u = h.nbrs[k];
                if (a[u] >= 0) continue;
                take(u);
            }
        }
    }
    return a;
}

void ec2vc_assign_device(sc_graph* g, int32_t p, const int32_t* na_host, uint64_t seed, int32_t* assign_dev) {
    validate_node_assignment(g, p, na_host);
    const int64_t m = g->m;
    if (m == 0) return;
    cudaStream_t s = g->ctx->stream;
    DevBuf<int32_t> na(std::max<int64_t>(g->n, 1)), first(1), draw(m);
    DevBuf<int64_t> idx(m);
    h2d(na.get(), na_host, g->n, s);
    const int32_t none = static_cast<int32_t>(std::min<int64_t>(m, INT32_MAX));
    h2d(first.get(), &none, 1, s);
    const unsigned grid = grid_for(m, kBlock);
    ec_flags_kernel<<<grid, kBlock, 0, s>>>(m, g->eu.get(), g->ev.get(), na.get(), first.get());
    SC_LAUNCH_CHECK();
    ec_draw_flags_kernel<<<grid, kBlock, 0, s>>>(m, g->eu.get(), g->ev.get(), na.get(), first.get(), draw.get());
    SC_LAUNCH_CHECK();
    size_t tmp = 0;
    SC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, draw.get(), idx.get(), m, s));
    SC_CUDA(cub::DeviceScan::ExclusiveSum(g->ctx->temp(tmp), tmp, draw.get(), idx.get(), m, s));
    ec_assign_kernel<<<grid, kBlock, 0, s>>>(m, g->eu.get(), g->ev.get(), na.get(), first.get(), idx.get(),
                                             substream(seed, "partition.ec2vc"), assign_dev);
    SC_LAUNCH_CHECK();
    count_launch(4);
}

void edge_cut_stats_device(sc_graph* g, int32_t p, const int32_t* na_host, int64_t* kept_counts, int64_t* num_cut,
                           int64_t* halo_counts, int32_t* kept_edges_host, int32_t* cut_edges_host,
                           int32_t* halo_nodes_host) {
    validate_node_assignment(g, p, na_host);
    const int64_t m = g->m;
    cudaStream_t s = g->ctx->stream;
    DevBuf<int32_t> na(std::max<int64_t>(g->n, 1));
    DevBuf<unsigned long long> counts(2 * size_t(p));
    SC_CUDA(cudaMemsetAsync(counts.get(), 0, counts.bytes(), s));
    h2d(na.get(), na_host, g->n, s);
    int64_t ncut = 0;
    DevBuf<int64_t> pos(std::max<int64_t>(m, 1) + 1);
    if (m > 0) {
        IsCut f{g->eu.get(), g->ev.get(), na.get(), m};
        cub::CountingInputIterator<int64_t> it(0);
        cub::TransformInputIterator<int64_t, IsCut, cub::CountingInputIterator<int64_t>> flags(it, f);
        size_t tmp = 0;
        SC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flags, pos.get(), m + 1, s));
        SC_CUDA(cub::DeviceScan::ExclusiveSum(g->ctx->temp(tmp), tmp, flags, pos.get(), m + 1, s));
        count_launch(2);
        d2h(&ncut, pos.get() + m, 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
    }
    DevBuf<uint64_t> keys(std::max<int64_t>(2 * ncut, 1)), sorted(std::max<int64_t>(2 * ncut, 1));
    DevBuf<int32_t> cuts(std::max<int64_t>(ncut, 1)), nodes(std::max<int64_t>(2 * ncut, 1));
    const int64_t nkept = m - ncut;
    DevBuf<uint64_t> kkeys(std::max<int64_t>(nkept, 1));
    if (m > 0) {
        halo_keys_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(m, g->eu.get(), g->ev.get(), na.get(), pos.get(),
                                                                keys.get(), cuts.get(), kkeys.get(), counts.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    DevBuf<int32_t> kept(std::max<int64_t>(nkept, 1));
    if (kept_edges_host && nkept > 0) {  // kept_edges: part-major, ascending edge id (stable by construction)
        DevBuf<uint64_t> ksorted(nkept);
        size_t tmp = 0;
        SC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, kkeys.get(), ksorted.get(), nkept, 0, 64, s));
        SC_CUDA(cub::DeviceRadixSort::SortKeys(g->ctx->temp(tmp), tmp, kkeys.get(), ksorted.get(), nkept, 0, 64, s));
        low_word_kernel<<<grid_for(nkept, kBlock), kBlock, 0, s>>>(nkept, ksorted.get(), kept.get());
        SC_LAUNCH_CHECK();
        count_launch(2);
        d2h(kept_edges_host, kept.get(), nkept, s);
        SC_CUDA(cudaStreamSynchronize(s));
    }
    int64_t uniq = 0;
    if (ncut > 0) {  // halo sets: sort (part, node) keys, unique
        size_t tmp = 0;
        SC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.get(), sorted.get(), 2 * ncut, 0, 64, s));
        SC_CUDA(cub::DeviceRadixSort::SortKeys(g->ctx->temp(tmp), tmp, keys.get(), sorted.get(), 2 * ncut, 0, 64, s));
        DevBuf<int64_t> nu(1);
        tmp = 0;
        SC_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, sorted.get(), keys.get(), nu.get(), 2 * ncut, s));
        SC_CUDA(cub::DeviceSelect::Unique(g->ctx->temp(tmp), tmp, sorted.get(), keys.get(), nu.get(), 2 * ncut, s));
        d2h(&uniq, nu.get(), 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
        halo_count_kernel<<<grid_for(uniq, kBlock), kBlock, 0, s>>>(uniq, keys.get(), counts.get() + p, nodes.get());
        SC_LAUNCH_CHECK();
        count_launch(3);
    }
    std::vector<unsigned long long> hc(2 * size_t(p));
    d2h(hc.data(), counts.get(), hc.size(), s);
    if (cut_edges_host && ncut) d2h(cut_edges_host, cuts.get(), ncut, s);
    if (halo_nodes_host && uniq) d2h(halo_nodes_host, nodes.get(), uniq, s);  // part-major, ascending
    SC_CUDA(cudaStreamSynchronize(s));
    *num_cut = ncut;
    for (int32_t i = 0; i < p; ++i) {
        if (kept_counts) kept_counts[i] = static_cast<int64_t>(hc[i]);
        if (halo_counts) halo_counts[i] = static_cast<int64_t>(hc[p + i]);
    }
}

}  // namespace sc
