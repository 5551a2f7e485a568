// sagecut_oracle.cpp — CPU restatement of the CoFree-GNN per-partition
// training step of the reference (`sagecut`, /root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY (see sagecut_oracle.h). Every function names the
// reference file:line it restates. It is deliberately plain: scalar loops,
// row-major flat arrays, the same Scalar for data as the reference's
// precision mode and the same f64 accumulators where the reference uses them.
#include "sagecut_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

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

using u64 = std::uint64_t;
using i32 = std::int32_t;
using i64 = std::int64_t;

// ---- rng.hpp:11-104 ------------------------------------------------------------
constexpr u64 kGamma = 0x9e3779b97f4a7c15ULL;
u64 mix64(u64 x) {  // rng.hpp:11-16
    x += kGamma;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
struct Rng {  // rng.hpp:20-80
    u64 s;
    bool has_spare = false;
    double spare = 0;
    explicit Rng(u64 seed) : s(seed) {}
    u64 next_u64() { return mix64((s += kGamma) - kGamma); }  // state += γ, then finalize
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_open_double() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
    u64 next_below(u64 n) {  // rng.hpp:43-49: reject r < 2^64 mod n
        const u64 threshold = (0 - n) % n;
        for (;;) {
            const u64 r = next_u64();
            if (r >= threshold) return r % n;
        }
    }
    double next_gaussian() {  // rng.hpp:52-63 Box-Muller with cached spare
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        const double u = next_open_double();
        const double v = next_double();
        const double r = std::sqrt(-2.0 * std::log(u));
        const double theta = 2.0 * 3.14159265358979323846 * v;
        spare = r * std::sin(theta);
        has_spare = true;
        return r * std::cos(theta);
    }
    bool next_bool() { return (next_u64() & 1u) != 0; }
    template <class T>
    void shuffle(std::vector<T>& xs) {  // rng.hpp:69-74 Fisher-Yates, i from n down to 2
        for (std::size_t i = xs.size(); i > 1; --i) {
            const auto j = static_cast<std::size_t>(next_below(i));
            std::swap(xs[i - 1], xs[j]);
        }
    }
};
u64 fnv1a64(const char* s) {  // rng.hpp:83-90
    u64 h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ULL;
    }
    return h;
}
u64 substream(u64 seed, const char* tag) { return mix64(seed ^ fnv1a64(tag)); }  // rng.hpp:94-96
u64 substream(u64 seed, const char* tag, u64 a) {                                 // rng.hpp:97-99
    return mix64(substream(seed, tag) ^ mix64(a + kGamma));
}
u64 substream(u64 seed, const char* tag, u64 a, u64 b) {  // rng.hpp:100-103
    return mix64(substream(seed, tag, a) ^ mix64(b + 0x2545f4914f6cdd1dULL));
}

// ---- graph.cpp:8-64 -------------------------------------------------------------
struct Graph {
    i32 n = 0;
    std::vector<std::pair<i32, i32>> edges;
    std::vector<i32> offsets, nbrs, eids, degrees;
    std::vector<double> features;  // n x d row-major
    int d = 0;
    std::vector<i32> labels;
    std::vector<double> multilabels;  // n x C of 0/1 (graph.hpp:64); empty when multi-class
    int num_classes = 0;
    std::vector<std::uint8_t> train, val, test;
    bool is_multilabel() const { return !multilabels.empty(); }  // graph.hpp:74
    bool has_labels() const { return !labels.empty() || is_multilabel(); }  // graph.hpp:72
};

Graph build_graph(i32 n, std::vector<std::pair<i32, i32>> raw) {
    if (n < 0) throw std::invalid_argument("build_graph: negative node count");
    std::vector<std::pair<i32, i32>> edges;
    edges.reserve(raw.size());
    for (auto e : raw) {
        if (e.first < 0 || e.second < 0 || e.first >= n || e.second >= n)
            throw std::invalid_argument("build_graph: edge endpoint out of range");
        if (e.first == e.second) continue;                      // drop self-loops
        if (e.first > e.second) std::swap(e.first, e.second);   // canonical u < v
        edges.push_back(e);
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    Graph g;
    g.n = n;
    g.edges = std::move(edges);
    g.degrees.assign(static_cast<std::size_t>(n), 0);
    for (auto& e : g.edges) {
        ++g.degrees[static_cast<std::size_t>(e.first)];
        ++g.degrees[static_cast<std::size_t>(e.second)];
    }
    g.offsets.assign(static_cast<std::size_t>(n) + 1, 0);
    for (i32 v = 0; v < n; ++v) g.offsets[v + 1] = g.offsets[v] + g.degrees[v];
    g.nbrs.resize(2 * g.edges.size());
    g.eids.resize(2 * g.edges.size());
    std::vector<i32> cur(g.offsets.begin(), g.offsets.end() - 1);
    for (std::size_t e = 0; e < g.edges.size(); ++e) {  // graph.cpp:47-55 cursor fill
        const auto [u, v] = g.edges[e];
        g.nbrs[cur[u]] = v;
        g.eids[cur[u]++] = static_cast<i32>(e);
        g.nbrs[cur[v]] = u;
        g.eids[cur[v]++] = static_cast<i32>(e);
    }
    return g;
}

// ---- synth.cpp:14-104 (fixture generator; O(n^2) exactly like the reference) ----
void attach_split_masks(Graph& g, u64 seed) {  // synth.cpp:14-34
    std::vector<i32> order(static_cast<std::size_t>(g.n));
    std::iota(order.begin(), order.end(), 0);
    Rng rng(substream(seed, "split"));
    rng.shuffle(order);
    const auto n = static_cast<std::size_t>(g.n);
    const std::size_t n_train = (n * 6) / 10, n_val = (n * 2) / 10;
    g.train.assign(n, 0);
    g.val.assign(n, 0);
    g.test.assign(n, 0);
    for (std::size_t i = 0; i < n; ++i) {
        const auto v = static_cast<std::size_t>(order[i]);
        if (i < n_train) g.train[v] = 1;
        else if (i < n_train + n_val) g.val[v] = 1;
        else g.test[v] = 1;
    }
}

Graph gen_homophilic_sbm(i32 n, int C, double p_in, double p_out, int feature_dim, double noise, u64 seed) {
    if (C < 1) throw std::invalid_argument("sbm: num_classes must be >= 1");
    if (n < C) throw std::invalid_argument("sbm: need at least one node per class");
    const int d = feature_dim > 0 ? feature_dim : C;
    if (d < C) throw std::invalid_argument("sbm: feature_dim must be >= num_classes");
    std::vector<i32> cls(static_cast<std::size_t>(n));
    for (i32 v = 0; v < n; ++v) cls[v] = v % C;
    Rng edge_rng(substream(seed, "sbm.edges"));
    std::vector<std::pair<i32, i32>> edges;
    for (i32 i = 0; i < n; ++i)
        for (i32 j = i + 1; j < n; ++j) {
            const double p = cls[i] == cls[j] ? p_in : p_out;
            if (edge_rng.next_double() < p) edges.emplace_back(i, j);
        }
    std::vector<i32> deg(static_cast<std::size_t>(n), 0);
    for (auto& e : edges) {
        ++deg[e.first];
        ++deg[e.second];
    }
    Rng rewire(substream(seed, "sbm.rewire"));  // synth.cpp:64-83
    for (i32 v = 0; v < n; ++v) {
        if (deg[v] > 0) continue;
        std::vector<i32> cand;
        for (i32 u = 0; u < n; ++u)
            if (u != v && cls[u] == cls[v]) cand.push_back(u);
        if (cand.empty())
            for (i32 u = 0; u < n; ++u)
                if (u != v) cand.push_back(u);
        const i32 u = cand[static_cast<std::size_t>(rewire.next_below(cand.size()))];
        edges.emplace_back(v, u);
        ++deg[v];
        ++deg[u];
    }
    Graph g = build_graph(n, std::move(edges));
    g.labels = cls;
    g.num_classes = C;
    g.d = d;
    Rng feat(substream(seed, "sbm.features"));  // synth.cpp:91-97
    g.features.assign(static_cast<std::size_t>(n) * d, 0.0);
    for (i32 v = 0; v < n; ++v) {
        g.features[static_cast<std::size_t>(v) * d + cls[v]] = 1.0;
        for (int c = 0; c < d; ++c) g.features[static_cast<std::size_t>(v) * d + c] += noise * feat.next_gaussian();
    }
    attach_split_masks(g, seed);
    return g;
}

// ---- partition.cpp:22-90, 92-114, 310-342 -------------------------------------
struct Part {
    std::vector<i32> nodes, g2l, local_deg, offsets, nbrs, eids, edge_gids;
    std::vector<std::pair<i32, i32>> edges;
};
struct VCut {
    int p = 0;
    std::vector<i32> assign;
    std::vector<Part> parts;
};

VCut build_vertex_cut(const Graph& g, int p, std::vector<i32> assign) {
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    if (assign.size() != g.edges.size())
        throw std::invalid_argument("edge assignment length does not match edge count");
    for (i32 a : assign)
        if (a < 0 || a >= p) throw std::invalid_argument("edge assignment references an invalid part");
    VCut vc;
    vc.p = p;
    vc.assign = std::move(assign);
    vc.parts.resize(static_cast<std::size_t>(p));
    std::vector<std::vector<std::uint8_t>> member(static_cast<std::size_t>(p),
                                                  std::vector<std::uint8_t>(static_cast<std::size_t>(g.n), 0));
    for (std::size_t e = 0; e < g.edges.size(); ++e) {  // :37-44 membership
        member[vc.assign[e]][g.edges[e].first] = 1;
        member[vc.assign[e]][g.edges[e].second] = 1;
    }
    int next = 0;  // :45-50 isolated nodes round-robin in ascending id
    for (i32 v = 0; v < g.n; ++v)
        if (g.degrees[v] == 0) {
            member[next][v] = 1;
            next = (next + 1) % p;
        }
    for (int i = 0; i < p; ++i) {  // :52-61 ascending-id local numbering
        Part& s = vc.parts[i];
        s.g2l.assign(static_cast<std::size_t>(g.n), -1);
        for (i32 v = 0; v < g.n; ++v)
            if (member[i][v]) {
                s.g2l[v] = static_cast<i32>(s.nodes.size());
                s.nodes.push_back(v);
            }
        s.local_deg.assign(s.nodes.size(), 0);
    }
    for (std::size_t e = 0; e < g.edges.size(); ++e) {  // :62-70 local edges, ascending global id
        Part& s = vc.parts[vc.assign[e]];
        const i32 lu = s.g2l[g.edges[e].first], lv = s.g2l[g.edges[e].second];
        s.edges.emplace_back(lu, lv);
        s.edge_gids.push_back(static_cast<i32>(e));
        ++s.local_deg[lu];
        ++s.local_deg[lv];
    }
    for (Part& s : vc.parts) {  // :72-88 local CSR by cursor in local-edge order
        const std::size_t nl = s.nodes.size();
        s.offsets.assign(nl + 1, 0);
        for (std::size_t v = 0; v < nl; ++v) s.offsets[v + 1] = s.offsets[v] + s.local_deg[v];
        s.nbrs.resize(2 * s.edges.size());
        s.eids.resize(2 * s.edges.size());
        std::vector<i32> cur(s.offsets.begin(), s.offsets.end() - 1);
        for (std::size_t e = 0; e < s.edges.size(); ++e) {
            const auto [u, v] = s.edges[e];
            s.nbrs[cur[u]] = v;
            s.eids[cur[u]++] = static_cast<i32>(e);
            s.nbrs[cur[v]] = u;
            s.eids[cur[v]++] = static_cast<i32>(e);
        }
    }
    return vc;
}

VCut partition_random(const Graph& g, int p, u64 seed) {  // :92-100
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    if (g.edges.empty()) throw std::invalid_argument("partition_random: graph has no edges");
    Rng rng(substream(seed, "partition.random"));
    std::vector<i32> a(g.edges.size());
    for (auto& x : a) x = static_cast<i32>(rng.next_below(static_cast<u64>(p)));
    return build_vertex_cut(g, p, std::move(a));
}

VCut partition_dbh(const Graph& g, int p, u64 seed) {  // :102-114
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    std::vector<i32> a(g.edges.size());
    for (std::size_t e = 0; e < g.edges.size(); ++e) {
        const auto [u, v] = g.edges[e];
        const i32 du = g.degrees[u], dv = g.degrees[v];
        const i32 pick = du != dv ? (du < dv ? u : v) : std::min(u, v);
        a[e] = static_cast<i32>(mix64(static_cast<u64>(pick) ^ seed) % static_cast<u64>(p));
    }
    return build_vertex_cut(g, p, std::move(a));
}

// partition.cpp:116-201 — greedy neighbour expansion, restated as the
// reference's literal boundary scan (O(picks x |boundary|); small graphs only).
VCut partition_ne(const Graph& g, int p, u64 /*seed*/, double slack, std::vector<std::string>& warnings) {
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    if (slack < 1.0) throw std::invalid_argument("partition_ne: balance_slack must be >= 1");
    const std::size_t m = g.edges.size();
    const std::size_t target = (m + static_cast<std::size_t>(p) - 1) / static_cast<std::size_t>(p);
    std::vector<i32> assign(m, p - 1);
    std::vector<std::uint8_t> done(m, 0), in_b(static_cast<std::size_t>(g.n), 0);
    std::vector<i32> deg(g.degrees);
    std::vector<i32> boundary;
    std::size_t left = m;
    i32 lowest = 0;
    for (int part = 0; part + 1 < p && left > 0; ++part) {
        boundary.clear();
        std::fill(in_b.begin(), in_b.end(), 0);
        std::size_t filled = 0;
        while (filled < target && left > 0) {
            i32 pick = -1, best = INT32_MAX;
            std::size_t keep = 0;
            for (std::size_t b = 0; b < boundary.size(); ++b) {  // :143-157
                const i32 v = boundary[b];
                if (deg[v] == 0) {
                    in_b[v] = 0;
                    continue;
                }
                boundary[keep++] = v;
                if (deg[v] < best || (deg[v] == best && v < pick)) {
                    best = deg[v];
                    pick = v;
                }
            }
            boundary.resize(keep);
            if (pick < 0) {  // :159-165 lowest-id node with unassigned edges
                while (lowest < g.n && deg[lowest] == 0) ++lowest;
                if (lowest >= g.n) break;
                pick = lowest;
            } else {
                in_b[pick] = 0;
                boundary.erase(std::find(boundary.begin(), boundary.end(), pick));
            }
            for (i32 k = g.offsets[pick]; k < g.offsets[pick + 1]; ++k) {  // :170-186
                const i32 e = g.eids[k];
                if (done[e]) continue;
                done[e] = 1;
                assign[e] = part;
                ++filled;
                --left;
                const i32 o = g.nbrs[k];
                --deg[pick];
                --deg[o];
                if (!in_b[o] && deg[o] > 0) {
                    in_b[o] = 1;
                    boundary.push_back(o);
                }
            }
        }
        const auto limit = static_cast<std::size_t>(slack * static_cast<double>(target));  // :188-193
        if (filled > limit)
            warnings.push_back("part " + std::to_string(part) + " overshoot: " + std::to_string(filled) +
                               " edges > slack limit " + std::to_string(limit));
    }
    return build_vertex_cut(g, p, std::move(assign));
}

// partition.cpp:203-231 — kept / cut edges and ascending halo sets.
struct ECut {
    int p = 0;
    std::vector<i32> node_assign;
    std::vector<std::vector<i32>> kept, halo;
    std::vector<i32> cut;
};
ECut edge_cut_from_assignment(const Graph& g, int p, std::vector<i32> na) {
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    if (na.size() != static_cast<std::size_t>(g.n))
        throw std::invalid_argument("node assignment length does not match node count");
    for (i32 a : na)
        if (a < 0 || a >= p) throw std::invalid_argument("node assignment references an invalid part");
    ECut ec;
    ec.p = p;
    ec.node_assign = std::move(na);
    ec.kept.resize(p);
    ec.halo.resize(p);
    for (std::size_t e = 0; e < g.edges.size(); ++e) {
        const auto [u, v] = g.edges[e];
        const i32 pu = ec.node_assign[u], pv = ec.node_assign[v];
        if (pu == pv) {
            ec.kept[pu].push_back(static_cast<i32>(e));
        } else {
            ec.cut.push_back(static_cast<i32>(e));
            ec.halo[pv].push_back(u);
            ec.halo[pu].push_back(v);
        }
    }
    for (auto& h : ec.halo) {
        std::sort(h.begin(), h.end());
        h.erase(std::unique(h.begin(), h.end()), h.end());
    }
    return ec;
}

// partition.cpp:233-278 — seeded BFS region growing (restart: uniform pick
// among the unassigned nodes in ascending id order).
ECut partition_edge_cut_greedy(const Graph& g, int p, u64 seed) {
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    const std::size_t n = static_cast<std::size_t>(g.n);
    Rng rng(substream(seed, "partition.edge_cut"));
    std::vector<i32> a(n, -1);
    const std::size_t base = n / static_cast<std::size_t>(p), rem = n % static_cast<std::size_t>(p);
    std::size_t assigned = 0;
    for (int part = 0; part < p && assigned < n; ++part) {
        const std::size_t target = base + (static_cast<std::size_t>(part) < rem ? 1 : 0);
        std::size_t size = 0;
        std::vector<i32> q;
        std::size_t head = 0;
        while (size < target && assigned < n) {
            if (head == q.size()) {
                std::vector<i32> free_nodes;
                for (i32 v = 0; v < g.n; ++v)
                    if (a[v] < 0) free_nodes.push_back(v);
                const i32 start = free_nodes[static_cast<std::size_t>(rng.next_below(free_nodes.size()))];
                a[start] = part;
                ++size;
                ++assigned;
                q.push_back(start);
                continue;
            }
            const i32 v = q[head++];
            for (i32 k = g.offsets[v]; k < g.offsets[v + 1]; ++k) {
                if (size >= target) break;
                const i32 u = g.nbrs[k];
                if (a[u] >= 0) continue;
                a[u] = part;
                ++size;
                ++assigned;
                q.push_back(u);
            }
        }
    }
    return edge_cut_from_assignment(g, p, std::move(a));
}

// partition.cpp:280-308
VCut edge_cut_to_vertex_cut(const Graph& g, const ECut& ec, u64 seed) {
    if (ec.node_assign.size() != static_cast<std::size_t>(g.n))
        throw std::invalid_argument("edge cut does not match graph");
    std::vector<i32> a(g.edges.size(), -1);
    for (int part = 0; part < ec.p; ++part)
        for (i32 e : ec.kept[part]) a[e] = part;
    i32 anchor = -1;
    if (!ec.cut.empty()) {
        const auto& first = g.edges[*std::min_element(ec.cut.begin(), ec.cut.end())];
        anchor = std::min(first.first, first.second);
    }
    Rng rng(substream(seed, "partition.ec2vc"));
    for (i32 e : ec.cut) {
        const auto [u, v] = g.edges[e];
        const i32 keep = (u == anchor || v == anchor) ? anchor : ((rng.next_u64() & 1u) ? u : v);
        a[e] = ec.node_assign[keep];
    }
    return build_vertex_cut(g, ec.p, std::move(a));
}

// ---- reweight.cpp:23-81 -----------------------------------------------------------
std::vector<std::vector<double>> weights(const Graph& g, const VCut& vc, int scheme) {
    std::vector<std::vector<double>> w;
    if (scheme == 0) {  // dar :23-45
        if (vc.assign.size() != g.edges.size())
            throw std::invalid_argument("dar_weights: partition does not match graph");
        for (const Part& s : vc.parts) {
            std::vector<double> x(s.nodes.size());
            for (std::size_t j = 0; j < s.nodes.size(); ++j) {
                const i32 gd = g.degrees[s.nodes[j]], ld = s.local_deg[j];
                if (gd == 0) {
                    if (ld != 0) throw std::logic_error("dar_weights: local edges on a degree-0 node");
                    x[j] = 1.0;
                } else {
                    x[j] = static_cast<double>(ld) / static_cast<double>(gd);
                }
            }
            w.push_back(std::move(x));
        }
    } else if (scheme == 1) {  // vanilla_inv :47-62
        std::vector<int> rf(static_cast<std::size_t>(g.n), 0);
        for (const Part& s : vc.parts)
            for (i32 v : s.nodes) ++rf[v];
        for (const Part& s : vc.parts) {
            std::vector<double> x(s.nodes.size());
            for (std::size_t j = 0; j < s.nodes.size(); ++j) x[j] = 1.0 / static_cast<double>(rf[s.nodes[j]]);
            w.push_back(std::move(x));
        }
    } else {  // unit :64-71
        for (const Part& s : vc.parts) w.emplace_back(s.nodes.size(), 1.0);
    }
    return w;
}

// ---- dropedge.cpp:9-37 --------------------------------------------------------------
std::vector<std::vector<std::uint8_t>> precompute_masks(std::size_t m, int k, double ratio, u64 seed) {
    if (k < 1) throw std::invalid_argument("precompute_masks: need at least one mask");
    if (ratio < 0.0 || ratio >= 1.0) throw std::invalid_argument("precompute_masks: ratio must lie in [0, 1)");
    const auto keep = static_cast<std::size_t>(std::ceil((1.0 - ratio) * static_cast<double>(m)));
    std::vector<std::vector<std::uint8_t>> out;
    std::vector<std::uint32_t> order(m);
    for (int i = 0; i < k; ++i) {
        std::iota(order.begin(), order.end(), 0u);
        Rng rng(substream(seed, "dropedge.mask", static_cast<u64>(i)));
        rng.shuffle(order);
        std::vector<std::uint8_t> mask(m, 0);
        for (std::size_t t = 0; t < keep; ++t) mask[order[t]] = 1;
        out.push_back(std::move(mask));
    }
    return out;
}

// ---- nn.hpp ----------------------------------------------------------------------------
template <class S>
struct Mat {  // row-major
    i64 r = 0, c = 0;
    std::vector<S> d;
    Mat() = default;
    Mat(i64 rr, i64 cc) : r(rr), c(cc), d(static_cast<std::size_t>(rr * cc), S(0)) {}
    S& operator()(i64 i, i64 j) { return d[static_cast<std::size_t>(i * c + j)]; }
    const S& operator()(i64 i, i64 j) const { return d[static_cast<std::size_t>(i * c + j)]; }
};

// C = A * B^T   (A: M x K, B: N x K)
template <class S>
Mat<S> mm_nt(const Mat<S>& A, const Mat<S>& B, i64 b_col0 = 0, i64 K = -1) {
    if (K < 0) K = B.c;
    Mat<S> C(A.r, B.r);
    for (i64 i = 0; i < A.r; ++i)
        for (i64 j = 0; j < B.r; ++j) {
            S acc(0);
            for (i64 k = 0; k < K; ++k) acc += A(i, k) * B(j, b_col0 + k);
            C(i, j) = acc;
        }
    return C;
}
// C = A * B[:, col0:col0+N]   (A: M x K, B: K x *)
template <class S>
Mat<S> mm_nn(const Mat<S>& A, const Mat<S>& B, i64 col0 = 0, i64 N = -1) {
    if (N < 0) N = B.c;
    Mat<S> C(A.r, N);
    for (i64 i = 0; i < A.r; ++i)
        for (i64 j = 0; j < N; ++j) {
            S acc(0);
            for (i64 k = 0; k < A.c; ++k) acc += A(i, k) * B(k, col0 + j);
            C(i, j) = acc;
        }
    return C;
}
// C = A^T * B   (A: K x M, B: K x N)
template <class S>
Mat<S> mm_tn(const Mat<S>& A, const Mat<S>& B) {
    Mat<S> C(A.c, B.c);
    for (i64 i = 0; i < A.c; ++i)
        for (i64 j = 0; j < B.c; ++j) {
            S acc(0);
            for (i64 k = 0; k < A.r; ++k) acc += A(k, i) * B(k, j);
            C(i, j) = acc;
        }
    return C;
}

template <class S>
struct Model {
    std::vector<Mat<S>> W, U;  // message (h x in), update (h x (h + in))
    Mat<S> head;               // C x embed
    std::size_t count() const {
        std::size_t n = head.d.size();
        for (std::size_t l = 0; l < W.size(); ++l) n += W[l].d.size() + U[l].d.size();
        return n;
    }
    template <class F>
    void each(F&& f) {
        for (std::size_t l = 0; l < W.size(); ++l) {
            f(W[l]);
            f(U[l]);
        }
        f(head);
    }
    template <class F>
    void each(F&& f) const {
        for (std::size_t l = 0; l < W.size(); ++l) {
            f(W[l]);
            f(U[l]);
        }
        f(head);
    }
    void to_flat(double* out) const {
        std::size_t k = 0;
        each([&](const Mat<S>& m) {
            for (auto x : m.d) out[k++] = static_cast<double>(x);
        });
    }
    void from_flat(const double* in) {
        std::size_t k = 0;
        each([&](Mat<S>& m) {
            for (auto& x : m.d) x = static_cast<S>(in[k++]);
        });
    }
};

template <class S>
Model<S> make_model(i64 in_dim, const std::vector<int>& hidden, i64 classes, u64 seed) {  // nn.hpp:73-102
    if (in_dim < 1 || classes < 1) throw std::invalid_argument("make_sage_model: dimensions must be positive");
    for (int h : hidden)
        if (h < 1) throw std::invalid_argument("make_sage_model: hidden dims must be positive");
    Rng rng(substream(seed, "init"));
    auto glorot = [&](i64 r, i64 c) {
        const double bound = std::sqrt(6.0 / static_cast<double>(r + c));
        Mat<S> m(r, c);
        for (i64 i = 0; i < r; ++i)
            for (i64 j = 0; j < c; ++j) m(i, j) = static_cast<S>(bound * (2.0 * rng.next_double() - 1.0));
        return m;
    };
    Model<S> m;
    i64 in = in_dim;
    for (int h : hidden) {
        m.W.push_back(glorot(h, in));
        m.U.push_back(glorot(h, h + in));
        in = h;
    }
    m.head = glorot(classes, in);
    return m;
}

struct Adj {  // AdjacencyView (graph.hpp:25-41) over a partition or the full graph
    i32 n;
    const i32 *offsets, *nbrs, *eids;
    std::size_t m;
};

template <class S>
struct Cache {
    std::vector<Mat<S>> inputs, msg_pre, means;
    Mat<S> emb;
    std::vector<S> inv;
};

template <class S>
Mat<S> forward(const Model<S>& model, const Adj& adj, const Mat<S>& x, const std::uint8_t* mask, Cache<S>& cache) {
    // nn.hpp:192-242
    if (x.r != adj.n) throw std::invalid_argument("sage_forward: feature rows != node count");
    const i64 in0 = model.W.empty() ? model.head.c : model.W[0].c;
    if (x.c != in0) throw std::invalid_argument("sage_forward: feature dim does not match model input dim");
    for (auto v : x.d)
        if (!std::isfinite(static_cast<double>(v))) throw std::invalid_argument("sage_forward: non-finite features");
    const i32 n = adj.n;
    cache.inv.assign(static_cast<std::size_t>(n), S(0));
    for (i32 v = 0; v < n; ++v) {  // masked_degrees nn.hpp:174-188, inv nn.hpp:209-215
        i32 d = 0;
        for (i32 k = adj.offsets[v]; k < adj.offsets[v + 1]; ++k)
            if (!mask || mask[adj.eids[k]]) ++d;
        cache.inv[v] = d > 0 ? S(1) / static_cast<S>(d) : S(0);
    }
    Mat<S> h = x;
    for (std::size_t l = 0; l < model.W.size(); ++l) {
        const Mat<S>& W = model.W[l];
        const Mat<S>& U = model.U[l];
        const i64 H = W.r, in = W.c;
        cache.inputs.push_back(h);
        Mat<S> pre = mm_nt(h, W);  // :220 msg_pre = h W^T
        Mat<S> msg = pre;
        for (auto& z : msg.d) z = std::max(z, S(0));  // :221 ReLU
        Mat<S> mean(n, H);
        for (i32 v = 0; v < n; ++v) {  // :222-230 masked neighbour sum, then *inv
            S* out = &mean(v, 0);
            for (i32 k = adj.offsets[v]; k < adj.offsets[v + 1]; ++k)
                if (!mask || mask[adj.eids[k]]) {
                    const S* src = &msg(adj.nbrs[k], 0);
                    for (i64 c = 0; c < H; ++c) out[c] += src[c];
                }
            for (i64 c = 0; c < H; ++c) out[c] *= cache.inv[v];
        }
        // :233-234  h' = mean U[:, :H]^T + h U[:, H:]^T  (two products, then add)
        Mat<S> a = mm_nt(mean, U, 0, H);
        Mat<S> b = mm_nt(h, U, H, in);
        for (std::size_t i = 0; i < a.d.size(); ++i) a.d[i] += b.d[i];
        cache.msg_pre.push_back(std::move(pre));
        cache.means.push_back(std::move(mean));
        h = std::move(a);
    }
    cache.emb = h;
    return mm_nt(h, model.head);  // :240
}

template <class S>
Model<S> backward(const Model<S>& model, const Cache<S>& cache, const Adj& adj, const Mat<S>& G,
                  const std::uint8_t* mask) {
    // nn.hpp:246-293
    const i32 n = adj.n;
    Model<S> gr;
    gr.head = mm_tn(G, cache.emb);  // :259
    Mat<S> dh = mm_nn(G, model.head);  // :260
    gr.W.resize(model.W.size());
    gr.U.resize(model.U.size());
    for (std::size_t l = model.W.size(); l-- > 0;) {
        const Mat<S>& W = model.W[l];
        const Mat<S>& U = model.U[l];
        const i64 H = W.r, in = W.c;
        const Mat<S>& h_in = cache.inputs[l];
        const Mat<S>& mean = cache.means[l];
        const Mat<S>& pre = cache.msg_pre[l];
        Mat<S> dUL = mm_tn(dh, mean), dUR = mm_tn(dh, h_in);  // :271-272
        gr.U[l] = Mat<S>(H, H + in);
        for (i64 i = 0; i < H; ++i) {
            for (i64 j = 0; j < H; ++j) gr.U[l](i, j) = dUL(i, j);
            for (i64 j = 0; j < in; ++j) gr.U[l](i, H + j) = dUR(i, j);
        }
        Mat<S> dmean = mm_nn(dh, U, 0, H);   // :274
        Mat<S> ddir = mm_nn(dh, U, H, in);   // :275
        Mat<S> dmsg(n, H);
        for (i32 v = 0; v < n; ++v) {  // :277-286 scatter inv[v]*dmean[v] to kept neighbours
            const S inv = cache.inv[v];
            if (inv == S(0)) continue;
            for (i32 k = adj.offsets[v]; k < adj.offsets[v + 1]; ++k)
                if (!mask || mask[adj.eids[k]]) {
                    S* dst = &dmsg(adj.nbrs[k], 0);
                    for (i64 c = 0; c < H; ++c) dst[c] += inv * dmean(v, c);
                }
        }
        Mat<S> dz = dmsg;  // :287-288 dz = 1[msg_pre > 0] * dmsg
        for (std::size_t i = 0; i < dz.d.size(); ++i) dz.d[i] = (pre.d[i] > S(0) ? S(1) : S(0)) * dmsg.d[i];
        gr.W[l] = mm_tn(dz, h_in);  // :289
        Mat<S> back = mm_nn(dz, W);  // :290 dh = dh_dir + dz W
        for (std::size_t i = 0; i < back.d.size(); ++i) back.d[i] = ddir.d[i] + back.d[i];
        dh = std::move(back);
    }
    return gr;
}

template <class S>
double softmax_ce(const Mat<S>& logits, const i32* y, const double* w, double normalizer, Mat<S>& grad) {
    // nn.hpp:317-345 (weights checked >= 0, rows with w == 0 skipped, f64 total)
    for (i64 r = 0; r < logits.r; ++r)
        if (!(w[r] >= 0.0)) throw std::invalid_argument("loss: node weights must be >= 0");
    if (!(normalizer > 0.0)) throw std::invalid_argument("loss: normalizer must be positive");
    grad = Mat<S>(logits.r, logits.c);
    double total = 0.0;
    for (i64 r = 0; r < logits.r; ++r) {
        if (y[r] < 0 || y[r] >= logits.c) throw std::invalid_argument("loss: class id out of range");
        if (w[r] == 0.0) continue;
        S mx = logits(r, 0);
        for (i64 c = 1; c < logits.c; ++c) mx = std::max(mx, logits(r, c));
        S se(0);
        for (i64 c = 0; c < logits.c; ++c) se += std::exp(logits(r, c) - mx);
        const S lse = mx + std::log(se);
        total += w[r] * static_cast<double>(lse - logits(r, y[r]));
        const S scale = static_cast<S>(w[r] / normalizer);
        for (i64 c = 0; c < logits.c; ++c) grad(r, c) = scale * (std::exp(logits(r, c) - lse) - S(c == y[r] ? 1 : 0));
    }
    return total / normalizer;
}

template <class S>
double bce(const Mat<S>& logits, const Mat<S>& t, const double* w, double normalizer, Mat<S>& grad) {
    // nn.hpp:348-378
    for (i64 r = 0; r < logits.r; ++r)
        if (!(w[r] >= 0.0)) throw std::invalid_argument("loss: node weights must be >= 0");
    if (!(normalizer > 0.0)) throw std::invalid_argument("loss: normalizer must be positive");
    grad = Mat<S>(logits.r, logits.c);
    double total = 0.0;
    for (i64 r = 0; r < logits.r; ++r) {
        if (w[r] == 0.0) continue;
        const S scale = static_cast<S>(w[r] / normalizer);
        for (i64 c = 0; c < logits.c; ++c) {
            const S z = logits(r, c), yv = t(r, c);
            if (yv != S(0) && yv != S(1)) throw std::invalid_argument("loss: bce targets must be 0 or 1");
            const S sp = std::max(z, S(0)) + std::log1p(std::exp(-std::abs(z)));
            total += w[r] * static_cast<double>(sp - z * yv);
            const S sg = z >= S(0) ? S(1) / (S(1) + std::exp(-z)) : std::exp(z) / (S(1) + std::exp(z));
            grad(r, c) = scale * (sg - yv);
        }
    }
    return total / normalizer;
}

template <class S>
void adam(Model<S>& model, const Model<S>& g, Model<S>& m1, Model<S>& m2, i64& step, double lr_d) {
    // nn.hpp:400-432
    bool finite = true;
    g.each([&](const Mat<S>& x) {
        for (auto v : x.d) finite = finite && std::isfinite(static_cast<double>(v));
    });
    if (!finite) throw std::invalid_argument("adam_step: non-finite gradient");
    ++step;
    const S b1 = static_cast<S>(0.9), b2 = static_cast<S>(0.999);
    const S c1 = static_cast<S>(1.0 - std::pow(0.9, static_cast<double>(step)));
    const S c2 = static_cast<S>(1.0 - std::pow(0.999, static_cast<double>(step)));
    const S lr = static_cast<S>(lr_d), eps = static_cast<S>(1e-8);
    std::vector<Mat<S>*> P, M, V;
    std::vector<const Mat<S>*> Gs;
    model.each([&](Mat<S>& x) { P.push_back(&x); });
    m1.each([&](Mat<S>& x) { M.push_back(&x); });
    m2.each([&](Mat<S>& x) { V.push_back(&x); });
    g.each([&](const Mat<S>& x) { Gs.push_back(&x); });
    for (std::size_t t = 0; t < P.size(); ++t)
        for (std::size_t i = 0; i < P[t]->d.size(); ++i) {
            const S gi = Gs[t]->d[i];
            S& m = M[t]->d[i];
            S& v = V[t]->d[i];
            m = b1 * m + (S(1) - b1) * gi;
            v = b2 * v + (S(1) - b2) * (gi * gi);
            const S mh = m / c1, vh = v / c2;
            P[t]->d[i] -= lr * mh / (std::sqrt(vh) + eps);
        }
}

template <class S>
Model<S> zeros_like(const Model<S>& m) {
    Model<S> z;
    for (std::size_t l = 0; l < m.W.size(); ++l) {
        z.W.emplace_back(m.W[l].r, m.W[l].c);
        z.U.emplace_back(m.U[l].r, m.U[l].c);
    }
    z.head = Mat<S>(m.head.r, m.head.c);
    return z;
}

// trainer.cpp:66-97 metric_from_logits: micro-F1 (positives at logit > 0) for
// multi-label graphs, else accuracy of the first arg-max; 0 for an empty mask.
template <class S>
double metric_from_logits(const Mat<S>& lg, const Graph& g, const std::uint8_t* mask) {
    std::size_t masked = 0;
    for (i32 v = 0; v < g.n; ++v) masked += mask[v];
    if (masked == 0) return 0.0;
    if (g.is_multilabel()) {
        std::int64_t tp = 0, fp = 0, fn = 0;
        for (i32 v = 0; v < g.n; ++v) {
            if (!mask[v]) continue;
            for (i64 c = 0; c < lg.c; ++c) {
                const bool pred = static_cast<double>(lg(v, c)) > 0.0;
                const bool truth = g.multilabels[static_cast<std::size_t>(v) * lg.c + c] != 0.0;
                tp += pred && truth;
                fp += pred && !truth;
                fn += !pred && truth;
            }
        }
        const std::int64_t denom = 2 * tp + fp + fn;
        return denom == 0 ? 0.0 : 2.0 * static_cast<double>(tp) / static_cast<double>(denom);
    }
    std::size_t correct = 0;
    for (i32 v = 0; v < g.n; ++v) {
        if (!mask[v]) continue;
        i64 best = 0;
        for (i64 c = 1; c < lg.c; ++c)
            if (static_cast<double>(lg(v, c)) > static_cast<double>(lg(v, best))) best = c;
        correct += best == g.labels[v];
    }
    return static_cast<double>(correct) / static_cast<double>(masked);
}

struct TrainerBase {
    virtual ~TrainerBase() = default;
    virtual void step(int epoch, double* loss, double* gnorm) = 0;
    virtual std::size_t count() const = 0;
    virtual void params(double*) const = 0;
    virtual void set_params(const double*) = 0;
    virtual void part_grads(int, double*) const = 0;
    virtual void gathered(double*) const = 0;
    virtual void part_logits(int, double*) const = 0;
    virtual double part_loss(int) const = 0;
    virtual int part_mask(int) const = 0;
    virtual void eval(double*, double*, double*) const = 0;
    virtual double time_part(int i, int epoch, int reps) = 0;
};

// trainer.hpp:202-313 (train_cofree_impl) — per-epoch body, eval kept separate.
template <class S>
struct Trainer final : TrainerBase {
    const Graph& g;
    const VCut& vc;
    std::vector<int> hidden;
    double lr;
    int loss_kind, use_de, K;
    double ratio;
    u64 seed;
    int workers;
    double normalizer = 0;
    struct In {
        Mat<S> x;
        std::vector<i32> y;
        Mat<S> t;
        std::vector<double> w;
        std::vector<std::vector<std::uint8_t>> masks;
    };
    std::vector<In> ins;
    Model<S> model, m1, m2;
    i64 adam_step = 0;
    std::vector<Model<S>> grads;
    std::vector<double> losses;
    std::vector<Mat<S>> logits;
    std::vector<int> chosen;
    Model<S> gath;

    Trainer(const Graph& gg, const VCut& v, std::vector<int> hid, double lr_, int loss, int reweight, int de, int k,
            double r, u64 s, int w)
        : g(gg), vc(v), hidden(std::move(hid)), lr(lr_), loss_kind(loss), use_de(de), K(k), ratio(r), seed(s),
          workers(w) {
        // validate_train_config trainer.cpp:21-36
        if (!(lr > 0.0)) throw std::invalid_argument("learning rate must be > 0");
        if (workers < 1) throw std::invalid_argument("workers must be >= 1");
        for (int h : hidden)
            if (h < 1) throw std::invalid_argument("hidden dims must be positive");
        if (use_de) {
            if (K < 1) throw std::invalid_argument("dropedge_k must be >= 1");
            if (ratio < 0.0 || ratio >= 1.0) throw std::invalid_argument("drop_ratio must lie in [0, 1)");
        }
        if (g.features.empty()) throw std::invalid_argument("training requires node features");
        if (!g.has_labels()) throw std::invalid_argument("training requires labels");
        if (g.train.empty()) throw std::invalid_argument("training requires split masks");
        if (loss_kind == 0 && g.labels.empty())  // trainer.hpp:207-208
            throw std::invalid_argument("softmax_ce requires multi-class labels");
        std::size_t cnt = 0;  // train_node_count trainer.cpp:59-64
        for (auto t : g.train) cnt += t;
        if (cnt == 0) throw std::invalid_argument("training requires a non-empty train mask");
        normalizer = static_cast<double>(cnt);
        if (vc.assign.size() != g.edges.size() || vc.parts.empty())
            throw std::invalid_argument("train_cofree: partition does not match graph");
        const auto W = weights(g, vc, reweight);
        ins.resize(vc.parts.size());
        for (std::size_t i = 0; i < vc.parts.size(); ++i) {  // trainer.hpp:218-243
            const Part& s = vc.parts[i];
            In& in = ins[i];
            in.x = Mat<S>(static_cast<i64>(s.nodes.size()), g.d);
            in.y.resize(s.nodes.size());
            in.w.resize(s.nodes.size());
            if (loss_kind == 1) in.t = Mat<S>(static_cast<i64>(s.nodes.size()), g.num_classes);
            for (std::size_t j = 0; j < s.nodes.size(); ++j) {
                const i32 v = s.nodes[j];
                for (int c = 0; c < g.d; ++c) in.x(j, c) = static_cast<S>(g.features[static_cast<std::size_t>(v) * g.d + c]);
                if (!g.is_multilabel()) in.y[j] = g.labels[v];
                if (loss_kind == 1) {  // label_targets graph.cpp:91-98: the multi-label matrix, or one-hot
                    if (g.is_multilabel())
                        for (int c = 0; c < g.num_classes; ++c)
                            in.t(j, c) = static_cast<S>(g.multilabels[static_cast<std::size_t>(v) * g.num_classes + c]);
                    else
                        in.t(j, g.labels[v]) = S(1);
                }
                in.w[j] = g.train[v] ? W[i][j] : 0.0;
            }
            if (use_de) in.masks = precompute_masks(s.edges.size(), K, ratio, substream(seed, "dropedge", i));
        }
        model = make_model<S>(g.d, hidden, g.num_classes, seed);
        m1 = zeros_like(model);
        m2 = zeros_like(model);
        grads.resize(vc.parts.size());
        losses.assign(vc.parts.size(), 0.0);
        logits.resize(vc.parts.size());
        chosen.assign(vc.parts.size(), -1);
    }

    void worker(std::size_t i, int epoch) {
        const Part& s = vc.parts[i];
        const In& in = ins[i];
        const std::uint8_t* mask = nullptr;
        chosen[i] = -1;
        if (use_de) {  // trainer.hpp:261-266
            Rng sel(substream(seed, "dropedge.select", i, static_cast<u64>(epoch)));
            const int k = static_cast<int>(sel.next_below(static_cast<u64>(K)));
            chosen[i] = k;
            mask = in.masks[static_cast<std::size_t>(k)].data();
        }
        const Adj adj{static_cast<i32>(s.nodes.size()), s.offsets.data(), s.nbrs.data(), s.eids.data(), s.edges.size()};
        Cache<S> cache;
        Mat<S> lg = forward(model, adj, in.x, mask, cache);
        Mat<S> G;
        losses[i] = loss_kind == 0 ? softmax_ce(lg, in.y.data(), in.w.data(), normalizer, G)
                                   : bce(lg, in.t, in.w.data(), normalizer, G);
        grads[i] = backward(model, cache, adj, G, mask);
        logits[i] = std::move(lg);
    }

    void step(int epoch, double* loss, double* gnorm) override {
        const std::size_t p = vc.parts.size();
        const int pool = std::min<int>(workers, static_cast<int>(p));
        if (pool <= 1) {
            for (std::size_t i = 0; i < p; ++i) worker(i, epoch);
        } else {
            std::vector<std::thread> th;
            std::vector<std::exception_ptr> err(static_cast<std::size_t>(pool));
            for (int w = 0; w < pool; ++w)
                th.emplace_back([&, w] {
                    try {
                        for (std::size_t i = static_cast<std::size_t>(w); i < p; i += static_cast<std::size_t>(pool))
                            worker(i, epoch);
                    } catch (...) {
                        err[static_cast<std::size_t>(w)] = std::current_exception();
                    }
                });
            for (auto& t : th) t.join();
            for (auto& e : err)
                if (e) std::rethrow_exception(e);
        }
        // gather_gradients trainer.hpp:79-94: ascending partition order
        gath = grads[0];
        for (std::size_t i = 1; i < p; ++i) {
            std::vector<Mat<S>*> dst;
            std::vector<const Mat<S>*> src;
            gath.each([&](Mat<S>& x) { dst.push_back(&x); });
            grads[i].each([&](const Mat<S>& x) { src.push_back(&x); });
            for (std::size_t t = 0; t < dst.size(); ++t)
                for (std::size_t k = 0; k < dst[t]->d.size(); ++k) dst[t]->d[k] += src[t]->d[k];
        }
        double sq = 0.0;  // grad_norm nn.hpp:145-152
        gath.each([&](const Mat<S>& x) {
            for (auto v : x.d) sq += static_cast<double>(v) * static_cast<double>(v);
        });
        *gnorm = std::sqrt(sq);
        double tot = 0.0;
        for (double l : losses) tot += l;
        *loss = tot;
        adam(model, gath, m1, m2, adam_step, lr);
    }

    // evaluate_splits trainer.hpp:132-140 + metric_from_logits trainer.cpp:66-97 (multi-class)
    void eval(double* tr, double* va, double* te) const override {
        const Adj adj{g.n, g.offsets.data(), g.nbrs.data(), g.eids.data(), g.edges.size()};
        Mat<S> x(g.n, g.d);
        for (std::size_t i = 0; i < x.d.size(); ++i) x.d[i] = static_cast<S>(g.features[i]);
        Cache<S> cache;
        const Mat<S> lg = forward(model, adj, x, nullptr, cache);
        *tr = metric_from_logits(lg, g, g.train.data());
        *va = metric_from_logits(lg, g, g.val.data());
        *te = metric_from_logits(lg, g, g.test.data());
    }

    double time_part(int i, int epoch, int reps) override {
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < reps; ++r) worker(static_cast<std::size_t>(i), epoch);
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
    }
    std::size_t count() const override { return model.count(); }
    void params(double* out) const override { model.to_flat(out); }
    void set_params(const double* in) override { model.from_flat(in); }
    void part_grads(int i, double* out) const override { grads[static_cast<std::size_t>(i)].to_flat(out); }
    void gathered(double* out) const override { gath.to_flat(out); }
    void part_logits(int i, double* out) const override {
        const auto& l = logits[static_cast<std::size_t>(i)];
        for (std::size_t k = 0; k < l.d.size(); ++k) out[k] = static_cast<double>(l.d[k]);
    }
    double part_loss(int i) const override { return losses[static_cast<std::size_t>(i)]; }
    int part_mask(int i) const override { return chosen[static_cast<std::size_t>(i)]; }
};

}  // namespace

extern "C" {

const char* or_last_error(void) { return g_err.c_str(); }
uint64_t or_mix64(uint64_t x) { return mix64(x); }
uint64_t or_substream(uint64_t seed, const char* tag, int nidx, uint64_t a, uint64_t b) {
    return nidx == 0 ? substream(seed, tag) : (nidx == 1 ? substream(seed, tag, a) : substream(seed, tag, a, b));
}
void or_rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t n, uint64_t* out_u, double* out_d) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) {
        if (kind == 0) out_u[i] = rng.next_u64();
        else if (kind == 1) out_u[i] = rng.next_below(arg);
        else if (kind == 2) out_d[i] = rng.next_double();
        else out_d[i] = rng.next_gaussian();
    }
}

void* or_graph_build(int32_t n, const int32_t* uv, int64_t m) {
    Graph* out = nullptr;
    if (guard([&] {
            std::vector<std::pair<i32, i32>> raw(static_cast<std::size_t>(m));
            for (int64_t e = 0; e < m; ++e) raw[static_cast<std::size_t>(e)] = {uv[2 * e], uv[2 * e + 1]};
            out = new Graph(build_graph(n, std::move(raw)));
        }))
        return nullptr;
    return out;
}
void* or_graph_sbm(int32_t n, int classes, double p_in, double p_out, int d, double noise, uint64_t seed) {
    Graph* out = nullptr;
    if (guard([&] { out = new Graph(gen_homophilic_sbm(n, classes, p_in, p_out, d, noise, seed)); })) return nullptr;
    return out;
}
void or_graph_free(void* g) { delete static_cast<Graph*>(g); }
int32_t or_graph_num_nodes(void* g) { return static_cast<Graph*>(g)->n; }
int64_t or_graph_num_edges(void* g) { return static_cast<int64_t>(static_cast<Graph*>(g)->edges.size()); }
void or_graph_edges(void* gp, int32_t* uv) {
    auto* g = static_cast<Graph*>(gp);
    for (std::size_t e = 0; e < g->edges.size(); ++e) {
        uv[2 * e] = g->edges[e].first;
        uv[2 * e + 1] = g->edges[e].second;
    }
}
void or_graph_csr(void* gp, int32_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* deg) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(offsets, g->offsets.data(), g->offsets.size() * 4);
    std::memcpy(nbrs, g->nbrs.data(), g->nbrs.size() * 4);
    std::memcpy(eids, g->eids.data(), g->eids.size() * 4);
    std::memcpy(deg, g->degrees.data(), g->degrees.size() * 4);
}
void or_graph_features(void* gp, double* out) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(out, g->features.data(), g->features.size() * 8);
}
void or_graph_labels(void* gp, int32_t* labels) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(labels, g->labels.data(), g->labels.size() * 4);
}
void or_graph_masks(void* gp, uint8_t* train, uint8_t* val, uint8_t* test) {
    auto* g = static_cast<Graph*>(gp);
    std::memcpy(train, g->train.data(), g->train.size());
    std::memcpy(val, g->val.data(), g->val.size());
    std::memcpy(test, g->test.data(), g->test.size());
}
int or_graph_set_data(void* gp, const float* features, int d, const int32_t* labels, int classes,
                      const uint8_t* train, const uint8_t* val, const uint8_t* test) {
    return guard([&] {
        auto* g = static_cast<Graph*>(gp);
        const auto n = static_cast<std::size_t>(g->n);
        g->d = d;
        g->features.resize(n * static_cast<std::size_t>(d));
        for (std::size_t i = 0; i < g->features.size(); ++i) g->features[i] = static_cast<double>(features[i]);
        g->labels.assign(labels, labels + n);
        g->num_classes = classes;
        g->train.assign(train, train + n);
        g->val.assign(val, val + n);
        g->test.assign(test, test + n);
    });
}

// load_labels' multi-label branch (graph_io.cpp:206-229): n x C 0/1 matrix, labels cleared.
int or_graph_set_multilabels(void* gp, const float* y, int classes) {
    return guard([&] {
        auto* g = static_cast<Graph*>(gp);
        const std::size_t k = static_cast<std::size_t>(g->n) * static_cast<std::size_t>(classes);
        g->multilabels.resize(k);
        for (std::size_t i = 0; i < k; ++i) {
            if (y[i] != 0.f && y[i] != 1.f) throw std::invalid_argument("loss: bce targets must be 0 or 1");
            g->multilabels[i] = static_cast<double>(y[i]);
        }
        g->num_classes = classes;
        g->labels.clear();
    });
}

// evaluate (trainer.cpp:101-112): SageModel<double> forward over the full graph,
// then metric_from_logits on one split mask.
int or_evaluate(void* gp, const double* theta, const int* hidden, int layers, const uint8_t* mask, double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        if (g.features.empty() || !g.has_labels())
            throw std::invalid_argument("evaluate: graph lacks features or labels");
        std::size_t masked = 0;
        for (i32 v = 0; v < g.n; ++v) masked += mask[v];
        if (masked == 0) throw std::invalid_argument("evaluate: empty mask");
        Model<double> m = make_model<double>(g.d, std::vector<int>(hidden, hidden + layers), g.num_classes, 0);
        m.from_flat(theta);
        const Adj adj{g.n, g.offsets.data(), g.nbrs.data(), g.eids.data(), g.edges.size()};
        Mat<double> x(g.n, g.d);
        x.d = g.features;
        Cache<double> cache;
        const Mat<double> lg = forward(m, adj, x, nullptr, cache);
        *out = metric_from_logits(lg, g, mask);
    });
}

// comm_volume (trainer.cpp:38-49); out = {floats_per_iteration, gradient_floats, embedding_floats}
int or_comm_volume(int mode, int num_parts, uint64_t params, uint64_t layers, uint64_t hidden, uint64_t halo,
                   uint64_t* out) {
    return guard([&] {
        if (num_parts < 1) throw std::invalid_argument("comm_volume: num_parts must be >= 1");
        const uint64_t grad = static_cast<uint64_t>(num_parts) * params;
        const uint64_t emb = mode == 1 ? 2ULL * layers * halo * hidden : 0ULL;
        out[0] = grad + emb;
        out[1] = grad;
        out[2] = emb;
    });
}
// expected_rf_random / imbalance_lower_bound (partition.cpp:344-362)
int or_expected_rf_random(int p, int64_t degree, double* out) {
    return guard([&] {
        if (p < 1) throw std::invalid_argument("expected_rf_random: num_parts must be >= 1");
        if (degree < 0) throw std::invalid_argument("expected_rf_random: degree must be >= 0");
        const double pd = static_cast<double>(p);
        *out = pd * (1.0 - std::pow(1.0 - 1.0 / pd, static_cast<double>(degree)));
    });
}
int or_imbalance_lower_bound(int p, int64_t max_degree, int64_t min_degree, double* out) {
    return guard([&] {
        if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
        if (min_degree < 1) throw std::invalid_argument("imbalance_lower_bound: min_degree must be >= 1");
        if (max_degree < min_degree) throw std::invalid_argument("imbalance_lower_bound: max_degree < min_degree");
        if (p == 1) {
            *out = 1.0;
            return;
        }
        const double pd = static_cast<double>(p);
        *out = (1.0 - std::pow(1.0 - 1.0 / pd, static_cast<double>(max_degree))) /
               (1.0 - std::pow(1.0 - 1.0 / pd, static_cast<double>(min_degree)));
    });
}

// The masked mean aggregation alone (nn.hpp:209-230) and its transpose
// (nn.hpp:277-288), float, over a CSR with int64 offsets (any size). mask:
// per local edge (eids index it) or null. Forward: out[v] = (sum over kept
// CSR slots of src[nbr], from 0, in CSR order) * inv[v], inv = 1/(float)deg.
// Backward (pull form of the scatter, same per-row order: CSR rows ascend):
// out[u] = (msg[u] > 0) ? sum over kept slots of src[nbr] : 0, where src is
// dmean already scaled by inv (the reference adds inv[v] * dmean[v]).
// Rows are split across `threads` std::threads (rows are independent).
void or_spmm(int bwd, int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const int32_t* eids,
             const uint8_t* mask, const float* src, const float* msg, float* out, int threads) {
    auto rows = [&](int64_t r0, int64_t r1) {
        std::vector<float> acc(static_cast<std::size_t>(H));
        for (int64_t v = r0; v < r1; ++v) {
            std::fill(acc.begin(), acc.end(), 0.f);
            int32_t deg = 0;
            for (int64_t k = off[v]; k < off[v + 1]; ++k) {
                if (mask && !mask[eids[k]]) continue;
                ++deg;
                const float* s = src + static_cast<int64_t>(nbrs[k]) * H;
                for (int32_t c = 0; c < H; ++c) acc[c] += s[c];
            }
            float* o = out + v * H;
            if (!bwd) {
                const float inv = deg > 0 ? 1.f / static_cast<float>(deg) : 0.f;
                for (int32_t c = 0; c < H; ++c) o[c] = acc[c] * inv;
            } else {
                const float* m = msg + v * H;
                for (int32_t c = 0; c < H; ++c) o[c] = m[c] > 0.f ? acc[c] : 0.f;
            }
        }
    };
    if (threads <= 1) {
        rows(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) th.emplace_back(rows, n * t / threads, n * (t + 1) / threads);
    for (auto& x : th) x.join();
}

void* or_partition(void* gp, int algo, int p, uint64_t seed) {
    VCut* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            if (algo == 0) out = new VCut(partition_random(g, p, seed));
            else if (algo == 1) out = new VCut(partition_dbh(g, p, seed));
            else if (algo == 2) {
                std::vector<std::string> w;
                out = new VCut(partition_ne(g, p, seed, 1.1, w));
            } else if (algo == 3) out = new VCut(edge_cut_to_vertex_cut(g, partition_edge_cut_greedy(g, p, seed), seed));
            else throw std::invalid_argument("oracle: unknown partition algorithm");
        }))
        return nullptr;
    return out;
}
void* or_build_vertex_cut(void* gp, int p, const int32_t* assign) {
    VCut* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            out = new VCut(build_vertex_cut(g, p, std::vector<i32>(assign, assign + g.edges.size())));
        }))
        return nullptr;
    return out;
}
// partition_ne with an explicit balance_slack; warnings joined by '\n' into
// wbuf (cap bytes, NUL-terminated).
void* or_partition_ne(void* gp, int p, uint64_t seed, double slack, char* wbuf, int64_t cap) {
    VCut* out = nullptr;
    if (guard([&] {
            std::vector<std::string> w;
            out = new VCut(partition_ne(*static_cast<Graph*>(gp), p, seed, slack, w));
            std::string j;
            for (const auto& x : w) j += (j.empty() ? "" : "\n") + x;
            if (wbuf && cap > 0) {
                std::strncpy(wbuf, j.c_str(), static_cast<std::size_t>(cap - 1));
                wbuf[cap - 1] = 0;
            }
        }))
        return nullptr;
    return out;
}
int or_edge_cut_greedy(void* gp, int p, uint64_t seed, int32_t* node_assign) {
    return guard([&] {
        const ECut ec = partition_edge_cut_greedy(*static_cast<Graph*>(gp), p, seed);
        std::memcpy(node_assign, ec.node_assign.data(), ec.node_assign.size() * 4);
    });
}
// kept_counts[p], num_cut, halo_counts[p]; cut_edges (num_cut) and halo_nodes
// (sum halo_counts, part-major, ascending) when non-null.
int or_edge_cut_stats(void* gp, int p, const int32_t* na, int64_t* kept_counts, int64_t* num_cut,
                      int64_t* halo_counts, int32_t* cut_edges, int32_t* halo_nodes) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        const ECut ec = edge_cut_from_assignment(g, p, std::vector<i32>(na, na + g.n));
        *num_cut = static_cast<int64_t>(ec.cut.size());
        for (int i = 0; i < p; ++i) {
            kept_counts[i] = static_cast<int64_t>(ec.kept[i].size());
            halo_counts[i] = static_cast<int64_t>(ec.halo[i].size());
        }
        if (cut_edges) std::memcpy(cut_edges, ec.cut.data(), ec.cut.size() * 4);
        if (halo_nodes)
            for (const auto& h : ec.halo) {
                std::memcpy(halo_nodes, h.data(), h.size() * 4);
                halo_nodes += h.size();
            }
    });
}
void* or_edge_cut_to_vertex_cut(void* gp, int p, const int32_t* na, uint64_t seed) {
    VCut* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            out = new VCut(edge_cut_to_vertex_cut(g, edge_cut_from_assignment(g, p, std::vector<i32>(na, na + g.n)),
                                                  seed));
        }))
        return nullptr;
    return out;
}
void or_partition_free(void* p) { delete static_cast<VCut*>(p); }
void or_partition_assignment(void* pp, int32_t* out) {
    auto* vc = static_cast<VCut*>(pp);
    std::memcpy(out, vc->assign.data(), vc->assign.size() * 4);
}
void or_part_sizes(void* pp, int i, int64_t* n_local, int64_t* n_edges) {
    auto& s = static_cast<VCut*>(pp)->parts[static_cast<std::size_t>(i)];
    *n_local = static_cast<int64_t>(s.nodes.size());
    *n_edges = static_cast<int64_t>(s.edges.size());
}
void or_part_arrays(void* pp, int i, int32_t* nodes, int32_t* edges_uv, int32_t* edge_gids, int32_t* local_deg,
                    int32_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* g2l) {
    auto& s = static_cast<VCut*>(pp)->parts[static_cast<std::size_t>(i)];
    std::memcpy(nodes, s.nodes.data(), s.nodes.size() * 4);
    for (std::size_t e = 0; e < s.edges.size(); ++e) {
        edges_uv[2 * e] = s.edges[e].first;
        edges_uv[2 * e + 1] = s.edges[e].second;
    }
    std::memcpy(edge_gids, s.edge_gids.data(), s.edge_gids.size() * 4);
    std::memcpy(local_deg, s.local_deg.data(), s.local_deg.size() * 4);
    std::memcpy(offsets, s.offsets.data(), s.offsets.size() * 4);
    std::memcpy(nbrs, s.nbrs.data(), s.nbrs.size() * 4);
    std::memcpy(eids, s.eids.data(), s.eids.size() * 4);
    if (g2l) std::memcpy(g2l, s.g2l.data(), s.g2l.size() * 4);
}
int or_replication_stats(void* pp, void* gp, int32_t* per_node_rf, double* rf, double* edge_balance,
                         double* node_balance, int64_t* duplicated) {
    // partition.cpp:310-342
    return guard([&] {
        const VCut& vc = *static_cast<VCut*>(pp);
        const Graph& g = *static_cast<Graph*>(gp);
        if (vc.assign.size() != g.edges.size())
            throw std::invalid_argument("replication_stats: partition does not match graph");
        std::fill(per_node_rf, per_node_rf + g.n, 0);
        std::size_t tot = 0, maxn = 0, maxe = 0;
        for (const Part& s : vc.parts) {
            tot += s.nodes.size();
            maxn = std::max(maxn, s.nodes.size());
            maxe = std::max(maxe, s.edges.size());
            for (i32 v : s.nodes) ++per_node_rf[v];
        }
        const double n = static_cast<double>(g.n), p = static_cast<double>(vc.p);
        *rf = static_cast<double>(tot) / n;
        *duplicated = static_cast<int64_t>(tot) - static_cast<int64_t>(g.n);
        *edge_balance = g.edges.empty() ? 0.0 : static_cast<double>(maxe) / (static_cast<double>(g.edges.size()) / p);
        *node_balance = tot == 0 ? 0.0 : static_cast<double>(maxn) / (static_cast<double>(tot) / p);
    });
}
int or_weights(void* gp, void* pp, int scheme, double* out) {
    return guard([&] {
        const auto w = weights(*static_cast<Graph*>(gp), *static_cast<VCut*>(pp), scheme);
        std::size_t k = 0;
        for (auto& part : w)
            for (double x : part) out[k++] = x;
    });
}
int or_precompute_masks(int64_t m, int k, double ratio, uint64_t seed, uint8_t* out) {
    return guard([&] {
        const auto masks = precompute_masks(static_cast<std::size_t>(m), k, ratio, seed);
        for (int i = 0; i < k; ++i) std::memcpy(out + static_cast<std::size_t>(i) * static_cast<std::size_t>(m), masks[i].data(), static_cast<std::size_t>(m));
    });
}
int or_select_mask(uint64_t seed, uint64_t part, uint64_t epoch, int k) {  // dropedge.cpp:35-37
    Rng rng(substream(seed, "dropedge.select", part, epoch));
    return static_cast<int>(rng.next_below(static_cast<u64>(k)));
}
int64_t or_init_params(int in_dim, const int* hidden, int layers, int classes, uint64_t seed, int f32, double* out) {
    int64_t count = -1;
    guard([&] {
        const std::vector<int> h(hidden, hidden + layers);
        if (f32) {
            auto m = make_model<float>(in_dim, h, classes, seed);
            if (out) m.to_flat(out);
            count = static_cast<int64_t>(m.count());
        } else {
            auto m = make_model<double>(in_dim, h, classes, seed);
            if (out) m.to_flat(out);
            count = static_cast<int64_t>(m.count());
        }
    });
    return count;
}
void* or_trainer_new(void* gp, void* pp, const int* hidden, int layers, double lr, int loss, int reweight,
                     int use_dropedge, int k, double ratio, uint64_t seed, int f32, int workers) {
    TrainerBase* out = nullptr;
    if (guard([&] {
            const Graph& g = *static_cast<Graph*>(gp);
            const VCut& vc = *static_cast<VCut*>(pp);
            std::vector<int> h(hidden, hidden + layers);
            if (f32) out = new Trainer<float>(g, vc, h, lr, loss, reweight, use_dropedge, k, ratio, seed, workers);
            else out = new Trainer<double>(g, vc, h, lr, loss, reweight, use_dropedge, k, ratio, seed, workers);
        }))
        return nullptr;
    return out;
}
void or_trainer_free(void* t) { delete static_cast<TrainerBase*>(t); }
int or_trainer_step(void* t, int epoch, double* loss, double* gnorm) {
    return guard([&] { static_cast<TrainerBase*>(t)->step(epoch, loss, gnorm); });
}
int64_t or_trainer_param_count(void* t) { return static_cast<int64_t>(static_cast<TrainerBase*>(t)->count()); }
void or_trainer_params(void* t, double* out) { static_cast<TrainerBase*>(t)->params(out); }
void or_trainer_set_params(void* t, const double* in) { static_cast<TrainerBase*>(t)->set_params(in); }
void or_trainer_part_grads(void* t, int i, double* out) { static_cast<TrainerBase*>(t)->part_grads(i, out); }
void or_trainer_gathered(void* t, double* out) { static_cast<TrainerBase*>(t)->gathered(out); }
void or_trainer_part_logits(void* t, int i, double* out) { static_cast<TrainerBase*>(t)->part_logits(i, out); }
double or_trainer_part_loss(void* t, int i) { return static_cast<TrainerBase*>(t)->part_loss(i); }
int or_trainer_part_mask(void* t, int i) { return static_cast<TrainerBase*>(t)->part_mask(i); }
void or_trainer_eval(void* t, double* tr, double* va, double* te) { static_cast<TrainerBase*>(t)->eval(tr, va, te); }
double or_trainer_time_part_step(void* t, int i, int epoch, int reps) {
    double s = -1;
    guard([&] { s = static_cast<TrainerBase*>(t)->time_part(i, epoch, reps); });
    return s;
}

}  // extern "C"
