// graph.cu — graph ingest, vertex-cut assignment and per-partition CSR build,
// all on the device (sm_100a). Integer/byte work: HBM-bound scans, sorts and
// scatters, no tensor cores.
//
// Bit-exact restatements of:
//   build_graph          proj/src/graph.cpp:8-64
//   partition_random     proj/src/partition.cpp:92-100
//   partition_dbh        proj/src/partition.cpp:102-114
//   build_vertex_cut     proj/src/partition.cpp:22-90
//   dar/vanilla/unit     proj/src/reweight.cpp:23-71
//   make_sage_model init proj/include/sagecut/nn.hpp:73-102
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.hpp"

namespace sc {

thread_local int64_t g_launches = 0;

namespace {

constexpr int kBlock = 256;

template <class T>
__global__ void fill_kernel(T* p, int64_t n, T v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
template <class T>
void fill(T* p, int64_t n, T v, cudaStream_t s) {
    if (n <= 0) return;
    fill_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(p, n, v);
    SC_LAUNCH_CHECK();
    count_launch();
}

__global__ void iota_kernel(int32_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        p[i] = static_cast<int32_t>(i);
}

struct I32ToI64 {
    __host__ __device__ int64_t operator()(int32_t x) const { return x; }
};

int bits_for(uint64_t x) {  // bits needed to represent values in [0, x]
    int b = 1;
    while (b < 64 && (x >> b) != 0) ++b;
    return b;
}

// ---- CSR build ----------------------------------------------------------------
// Row x of the reference's cursor-filled CSR lists first the edges (a, x), a < x,
// in edge order (= ascending a, since edges are sorted by (u, v)), then the
// edges (x, b) in edge order (= ascending b). Both halves are placed directly:
// the upper half by arithmetic (edges with u == x are contiguous), the lower
// half through one stable radix sort of the edges by v.
__global__ void count_uv_kernel(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                int32_t* cnt_lower, int32_t* cnt_upper) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        atomicAdd(&cnt_upper[u[e]], 1);
        atomicAdd(&cnt_lower[v[e]], 1);
    }
}

__global__ void degree_kernel(int64_t n, const int32_t* cl, const int32_t* cu, int32_t* deg, int64_t* deg64) {
    for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x) {
        const int32_t d = cl[x] + cu[x];
        if (deg) deg[x] = d;
        deg64[x] = d;
    }
}

__global__ void fill_upper_kernel(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                                  const int64_t* __restrict__ off, const int32_t* __restrict__ cl,
                                  const int64_t* __restrict__ upstart, int32_t* nbrs, int32_t* eids) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        const int32_t x = u[e];
        const int64_t slot = off[x] + cl[x] + (e - upstart[x]);
        nbrs[slot] = v[e];
        eids[slot] = static_cast<int32_t>(e);
    }
}

__global__ void fill_lower_kernel(int64_t m, const int32_t* __restrict__ vs, const int32_t* __restrict__ es,
                                  const int32_t* __restrict__ u, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ lowstart, int32_t* nbrs, int32_t* eids) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m; k += int64_t(gridDim.x) * blockDim.x) {
        const int32_t x = vs[k];
        const int32_t e = es[k];
        const int64_t slot = off[x] + (k - lowstart[x]);
        nbrs[slot] = u[e];
        eids[slot] = e;
    }
}

}  // namespace

void build_csr(sc_ctx* ctx, int64_t n, int64_t m, const int32_t* u, const int32_t* v, int64_t* offsets,
               int32_t* nbrs, int32_t* eids, int32_t* degrees_out) {
    cudaStream_t s = ctx->stream;
    DevBuf<int32_t> cl(n + 1), cu(n + 1);
    DevBuf<int64_t> deg64(n + 1), lowstart(n + 1), upstart(n + 1);
    SC_CUDA(cudaMemsetAsync(cl.get(), 0, (n + 1) * 4, s));
    SC_CUDA(cudaMemsetAsync(cu.get(), 0, (n + 1) * 4, s));
    if (m > 0) {
        count_uv_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(m, u, v, cl.get(), cu.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    if (n > 0) {
        degree_kernel<<<grid_for(n, kBlock), kBlock, 0, s>>>(n, cl.get(), cu.get(), degrees_out, deg64.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    SC_CUDA(cudaMemsetAsync(deg64.get() + n, 0, 8, s));
    // offsets = exclusive scan of degrees over n+1 entries (last = 2m)
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg64.get(), offsets, n + 1, s);
    cub::DeviceScan::ExclusiveSum(ctx->temp(tb), tb, deg64.get(), offsets, n + 1, s);
    count_launch(2);
    auto cnt_iter_l = cl.get();
    auto cnt_iter_u = cu.get();
    // lowstart/upstart: exclusive scans of the int32 counts into int64
    cub::TransformInputIterator<int64_t, I32ToI64, const int32_t*> itl(cnt_iter_l, I32ToI64{});
    cub::TransformInputIterator<int64_t, I32ToI64, const int32_t*> itu(cnt_iter_u, I32ToI64{});
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, itl, lowstart.get(), n + 1, s);
    cub::DeviceScan::ExclusiveSum(ctx->temp(tb), tb, itl, lowstart.get(), n + 1, s);
    cub::DeviceScan::ExclusiveSum(ctx->temp(tb), tb, itu, upstart.get(), n + 1, s);
    count_launch(4);
    if (m == 0) return;
    DevBuf<int32_t> idx(m), vs(m), es(m);
    iota_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(idx.get(), m);
    SC_LAUNCH_CHECK();
    count_launch();
    tb = 0;
    const int eb = bits_for(static_cast<uint64_t>(n));
    cub::DeviceRadixSort::SortPairs(nullptr, tb, v, vs.get(), idx.get(), es.get(), m, 0, eb, s);
    cub::DeviceRadixSort::SortPairs(ctx->temp(tb), tb, v, vs.get(), idx.get(), es.get(), m, 0, eb, s);
    count_launch(4);
    fill_upper_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(m, u, v, offsets, cl.get(), upstart.get(), nbrs, eids);
    SC_LAUNCH_CHECK();
    fill_lower_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(m, vs.get(), es.get(), u, offsets, lowstart.get(), nbrs,
                                                            eids);
    SC_LAUNCH_CHECK();
    count_launch(2);
    // temporaries are freed at scope exit; keep the stream ordered first
    SC_CUDA(cudaStreamSynchronize(s));
}

// ---- build_graph (graph.cpp:8-64) ----------------------------------------------------
namespace {
constexpr uint64_t kSelfLoop = ~0ULL;
__global__ void canon_kernel(int64_t m, int32_t n, const int32_t* __restrict__ raw, uint64_t* keys, int* bad) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        int32_t a = raw[2 * i], b = raw[2 * i + 1];
        if (a < 0 || b < 0 || a >= n || b >= n) {
            *bad = 1;
            keys[i] = kSelfLoop;
            continue;
        }
        if (a == b) {
            keys[i] = kSelfLoop;
            continue;
        }
        if (a > b) {
            const int32_t t = a;
            a = b;
            b = t;
        }
        keys[i] = (static_cast<uint64_t>(a) << 32) | static_cast<uint32_t>(b);
    }
}
struct NotSelfLoop {
    __host__ __device__ bool operator()(uint64_t k) const { return k != kSelfLoop; }
};
__global__ void split_keys_kernel(int64_t m, const uint64_t* keys, int32_t* u, int32_t* v) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
        u[i] = static_cast<int32_t>(keys[i] >> 32);
        v[i] = static_cast<int32_t>(keys[i] & 0xffffffffu);
    }
}
}  // namespace

std::unique_ptr<sc_graph> build_graph_device(sc_ctx* ctx, int32_t n, const int32_t* raw_dev, int64_t m_raw,
                                             int64_t* self_loops, int64_t* dups) {
    if (n < 0) throw std::invalid_argument("build_graph: negative node count");
    cudaStream_t s = ctx->stream;
    auto g = std::make_unique<sc_graph>();
    g->ctx = ctx;
    g->n = n;
    DevBuf<uint64_t> keys(m_raw > 0 ? m_raw : 1), keys2(m_raw > 0 ? m_raw : 1);
    DevBuf<int> flags(2);
    DevBuf<int64_t> nsel(1);
    SC_CUDA(cudaMemsetAsync(flags.get(), 0, 8, s));
    int64_t m_kept = 0, m_unique = 0;
    if (m_raw > 0) {
        canon_kernel<<<grid_for(m_raw, kBlock), kBlock, 0, s>>>(m_raw, n, raw_dev, keys.get(), flags.get());
        SC_LAUNCH_CHECK();
        count_launch();
        int bad = 0;
        d2h(&bad, flags.get(), 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
        if (bad) throw std::invalid_argument("build_graph: edge endpoint out of range");
        size_t tb = 0;
        cub::DeviceSelect::If(nullptr, tb, keys.get(), keys2.get(), nsel.get(), m_raw, NotSelfLoop{}, s);
        cub::DeviceSelect::If(ctx->temp(tb), tb, keys.get(), keys2.get(), nsel.get(), m_raw, NotSelfLoop{}, s);
        d2h(&m_kept, nsel.get(), 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
        const int hb = bits_for(static_cast<uint64_t>(n));
        tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, keys2.get(), keys.get(), m_kept, 0, 32 + hb, s);
        cub::DeviceRadixSort::SortKeys(ctx->temp(tb), tb, keys2.get(), keys.get(), m_kept, 0, 32 + hb, s);
        tb = 0;
        cub::DeviceSelect::Unique(nullptr, tb, keys.get(), keys2.get(), nsel.get(), m_kept, s);
        cub::DeviceSelect::Unique(ctx->temp(tb), tb, keys.get(), keys2.get(), nsel.get(), m_kept, s);
        d2h(&m_unique, nsel.get(), 1, s);
        SC_CUDA(cudaStreamSynchronize(s));
        count_launch(8);
    }
    if (self_loops) *self_loops = m_raw - m_kept;
    if (dups) *dups = m_kept - m_unique;
    g->m = m_unique;
    g->eu.alloc(std::max<int64_t>(m_unique, 1));
    g->ev.alloc(std::max<int64_t>(m_unique, 1));
    if (m_unique > 0) {
        split_keys_kernel<<<grid_for(m_unique, kBlock), kBlock, 0, s>>>(m_unique, keys2.get(), g->eu.get(),
                                                                        g->ev.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    g->degrees.alloc(std::max<int32_t>(n, 1));
    g->offsets.alloc(static_cast<size_t>(n) + 1);
    g->nbrs.alloc(std::max<int64_t>(2 * m_unique, 1));
    g->eids.alloc(std::max<int64_t>(2 * m_unique, 1));
    build_csr(ctx, n, m_unique, g->eu.get(), g->ev.get(), g->offsets.get(), g->nbrs.get(), g->eids.get(),
              g->degrees.get());
    return g;
}

// ---- edge -> part assignment -------------------------------------------------------
namespace {
// partition_random: edge e consumes the (e + shift)-th draw of the stream, where
// shift counts next_below rejections before e. Draws r < 2^64 mod p are
// rejected (rng.hpp:43-49); the first rejection at or after `start` is reported.
__global__ void random_assign_kernel(int64_t m, uint32_t p, uint64_t s, uint64_t thr, int64_t start, int64_t shift,
                                     int32_t* assign, unsigned long long* first_reject) {
    for (int64_t e = start + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = draw_u64(s, static_cast<uint64_t>(e + shift));
        if (r < thr) atomicMin(first_reject, static_cast<unsigned long long>(e));
        assign[e] = static_cast<int32_t>(r % p);
    }
}
__global__ void dbh_assign_kernel(int64_t m, uint32_t p, uint64_t seed, const int32_t* __restrict__ u,
                                  const int32_t* __restrict__ v, const int32_t* __restrict__ deg, int32_t* assign) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        const int32_t a = u[e], b = v[e];
        const int32_t da = deg[a], db = deg[b];
        const int32_t pick = da != db ? (da < db ? a : b) : min(a, b);
        assign[e] = static_cast<int32_t>(mix64(static_cast<uint64_t>(static_cast<int64_t>(pick)) ^ seed) % p);
    }
}
}  // namespace

void assign_random(sc_graph* g, int32_t p, uint64_t seed, int32_t* assign) {
    cudaStream_t st = g->ctx->stream;
    const uint64_t s = substream(seed, "partition.random");
    const uint64_t thr = below_threshold(static_cast<uint64_t>(p));
    DevBuf<unsigned long long> first(1);
    int64_t start = 0, shift = 0;
    for (;;) {
        const unsigned long long none = static_cast<unsigned long long>(g->m);
        h2d(first.get(), &none, 1, st);
        random_assign_kernel<<<grid_for(g->m - start, kBlock), kBlock, 0, st>>>(
            g->m, static_cast<uint32_t>(p), s, thr, start, shift, assign, first.get());
        SC_LAUNCH_CHECK();
        count_launch();
        if (thr == 0) break;  // p a power of two: next_below never rejects
        unsigned long long f = 0;
        d2h(&f, first.get(), 1, st);
        SC_CUDA(cudaStreamSynchronize(st));
        if (f >= static_cast<unsigned long long>(g->m)) break;
        start = static_cast<int64_t>(f);  // redo from the rejected edge with one more draw consumed
        shift += 1;
    }
}

void assign_dbh(sc_graph* g, int32_t p, uint64_t seed, int32_t* assign) {
    if (g->m == 0) return;
    dbh_assign_kernel<<<grid_for(g->m, kBlock), kBlock, 0, g->ctx->stream>>>(
        g->m, static_cast<uint32_t>(p), seed, g->eu.get(), g->ev.get(), g->degrees.get(), assign);
    SC_LAUNCH_CHECK();
    count_launch();
}

// ---- build_vertex_cut (partition.cpp:22-90) ------------------------------------------------
namespace {
__global__ void check_assign_kernel(int64_t m, int32_t p, const int32_t* a, int* bad) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x)
        if (a[e] < 0 || a[e] >= p) *bad = 1;
}
// per-part edge counts: a shared-memory histogram per block (p <= kHistParts), then one global add per
// (block, part) — instead of m global atomics on p counters
constexpr int kHistParts = 4096;
__global__ void count_parts_kernel(int64_t m, int32_t p, const int32_t* __restrict__ a, int32_t* part_count) {
    __shared__ int32_t h[kHistParts];
    const bool shared = p <= kHistParts;
    if (shared)
        for (int i = threadIdx.x; i < p; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m; e += int64_t(gridDim.x) * blockDim.x) {
        if (shared) atomicAdd(&h[a[e]], 1);
        else atomicAdd(&part_count[a[e]], 1);
    }
    __syncthreads();
    if (shared)
        for (int i = threadIdx.x; i < p; i += blockDim.x)
            if (h[i]) atomicAdd(&part_count[i], h[i]);
}
// Endpoints of part i's edges (perm[0 .. mi) = its global edge ids), then the isolated nodes it
// receives round-robin in ascending id, starting at part 0 (:45-50): iso[i], iso[i + p], ...
__global__ void part_endpoints_kernel(int64_t mi, const int32_t* __restrict__ perm, const int32_t* __restrict__ u,
                                      const int32_t* __restrict__ v, const int32_t* __restrict__ iso, int64_t niso_i,
                                      int32_t i, int32_t p, int32_t* out) {
    const int64_t total = 2 * mi + niso_i;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        if (k < 2 * mi) {
            const int32_t e = perm[k >> 1];
            out[k] = (k & 1) ? v[e] : u[e];
        } else {
            out[k] = iso[i + (k - 2 * mi) * p];
        }
    }
}
// per_node_rf (:316-321): one increment per part that contains the node (nodes are unique per part)
__global__ void rf_inc_kernel(int64_t nl, const int32_t* __restrict__ nodes, int32_t* rf) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nl; j += int64_t(gridDim.x) * blockDim.x)
        rf[nodes[j]] += 1;
}
__global__ void scatter_g2l_kernel(int64_t nl, const int32_t* __restrict__ nodes, int32_t* g2l, bool clear) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nl; j += int64_t(gridDim.x) * blockDim.x)
        g2l[nodes[j]] = clear ? -1 : static_cast<int32_t>(j);
}
struct IsDeg0 {
    const int32_t* deg;
    __host__ __device__ bool operator()(int32_t x) const { return deg[x] == 0; }
};
__global__ void local_edges_kernel(int64_t mi, const int32_t* __restrict__ perm, const int32_t* __restrict__ u,
                                   const int32_t* __restrict__ v, const int32_t* __restrict__ g2l, int32_t* lu,
                                   int32_t* lv, int32_t* gids) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < mi; k += int64_t(gridDim.x) * blockDim.x) {
        const int32_t e = perm[k];
        lu[k] = g2l[u[e]];
        lv[k] = g2l[v[e]];
        gids[k] = e;
    }
}
}  // namespace

std::unique_ptr<sc_vcut> build_vertex_cut_device(sc_graph* g, int32_t p, DevBuf<int32_t>&& assign) {
    if (p < 1) throw std::invalid_argument("num_parts must be >= 1");
    sc_ctx* ctx = g->ctx;
    cudaStream_t s = ctx->stream;
    const int64_t n = g->n, m = g->m;
    auto vc = std::make_unique<sc_vcut>();
    vc->g = g;
    vc->p = p;
    vc->assign = std::move(assign);
    DevBuf<int> bad(1);
    SC_CUDA(cudaMemsetAsync(bad.get(), 0, 4, s));
    if (m > 0) {
        check_assign_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(m, p, vc->assign.get(), bad.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    int hbad = 0;
    d2h(&hbad, bad.get(), 1, s);
    SC_CUDA(cudaStreamSynchronize(s));
    if (hbad) throw std::invalid_argument("edge assignment references an invalid part");

    // Sparse construction: no p x n arrays. Edge ids are stably sorted by part (ascending global
    // order within a part, :62-70); each part's node set is the sorted unique set of its edges'
    // endpoints plus its round-robin isolated nodes (= the reference's ascending membership scan,
    // :37-58); local ids come from a scratch n-array scattered and cleared per held part.
    DevBuf<int32_t> part_count(p);
    SC_CUDA(cudaMemsetAsync(part_count.get(), 0, p * 4, s));
    if (m > 0) {
        count_parts_kernel<<<grid_for(m, kBlock, int64_t(num_sms()) * 8), kBlock, 0, s>>>(m, p, vc->assign.get(),
                                                                                         part_count.get());
        SC_LAUNCH_CHECK();
        count_launch();
    }
    // isolated nodes, ascending
    DevBuf<int32_t> iso(std::max<int64_t>(n, 1));
    DevBuf<int64_t> niso_dev(1);
    int64_t niso = 0;
    if (n > 0) {
        cub::CountingInputIterator<int32_t> ids(0);
        size_t tb = 0;
        cub::DeviceSelect::If(nullptr, tb, ids, iso.get(), niso_dev.get(), n, IsDeg0{g->degrees.get()}, s);
        cub::DeviceSelect::If(ctx->temp(tb), tb, ids, iso.get(), niso_dev.get(), n, IsDeg0{g->degrees.get()}, s);
        d2h(&niso, niso_dev.get(), 1, s);
        count_launch(2);
    }
    vc->own_rank = g->own_rank;
    vc->own_world = g->own_world;
    vc->parts.resize(p);
    vc->per_node_rf.alloc(std::max<int64_t>(n, 1));
    SC_CUDA(cudaMemsetAsync(vc->per_node_rf.get(), 0, vc->per_node_rf.bytes(), s));
    std::vector<int32_t> counts(p, 0);
    d2h(counts.data(), part_count.get(), p, s);
    DevBuf<int32_t> perm(std::max<int64_t>(m, 1));
    if (m > 0) {
        DevBuf<int32_t> idx(m), keys_out(m);
        iota_kernel<<<grid_for(m, kBlock), kBlock, 0, s>>>(idx.get(), m);
        SC_LAUNCH_CHECK();
        size_t tb = 0;
        const int eb = bits_for(static_cast<uint64_t>(p));
        cub::DeviceRadixSort::SortPairs(nullptr, tb, vc->assign.get(), keys_out.get(), idx.get(), perm.get(), m, 0, eb,
                                        s);
        cub::DeviceRadixSort::SortPairs(ctx->temp(tb), tb, vc->assign.get(), keys_out.get(), idx.get(), perm.get(), m,
                                        0, eb, s);
        count_launch(3);
        SC_CUDA(cudaStreamSynchronize(s));  // idx / keys_out are freed on scope exit
    }
    SC_CUDA(cudaStreamSynchronize(s));
    int64_t max_ends = 1;
    for (int32_t i = 0; i < p; ++i) {
        const int64_t niso_i = niso > i ? (niso - i + p - 1) / p : 0;
        max_ends = std::max<int64_t>(max_ends, 2 * int64_t(counts[i]) + niso_i);
    }
    DevBuf<int32_t> ends(max_ends), ends_sorted(max_ends), uniq(max_ends);
    DevBuf<int64_t> nuniq(1);
    bool any_held = false;
    for (int32_t i = 0; i < p; ++i) any_held |= g->owns(i);
    DevBuf<int32_t> g2l_scr;  // -1 everywhere between held parts
    if (any_held && n > 0) {
        g2l_scr.alloc(n);
        fill(g2l_scr.get(), n, int32_t(-1), s);
    }
    const int nb = bits_for(static_cast<uint64_t>(std::max<int64_t>(n, 1)));
    int64_t start = 0;
    for (int32_t i = 0; i < p; ++i) {
        PartDev& pd = vc->parts[i];
        pd.held = g->owns(i);
        pd.m_local = counts[i];
        const int64_t mi = pd.m_local;
        const int64_t niso_i = niso > i ? (niso - i + p - 1) / p : 0;
        const int64_t ne = 2 * mi + niso_i;
        int64_t nl = 0;
        if (ne > 0) {
            part_endpoints_kernel<<<grid_for(ne, kBlock), kBlock, 0, s>>>(mi, perm.get() + start, g->eu.get(),
                                                                           g->ev.get(), iso.get(), niso_i, i, p,
                                                                           ends.get());
            SC_LAUNCH_CHECK();
            size_t tb = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tb, ends.get(), ends_sorted.get(), ne, 0, nb, s);
            cub::DeviceRadixSort::SortKeys(ctx->temp(tb), tb, ends.get(), ends_sorted.get(), ne, 0, nb, s);
            tb = 0;
            cub::DeviceSelect::Unique(nullptr, tb, ends_sorted.get(), uniq.get(), nuniq.get(), ne, s);
            cub::DeviceSelect::Unique(ctx->temp(tb), tb, ends_sorted.get(), uniq.get(), nuniq.get(), ne, s);
            d2h(&nl, nuniq.get(), 1, s);
            SC_CUDA(cudaStreamSynchronize(s));
            if (nl > 0) rf_inc_kernel<<<grid_for(nl, kBlock), kBlock, 0, s>>>(nl, uniq.get(), vc->per_node_rf.get());
            SC_LAUNCH_CHECK();
            count_launch(6);
        }
        pd.n_local = nl;
        if (!pd.held) {
            start += mi;
            continue;
        }
        pd.nodes.alloc(std::max<int64_t>(nl, 1));
        if (nl > 0) {
            SC_CUDA(cudaMemcpyAsync(pd.nodes.get(), uniq.get(), nl * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
            scatter_g2l_kernel<<<grid_for(nl, kBlock), kBlock, 0, s>>>(nl, pd.nodes.get(), g2l_scr.get(), false);
            SC_LAUNCH_CHECK();
            count_launch();
        }
        pd.lu.alloc(std::max<int64_t>(mi, 1));
        pd.lv.alloc(std::max<int64_t>(mi, 1));
        pd.edge_gids.alloc(std::max<int64_t>(mi, 1));
        if (mi > 0) {
            local_edges_kernel<<<grid_for(mi, kBlock), kBlock, 0, s>>>(mi, perm.get() + start, g->eu.get(), g->ev.get(),
                                                                       g2l_scr.get(), pd.lu.get(), pd.lv.get(),
                                                                       pd.edge_gids.get());
            SC_LAUNCH_CHECK();
            count_launch();
        }
        if (nl > 0) {
            scatter_g2l_kernel<<<grid_for(nl, kBlock), kBlock, 0, s>>>(nl, pd.nodes.get(), g2l_scr.get(), true);
            SC_LAUNCH_CHECK();
            count_launch();
        }
        start += mi;
        pd.local_deg.alloc(std::max<int64_t>(pd.n_local, 1));
        pd.offsets.alloc(pd.n_local + 1);
        pd.nbrs.alloc(std::max<int64_t>(2 * mi, 1));
        pd.eids.alloc(std::max<int64_t>(2 * mi, 1));
        build_csr(ctx, pd.n_local, mi, pd.lu.get(), pd.lv.get(), pd.offsets.get(), pd.nbrs.get(), pd.eids.get(),
                  pd.local_deg.get());
    }
    SC_CUDA(cudaStreamSynchronize(s));
    return vc;
}

// global_to_local of a held part (partition.hpp:20): -1 everywhere, then j at nodes[j]
void part_g2l_device(const sc_vcut* vc, int32_t part, int32_t* out_dev) {
    const PartDev& pd = vc->held(part);
    cudaStream_t s = vc->g->ctx->stream;
    const int64_t n = vc->g->n;
    if (n == 0) return;
    fill(out_dev, n, int32_t(-1), s);
    if (pd.n_local > 0) {
        scatter_g2l_kernel<<<grid_for(pd.n_local, kBlock), kBlock, 0, s>>>(pd.n_local, pd.nodes.get(), out_dev, false);
        SC_LAUNCH_CHECK();
        count_launch(2);
    }
}

// ---- reweight.cpp:23-71 --------------------------------------------------------------
namespace {
__global__ void weights_kernel(int64_t nl, int scheme, const int32_t* __restrict__ nodes,
                               const int32_t* __restrict__ ld, const int32_t* __restrict__ gdeg,
                               const int32_t* __restrict__ rf, double* w, int* logic_err) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < nl; j += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = nodes[j];
        double x = 1.0;
        if (scheme == 0) {
            const int32_t gd = gdeg[v];
            if (gd == 0) {
                if (ld[j] != 0) *logic_err = 1;
                x = 1.0;  // round-robin isolated node keeps its supervision
            } else {
                x = static_cast<double>(ld[j]) / static_cast<double>(gd);
            }
        } else if (scheme == 1) {
            x = 1.0 / static_cast<double>(rf[v]);
        }
        w[j] = x;
    }
}
}  // namespace

void compute_weights_device(sc_vcut* vc, int scheme, int32_t part, double* out_dev) {
    const PartDev& pd = vc->held(part);
    if (pd.n_local == 0) return;
    DevBuf<int> err(1);
    cudaStream_t s = vc->g->ctx->stream;
    SC_CUDA(cudaMemsetAsync(err.get(), 0, 4, s));
    weights_kernel<<<grid_for(pd.n_local, kBlock), kBlock, 0, s>>>(pd.n_local, scheme, pd.nodes.get(),
                                                                   pd.local_deg.get(), vc->g->degrees.get(),
                                                                   vc->per_node_rf.get(), out_dev, err.get());
    SC_LAUNCH_CHECK();
    count_launch();
    int h = 0;
    d2h(&h, err.get(), 1, s);
    SC_CUDA(cudaStreamSynchronize(s));
    if (h) throw std::logic_error("dar_weights: local edges on a degree-0 node");
}

// ---- make_sage_model init (nn.hpp:73-102) ----------------------------------------------
// Draw k of the init stream goes to flat parameter k (matrices in for_each_matrix
// order, each row-major); the matrix of k (its Glorot bound) is found by binary
// search over the nmat + 1 matrix offsets, so any layer count works.
namespace {
__global__ void init_kernel(int64_t total, uint64_t s, int32_t nmat, const int64_t* __restrict__ start,
                            const double* __restrict__ bound, float* out) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
        int32_t lo = 0, hi = nmat - 1;  // last matrix with start <= k
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (start[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        const double r = u64_to_double(draw_u64(s, static_cast<uint64_t>(k)));
        out[k] = static_cast<float>(bound[lo] * (2.0 * r - 1.0));
    }
}
}  // namespace

void init_params_device(sc_ctx* ctx, int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t classes,
                        uint64_t seed, float* out_dev) {
    if (in_dim < 1 || classes < 1) throw std::invalid_argument("make_sage_model: dimensions must be positive");
    std::vector<int64_t> start;
    std::vector<double> bound;
    int64_t off = 0;
    int64_t in = in_dim;
    auto add = [&](int64_t r, int64_t c) {
        start.push_back(off);
        bound.push_back(std::sqrt(6.0 / static_cast<double>(r + c)));
        off += r * c;
    };
    for (int32_t l = 0; l < layers; ++l) {
        if (hidden[l] < 1) throw std::invalid_argument("make_sage_model: hidden dims must be positive");
        add(hidden[l], in);
        add(hidden[l], hidden[l] + in);
        in = hidden[l];
    }
    add(classes, in);
    const int32_t nmat = static_cast<int32_t>(start.size());
    cudaStream_t s = ctx->stream;
    DevBuf<int64_t> d_start(nmat);
    DevBuf<double> d_bound(nmat);
    h2d(d_start.get(), start.data(), nmat, s);
    h2d(d_bound.get(), bound.data(), nmat, s);
    init_kernel<<<grid_for(off, kBlock), kBlock, 0, s>>>(off, substream(seed, "init"), nmat, d_start.get(),
                                                         d_bound.get(), out_dev);
    SC_LAUNCH_CHECK();
    count_launch();
    SC_CUDA(cudaStreamSynchronize(s));  // the offset tables are freed on return
}

}  // namespace sc
