// trainer.cu — train_cofree_impl (proj/include/sagecut/trainer.hpp:202-313) on
// the device: one rank per GPU owns partitions i with i % world == rank, runs
// their forward / loss / backward back to back on one stream, all-gathers each
// per-partition gradient bucket (one parameter matrix) over NCCL on a comm
// stream as soon as backward produces it, then every rank sums the slots in
// ascending partition order (the reference's gather_gradients,
// trainer.hpp:79-94) and applies the same Adam step.
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "gemm_tc.cuh"
#include "internal.hpp"
#include "nn.cuh"
#include "trainer.hpp"

namespace sc {

#define SC_NCCL(expr)                                                                                        \
    do {                                                                                                     \
        ncclResult_t sc_r_ = (expr);                                                                         \
        if (sc_r_ != ncclSuccess) throw ::sc::NcclError(std::string(#expr) + ": " + ncclGetErrorString(sc_r_)); \
    } while (0)

// ---- per-kernel event profiler (bench.py roofline) ---------------------------
void Profiler::begin(const char* name, double bytes, cudaStream_t s, double flops) {
    if (!enabled) return;
    if (used == events.size()) {
        cudaEvent_t a, b;
        SC_CUDA(cudaEventCreate(&a));
        SC_CUDA(cudaEventCreate(&b));
        events.push_back({a, b});
    }
    cur_name = name;
    cur_bytes = bytes;
    cur_flops = flops;
    SC_CUDA(cudaEventRecord(events[used].first, s));
}
void Profiler::end(cudaStream_t s) {
    if (!enabled) return;
    SC_CUDA(cudaEventRecord(events[used].second, s));
    records.push_back({cur_name, cur_bytes, cur_flops, used});
    ++used;
}
void Profiler::collect() {
    if (!enabled) return;
    totals.clear();
    for (const auto& r : records) {
        float ms = 0.f;
        SC_CUDA(cudaEventElapsedTime(&ms, events[r.slot].first, events[r.slot].second));
        auto& t = totals[r.name];
        t.ms += ms;
        t.bytes += r.bytes;
        t.flops += r.flops;
        t.calls += 1;
    }
    records.clear();
    used = 0;
}
Profiler::~Profiler() {
    for (auto& e : events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
}

}  // namespace sc

using namespace sc;

cudaEvent_t sc_trainer::fork_event() {
    if (fork_used == fork_events.size()) {
        cudaEvent_t e;
        SC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        fork_events.push_back(e);
    }
    return fork_events[fork_used++ % fork_events.size()];
}

sc_trainer::~sc_trainer() {
    if (comm) ncclCommDestroy(comm);
    for (cudaEvent_t e : fork_events) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (host) cudaFreeHost(host);
    if (xhost) cudaFreeHost(xhost);
    for (cudaEvent_t e : xfer_events) cudaEventDestroy(e);
    if (comm_done) cudaEventDestroy(comm_done);
    if (comm_stream) cudaStreamDestroy(comm_stream);
}

namespace sc {

namespace {
// Model layout (SageModel::for_each_matrix order), parameters initialised by
// make_sage_model, optimizer state, gradient buckets and the per-operand
// |max| slots: everything but the partitions.
void init_model(sc_trainer* t) {
    sc_graph* g = t->g;
    t->d = g->dim;
    t->dp = (t->d + 3) / 4 * 4;
    t->C = g->num_classes;
    t->Cp = (t->C + 3) / 4 * 4;  // logits / dlogits row stride: 16-byte rows for the tensor-core kernels
    int64_t off = 0;
    int in = t->d;
    t->lay.clear();
    for (int l = 0; l < t->L; ++l) {
        LayerOff lo;
        lo.in = in;
        lo.H = t->hidden[l];
        lo.W = off;
        off += int64_t(lo.H) * in;
        lo.U = off;
        off += int64_t(lo.H) * (lo.H + in);
        t->lay.push_back(lo);
        in = lo.H;
    }
    t->E = in;
    t->head_off = off;
    off += int64_t(t->C) * t->E;
    t->P = off;
    t->theta.alloc(t->P);
    init_params_device(t->ctx, t->d, t->hidden.data(), t->L, t->C, t->seed, t->theta.get());
    t->amax.alloc(sc_trainer::kSlotBase + 2 * std::max(t->L, 1));
    t->tc.init(t);
    const char* e = std::getenv("SC_FUSE_TOP");
    t->fuse_top = t->L >= 1 && t->tc.enabled && !(e && e[0] == '0');
    if (t->fuse_top) {
        const LayerOff& lo = t->lay[t->L - 1];
        t->Z.alloc(int64_t(t->Cp) * (lo.H + lo.in));
        SC_CUDA(cudaMemsetAsync(t->Z.get(), 0, t->Z.bytes(), t->ctx->stream));
        t->Xp.alloc(int64_t(t->C) * (lo.H + lo.in));
        t->z_version = 0;
        e = std::getenv("SC_PTA");
        t->pta = 2 * t->Cp <= lo.H && !(e && e[0] == '0');
    }
}

// Z = head U_{L-1} (C x (H + in)) for the current weights (composed top layer)
void ensure_z(sc_trainer* t, cudaStream_t s) {
    if (t->z_version == t->tc.version) return;
    const LayerOff& lo = t->lay[t->L - 1];
    const int zl = lo.H + lo.in;
    small_gemm(t->C, zl, lo.H, t->theta.get() + t->head_off, t->E, false, t->theta.get() + lo.U, zl, false,
               t->Z.get(), zl, s);
    t->z_version = t->tc.version;
}
}  // namespace

void trainer_init(sc_trainer* t) {
    sc_graph* g = t->g;
    sc_vcut* vc = t->vc;
    if (!(t->lr > 0.0)) throw std::invalid_argument("learning rate must be > 0");
    if (t->L < 0) throw std::invalid_argument("layers must be >= 0");
    for (int h : t->hidden)
        if (h < 1) throw std::invalid_argument("hidden dims must be positive");
    if (t->use_dropedge) {
        if (t->K < 1) throw std::invalid_argument("dropedge_k must be >= 1");
        if (t->ratio < 0.0 || t->ratio >= 1.0) throw std::invalid_argument("drop_ratio must lie in [0, 1)");
    }
    if (g->dim == 0) throw std::invalid_argument("training requires node features");
    if (g->num_classes == 0) throw std::invalid_argument("training requires labels");
    if (t->loss == 0 && g->multilabel)  // trainer.hpp:207-208
        throw std::invalid_argument("softmax_ce requires multi-class labels");
    if (vc->g != g || vc->parts.empty()) throw std::invalid_argument("train_cofree: partition does not match graph");
    if (g->train_count == 0) throw std::invalid_argument("training requires a non-empty train mask");
    if (t->world < 1 || t->rank < 0 || t->rank >= t->world) throw std::invalid_argument("bad rank/world");
    for (int i = t->rank; i < vc->p; i += t->world)  // every partition this rank trains must be materialised
        (void)vc->held(i);
    cudaStream_t s = t->ctx->stream;
    t->normalizer = static_cast<double>(g->train_count);
    t->p = vc->p;
    init_model(t);
    t->m1.alloc(t->P);
    t->m2.alloc(t->P);
    t->gathered.alloc(t->P);
    // gradient buckets: one per matrix, for_each_matrix order (W_l, U_l, ..., head)
    t->b_off.clear();
    for (const LayerOff& lo : t->lay) {
        t->b_off.push_back(lo.W);
        t->b_off.push_back(lo.U);
    }
    t->b_off.push_back(t->head_off);
    t->b_off.push_back(t->P);
    t->b_off_dev.alloc(t->b_off.size());
    SC_CUDA(cudaMemcpyAsync(t->b_off_dev.get(), t->b_off.data(), t->b_off.size() * sizeof(int64_t),
                            cudaMemcpyHostToDevice, s));
    t->pp = (t->p + t->world - 1) / t->world * t->world;
    t->slots.alloc(int64_t(t->pp) * t->P);
    SC_CUDA(cudaMemsetAsync(t->m1.get(), 0, t->m1.bytes(), s));
    SC_CUDA(cudaMemsetAsync(t->m2.get(), 0, t->m2.bytes(), s));
    SC_CUDA(cudaMemsetAsync(t->slots.get(), 0, t->slots.bytes(), s));

    // per-partition inputs (trainer.hpp:218-243)
    {
        int64_t rows = 0;
        for (int i = t->rank; i < t->p; i += t->world) rows += vc->parts[i].n_local;
        size_t free_b = 0, total_b = 0;
        SC_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const double budget = 0.15 * static_cast<double>(free_b);  // each cache: at most 15 % of free memory
        const char* e = std::getenv("SC_SHARED_X0");
        t->shared_x0 = e ? std::atoi(e) != 0 : 4.0 * rows * t->dp > budget;
        e = std::getenv("SC_SHARED_LOGITS");
        t->shared_logits = e ? std::atoi(e) != 0 : 4.0 * rows * t->Cp > budget;
    }
    int64_t n_max = 1, nnz_max = 1;
    t->local.clear();
    for (int i = t->rank; i < t->p; i += t->world) t->local.push_back(i);
    t->ps.resize(t->p);
    for (int i = 0; i < t->p; ++i) {
        PartState& st = t->ps[i];
        const PartDev& pd = vc->parts[i];
        st.n = pd.n_local;
        st.nnz = 2 * pd.m_local;
        const bool mine = (i % t->world) == t->rank;
        if (!mine) continue;
        n_max = std::max(n_max, st.n);
        nnz_max = std::max(nnz_max, st.nnz);
        st.w.alloc(std::max<int64_t>(st.n, 1));
        st.scale.alloc(std::max<int64_t>(st.n, 1));
        compute_weights_device(vc, t->reweight, i, st.w.get());
        loss_weights(t, i);
        // |dloss/dlogits| <= scale = w / normalizer (|softmax - onehot|, |sigmoid - y| <= 1)
        st.g_amax.alloc(1);
        SC_CUDA(cudaMemsetAsync(st.g_amax.get(), 0, sizeof(float), s));
        absmax(st.n, st.scale.get(), st.g_amax.get(), s);
        if (!t->shared_logits) st.logits.alloc(std::max<int64_t>(st.n * t->Cp, 1));
        build_heavy_rows(t->ctx, st.n, pd.offsets.get(), st.heavy);
        if (!t->shared_x0) st.x0.alloc(std::max<int64_t>(st.n * t->dp, 1));
        if (t->use_dropedge) {
            st.words = (st.nnz + 31) / 32;
            st.bits.alloc(std::max<int64_t>(st.words * t->K, 1));
            DevBuf<uint8_t> masks(std::max<int64_t>(pd.m_local * t->K, 1));
            // partition_mask_set (trainer.hpp:117-121)
            precompute_masks_device(t->ctx, pd.m_local, t->K, t->ratio, substream(t->seed, "dropedge", uint64_t(i)),
                                    masks.get());
            for (int k = 0; k < t->K; ++k)
                mask_to_bits(st.nnz, pd.eids.get(), masks.get() + int64_t(k) * pd.m_local, st.bits.get() + k * st.words,
                             s);
            SC_CUDA(cudaStreamSynchronize(s));
        }
    }
    t->part_loss.alloc(t->pp);
    SC_CUDA(cudaMemsetAsync(t->part_loss.get(), 0, t->part_loss.bytes(), s));
    t->out2.alloc(2);
    if (!t->host) {
        void* h = nullptr;
        SC_CUDA(cudaMallocHost(&h, sizeof(sc_trainer::HostOut)));
        t->host = static_cast<sc_trainer::HostOut*>(h);
        *t->host = sc_trainer::HostOut{{0, 0}, 0};
    }
    t->nonfinite.alloc(1);
    t->red_partial.alloc(1024);
    if (t->shared_x0) t->x0_shared.alloc(std::max<int64_t>(n_max * t->dp, 1));
    if (t->shared_logits) t->logits_shared.alloc(std::max<int64_t>(n_max * t->Cp, 1));
    {  // compact activations when the full per-layer set would not leave headroom
        const char* e = std::getenv("SC_COMPACT_ACTS");
        t->compact = false;
        if (e) {
            t->compact = std::atoi(e) != 0;
        } else {
            size_t free_b = 0, total_b = 0;
            SC_CUDA(cudaMemGetInfo(&free_b, &total_b));
            const double full = 4.0 * static_cast<double>(carve_train(t, nullptr, n_max));
            t->compact = full > 0.85 * static_cast<double>(free_b) - 2e9;
        }
    }
    ensure_rows(t, n_max);
    int64_t max_seg = 0;
    for (int i : t->local) max_seg = std::max<int64_t>(max_seg, t->ps[i].heavy.nseg);
    int32_t maxH = 1;
    for (auto& lo : t->lay) maxH = std::max(maxH, lo.H);
    if (max_seg) t->heavy_ws.alloc(max_seg * maxH);
    int32_t maxN1 = t->C, maxN2 = t->E;
    for (auto& lo : t->lay) {
        maxN1 = std::max(maxN1, 2 * lo.H);  // the dual dU + dW launch: A = [dh | dz]
        maxN2 = std::max(maxN2, lo.H + lo.in);
    }
    t->ws_floats = gemm_tn_workspace_floats(maxN1, maxN2);
    t->ws.alloc(t->ws_floats);
    if (const char* o = std::getenv("SC_OVERLAP")) t->overlap = std::atoi(o) != 0;
    if (t->overlap) {
        t->ws_side.alloc(t->ws_floats);
        int least = 0, greatest = 0;
        SC_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SC_CUDA(cudaStreamCreateWithPriority(&t->side, cudaStreamNonBlocking, greatest));
    }
    SC_CUDA(cudaStreamSynchronize(s));
}

void trainer_init_eval_only(sc_trainer* t) {
    sc_graph* g = t->g;
    if (t->L < 0) throw std::invalid_argument("layers must be >= 0");
    for (int h : t->hidden)
        if (h < 1) throw std::invalid_argument("make_sage_model: hidden dims must be positive");
    if (g->dim == 0 || g->num_classes == 0) throw std::invalid_argument("evaluate: graph lacks features or labels");
    t->eval_only = true;
    init_model(t);
    SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
}

// loss weight = train_mask ? scheme weight : 0; scale = (float)(w / normalizer)
__global__ void loss_weight_kernel(int64_t n, const int32_t* nodes, const uint8_t* train, double* w, float* scale,
                                   double normalizer) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
        const double x = train[nodes[j]] ? w[j] : 0.0;
        w[j] = x;
        scale[j] = static_cast<float>(x / normalizer);
    }
}

void loss_weights(sc_trainer* t, int i) {
    PartState& st = t->ps[i];
    if (st.n == 0) return;
    loss_weight_kernel<<<grid_for(st.n, 256), 256, 0, t->ctx->stream>>>(
        st.n, t->vc->parts[i].nodes.get(), t->g->train.get(), st.w.get(), st.scale.get(), t->normalizer);
    SC_LAUNCH_CHECK();
    count_launch();
}

namespace {
// 256-byte-aligned sub-buffers of one allocation (base null: sizing pass).
struct Carver {
    float* base = nullptr;
    size_t off = 0;
    float* take(size_t floats) {
        float* p = base ? base + off : nullptr;
        off += (std::max<size_t>(floats, 1) + 63) / 64 * 64;
        return p;
    }
};
int32_t max_hidden(const sc_trainer* t) {
    int32_t h = std::max<int32_t>(t->E, 1);
    for (auto& lo : t->lay) h = std::max(h, lo.H);
    return h;
}
}  // namespace

size_t carve_train(sc_trainer* t, float* base, int64_t n) {
    Carver c{base};
    const int32_t maxH = max_hidden(t);
    int32_t maxW = std::max<int32_t>(std::max(t->E, t->d), maxH);
    for (auto& lo : t->lay) maxW = std::max(maxW, std::max(lo.H, lo.in));
    t->X.assign(t->L + 1, nullptr);
    t->MSG.assign(t->L, nullptr);
    t->MEAN.assign(t->L, nullptr);
    t->POS.assign(t->L, nullptr);
    // X[L] (the embedding) is never formed when the top layer is composed with the head
    for (int l = 0; l < t->L; ++l)
        if (!(t->fuse_top && l == t->L - 1)) t->X[l + 1] = c.take(size_t(n) * t->lay[l].H);
    float* shared_msg = t->compact && t->L > 0 ? c.take(size_t(n) * maxH) : nullptr;
    for (int l = 0; l < t->L; ++l) {
        t->MSG[l] = t->compact ? shared_msg : c.take(size_t(n) * t->lay[l].H);
        t->MEAN[l] = c.take(size_t(n) * t->lay[l].H);
        // sign bits: compact activations (every layer), or the projected top layer's dz mask
        if (t->compact || (t->pta && l == t->L - 1))
            t->POS[l] = reinterpret_cast<uint32_t*>(c.take(size_t(n) * ((t->lay[l].H + 31) / 32)));
    }
    t->inv = c.take(n);
    t->G = c.take(size_t(n) * t->Cp);
    t->dh = c.take(size_t(n) * maxW);
    t->dmean = c.take(size_t(n) * maxW);  // also the dh ping-pong partner (backward)
    t->dz = c.take(size_t(n) * maxH);
    return c.off;
}

void ensure_rows(sc_trainer* t, int64_t n) {
    if (n <= t->rows_cap) return;
    t->rows_cap = n;
    const size_t need = carve_train(t, nullptr, n);
    t->arena.ensure(need);
    carve_train(t, t->arena.get(), n);
    t->row_loss.alloc(n);
    t->eval_logits.release();
}

namespace {

struct Rows {
    int64_t n;
    const int64_t* offsets;
    const int32_t* nbrs;
    const uint32_t* bits;
    const int32_t* nodes;  // local -> global row (features / labels); null = identity
    int64_t nnz;           // CSR slots
    int64_t kept;          // CSR slots kept by the selected DropEdge mask
    const float* g_amax;   // bound on max|dloss/dlogits| (= max loss scale)
    const float* x0;       // layer-0 input rows (the partition's gathered features)
    int64_t x0_ld;         // their pitch (dp for gathered rows: zero-padded to 16 bytes)
    const HeavyRows* hv;   // hub rows (segmented aggregation)
};

// Algorithmic HBM bytes of one aggregation launch: offsets,
// neighbour ids, mask bits, inv_deg (fwd) or ReLU-mask rows (bwd), one gathered
// fp32 row per kept slot, and the output rows.
double spmm_bytes(const Rows& R, int H, bool bwd) {
    double b = 8.0 * (R.n + 1) + 4.0 * R.nnz + (R.bits ? (R.nnz + 7) / 8 : 0) + 4.0 * H * R.kept + 4.0 * H * R.n;
    b += bwd ? 4.0 * H * R.n : 4.0 * R.n;
    return b;
}

// Activation buffers of one forward pass: X[l] (layer inputs, l >= 1), MSG[l],
// MEAN[l], inv. Training keeps one buffer per layer (the backward's cache);
// evaluation may alias them (ping-pong X, one MSG, one MEAN).
struct Acts {
    std::vector<float*> X, MSG, MEAN;
    std::vector<uint32_t*> POS;  // ReLU sign bits of MSG[l] (compact training), else null
    float* inv = nullptr;
};
Acts train_acts(sc_trainer* t) {
    Acts a;
    a.X = t->X;
    a.MSG = t->MSG;
    a.MEAN = t->MEAN;
    a.POS = t->POS;
    a.inv = t->inv;
    return a;
}

// sage_forward (nn.hpp:192-242). Writes logits; the cache lands in A.
void forward(sc_trainer* t, const Rows& R, float* logits, const Acts& A) {
    cudaStream_t s = t->ctx->stream;
    Profiler& P = t->prof;
    const int64_t n = R.n;
    P.begin("inv_degree", double(n) * 12 + double(R.offsets ? 8 : 0) * n, s);
    inv_degree(n, R.offsets, R.bits, A.inv, s);
    P.end(s);
    const MatA x0{R.x0, R.x0_ld, nullptr, t->d};
    for (int l = 0; l < t->L; ++l) {
        const LayerOff& lo = t->lay[l];
        const MatA xin = l == 0 ? x0 : MatA{A.X[l], lo.in, nullptr, lo.in};
        const float* xin_amax = l == 0 ? t->g->feat_amax.get() : t->amax_x(l);
        // msg = relu(h W^T)   (nn.hpp:220-221)
        P.begin("gemm_msg", 4.0 * n * (lo.in + lo.H), s, 2.0 * n * lo.in * lo.H);
        t->tc.nt(t, xin, xin_amax, MatB{t->theta.get() + lo.W, lo.in, false}, nullptr, nullptr, nullptr,
                 A.MSG[l], lo.H, n, lo.H, kEpiRelu, nullptr, t->amax_msg(l), A.POS.empty() ? nullptr : A.POS[l]);
        P.end(s);
        if (t->pta && l == t->L - 1) {
            // logits = h Z_R^T + inv * sum_kept (msg Z_L^T)[nbr]: the projection P = msg Z_L^T (Cp wide,
            // into MEAN[l]'s buffer) is aggregated instead of msg (nn.hpp:222-234, 240 re-associated)
            ensure_z(t, s);
            const int zl = lo.H + lo.in;
            float* proj = A.MEAN[l];
            P.begin("gemm_head", 4.0 * n * (lo.H + lo.in + 2 * t->Cp), s, 2.0 * n * zl * t->C);
            t->tc.nt(t, MatA{A.MSG[l], lo.H, nullptr, lo.H}, t->amax_msg(l), MatB{t->Z.get(), zl, false}, nullptr,
                     nullptr, nullptr, proj, t->Cp, n, t->Cp, kEpiNone, nullptr, nullptr);
            t->tc.nt(t, xin, xin_amax, MatB{t->Z.get() + lo.H, zl, false}, nullptr, nullptr, nullptr, logits, t->Cp, n,
                     t->Cp, kEpiNone, nullptr, nullptr);
            P.end(s);
            P.begin("spmm_fwd_top", spmm_bytes(R, t->Cp, false) + 4.0 * n * t->Cp, s);
            spmm_fwd_add(n, t->Cp, R.offsets, R.nbrs, R.bits, A.inv, proj, logits, s, R.hv, t->heavy_ws.get());
            P.end(s);
            return;
        }
        // mean = inv * sum_kept msg[nbr]   (nn.hpp:222-230)
        P.begin("spmm_fwd", spmm_bytes(R, lo.H, false), s);
        spmm_fwd(n, lo.H, R.offsets, R.nbrs, R.bits, A.inv, A.MSG[l], A.MEAN[l], s, R.hv, t->heavy_ws.get());
        P.end(s);
        if (t->fuse_top && l == t->L - 1) {
            // logits = h_L head^T = mean Z_L^T + h Z_R^T   (nn.hpp:233-234, 240 composed)
            ensure_z(t, s);
            const int zl = lo.H + lo.in;
            const MatA mean{A.MEAN[l], lo.H, nullptr, lo.H};
            const MatB zL{t->Z.get(), zl, false}, zR{t->Z.get() + lo.H, zl, false};
            P.begin("gemm_head", 4.0 * n * (lo.H + lo.in + t->C), s, 2.0 * n * zl * t->C);
            t->tc.nt(t, mean, t->amax_msg(l), zL, &xin, xin_amax, &zR, logits, t->Cp, n, t->C, kEpiNone, nullptr,
                     nullptr);
            P.end(s);
            return;
        }
        // h' = mean U_L^T + h U_R^T   (nn.hpp:233-234)
        const MatB uL{t->theta.get() + lo.U, lo.H + lo.in, false};
        const MatB uR{t->theta.get() + lo.U + lo.H, lo.H + lo.in, false};
        const MatA mean{A.MEAN[l], lo.H, nullptr, lo.H};
        P.begin("gemm_update", 4.0 * n * (2 * lo.H + lo.in), s, 2.0 * n * (lo.H + lo.in) * lo.H);
        // |mean| <= max|msg| (a mean of msg rows): msg's bound scales it.
        t->tc.nt(t, mean, t->amax_msg(l), uL, &xin, xin_amax, &uR, A.X[l + 1], lo.H, n, lo.H, kEpiNone, nullptr,
                 t->amax_x(l + 1));
        P.end(s);
    }
    const MatA emb = t->L == 0 ? x0 : MatA{A.X[t->L], t->E, nullptr, t->E};
    P.begin("gemm_head", 4.0 * n * (t->E + t->C), s, 2.0 * n * t->E * t->C);
    const float* emb_amax = t->L == 0 ? t->g->feat_amax.get() : t->amax_x(t->L);
    t->tc.nt(t, emb, emb_amax, MatB{t->theta.get() + t->head_off, t->E, false}, nullptr, nullptr, nullptr, logits,
             t->Cp, n, t->C, kEpiNone, nullptr, nullptr);
    P.end(s);
}

// Layers l = top .. 0 of sage_backward (nn.hpp:262-291) given dh of layer `top` in `dh` (amax in
// dh_amax); layer top's dmean / dU come from the caller when `top_done` (composed top layer).
// top_done: 0 none; 1 the composed top layer's dmean is in dh2 and its dU done (backward_fused);
// 2 also its dz (projected top-layer aggregation).
void backward_layers(sc_trainer* t, const Rows& R, int i, int top, float* dh, float* dh_amax, float* dh2,
                     float* dh2_amax, int top_done);

// The composed top layer's backward (see sc_trainer::fuse_top), then layers L-2 .. 0 as usual.
void backward_fused(sc_trainer* t, const Rows& R, int i) {
    const int round = i / t->world;
    cudaStream_t s = t->ctx->stream;
    Profiler& P = t->prof;
    const int64_t n = R.n;
    const int T = t->L - 1;
    const LayerOff& lo = t->lay[T];
    const int zl = lo.H + lo.in;
    const MatT x0t{R.x0, R.x0_ld, nullptr, t->d};
    const MatT xint = T == 0 ? x0t : MatT{t->X[T], lo.in, nullptr, lo.in};
    const float* xin_amax = T == 0 ? t->g->feat_amax.get() : t->amax_x(T);
    const MatT meant{t->MEAN[T], lo.H, nullptr, lo.H};
    const MatT gt{t->G, t->Cp, nullptr, t->C};
    const MatA ga{t->G, t->Cp, nullptr, t->C};
    // Xp = G^T [mean | h_in]; dHead = Xp U^T (nn.hpp:259 with emb = mean U_L^T + h U_R^T);
    // dU = head^T Xp (:271-272 with dh = G head)
    ensure_z(t, s);
    float* dh2 = t->dmean;
    float* dh2_amax = t->amax_slot(sc_trainer::kSlotDh1);
    float* ghat_amax = t->amax_slot(sc_trainer::kSlotDh0);
    if (t->pta) {
        // G^T mean = G^T D^-1 A msg = Ghat^T msg with Ghat = A^T (inv * G): one Cp-wide pull aggregation
        // (A symmetric; the same kept-slot sums as :277-286) instead of the H-wide mean / dmean.
        float* ghat = t->dh;
        P.begin("spmm_bwd_top", spmm_bytes(R, t->Cp, false), s);
        SC_CUDA(cudaMemsetAsync(ghat_amax, 0, sizeof(float), s));
        spmm_sum_scaled(n, t->Cp, R.offsets, R.nbrs, R.bits, t->inv, t->G, ghat, s, ghat_amax, R.hv,
                        t->heavy_ws.get());
        P.end(s);
        const MatT msgt{t->MSG[T], lo.H, nullptr, lo.H};
        P.begin("wgrad", 4.0 * n * (2 * t->C + zl), s, 2.0 * n * t->C * zl);
        t->tc.tn(t, MatT{ghat, t->Cp, nullptr, t->C}, ghat_amax, msgt, t->amax_msg(T), nullptr, nullptr, n,
                 t->Xp.get(), zl);
        t->tc.tn(t, gt, R.g_amax, xint, xin_amax, nullptr, nullptr, n, t->Xp.get() + lo.H, zl);
        P.end(s);
    } else {
        P.begin("wgrad", 4.0 * n * (t->C + zl), s, 2.0 * n * t->C * zl);
        t->tc.tn(t, gt, R.g_amax, meant, t->amax_msg(T), &xint, xin_amax, n, t->Xp.get(), zl);
        P.end(s);
    }
    P.begin("wgrad_small", 4.0 * t->C * zl * 2 + 4.0 * lo.H * zl, s, 2.0 * t->C * zl * lo.H * 2);
    small_gemm(t->C, t->E, zl, t->Xp.get(), zl, false, t->theta.get() + lo.U, zl, true, t->slot_ptr(2 * t->L, i),
               t->E, s);
    small_gemm(lo.H, zl, t->C, t->theta.get() + t->head_off, t->E, true, t->Xp.get(), zl, false,
               t->slot_ptr(2 * T + 1, i), zl, s);
    P.end(s);
    exchange_bucket(t, 2 * t->L, round);
    exchange_bucket(t, 2 * T + 1, round);
    if (t->pta) {
        // dz = 1[msg > 0] * A^T (inv * G Z_L) = 1[msg > 0] * (Ghat Z_L)   (:274-288 re-associated)
        float* dz_amax = t->amax_slot(sc_trainer::kSlotDz);
        SC_CUDA(cudaMemsetAsync(dz_amax, 0, sizeof(float), s));
        P.begin("gemm_dgrad", 4.0 * n * (t->Cp + 2 * lo.H), s, 2.0 * n * t->C * lo.H);
        t->tc.nt(t, MatA{t->dh, t->Cp, nullptr, t->C}, ghat_amax, MatB{t->Z.get(), zl, true}, nullptr, nullptr,
                 nullptr, t->dz, lo.H, n, lo.H, kEpiMask, nullptr, dz_amax, nullptr, nullptr, t->POS[T]);
        P.end(s);
        backward_layers(t, R, i, T, t->dh, ghat_amax, dh2, dh2_amax, 2);
        return;
    }
    // dmean_s = inv * (dh U_L) = inv * (G Z_L)   (:274)
    P.begin("gemm_dgrad", 4.0 * n * (t->C + lo.H + 1), s, 2.0 * n * t->C * lo.H);
    t->tc.nt(t, ga, R.g_amax, MatB{t->Z.get(), zl, true}, nullptr, nullptr, nullptr, dh2, lo.H, n, lo.H,
             kEpiRowScale, t->inv, nullptr);
    P.end(s);
    backward_layers(t, R, i, T, t->dh, t->amax_slot(sc_trainer::kSlotDh0), dh2, dh2_amax, 1);
}

// sage_backward (nn.hpp:246-293) into partition i's gradient slot; each
// finished bucket is handed to the comm stream (exchange round i / world).
void backward(sc_trainer* t, const Rows& R, int i) {
    const int round = i / t->world;
    cudaStream_t s = t->ctx->stream;
    // side stream for the weight-gradient GEMMs that need only dh (see trainer.hpp)
    cudaStream_t w = t->overlap ? t->side : s;
    float* ws_w = t->overlap ? t->ws_side.get() : t->ws.get();
    auto hand_off = [&](cudaStream_t from, cudaStream_t to) {
        if (from == to) return;
        cudaEvent_t ev = t->fork_event();
        SC_CUDA(cudaEventRecord(ev, from));
        SC_CUDA(cudaStreamWaitEvent(to, ev, 0));
    };
    Profiler& P = t->prof;
    const int64_t n = R.n;
    const MatT x0t{R.x0, R.x0_ld, nullptr, t->d};
    if (t->fuse_top) {
        backward_fused(t, R, i);
        return;
    }
    const MatT embt = t->L == 0 ? x0t : MatT{t->X[t->L], t->E, nullptr, t->E};
    // head grad = G^T emb (side) ; dh = G head (main)   (:259-260)
    hand_off(s, w);
    P.begin("wgrad", 4.0 * n * (t->C + t->E), w, 2.0 * n * t->C * t->E);
    const float* x0_amax = t->g->feat_amax.get();
    const float* emb_amax = t->L == 0 ? x0_amax : t->amax_x(t->L);
    t->tc.tn(t, MatT{t->G, t->Cp, nullptr, t->C}, R.g_amax, embt, emb_amax, nullptr, nullptr, n,
             t->slot_ptr(2 * t->L, i), t->E, w, ws_w);
    P.end(w);
    exchange_bucket(t, 2 * t->L, round, w);
    // dh ping-pongs with dmean's buffer: each layer's dmean (dh2 below) is dead once the
    // transposed aggregation has read it, and the next dh is written there.
    float* dh = t->dh;
    float* dh2 = t->dmean;
    float* dh_amax = t->amax_slot(sc_trainer::kSlotDh0);
    float* dh2_amax = t->amax_slot(sc_trainer::kSlotDh1);
    if (t->L == 0) {
        hand_off(w, s);
        return;
    }
    P.begin("gemm_dgrad", 4.0 * n * (t->C + t->E), s, 2.0 * n * t->C * t->E);
    t->tc.nt(t, MatA{t->G, t->Cp, nullptr, t->C}, R.g_amax, MatB{t->theta.get() + t->head_off, t->E, true},
             nullptr, nullptr, nullptr, dh, t->E, n, t->E, kEpiNone, nullptr, dh_amax);
    P.end(s);
    backward_layers(t, R, i, t->L - 1, dh, dh_amax, dh2, dh2_amax, 0);
}

void backward_layers(sc_trainer* t, const Rows& R, int i, int top, float* dh, float* dh_amax, float* dh2,
                     float* dh2_amax, int top_done) {
    const int round = i / t->world;
    cudaStream_t s = t->ctx->stream;
    cudaStream_t w = t->overlap ? t->side : s;
    float* ws_w = t->overlap ? t->ws_side.get() : t->ws.get();
    auto hand_off = [&](cudaStream_t from, cudaStream_t to) {
        if (from == to) return;
        cudaEvent_t ev = t->fork_event();
        SC_CUDA(cudaEventRecord(ev, from));
        SC_CUDA(cudaStreamWaitEvent(to, ev, 0));
    };
    Profiler& P = t->prof;
    const int64_t n = R.n;
    const MatT x0t{R.x0, R.x0_ld, nullptr, t->d};
    const float* x0_amax = t->g->feat_amax.get();
    for (int l = top; l >= 0; --l) {
        const LayerOff& lo = t->lay[l];
        const bool composed = top_done > 0 && l == top;  // dmean and dU already done (backward_fused)
        const bool dz_ready = top_done == 2 && l == top;
        const MatT xint = l == 0 ? x0t : MatT{t->X[l], lo.in, nullptr, lo.in};
        const MatT dht{dh, lo.H, nullptr, lo.H};
        const MatT meant{t->MEAN[l], lo.H, nullptr, lo.H};
        const float* xin_amax = l == 0 ? x0_amax : t->amax_x(l);
        if (!composed) {
            // dmean_s = inv * (dh U_L)   (:274, pre-scaled for the pull aggregation)
            P.begin("gemm_dgrad", 4.0 * n * (2 * lo.H + 1), s, 2.0 * n * lo.H * lo.H);
            t->tc.nt(t, MatA{dh, lo.H, nullptr, lo.H}, dh_amax, MatB{t->theta.get() + lo.U, lo.H + lo.in, true},
                     nullptr, nullptr, nullptr, dh2, lo.H, n, lo.H, kEpiRowScale, t->inv, nullptr);
            P.end(s);
        }
        // One launch for dU = dh^T [mean | h_in] (:271-272) and dW = dz^T h_in (:289) after the
        // transposed aggregation, so h_in (and the tiles' conversions) stream once for both;
        // otherwise dU runs first (optionally on the side stream) and dW after.
        float* dz_amax = t->amax_slot(sc_trainer::kSlotDz);
        const MatT dzt{t->dz, lo.H, nullptr, lo.H};
        const bool dual = !composed && !t->overlap && t->tc.enabled && t->tc.dual &&
                          tn_dual_supported(dht, dzt, meant, xint);
        if (!dual && !composed) {
            hand_off(s, w);
            P.begin("wgrad", 4.0 * n * (2 * lo.H + lo.in), w, 2.0 * n * lo.H * (lo.H + lo.in));
            t->tc.tn(t, dht, dh_amax, meant, t->amax_msg(l), &xint, xin_amax, n, t->slot_ptr(2 * l + 1, i),
                     lo.H + lo.in, w, ws_w);
            P.end(w);
            exchange_bucket(t, 2 * l + 1, round, w);
        }
        // dz = 1[msg > 0] * sum_kept dmean_s[nbr]   (:277-288)
        if (!dz_ready) {
            SC_CUDA(cudaMemsetAsync(dz_amax, 0, sizeof(float), s));
            P.begin("spmm_bwd", spmm_bytes(R, lo.H, true), s);
            spmm_bwd(n, lo.H, R.offsets, R.nbrs, R.bits, dh2, t->compact ? nullptr : t->MSG[l], t->dz, s, dz_amax,
                     R.hv, t->heavy_ws.get(), t->POS[l]);
            P.end(s);
        }
        if (dual) {
            P.begin("wgrad", 4.0 * n * (3 * lo.H + lo.in), s, 2.0 * n * lo.H * (lo.H + 2 * lo.in));
            if (!t->tc.tn_dual(t, dht, dh_amax, dzt, dz_amax, meant, t->amax_msg(l), xint, xin_amax, n,
                               t->slot_ptr(2 * l + 1, i), lo.H + lo.in, t->slot_ptr(2 * l, i), lo.in))
                throw std::logic_error("dual weight-gradient launch refused a supported shape");
            P.end(s);
            exchange_bucket(t, 2 * l + 1, round);
        } else {
            // dW = dz^T h_in   (:289)
            P.begin("wgrad", 4.0 * n * (lo.H + lo.in), s, 2.0 * n * lo.H * lo.in);
            t->tc.tn(t, dzt, dz_amax, xint, xin_amax, nullptr, nullptr, n, t->slot_ptr(2 * l, i), lo.in);
            P.end(s);
        }
        exchange_bucket(t, 2 * l, round);
        if (l > 0) {  // dh = dh U_R + dz W   (:275, :290); layer 0's is unused
            const MatA dzA{t->dz, lo.H, nullptr, lo.H};
            const MatB wB{t->theta.get() + lo.W, lo.in, true};
            SC_CUDA(cudaMemsetAsync(dh2_amax, 0, sizeof(float), s));
            if (composed) {  // dh U_R = G head U_R = G Z_R
                const int zl = lo.H + lo.in;
                P.begin("gemm_dgrad", 4.0 * n * (t->C + lo.H + lo.in), s, 2.0 * n * (t->C + lo.H) * lo.in);
                t->tc.nt(t, MatA{t->G, t->Cp, nullptr, t->C}, R.g_amax, MatB{t->Z.get() + lo.H, zl, true}, &dzA,
                         dz_amax, &wB, dh2, lo.in, n, lo.in, kEpiNone, nullptr, dh2_amax);
            } else {
                const MatA dhA{dh, lo.H, nullptr, lo.H};
                P.begin("gemm_dgrad", 4.0 * n * (2 * lo.H + lo.in), s, 2.0 * n * 2 * lo.H * lo.in);
                t->tc.nt(t, dhA, dh_amax, MatB{t->theta.get() + lo.U + lo.H, lo.H + lo.in, true}, &dzA, dz_amax, &wB,
                         dh2, lo.in, n, lo.in, kEpiNone, nullptr, dh2_amax);
            }
            P.end(s);
            std::swap(dh, dh2);
            std::swap(dh_amax, dh2_amax);
        }
        hand_off(w, s);  // dU(l) read the old dh / dh_amax, which the next layer overwrites
    }
}

}  // namespace

void run_partition(sc_trainer* t, int i, int epoch) {
    cudaStream_t s = t->ctx->stream;
    PartState& st = t->ps[i];
    const PartDev& pd = t->vc->parts[i];
    const uint32_t* bits = nullptr;
    st.chosen = -1;
    if (t->use_dropedge) {  // trainer.hpp:261-266
        HostRng rng(substream(t->seed, "dropedge.select", uint64_t(i), uint64_t(epoch)));
        st.chosen = static_cast<int>(rng.next_below(uint64_t(t->K)));
        bits = st.bits.get() + int64_t(st.chosen) * st.words;
    }
    const int64_t kept =
        bits ? 2 * static_cast<int64_t>(std::ceil((1.0 - t->ratio) * static_cast<double>(pd.m_local))) : st.nnz;
    float* x0 = t->shared_x0 ? t->x0_shared.get() : st.x0.get();
    if (t->shared_x0 || st.x0_version != t->g->feat_version) {  // the partition's feature rows, contiguous
        t->prof.begin("gather_x0", 8.0 * st.n * t->d, s);                   // (train_cofree :225-227)
        gather_rows(st.n, t->d, pd.nodes.get(), t->g->features.get(), x0, s, t->dp);
        t->prof.end(s);
        st.x0_version = t->g->feat_version;
    }
    float* logits = t->shared_logits ? t->logits_shared.get() : st.logits.get();
    t->last_part = i;
    const Rows R{st.n, pd.offsets.get(), pd.nbrs.get(), bits, pd.nodes.get(), st.nnz, kept, st.g_amax.get(),
                 x0, t->dp, &st.heavy};
    SC_CUDA(cudaMemsetAsync(t->amax.get(), 0, t->amax.bytes(), s));  // per-partition operand |max| slots
    forward(t, R, logits, train_acts(t));
    t->prof.begin("loss", double(st.n) * (8.0 * t->C + 24), s);
    if (t->loss == 0)
        softmax_ce(st.n, t->C, t->Cp, logits, t->g->labels.get(), pd.nodes.get(), st.w.get(), st.scale.get(),
                   t->G, t->row_loss.get(), s);
    else
        bce(st.n, t->C, t->Cp, logits, t->g->labels.get(), t->g->multilabel ? t->g->targets.get() : nullptr,
            pd.nodes.get(), st.w.get(), st.scale.get(), t->G, t->row_loss.get(), s);
    sum_f64(st.n, t->row_loss.get(), t->red_partial.get(), t->part_loss.get() + i, t->normalizer, s);
    t->prof.end(s);
    exchange_bucket(t, -1, i / t->world);
    backward(t, R, i);
}

void trainer_stage_features(sc_trainer* t, const float* features, bool is_device) {
    sc_graph* g = t->g;
    if (g->dim == 0) throw std::invalid_argument("stage_features: graph has no feature buffer");
    if (g->staged) throw std::invalid_argument("stage_features: features already staged (step first)");
    if (!g->copy_stream) {
        SC_CUDA(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
        SC_CUDA(cudaEventCreateWithFlags(&g->staged_ev, cudaEventDisableTiming));
        SC_CUDA(cudaEventCreateWithFlags(&g->released_ev, cudaEventDisableTiming));
    }
    cudaStream_t c = g->copy_stream;
    const int64_t nd = int64_t(g->n) * g->dim;
    g->features_next.ensure(std::max<int64_t>(nd, 1));
    if (g->released_recorded) SC_CUDA(cudaStreamWaitEvent(c, g->released_ev, 0));  // old buffer no longer read
    // Only the copy engine works here: kernels on this stream would take SM slots from the
    // step's persistent GEMMs. |max| and the x0 gathers run on the compute stream at commit.
    SC_CUDA(cudaMemcpyAsync(g->features_next.get(), features, sizeof(float) * nd,
                            is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c));
    SC_CUDA(cudaEventRecord(g->staged_ev, c));
    g->staged = true;
}

void commit_staged_features(sc_trainer* t) {
    sc_graph* g = t->g;
    if (!g->staged) return;
    cudaStream_t s = t->ctx->stream;
    SC_CUDA(cudaStreamWaitEvent(s, g->staged_ev, 0));
    SC_CUDA(cudaEventRecord(g->released_ev, s));  // everything that read the old buffer is enqueued before this
    std::swap(g->features, g->features_next);
    ++g->feat_version;  // partitions re-gather their x0 rows lazily (run_partition)
    SC_CUDA(cudaMemsetAsync(g->feat_amax.get(), 0, sizeof(float), s));
    absmax(int64_t(g->n) * g->dim, g->features.get(), g->feat_amax.get(), s);
    g->released_recorded = true;
    g->staged = false;
}

void trainer_step_async(sc_trainer* t, int epoch) {
    cudaStream_t s = t->ctx->stream;
    commit_staged_features(t);
    t->prof.records.clear();
    t->prof.used = 0;
    if (t->world > 1 && !t->comm && !t->xfn && !t->emulate)
        throw std::invalid_argument("sc_trainer_init_comm (or an exchange callback) must precede stepping at world > 1");
    // Exchange round j trains partition j*world + rank on every rank; each
    // finished gradient bucket (and the partition loss) is all-gathered on the
    // comm stream while the rest of backward runs. Every slot has exactly one
    // writer, so the exchange moves bits and the ordered sum below is bitwise
    // the reference's single-process gather for any GPU count.
    t->xfer_used = 0;
    t->fork_used = 0;
    t->audit_floats = uint64_t(t->local.size()) * uint64_t(t->P);  // each local partition hands |theta| floats over
    const int rounds = t->pp / t->world;
    for (int j = 0; j < rounds; ++j) {
        const int i = j * t->world + t->rank;
        if (i < t->p) {
            run_partition(t, i, epoch);
        } else {  // no partition this round (p % world != 0): same collective sequence, padding slots
            exchange_bucket(t, -1, j);
            for (int b = t->nb() - 1; b >= 0; --b) exchange_bucket(t, b, j);
        }
    }
    if (t->comm) {  // exposed tail of the exchange: the last buckets' all-gathers
        t->prof.begin("exchange_tail", 4.0 * t->p * t->P, s);
        SC_CUDA(cudaEventRecord(t->comm_done, t->comm_stream));
        SC_CUDA(cudaStreamWaitEvent(s, t->comm_done, 0));
        t->prof.end(s);
    }
    SC_CUDA(cudaMemsetAsync(t->nonfinite.get(), 0, 4, s));
    t->prof.begin("gather_adam", 4.0 * t->P * (t->p + 6), s);
    gather_grads(t->P, t->p, t->pp, t->nb(), t->b_off_dev.get(), t->slots.get(), t->gathered.get(),
                 t->red_partial.get(), t->nonfinite.get(), s);
    finalize_step(t->red_partial.get(), t->part_loss.get(), t->p, t->out2.get(), s);
    // adam_step (nn.hpp:400-432): corrections in f64, cast to float
    const int64_t step = t->adam_step + 1;
    const float c1 = static_cast<float>(1.0 - std::pow(0.9, static_cast<double>(step)));
    const float c2 = static_cast<float>(1.0 - std::pow(0.999, static_cast<double>(step)));
    adam(t->P, t->theta.get(), t->m1.get(), t->m2.get(), t->gathered.get(), 0.9f, 0.999f, c1, c2,
         static_cast<float>(t->lr), static_cast<float>(1e-8), t->nonfinite.get(), s);
    t->tc.invalidate();  // weights changed: rebuild the pre-split weight images on next use
    t->prof.end(s);
    d2h(t->host->out, t->out2.get(), 2, s);
    d2h(&t->host->nonfinite, t->nonfinite.get(), 1, s);
    t->pending = true;
}

void trainer_finish(sc_trainer* t, double* loss, double* gnorm) {
    if (t->pending) {
        SC_CUDA(cudaStreamSynchronize(t->ctx->stream));
        t->pending = false;
        t->prof.collect();
        if (t->host->nonfinite) throw std::invalid_argument("adam_step: non-finite gradient");
        ++t->adam_step;
        t->last_loss = t->host->out[1];
        t->last_gnorm = t->host->out[0];
    }
    if (loss) *loss = t->last_loss;
    if (gnorm) *gnorm = t->last_gnorm;
}

namespace {
// Full-graph forward (evaluate_splits, trainer.hpp:132-140) into t->eval_logits
// with the current parameters; returns nothing, logits stay on the device.
void eval_forward(sc_trainer* t) {
    cudaStream_t s = t->ctx->stream;
    sc_graph* g = t->g;
    const int64_t n = g->n;
    if (t->eval_logits.size() < size_t(n) * t->Cp) t->eval_logits.alloc(std::max<int64_t>(n * t->Cp, 1));
    int32_t maxH = 1;
    for (auto& lo : t->lay) maxH = std::max(maxH, lo.H);
    if (!t->eval_heavy_built) {
        build_heavy_rows(t->ctx, n, g->offsets.get(), t->eval_heavy);
        t->eval_heavy_built = true;
        if (size_t(t->eval_heavy.nseg) * maxH > t->heavy_ws.size()) t->heavy_ws.alloc(size_t(t->eval_heavy.nseg) * maxH);
    }
    // Forward-only set carved from the training arena (the step is complete, its cache is
    // dead): ping-pong layer outputs, one msg, one mean, inv. The arena grows if n needs more.
    Acts A;
    {
        auto carve_eval = [&](float* base) {
            Carver c{base};
            float* x[2] = {c.take(size_t(n) * maxH), c.take(size_t(n) * maxH)};
            float* msg = c.take(size_t(n) * maxH);
            float* mean = c.take(size_t(n) * maxH);
            A.X.assign(t->L + 1, nullptr);
            for (int l = 1; l <= t->L; ++l) A.X[l] = x[l & 1];
            A.MSG.assign(t->L, msg);
            A.MEAN.assign(t->L, mean);
            A.inv = c.take(n);
            return c.off;
        };
        const size_t need = carve_eval(nullptr);
        if (t->arena.size() < need) {
            SC_CUDA(cudaStreamSynchronize(s));  // nothing in flight reads the old arena
            t->arena.alloc(need);
            if (t->rows_cap > 0) carve_train(t, t->arena.get(), t->rows_cap);
        }
        carve_eval(t->arena.get());
    }
    // layer-0 rows: the features themselves, or a 16-byte-row copy so the GEMMs stay on TMA
    const float* x0 = g->features.get();
    int64_t x0_ld = g->dim;
    if (t->dp != t->d) {
        if (t->eval_x0_version != g->feat_version || t->eval_x0.size() < size_t(n) * t->dp) {
            t->eval_x0.ensure(std::max<int64_t>(n * t->dp, 1));
            gather_rows(n, t->d, nullptr, g->features.get(), t->eval_x0.get(), s, t->dp);
            t->eval_x0_version = g->feat_version;
        }
        x0 = t->eval_x0.get();
        x0_ld = t->dp;
    }
    const Rows R{n, g->offsets.get(), g->nbrs.get(), nullptr, nullptr, 2 * g->m, 2 * g->m, nullptr, x0, x0_ld,
                 &t->eval_heavy};
    const bool was = t->prof.enabled;
    t->prof.enabled = false;
    SC_CUDA(cudaMemsetAsync(t->amax.get(), 0, t->amax.bytes(), s));  // operand |max| slots of this pass
    forward(t, R, t->eval_logits.get(), A);
    t->prof.enabled = was;
}

// metric_from_logits (trainer.cpp:66-97) over each device mask.
void eval_metrics(sc_trainer* t, const uint8_t* const* masks, int nm, double* out) {
    cudaStream_t s = t->ctx->stream;
    sc_graph* g = t->g;
    DevBuf<unsigned long long> cnt(4 * nm);
    SC_CUDA(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
    for (int i = 0; i < nm; ++i) {
        if (g->multilabel)
            f1_counts(g->n, t->C, t->Cp, t->eval_logits.get(), g->targets.get(), masks[i], cnt.get() + 4 * i, s);
        else
            count_correct(g->n, t->C, t->Cp, t->eval_logits.get(), g->labels.get(), masks[i], cnt.get() + 4 * i, s);
    }
    std::vector<unsigned long long> h(4 * nm);
    d2h(h.data(), cnt.get(), 4 * nm, s);
    SC_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < nm; ++i) {
        const unsigned long long* c = h.data() + 4 * i;
        if (g->multilabel) {  // micro-F1 with positives at logit > 0
            const unsigned long long denom = 2 * c[0] + c[1] + c[2];
            out[i] = (c[3] == 0 || denom == 0) ? 0.0 : 2.0 * double(c[0]) / double(denom);
        } else {
            out[i] = c[1] ? double(c[0]) / double(c[1]) : 0.0;
        }
    }
}
}  // namespace

void trainer_evaluate(sc_trainer* t, double* tr, double* va, double* te) {
    trainer_finish(t, nullptr, nullptr);  // metrics of a settled step only
    eval_forward(t);
    const uint8_t* masks[3] = {t->g->train.get(), t->g->val.get(), t->g->test.get()};
    double out[3];
    eval_metrics(t, masks, 3, out);
    *tr = out[0];
    *va = out[1];
    *te = out[2];
}

double trainer_evaluate_mask(sc_trainer* t, const uint8_t* mask_dev) {
    trainer_finish(t, nullptr, nullptr);
    eval_forward(t);
    double out = 0.0;
    eval_metrics(t, &mask_dev, 1, &out);
    return out;
}

void trainer_init_comm(sc_trainer* t, const uint8_t id[128]) {
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    SC_CUDA(cudaSetDevice(t->ctx->device));
    SC_NCCL(ncclCommInitRank(&t->comm, t->world, uid, t->rank));
    if (!t->comm_stream) SC_CUDA(cudaStreamCreateWithFlags(&t->comm_stream, cudaStreamNonBlocking));
    if (!t->comm_done) SC_CUDA(cudaEventCreateWithFlags(&t->comm_done, cudaEventDisableTiming));
}

namespace {
// The same all-gather through the caller's host transport: wait for the
// producer, stage this rank's bytes in pinned memory, call out, copy the
// gathered range back. Synchronous (test / fallback transport, not the fast path).
void exchange_host(sc_trainer* t, int b, int round, cudaStream_t s) {
    const int first = round * t->world;
    const int kind = b < 0 ? 1 : 0;
    const size_t per = b < 0 ? sizeof(double) : sizeof(float) * size_t(t->b_len(b));
    unsigned char* base = b < 0 ? reinterpret_cast<unsigned char*>(t->part_loss.get() + first)
                                : reinterpret_cast<unsigned char*>(t->slot_ptr(b, first));
    const size_t need = per * (size_t(t->world) + 1);
    if (t->xhost_bytes < need) {
        if (t->xhost) SC_CUDA(cudaFreeHost(t->xhost));
        t->xhost = nullptr;
        SC_CUDA(cudaMallocHost(&t->xhost, need));
        t->xhost_bytes = need;
    }
    unsigned char* send = static_cast<unsigned char*>(t->xhost);
    unsigned char* recv = send + per;
    SC_CUDA(cudaMemcpyAsync(send, base + per * t->rank, per, cudaMemcpyDeviceToHost, s));
    SC_CUDA(cudaStreamSynchronize(s));
    if (t->xfn(t->xuser, kind, round, b, send, recv, static_cast<int64_t>(per)) != 0)
        throw std::runtime_error("gradient exchange callback failed (round " + std::to_string(round) + ", bucket " +
                                 std::to_string(b) + ")");
    SC_CUDA(cudaMemcpyAsync(base, recv, per * t->world, cudaMemcpyHostToDevice, s));
    SC_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

void exchange_bucket(sc_trainer* t, int b, int round, cudaStream_t producer) {
    cudaStream_t s = producer ? producer : t->ctx->stream;
    if (t->emulate) return;  // no peers: the other ranks' slots stay zero
    if (t->xfn) {
        exchange_host(t, b, round, s);
        return;
    }
    if (!t->comm) return;  // world == 1 without a communicator: nothing to exchange
    if (t->xfer_used == t->xfer_events.size()) {
        cudaEvent_t e;
        SC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        t->xfer_events.push_back(e);
    }
    cudaEvent_t ev = t->xfer_events[t->xfer_used++];
    SC_CUDA(cudaEventRecord(ev, s));
    SC_CUDA(cudaStreamWaitEvent(t->comm_stream, ev, 0));
    const int first = round * t->world;  // the round's partitions first .. first + world - 1 are contiguous
    if (b < 0) {
        double* base = t->part_loss.get() + first;
        SC_NCCL(ncclAllGather(base + t->rank, base, 1, ncclFloat64, t->comm, t->comm_stream));
    } else {
        const int64_t len = t->b_len(b);
        float* base = t->slot_ptr(b, first);
        SC_NCCL(ncclAllGather(base + int64_t(t->rank) * len, base, size_t(len), ncclFloat32, t->comm,
                              t->comm_stream));
    }
}

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId uid;
    SC_NCCL(ncclGetUniqueId(&uid));
    std::memcpy(out, uid.internal, 128);
}

}  // namespace sc
