// trainer.hpp — sc_trainer state (train_cofree_impl, proj/include/sagecut/trainer.hpp:202-313).
#pragma once

#include <nccl.h>

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "gemm_tc.cuh"
#include "internal.hpp"
#include "nn.cuh"

namespace sc {

struct LayerOff {
    int in = 0, H = 0;
    int64_t W = 0, U = 0;  // offsets of message / update in the flat parameter vector
};

struct PartState {
    int64_t n = 0, nnz = 0;
    DevBuf<double> w;      // loss weight (train ? scheme weight : 0)
    DevBuf<float> scale;   // (float)(w / normalizer)
    DevBuf<uint32_t> bits; // K CSR-slot bitmaps
    int64_t words = 0;
    DevBuf<float> logits;  // n x C, last step
    DevBuf<float> g_amax;  // bound on max|dloss/dlogits| (tensor-core operand scale)
    DevBuf<float> x0;      // layer-0 input: this partition's feature rows (n x d), gathered once per
    uint64_t x0_version = 0;  // feature version, so the GEMMs stream contiguous rows
    HeavyRows heavy;          // hub rows of the local CSR (segmented aggregation)
    int chosen = -1;
};

struct Profiler {
    struct Rec {
        const char* name;
        double bytes, flops;
        size_t slot;
    };
    struct Total {
        double ms = 0, bytes = 0, flops = 0;
        int calls = 0;
    };
    bool enabled = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
    std::vector<Rec> records;
    size_t used = 0;
    const char* cur_name = nullptr;
    double cur_bytes = 0, cur_flops = 0;
    std::map<std::string, Total> totals;
    // bytes: algorithmic HBM bytes; flops: algorithmic 2MNK of a GEMM (fp32-equivalent products)
    void begin(const char* name, double bytes, cudaStream_t s, double flops = 0);
    void end(cudaStream_t s);
    void collect();
    ~Profiler();
};

}  // namespace sc

struct sc_trainer {
    sc_ctx* ctx = nullptr;
    sc_graph* g = nullptr;
    sc_vcut* vc = nullptr;
    int rank = 0, world = 1;
    // config
    int L = 0;
    std::vector<int> hidden;
    double lr = 0.01;
    int loss = 0, reweight = 0, use_dropedge = 0, K = 10;
    double ratio = 0.5;
    uint64_t seed = 0;
    int deterministic = 1, gemm_mode = 0;
    // dims
    int d = 0, C = 0, Cp = 0, E = 0, p = 0;
    int dp = 0;  // x0 row pitch: d rounded up to 4 floats (16-byte rows for the TMA-fed GEMMs)
    std::vector<sc::LayerOff> lay;
    int64_t head_off = 0, P = 0;
    double normalizer = 1.0;
    // parameters / optimizer / gradients
    sc::DevBuf<float> theta, m1, m2, gathered;
    // Per-partition gradient slots, bucket-major: bucket b (= parameter matrix
    // b in for_each_matrix order: W_0, U_0, ..., W_{L-1}, U_{L-1}, head) holds
    // pp = ceil(p / world) * world consecutive copies of its b_len[b] floats,
    // one per partition, so the copies of one exchange round
    // (partitions j*world .. j*world + world-1) are one contiguous range.
    sc::DevBuf<float> slots;
    int pp = 0;
    std::vector<int64_t> b_off;      // nb + 1 offsets into the flat parameter vector
    sc::DevBuf<int64_t> b_off_dev;
    int nb() const { return static_cast<int>(b_off.size()) - 1; }
    int64_t b_len(int b) const { return b_off[b + 1] - b_off[b]; }
    float* slot_ptr(int b, int i) { return slots.get() + b_off[b] * pp + int64_t(i) * b_len(b); }
    int64_t adam_step = 0;
    // partitions
    std::vector<int> local;
    std::vector<sc::PartState> ps;
    // Per-row activation / gradient buffers (rows_cap rows), carved from ONE arena
    // (carve_train): X[l] (l >= 1), MSG[l], MEAN[l], inv, G, dh, dmean, dz. The
    // backward's dh ping-pong reuses dmean's buffer (dmean is dead once the
    // transposed aggregation has read it). Full-graph evaluation carves its
    // forward-only set (two ping-pong layer outputs, one msg, one mean, inv) from
    // the same arena, growing it if needed, so the two never hold memory at once.
    // compact (large graphs, or SC_COMPACT_ACTS=1): one msg buffer shared by every
    // layer plus the ReLU decisions as sign bits POS[l] ([rows][ceil(H/32)] words,
    // written by the msg GEMM's epilogue) for the backward.
    int64_t rows_cap = 0;
    bool compact = false;
    sc::DevBuf<float> arena;
    std::vector<float*> X, MSG, MEAN;
    std::vector<uint32_t*> POS;
    float *inv = nullptr, *G = nullptr, *dh = nullptr, *dmean = nullptr, *dz = nullptr;
    sc::DevBuf<float> eval_logits, ws, ws_side;
    sc::DevBuf<float> heavy_ws;   // segment partial sums of the heavy-row aggregation
    sc::HeavyRows eval_heavy;     // heavy rows of the full graph (evaluate_splits)
    bool eval_heavy_built = false;
    sc::DevBuf<float> eval_x0;  // the full feature matrix with 16-byte rows (d % 4 != 0)
    uint64_t eval_x0_version = 0;
    bool eval_only = false;     // sc_evaluate's forward-only engine (no partitions, no optimizer)
    // Per-partition caches that only save time: each local partition's gathered layer-0 rows
    // (x0) and its last logits. When they would take more than their budget of device memory
    // (large graphs: R-MAT 20M / 1B at p = 16) all partitions share one buffer instead: x0 is
    // then gathered again for every partition every step (~n_i d 8 bytes), and only the last
    // trained partition's logits stay readable (sc_trainer_get_part_logits).
    bool shared_x0 = false, shared_logits = false;
    sc::DevBuf<float> x0_shared, logits_shared;
    int last_part = -1;
    // CommAudit (trainer.hpp:61-76): parameter-gradient floats this rank's
    // partitions handed to the exchange in the last epoch (p * |theta| at world 1).
    uint64_t audit_floats = 0;
    // Backward runs the weight-gradient GEMMs that only need dh (head: G^T emb;
    // update: dh^T [mean | h]) on a high-priority side stream, concurrently with
    // the dgrad -> transposed aggregation -> dW chain on the main stream.
    // Opt-in (SC_OVERLAP=1): on B200 the two contend for HBM and the epoch
    // gains <1 % (profiles/r01_overlap_ab.txt), while the aggregation's own
    // duration, and so its roofline figure, doubles.
    bool overlap = false;
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> fork_events;
    size_t fork_used = 0;
    cudaEvent_t fork_event();
    int64_t ws_floats = 0;
    sc::DevBuf<double> row_loss, part_loss, out2, red_partial;
    sc::DevBuf<int> nonfinite;
    // max|x| of every tensor-core A operand, reduced by its producing kernel
    // and read by the consuming GEMM to pick its power-of-two operand scale.
    enum { kSlotDh0 = 0, kSlotDh1 = 1, kSlotDz = 2, kSlotBase = 3 };
    sc::DevBuf<float> amax;
    float* amax_slot(int i) { return amax.get() + i; }
    float* amax_x(int l) { return amax.get() + kSlotBase + (l - 1); }  // layer input X[l], l in [1, L]
    float* amax_msg(int l) { return amax.get() + kSlotBase + L + l; }  // MSG[l], l in [0, L)
    // Pinned (cudaMallocHost) read-back slots: a D2H into pageable memory would
    // block the host until the whole step has run, so nothing (e.g. the next
    // step's feature copy) could be enqueued behind it.
    struct HostOut {
        double out[2];
        int nonfinite;
    };
    HostOut* host = nullptr;
    bool pending = false;
    double last_loss = 0, last_gnorm = 0;
    sc::TcGemm tc;
    sc::Profiler prof;
    // Composed top layer (tensor-core path, L >= 1, SC_FUSE_TOP != 0): the last layer's update
    // h_L = mean U_L^T + h U_R^T and the head logits = h_L head^T are both linear, so
    // logits = mean Z_L^T + h Z_R^T with Z = head U_{L-1} (C x (H + in), once per weight version),
    // and h_L is never formed. Backward: Xp = G^T [mean | h] (one TN GEMM with C output rows) gives
    // dHead = Xp U^T and dU_{L-1} = head^T Xp; dmean = inv (G Z_L); dh_{L-1} = G Z_R + dz W.
    bool fuse_top = false;
    // ... and (pta, when the padded class count is at most half the top layer's width) the top
    // layer's aggregation runs on projected rows: logits = h Z_R^T + A_norm (msg Z_L^T), whose rows are
    // Cp wide instead of H (nn.hpp:222-234 re-associated; A_norm the masked mean). Backward: Ghat =
    // A^T (inv * G) (Cp-wide pull), Xp = [Ghat^T msg | G^T h], dz = 1[msg > 0] (Ghat Z_L).
    bool pta = false;
    sc::DevBuf<float> Z, Xp;  // Z: Cp rows (rows C .. Cp-1 zero), so Cp-wide products have zero padding
    uint64_t z_version = 0;
    // Host transport (sc_trainer_set_exchange), used instead of NCCL when set.
    using ExchangeFn = int32_t (*)(void*, int32_t, int32_t, int32_t, const void*, void*, int64_t);
    ExchangeFn xfn = nullptr;
    bool emulate = false;  // sc_trainer_emulate_rank: one rank of a world > 1 job, exchange skipped
    void* xuser = nullptr;
    void* xhost = nullptr;       // pinned staging: send (one rank's bytes) + recv (world x)
    size_t xhost_bytes = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;      // gradient exchange, overlapped with backward
    std::vector<cudaEvent_t> xfer_events;    // compute -> comm stream hand-offs (reused per step)
    size_t xfer_used = 0;
    cudaEvent_t comm_done = nullptr;
    ~sc_trainer();
};

namespace sc {
void trainer_init(sc_trainer* t);
void loss_weights(sc_trainer* t, int i);
void ensure_rows(sc_trainer* t, int64_t n);
// Lay the training buffers for `rows` rows out from base (null: sizing pass); returns floats used.
size_t carve_train(sc_trainer* t, float* base, int64_t rows);
void run_partition(sc_trainer* t, int i, int epoch);
void trainer_step_async(sc_trainer* t, int epoch);
void trainer_finish(sc_trainer* t, double* loss, double* gnorm);
void trainer_evaluate(sc_trainer* t, double* tr, double* va, double* te);
// evaluate (trainer.cpp:101-112): the current model's full-graph metric over one
// split mask (device); accuracy, or micro-F1 on multi-label graphs.
double trainer_evaluate_mask(sc_trainer* t, const uint8_t* mask_dev);
// Forward-only engine over g for a given model (sc_evaluate).
void trainer_init_eval_only(sc_trainer* t);
void trainer_init_comm(sc_trainer* t, const uint8_t id[128]);
// Stage the next step's features (host or device source): the copy runs on the
// graph's copy stream (copy engine only), overlapping the current step; the
// next trainer_step_async commits them (swap, |max|, lazy x0 re-gathers).
void trainer_stage_features(sc_trainer* t, const float* features, bool is_device);
void commit_staged_features(sc_trainer* t);
// Exchange bucket b (or the losses, b = -1) of exchange round j across ranks
// on the comm stream once the compute stream has produced it.
void exchange_bucket(sc_trainer* t, int b, int round, cudaStream_t producer = nullptr);
void nccl_unique_id(uint8_t out[128]);
}  // namespace sc
