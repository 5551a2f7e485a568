/* sagecut_cuda.h — C ABI of libsagecut_cuda.so, the B200-native drop-in for the
 * CoFree-GNN per-partition training step of the reference `sagecut`
 * (/root/reference/proj, arXiv 2308.03209).
 *
 * The reference has no FFI: its boundary is the C++ API in namespace sagecut
 * (partition.hpp, reweight.hpp, dropedge.hpp, nn.hpp, trainer.hpp), called by
 * proj/tools/main.cpp and the tests. Each entry point below replaces one of
 * those functions (cited per declaration); a C++ facade that re-exports the
 * reference signatures on top of this ABI is include/sagecut_b200.hpp, and the
 * ctypes mirror used by tests/ and bench.py is paper_2308_03209_b200/sagecut.py.
 *
 * Conventions
 *   - plain pointers + sizes; host buffers unless a name says _dev;
 *   - device state lives in opaque handles with explicit *_destroy;
 *   - edges are int32 [m][2] pairs; matrices are row-major;
 *   - parameters are ONE flat fp32 vector in SageModel::for_each_matrix order
 *     (layer0.message, layer0.update, ..., head), each matrix row-major;
 *   - every function returns an sc_status; on failure sc_last_error() holds the
 *     reference's message text where the reference throws
 *     (std::invalid_argument -> SC_EINVAL, std::runtime_error -> SC_ERUNTIME,
 *     std::logic_error -> SC_EINTERNAL), mirroring the CLI's exit-code map
 *     (proj/tools/main.cpp:822-834).
 */
#ifndef SAGECUT_CUDA_H
#define SAGECUT_CUDA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SC_OK = 0,
    SC_EINVAL = 1,     /* std::invalid_argument */
    SC_ERUNTIME = 2,   /* std::runtime_error */
    SC_EINTERNAL = 3,  /* std::logic_error / bug */
    SC_ECUDA = 4,      /* CUDA runtime / launch failure */
    SC_ENCCL = 5       /* NCCL failure */
} sc_status;

typedef struct sc_ctx sc_ctx;         /* one device + streams + scratch      */
typedef struct sc_graph sc_graph;     /* sagecut::Graph on the device        */
typedef struct sc_vcut sc_vcut;       /* sagecut::VertexCutPartition         */
typedef struct sc_trainer sc_trainer; /* train_cofree_impl state             */

const char* sc_last_error(void);
const char* sc_version(void);

/* ---- context ------------------------------------------------------------ */
sc_status sc_ctx_create(int device, sc_ctx** out);
sc_status sc_ctx_destroy(sc_ctx* ctx);
sc_status sc_ctx_sync(sc_ctx* ctx);
/* Kernel launches issued by this library on ctx since creation (counter). */
int64_t sc_ctx_launch_count(sc_ctx* ctx);
/* CUDA-event timer on ctx's stream: start records an event, stop records a
 * second one, synchronizes, and returns the elapsed device time. */
sc_status sc_ctx_timer_start(sc_ctx* ctx);
sc_status sc_ctx_timer_stop(sc_ctx* ctx, double* ms);

/* ---- graph (proj/include/sagecut/graph.hpp:53-96, proj/src/graph.cpp) ---- */
/* build_graph (graph.cpp:8-64): drop self-loops, canonicalise u<v, sort,
 * dedup, CSR with ascending neighbour rows. raw_uv is a host buffer. */
sc_status sc_build_graph(sc_ctx* ctx, int32_t num_nodes, const int32_t* raw_uv, int64_t m_raw, sc_graph** out,
                         int64_t* dropped_self_loops, int64_t* merged_duplicates);
/* Same, from a raw edge list already resident on the device. */
sc_status sc_build_graph_dev(sc_ctx* ctx, int32_t num_nodes, const int32_t* raw_uv_dev, int64_t m_raw,
                             sc_graph** out, int64_t* dropped_self_loops, int64_t* merged_duplicates);
/* Attach features (fp32 n x d), class ids, and the train/val/test masks
 * (Graph::features, labels, num_classes, train/val/test_mask). Host buffers. */
/* Graph::features / labels / masks (graph.hpp:58-66). features may be NULL: a zero n x dim
 * matrix is allocated (fill it with sc_graph_set_feature_rows). */
sc_status sc_graph_set_data(sc_graph* g, const float* features, int32_t dim, const int32_t* labels,
                            int32_t num_classes, const uint8_t* train, const uint8_t* val, const uint8_t* test);
/* Multi-label targets (Graph::multilabels, graph.hpp:64; load_labels' multi-label
 * branch, graph_io.cpp:206-229): n x C row-major, every entry 0 or 1 (else SC_EINVAL
 * "loss: bce targets must be 0 or 1", nn.hpp:366-367). Replaces the class ids;
 * the graph then trains with bce only (softmax_ce -> "softmax_ce requires
 * multi-class labels", trainer.hpp:207-208) and evaluates with micro-F1
 * (trainer.cpp:72-87). Call after sc_graph_set_data (features + masks). */
sc_status sc_graph_set_multilabels(sc_graph* g, const float* targets, int32_t num_classes);
/* Replace only the features (e.g. a new batch of the same graph). Host or device source. */
sc_status sc_graph_set_features(sc_graph* g, const float* features, int is_device);
/* Write feature rows [row0, row0 + rows) (host or device source), e.g. a matrix too large to
 * stage whole; sc_graph_set_data with features == NULL allocates a zero matrix to fill this way
 * (load_features' row-by-row fill, graph_io.cpp:82-160). The operand scale max|features| is
 * raised by the new rows (exact when every row is written once over zeros). */
sc_status sc_graph_set_feature_rows(sc_graph* g, int64_t row0, int64_t rows, const float* src, int is_device);
sc_status sc_graph_info(sc_graph* g, int32_t* num_nodes, int64_t* num_edges, int32_t* dim, int32_t* num_classes);
sc_status sc_graph_copy_edges(sc_graph* g, int32_t* uv);
sc_status sc_graph_copy_csr(sc_graph* g, int64_t* offsets, int32_t* neighbors, int32_t* edge_ids, int32_t* degrees);
sc_status sc_graph_destroy(sc_graph* g);

/* ---- dataset files (proj/include/sagecut/graph_io.hpp, proj/src/graph_io.cpp) ---- */
/* load_graph (graph_io.cpp:41-80): "u v" text lines ('#' comments, blank lines
 * skipped), then build_graph on the device. num_nodes < 0: 1 + the largest id
 * (LoadOptions::num_nodes); strict: SC_ERUNTIME if a node id never appears.
 * Parse errors: SC_ERUNTIME "<path>:<line>: <what>" as the reference. */
sc_status sc_load_graph(sc_ctx* ctx, const char* path, int32_t num_nodes, int32_t strict, sc_graph** out,
                        int64_t* dropped_self_loops, int64_t* merged_duplicates);
/* The edge-list parse of load_graph alone (host only): raw (u, v) pairs in file
 * order (cap = pairs the buffer holds; uv = NULL to size) and the node count. */
sc_status sc_read_edge_list(const char* path, int32_t num_nodes, int32_t* uv, int64_t cap, int64_t* m, int32_t* n);
/* load_features (graph_io.cpp:82-160): CSV or "CFM1" binary (sniffed), as fp32
 * row-major. Call with out = NULL to get rows / cols, then with a buffer. */
sc_status sc_load_features(const char* path, int32_t expected_nodes, float* out, int64_t cap, int64_t* rows,
                           int64_t* cols);
/* load_labels (graph_io.cpp:188-242): class ids (labels, n) or a multi-label 0/1
 * matrix (targets, n x num_classes; *is_multilabel = 1). NULL outputs: query only. */
sc_status sc_load_labels(const char* path, int32_t num_nodes, int32_t* labels, float* targets, int64_t cap,
                         int32_t* num_classes, int32_t* is_multilabel);
/* load_masks (graph_io.cpp:256-283): "train|val|test <id>" lines -> n-byte masks. */
sc_status sc_load_masks(const char* path, int32_t num_nodes, uint8_t* train, uint8_t* val, uint8_t* test);
/* save_edge_list / save_features_csv|binary / save_labels / save_masks
 * (graph_io.cpp:75-80, 162-186, 244-254, 285-296), byte-compatible. */
sc_status sc_save_edge_list(sc_graph* g, const char* path);
sc_status sc_save_features(const char* path, const float* features, int64_t rows, int64_t cols, int32_t binary);
sc_status sc_save_labels(const char* path, int32_t num_nodes, const int32_t* labels, const float* targets,
                         int32_t num_classes);
sc_status sc_save_masks(const char* path, int32_t num_nodes, const uint8_t* train, const uint8_t* val,
                        const uint8_t* test);

/* ---- vertex cut (proj/include/sagecut/partition.hpp, proj/src/partition.cpp) */
/* partition_random (partition.cpp:92-100): edge e takes the e-th next_below(p)
 * draw of Rng(substream(seed,"partition.random")). */
sc_status sc_partition_random(sc_graph* g, int32_t num_parts, uint64_t seed, sc_vcut** out);
/* partition_dbh (partition.cpp:102-114). */
sc_status sc_partition_dbh(sc_graph* g, int32_t num_parts, uint64_t seed, sc_vcut** out);
/* build_vertex_cut (partition.cpp:22-90) from a caller-supplied assignment. */
sc_status sc_build_vertex_cut(sc_graph* g, int32_t num_parts, const int32_t* edge_assignment, sc_vcut** out);
/* partition_ne (partition.cpp:116-201), output-identical: greedy neighbour
 * expansion with a lazy-deletion (unassigned-degree, id) min-heap instead of
 * the reference's boundary rescan. Overshoot reports -> sc_vcut_warnings. */
sc_status sc_partition_ne(sc_graph* g, int32_t num_parts, uint64_t seed, double balance_slack, sc_vcut** out);
/* partition_edge_cut_greedy (partition.cpp:233-278): node -> part (n, host). */
sc_status sc_partition_edge_cut_greedy(sc_graph* g, int32_t num_parts, uint64_t seed, int32_t* node_assignment);
/* edge_cut_from_assignment (partition.cpp:203-231): kept_counts[p] (may be
 * NULL), *num_cut, halo_counts[p] (may be NULL); when non-NULL, kept_edges
 * (m - num_cut: kept_edges part-major, each ascending), cut_edges (num_cut,
 * ascending) and halo_nodes (sum halo_counts: halo_sets part-major, each
 * ascending). Call once with NULL lists to size them. */
sc_status sc_edge_cut_from_assignment(sc_graph* g, int32_t num_parts, const int32_t* node_assignment,
                                      int64_t* kept_counts, int64_t* num_cut, int64_t* halo_counts,
                                      int32_t* kept_edges, int32_t* cut_edges, int32_t* halo_nodes);
/* edge_cut_to_vertex_cut (partition.cpp:280-308) of the edge cut induced by
 * node_assignment (n, host). */
sc_status sc_edge_cut_to_vertex_cut(sc_graph* g, int32_t num_parts, const int32_t* node_assignment, uint64_t seed,
                                    sc_vcut** out);
/* VertexCutPartition::warnings joined by '\n' (NUL-terminated, truncated to
 * cap); *needed = full length + 1. */
sc_status sc_vcut_warnings(sc_vcut* vc, char* buf, int64_t cap, int64_t* needed);
sc_status sc_vcut_num_parts(sc_vcut* vc, int32_t* num_parts);
sc_status sc_vcut_assignment(sc_vcut* vc, int32_t* out);
sc_status sc_vcut_part_sizes(sc_vcut* vc, int32_t part, int64_t* n_local, int64_t* n_edges);
/* Partition ownership for multi-GPU training (one process per GPU): vertex cuts
 * built on g after this call materialise only the parts i with
 * i % world == rank (the ones that rank trains, trainer.hpp:283-288's worker
 * assignment); every other part keeps its sizes (and its nodes' replication
 * counts) but no device arrays, so a rank holds ~p/world partitions instead of
 * all p. Accessing a part that is not held gives SC_EINVAL. Default: (0, 1). */
sc_status sc_graph_set_part_ownership(sc_graph* g, int32_t rank, int32_t world);
sc_status sc_vcut_part_held(sc_vcut* vc, int32_t part, int32_t* held);
/* PartSubgraph fields (partition.hpp:14-31); any pointer may be NULL. */
sc_status sc_vcut_part_copy(sc_vcut* vc, int32_t part, int32_t* nodes, int32_t* edges_uv, int32_t* edge_global_ids,
                            int32_t* local_degrees, int64_t* offsets, int32_t* neighbors, int32_t* edge_ids,
                            int32_t* global_to_local);
/* replication_stats (partition.cpp:310-342). */
sc_status sc_replication_stats(sc_vcut* vc, int32_t* per_node_rf, double* rf, double* edge_balance,
                               double* node_balance, int64_t* duplicated_nodes);
sc_status sc_vcut_destroy(sc_vcut* vc);

/* ---- reweighting (proj/src/reweight.cpp:23-81) ---------------------------- */
/* scheme: 0 dar, 1 vanilla_inv, 2 none. out: concatenated per part (sum n_i). */
sc_status sc_compute_weights(sc_vcut* vc, int32_t scheme, double* out);

/* ---- DropEdge-K (proj/src/dropedge.cpp:9-37) ------------------------------- */
/* precompute_masks: K masks over num_edges local edges, each keeping exactly
 * ceil((1-ratio)*num_edges); bit-exact with the reference's Fisher-Yates
 * stream (computed on the device). out: K x num_edges bytes (host). */
sc_status sc_precompute_masks(sc_ctx* ctx, int64_t num_edges, int32_t k, double ratio, uint64_t seed, uint8_t* out);
/* select_mask with Rng(substream(seed,"dropedge.select",part,epoch))
 * (trainer.hpp:261-266). */
int32_t sc_select_mask(uint64_t seed, uint64_t part, uint64_t epoch, int32_t k);
uint64_t sc_substream(uint64_t seed, const char* tag, int32_t nidx, uint64_t a, uint64_t b);

/* ---- model (proj/include/sagecut/nn.hpp:73-102) ---------------------------- */
int64_t sc_param_count(int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t num_classes);
/* make_sage_model<float>: Glorot draws from Rng(substream(seed,"init")). */
sc_status sc_init_params(sc_ctx* ctx, int32_t in_dim, const int32_t* hidden, int32_t layers, int32_t num_classes,
                         uint64_t seed, float* out);

/* ---- trainer (proj/include/sagecut/trainer.hpp:20-33, 202-313) ------------- */
typedef struct {
    int32_t layers;          /* TrainConfig::layers */
    const int32_t* hidden;   /* resolved per-layer hidden dims (length layers) */
    double learning_rate;    /* TrainConfig::learning_rate */
    int32_t loss;            /* 0 softmax_ce, 1 bce */
    int32_t reweight;        /* 0 dar, 1 vanilla_inv, 2 none */
    int32_t use_dropedge;
    int32_t dropedge_k;
    double drop_ratio;
    uint64_t seed;
    int32_t deterministic;   /* accepted for API compatibility: the exchange all-gathers
                                per-partition slots and sums them in ascending partition
                                order, which is always bitwise invariant to the GPU count
                                and costs the same bytes as a reduction at p = world */
    int32_t gemm;            /* 0: auto (tcgen05 where shapes allow), 1: SIMT fp32 only */
} sc_train_config;

/* Partitions i with i % world == rank are trained on this rank's device. */
sc_status sc_trainer_create(sc_ctx* ctx, sc_graph* g, sc_vcut* vc, const sc_train_config* cfg, int32_t rank,
                            int32_t world, sc_trainer** out);
/* NCCL: rank 0 calls sc_nccl_unique_id and ships the 128 bytes to the others
 * (optional at world == 1: a single-rank communicator runs the same exchange). */
sc_status sc_nccl_unique_id(uint8_t out[128]);
sc_status sc_trainer_init_comm(sc_trainer* t, const uint8_t id[128]);
/* Time ONE rank's share of a world > 1 job on a single GPU (no peers): the trainer runs this
 * rank's partitions and exchange rounds exactly as it would in the job, but the all-gathers are
 * skipped, so the other ranks' gradient slots stay zero and the gathered gradient / Adam step
 * cover this rank's partitions only (timing and memory only, not a training result). */
sc_status sc_trainer_emulate_rank(sc_trainer* t);
/* Host transport for the gradient exchange, instead of NCCL (multi-process
 * runs without a GPU per rank, e.g. several ranks time-sharing one device in
 * tests, or any collective library the caller already runs). Called once per
 * (exchange round, bucket) on the stepping thread with this rank's
 * contribution in `send` (bytes_per_rank bytes, host) and must return, in
 * `recv`, all ranks' contributions concatenated in rank order (an all-gather,
 * world * bytes_per_rank bytes); kind 0 = one partition's f32 gradient bucket
 * (bucket = parameter matrix in for_each_matrix order), kind 1 = the round's
 * f64 partition losses (bucket = -1). Non-zero return = failure (SC_ERUNTIME).
 * The bits moved are the same as over NCCL, so results stay bitwise
 * independent of the rank count. fn = NULL restores NCCL. */
typedef int32_t (*sc_exchange_fn)(void* user, int32_t kind, int32_t round, int32_t bucket, const void* send,
                                  void* recv, int64_t bytes_per_rank);
sc_status sc_trainer_set_exchange(sc_trainer* t, sc_exchange_fn fn, void* user);
/* One epoch of train_cofree_impl (trainer.hpp:255-302): every local
 * partition's forward / loss / backward, the gradient exchange, grad_norm and
 * one Adam step. Outputs are host scalars (the only D2H of the step). */
sc_status sc_trainer_step(sc_trainer* t, int32_t epoch, double* loss, double* grad_norm);
/* Stage the NEXT step's n x d features (host: pinned for a true async copy;
 * or device): the copy runs on a copy stream while the current step computes,
 * and the next sc_trainer_step / _step_async commits them (the features the
 * reference's PartitionInputs gather, trainer.hpp:225-227). One staging per step. */
sc_status sc_trainer_stage_features(sc_trainer* t, const float* features, int32_t is_device);
/* Same, but enqueue only (no host sync); results via sc_trainer_last(). */
sc_status sc_trainer_step_async(sc_trainer* t, int32_t epoch);
sc_status sc_trainer_last(sc_trainer* t, double* loss, double* grad_norm);
sc_status sc_trainer_param_count(sc_trainer* t, int64_t* n);
sc_status sc_trainer_get_params(sc_trainer* t, float* out);
sc_status sc_trainer_set_params(sc_trainer* t, const float* in);
sc_status sc_trainer_get_grads(sc_trainer* t, float* out);              /* gathered */
sc_status sc_trainer_get_part_grads(sc_trainer* t, int32_t part, float* out);
sc_status sc_trainer_get_part_logits(sc_trainer* t, int32_t part, float* out);
sc_status sc_trainer_get_part_loss(sc_trainer* t, int32_t part, double* loss);
sc_status sc_trainer_get_part_mask(sc_trainer* t, int32_t part, int32_t* mask_index);
/* evaluate_splits (trainer.hpp:132-140): full-graph forward + accuracy. */
sc_status sc_trainer_evaluate(sc_trainer* t, double* train, double* val, double* test);
/* evaluate (trainer.cpp:101-112) of the trainer's current model over one split
 * mask (n bytes, host): accuracy, or micro-F1 on multi-label graphs. SC_EINVAL
 * "evaluate: empty mask" when no node is masked. */
sc_status sc_trainer_evaluate_mask(sc_trainer* t, const uint8_t* mask, double* metric);
/* evaluate (trainer.cpp:101-112) of a given model: flat f32 parameters in
 * for_each_matrix order for in_dim = the graph's feature dim, hidden[layers],
 * num_classes = the graph's classes; forward-only on the device. */
sc_status sc_evaluate(sc_ctx* ctx, sc_graph* g, const float* theta, const int32_t* hidden, int32_t layers,
                      const uint8_t* mask, double* metric);
/* CommAudit (trainer.hpp:61-76, TrainResult::audit): parameter-gradient floats this
 * rank's partitions handed to the exchange in the last step (p * |theta| at
 * world 1) and node-embedding floats (always 0: none cross partitions). */
sc_status sc_trainer_comm_audit(sc_trainer* t, uint64_t* gradient_floats, uint64_t* embedding_floats);
/* GEMMs that ran on the fp32 SIMT kernels although the tensor-core path was
 * enabled (operand layout not TMA-compatible), since the trainer was created. */
sc_status sc_trainer_fallback_count(sc_trainer* t, int64_t* count);
/* Memory layout the trainer chose (no reference counterpart: the reference keeps
 * every per-layer cache in host RAM, nn.hpp:160-170). flags bit 0: compact
 * activations (one msg buffer + ReLU sign bits); bit 1: shared x0 rows; bit 2:
 * shared logits. arena_bytes: the per-row activation arena. */
sc_status sc_trainer_memory_mode(sc_trainer* t, int32_t* flags, int64_t* arena_bytes);
/* Per-kernel timing of the last step (CUDA events), for bench.py's roofline. */
sc_status sc_trainer_profile(sc_trainer* t, int32_t enable);
sc_status sc_trainer_kernel_times(sc_trainer* t, const char** names, double* ms, double* bytes, int32_t cap,
                                  int32_t* count);
/* Algorithmic GEMM flops (2MNK, fp32-equivalent products) per kernel group, in
 * the order of sc_trainer_kernel_times (0 for non-GEMM groups). */
sc_status sc_trainer_kernel_flops(sc_trainer* t, double* flops, int32_t cap, int32_t* count);
sc_status sc_trainer_destroy(sc_trainer* t);

/* ---- analytic models (host only) ------------------------------------------- */
/* comm_volume (trainer.cpp:38-49): mode 0 cofree (p * |theta| gradient floats per
 * iteration), 1 halo_sync_model (+ 2 * L * total_halo * hidden embedding floats). */
sc_status sc_comm_volume(int32_t mode, int32_t num_parts, uint64_t param_count, uint64_t num_layers,
                         uint64_t hidden_dim, uint64_t total_halo, uint64_t* floats_per_iteration,
                         uint64_t* gradient_floats, uint64_t* embedding_floats);
/* expected_rf_random (partition.cpp:344-349): p (1 - (1 - 1/p)^degree). */
sc_status sc_expected_rf_random(int32_t num_parts, int64_t degree, double* out);
/* imbalance_lower_bound (partition.cpp:351-362). */
sc_status sc_imbalance_lower_bound(int32_t num_parts, int64_t max_degree, int64_t min_degree, double* out);

/* ---- files (byte-compatible with the reference's writers) ------------------ */
/* save_partition (partition_io.cpp:12-29): JSON {num_parts, edge_assignment,
 * parts[{nodes[, weights]}][, weight_scheme]}, nlohmann dump(2). weight_scheme:
 * -1 = no weights, else 0 dar / 1 vanilla_inv / 2 none (compute_weights). */
sc_status sc_save_partition(sc_vcut* vc, const char* path, int32_t weight_scheme);
/* load_partition (partition_io.cpp:31-56): rebuilds the vertex cut from the
 * stored assignment and checks the stored node sets (SC_ERUNTIME on mismatch). */
sc_status sc_load_partition(sc_graph* g, const char* path, sc_vcut** out);
/* save_edge_cut (partition_io.cpp:58-68) of the edge cut induced by node_assignment. */
sc_status sc_save_edge_cut(sc_graph* g, int32_t num_parts, const int32_t* node_assignment, const char* path);
/* save_checkpoint (checkpoint.cpp:44-57) of the trainer's model as SageModel<double>
 * ("CFCK", u64 L, per layer message + update, head; u64 rows, u64 cols, row-major f64 LE). */
sc_status sc_trainer_save_checkpoint(sc_trainer* t, const char* path);
/* load_checkpoint (checkpoint.cpp:59-84) into the trainer's parameters (cast to f32;
 * SC_EINVAL when the shapes differ from the trainer's model). */
sc_status sc_trainer_load_checkpoint(sc_trainer* t, const char* path);
/* save_checkpoint of a flat f32 parameter vector (for_each_matrix order) with
 * the model's dims; load: count = number of parameters (pass theta = NULL to
 * size), values cast to f32 in the same order. */
sc_status sc_save_checkpoint_params(const float* theta, int32_t in_dim, const int32_t* hidden, int32_t layers,
                                    int32_t num_classes, const char* path);
sc_status sc_load_checkpoint_params(const char* path, float* theta, int64_t cap, int64_t* count);
typedef struct {         /* EpochMetrics (trainer.hpp:38-46) */
    int32_t epoch;
    double train_loss, train_metric, val_metric, test_metric, grad_norm;
    uint64_t comm_floats;
} sc_epoch_metrics;
/* write_metrics_jsonl (trainer.cpp:126-140). */
sc_status sc_write_metrics_jsonl(const char* path, int32_t n, const sc_epoch_metrics* rows);

/* ---- diagnostics (kernel-level parity tests) ------------------------------- */
/* C[M x N] = A1[rows1] B1' (+ A2 B2') with epilogue epi (0 none, 1 relu,
 * 2 row-scale by `scale`), through the tcgen05 bf16x3 kernel (mode 0) or the
 * fp32 SIMT kernel (mode 1). B' = B^T when b_nn == 0 (B is N x K), B when
 * b_nn == 1 (B is K x N). A1 has a1_rows rows of lda1 floats; rows1 (length
 * M, optional) gathers them. All buffers are host memory. */
sc_status sc_debug_gemm(sc_ctx* ctx, int32_t mode, int64_t M, int32_t N, int32_t K1, const float* A1,
                        int64_t a1_rows, int64_t lda1, const int32_t* rows1, const float* B1, int64_t ldb1,
                        int32_t b1_nn, int32_t K2, const float* A2, int64_t lda2, const float* B2, int64_t ldb2,
                        int32_t b2_nn, int32_t epi, const float* scale, float* C);
/* Weight-gradient product C[N1 x (N2a + N2b)] = A^T [B1 | B2[rows2]] over M
 * rows: tcgen05 fp16x3 split-K (mode 0) or fp32 SIMT split-K (mode 1).
 * A: M x N1, B1: M x N2a, B2: b2_rows x N2b (optional), rows2: M gather
 * indices into B2 (optional). Host buffers. */
sc_status sc_debug_gemm_tn(sc_ctx* ctx, int32_t mode, int64_t M, const float* A, int32_t N1, const float* B1,
                           int32_t N2a, const float* B2, int64_t b2_rows, int32_t N2b, const int32_t* rows2, float* C);

/* The dual weight-gradient launch alone (one layer's dU and dW, nn.hpp:271-272 +
 * :289): C1 = A1^T [B1 | B2] (N1a x (N2a + N2b)) and C2 = A2^T B2 (N1b x N2b)
 * over M rows in ONE tcgen05 fp16x3 split-K launch. Host buffers, row-major
 * M x N matrices; SC_EINVAL if the shapes do not fit the dual launch
 * (N1a and N2a multiples of 256). */
sc_status sc_debug_gemm_tn_dual(sc_ctx* ctx, int64_t M, const float* A1, int32_t N1a, const float* A2, int32_t N1b,
                               const float* B1, int32_t N2a, const float* B2, int32_t N2b, float* C1, float* C2);
/* The masked mean aggregation alone (nn.hpp:209-230; bwd = 0) or its
 * transpose with the ReLU gate (nn.hpp:277-288, pull form; bwd = 1), through the
 * trainer's kernels (spmm_fwd / spmm_bwd incl. the segmented hub-row path), on a
 * CSR with int64 offsets (n + 1), neighbours and local edge ids (offsets[n]),
 * an optional per-local-edge keep mask (num_edges bytes, as the reference's
 * DropEdge masks index edges). src: n x H (fwd: msg; bwd: dmean already scaled
 * by inv); msg (bwd): the forward's messages (gate = msg > 0); out: n x H. Host
 * buffers. bwd = 2 / 3: the projected top layer's aggregations (trainer.hpp pta):
 * 2 = sum_kept inv[nbr] src[nbr] (no gate), 3 = msg + inv * sum_kept src[nbr]
 * (msg = the addend), inv the masked inverse degrees. */
sc_status sc_debug_spmm(sc_ctx* ctx, int32_t bwd, int64_t n, int32_t H, const int64_t* offsets,
                        const int32_t* nbrs, const int32_t* eids, int64_t num_edges, const uint8_t* edge_mask,
                        const float* src, const float* msg, float* out);
/* Copy `bytes` of a trainer activation buffer ("X" layer 1..L, "MSG" / "MEAN"
 * layer 0..L-1, "inv", "G") to device memory: after a step they hold the last
 * local partition's forward cache (parity diagnostics). */
sc_status sc_trainer_debug_buffer(sc_trainer* t, const char* name, int32_t layer, void* dst_dev, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif
