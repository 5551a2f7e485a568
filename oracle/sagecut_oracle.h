/* sagecut_oracle.h — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load liboracle.so, and only as the checker. The product
 * (paper_2308_03209_b200/) never links or calls it.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below
 * against golden vectors dumped from the REAL reference (oracle/_ref, built
 * from /root/reference/proj/src by oracle/Makefile and validated by running the
 * reference's own unit + acceptance suites against the Eigen shim).
 *
 * Layout conventions (shared with the product C-ABI, include/sagecut_cuda.h):
 *   edges      int32 [m][2] canonical (u < v, sorted, deduped)
 *   matrices   row-major
 *   parameters one flat vector in SageModel::for_each_matrix order
 *              (layer0.message, layer0.update, layer1.message, ..., head),
 *              each matrix row-major — the order make_sage_model draws in
 *              (proj/include/sagecut/nn.hpp:73-102).
 */
#ifndef SAGECUT_ORACLE_H
#define SAGECUT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

/* rng.hpp */
uint64_t or_mix64(uint64_t x);
uint64_t or_substream(uint64_t seed, const char* tag, int nidx, uint64_t a, uint64_t b);
void or_rng_draws(uint64_t seed, int kind, uint64_t arg, int64_t n, uint64_t* out_u, double* out_d);

/* graphs */
void* or_graph_build(int32_t n, const int32_t* uv, int64_t m);
void* or_graph_sbm(int32_t n, int classes, double p_in, double p_out, int d, double noise, uint64_t seed);
void or_graph_free(void* g);
int32_t or_graph_num_nodes(void* g);
int64_t or_graph_num_edges(void* g);
void or_graph_edges(void* g, int32_t* uv);
void or_graph_csr(void* g, int32_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* deg);
void or_graph_features(void* g, double* out);
void or_graph_labels(void* g, int32_t* labels);
void or_graph_masks(void* g, uint8_t* train, uint8_t* val, uint8_t* test);
int or_graph_set_data(void* g, const float* features, int d, const int32_t* labels, int classes,
                      const uint8_t* train, const uint8_t* val, const uint8_t* test);

int or_graph_set_multilabels(void* g, const float* y, int classes);

/* trainer.cpp:38-49, 101-112; partition.cpp:344-362 */
int or_evaluate(void* g, const double* theta, const int* hidden, int layers, const uint8_t* mask, double* out);
int or_comm_volume(int mode, int num_parts, uint64_t params, uint64_t layers, uint64_t hidden, uint64_t halo,
                   uint64_t* out);
int or_expected_rf_random(int p, int64_t degree, double* out);
int or_imbalance_lower_bound(int p, int64_t max_degree, int64_t min_degree, double* out);

/* nn.hpp:209-230 / 277-288: aggregation alone (float), int64 offsets */
void or_spmm(int bwd, int64_t n, int32_t H, const int64_t* off, const int32_t* nbrs, const int32_t* eids,
             const uint8_t* mask, const float* src, const float* msg, float* out, int threads);

/* partition.cpp */
void* or_partition(void* g, int algo /*0 random, 1 dbh, 2 ne (slack 1.1), 3 edge-cut greedy -> ec2vc*/, int p,
                   uint64_t seed);
void* or_partition_ne(void* g, int p, uint64_t seed, double slack, char* warnings, int64_t cap);
int or_edge_cut_greedy(void* g, int p, uint64_t seed, int32_t* node_assign);
int or_edge_cut_stats(void* g, int p, const int32_t* node_assign, int64_t* kept_counts, int64_t* num_cut,
                      int64_t* halo_counts, int32_t* cut_edges, int32_t* halo_nodes);
void* or_edge_cut_to_vertex_cut(void* g, int p, const int32_t* node_assign, uint64_t seed);
void* or_build_vertex_cut(void* g, int p, const int32_t* assign);
void or_partition_free(void* p);
void or_partition_assignment(void* p, int32_t* out);
void or_part_sizes(void* p, int i, int64_t* n_local, int64_t* n_edges);
void or_part_arrays(void* p, int i, int32_t* nodes, int32_t* edges_uv, int32_t* edge_gids, int32_t* local_deg,
                    int32_t* offsets, int32_t* nbrs, int32_t* eids, int32_t* g2l);
int or_replication_stats(void* p, void* g, int32_t* per_node_rf, double* rf, double* edge_balance,
                         double* node_balance, int64_t* duplicated);

/* reweight.cpp / dropedge.cpp */
int or_weights(void* g, void* p, int scheme, double* out);
int or_precompute_masks(int64_t num_edges, int k, double ratio, uint64_t seed, uint8_t* out);
int or_select_mask(uint64_t seed, uint64_t part, uint64_t epoch, int k);

/* nn.hpp */
int64_t or_init_params(int in_dim, const int* hidden, int layers, int classes, uint64_t seed, int f32, double* out);

/* trainer.hpp:202-313 */
void* or_trainer_new(void* g, void* p, const int* hidden, int layers, double lr, int loss, int reweight,
                     int use_dropedge, int k, double ratio, uint64_t seed, int f32, int workers);
void or_trainer_free(void* t);
int or_trainer_step(void* t, int epoch, double* loss, double* gnorm);
int64_t or_trainer_param_count(void* t);
void or_trainer_params(void* t, double* out);
void or_trainer_set_params(void* t, const double* in);
void or_trainer_part_grads(void* t, int i, double* out);
void or_trainer_gathered(void* t, double* out);
void or_trainer_part_logits(void* t, int i, double* out);
double or_trainer_part_loss(void* t, int i);
int or_trainer_part_mask(void* t, int i);
void or_trainer_eval(void* t, double* train, double* val, double* test);
double or_trainer_time_part_step(void* t, int i, int epoch, int reps);

#ifdef __cplusplus
}
#endif
#endif
