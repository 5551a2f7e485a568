// nn.cuh — kernels of the per-partition training step (declarations).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"

namespace sc {

// Aggregation rows with more than kHeavySlots CSR slots (skewed degrees) are
// split into kSegSlots-slot segments so no single warp walks a hub row.
constexpr int64_t kHeavySlots = 4096;
constexpr int64_t kSegSlots = 1024;
// Narrow rows (<= 128 floats) of at most kNarrowSlots CSR slots are aggregated several per warp; the
// longer ones (the "mid" rows, up to kHeavySlots) a warp each, from a list.
constexpr int64_t kNarrowSlots = 64;
struct HeavyRows {
    DevBuf<int32_t> mid;        // nmid rows with kNarrowSlots < slots <= kHeavySlots, ascending
    int32_t nmid = 0;
    bool built = false;
    DevBuf<int32_t> rows;       // nh heavy rows, ascending
    DevBuf<int32_t> seg_first;  // nh + 1: segments of row h are [seg_first[h], seg_first[h+1])
    DevBuf<int32_t> seg_row;    // nseg
    DevBuf<int64_t> seg_begin;  // nseg: first CSR slot of the segment
    int32_t nh = 0, nseg = 0;
};
// Heavy-row table of a CSR (offsets on the device).
void build_heavy_rows(sc_ctx* ctx, int64_t n, const int64_t* offsets, HeavyRows& hv);

// A operand of a row-major GEMM: A[r][k] = ptr[(rows ? rows[r] : r) * ld + k].
struct MatA {
    const float* ptr = nullptr;
    int64_t ld = 0;
    const int32_t* rows = nullptr;  // optional row gather (partition -> global features)
    int32_t K = 0;
};
// B operand: NT: B is [N x K] (ld between rows of N); NN: B is [K x N] (ld between rows of K).
struct MatB {
    const float* ptr = nullptr;
    int64_t ld = 0;
    bool nn = false;
};

// kEpiMask: C = 1[msg > 0] * acc, the ReLU decision of the N-wide msg row (mask_msg, row stride N) or
// its sign bits (mask_pos, [M][ceil(N / 32)] words) — the transposed aggregation's dz (nn.hpp:287-288).
enum Epilogue : int { kEpiNone = 0, kEpiRelu = 1, kEpiRowScale = 2, kEpiMask = 3 };

// C[M x N] = A1 * op(B1) (+ A2 * op(B2)), fp32 in/out, fp32 accumulate, then epilogue.
// amax_out (optional): atomically max-reduced with |C| (the next GEMM's operand scale).
void gemm_nt(const MatA& a1, const MatB& b1, const MatA* a2, const MatB* b2, float* C, int64_t ldc, int64_t M,
             int32_t N, int epi, const float* row_scale, cudaStream_t s, float* amax_out = nullptr,
             const float* mask_msg = nullptr, const uint32_t* mask_pos = nullptr);

// dst[r][:] = src[rows[r]][:] (n x d); dst_ld > d pads each destination row with zeros
// (and then rows may be null: identity).
void gather_rows(int64_t n, int32_t d, const int32_t* rows, const float* src, float* dst, cudaStream_t s,
                 int32_t dst_ld = 0);

// *out = max(*out, max |x[0..n)|) (non-negative floats compare like their bit patterns).
void absmax(int64_t n, const float* x, float* out, cudaStream_t s);
// C[M x N] = op(A) op(B) in fp32 with fp64 accumulation (small weight-space products).
void small_gemm(int M, int N, int K, const float* A, int64_t lda, bool ta, const float* B, int64_t ldb, bool tb,
                float* C, int64_t ldc, cudaStream_t s);

// Weight gradient: C[N1 x N2] = A^T [N1 x M] * Bcat [M x N2], where Bcat's
// columns [0, n2a) come from b1 and [n2a, N2) from b2 (b2 may gather rows).
// Split-K over M with a fixed-order reduction (deterministic). C has row stride ldc.
struct MatT {
    const float* ptr = nullptr;
    int64_t ld = 0;
    const int32_t* rows = nullptr;
    int32_t cols = 0;
};
void gemm_tn(const MatT& a, const MatT& b1, const MatT* b2, int64_t M, float* C, int64_t ldc, float* workspace,
             int64_t workspace_floats, cudaStream_t s);
int64_t gemm_tn_workspace_floats(int32_t N1, int32_t N2);

// Per-node inverse masked degree (nn.hpp:174-188, 209-215): inv = d > 0 ? 1/d : 0.
void inv_degree(int64_t n, const int64_t* offsets, const uint32_t* mask_bits, float* inv, cudaStream_t s);
// mean[v] = inv[v] * sum_{k in CSR(v), kept} msg[nbr_k]   (nn.hpp:222-230).
// hv (optional): the CSR's heavy rows, aggregated through `partial`
// (hv->nseg x H floats).
void spmm_fwd(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* mask_bits,
              const float* inv, const float* msg, float* mean, cudaStream_t s, const HeavyRows* hv = nullptr,
              float* partial = nullptr);
// dz[u] = 1[msg[u] > 0] * sum_{v in CSR(u), kept} dmean_s[v]   (nn.hpp:277-288, pull form).
// relu_pos (compact activations): the ReLU decisions as sign bits, [n][ceil(H / 32)]
// words (bit c % 32 of word c / 32), read instead of the msg rows (msg may be null).
// out += inv * sum_kept src[nbr] (the composed top layer's forward aggregation of projected rows)
void spmm_fwd_add(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* mask_bits,
                  const float* inv, const float* src, float* out, cudaStream_t s, const HeavyRows* hv, float* partial);
// out = sum_kept inv[nbr] src[nbr] (pull form of the transposed aggregation, nn.hpp:277-286, without the
// ReLU mask; rows of at most 128 floats)
void spmm_sum_scaled(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* mask_bits,
                     const float* inv, const float* src, float* out, cudaStream_t s, float* amax_out,
                     const HeavyRows* hv, float* partial);
void spmm_bwd(int64_t n, int32_t H, const int64_t* offsets, const int32_t* nbrs, const uint32_t* mask_bits,
              const float* dmean_s, const float* msg, float* dz, cudaStream_t s, float* amax_out = nullptr,
              const HeavyRows* hv = nullptr, float* partial = nullptr, const uint32_t* relu_pos = nullptr);
// pos[r][w] bit q = C[r][32 w + q] > 0 (for GEMM paths whose epilogue does not emit the bits).
void relu_sign_bits(int64_t M, int32_t N, const float* C, int64_t ldc, uint32_t* pos, cudaStream_t s);
// CSR-slot bitmap of a local-edge-indexed byte mask: bit k = mask[eids[k]].
void mask_to_bits(int64_t nnz, const int32_t* eids, const uint8_t* mask, uint32_t* bits, cudaStream_t s);

// Loss + dloss/dlogits (nn.hpp:317-378). Rows with w == 0 get zero gradient.
// row_loss[r] = w * (lse - z_y) (CE) in f64; scale[r] = (float)(w / normalizer).
// ld: row stride of logits and G (>= C)
void softmax_ce(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const int32_t* rows,
                const double* w, const float* scale, float* G, double* row_loss, cudaStream_t s);
// targets (optional): the graph's n x C 0/1 multi-label matrix, else one-hot of labels.
void bce(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const uint8_t* targets,
         const int32_t* rows, const double* w, const float* scale, float* G, double* row_loss, cudaStream_t s);
// Deterministic f64 sum of x[0..n), divided by `divisor`, into *out (fixed-shape two-pass reduction).
void sum_f64(int64_t n, const double* x, double* partial, double* out, double divisor, cudaStream_t s);

// gathered[k] = sum_{i < p} slot_i[k] in ascending i (trainer.hpp:79-94) over
// bucket-major slots (bucket b = parameter matrix b holds pp >= p per-partition
// copies; b_off: nb + 1 device offsets, the last = P); f64 sum of squares +
// non-finite flag for grad_norm / adam_step's check.
void gather_grads(int64_t P, int32_t p, int32_t pp, int32_t nb, const int64_t* b_off, const float* slots,
                  float* gathered, double* partial, int* nonfinite, cudaStream_t s);
// out[0] = sqrt(sum partial) (grad_norm), out[1] = sum part_loss[0..p) in order.
void finalize_step(const double* partial, const double* part_loss, int32_t p, double* out, cudaStream_t s);
// Adam (nn.hpp:400-432); skipped entirely when *nonfinite is set.
void adam(int64_t P, float* theta, float* m1, float* m2, const float* g, float b1, float b2, float c1, float c2,
          float lr, float eps, const int* nonfinite, cudaStream_t s);

// Accuracy of argmax(logits) over masked rows (trainer.cpp:66-97, multi-class).
void count_correct(int64_t n, int32_t C, int32_t ld, const float* logits, const int32_t* labels, const uint8_t* mask,
                   unsigned long long* correct_and_total, cudaStream_t s);

// Micro-F1 counts (trainer.cpp:72-87): out[0..3] += (tp, fp, fn, masked rows).
void f1_counts(int64_t n, int32_t C, int32_t ld, const float* logits, const uint8_t* targets, const uint8_t* mask,
               unsigned long long* out, cudaStream_t s);

}  // namespace sc
